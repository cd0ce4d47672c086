#!/usr/bin/env python
"""HalftimeHash B200 benchmark (driver contract: one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload cfg1|cfg2|cfg3|cfg4|cfg5] [--no-extra] [--e2e-steps E]
                  [--exchange auto|flags|p2p|nccl]

Headline workload: config 4 of BASELINE.json -- 8192 strings x 1 MiB per GPU
(8 GiB, 40-byte variant), the largest batch config and the one quoted per GPU
and per box; strings are sharded round-robin across ranks (weak scaling, no
data-path collective).  A "step" is one pass of the hash over the whole
batch: exactly one hash_kernel launch.  Inputs (8 GiB) exceed L2 (126 MB),
so no flush is needed between steps.  At N=1 rank 0 also measures the other
configs (cfg1, cfg2, cfg3, cfg5, and config 5's multi-GPU exchange emulated
on one GPU) into "workloads" (cfg1/cfg2 with an L2 flush between timed
iterations).

--gpus N > 1 without torchrun's environment re-launches this script under
``torch.distributed.run --nproc-per-node N`` (127.0.0.1); under torchrun,
WORLD_SIZE must equal --gpus.  Config 5 on N > 1 GPUs splits the one string
across the ranks (strong scaling) with the in-stream peer-flag exchange.

--impl reference times the reference's CPU implementation on all host cores
over a bounded sample of the same workload: the reference package itself
(halftimehash 0.1.0 ``_hash_words_np``, hasher.py:331-413, installed in
baseline/_ref) when present, else its numpy restatement oracle/oracle_np.py.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402

METRIC = "GB/s hashed"
UNIT = "GB/s"

# the dominant kernel of each workload (launch configuration picked by the C-ABI)
KERNELS = {
    "cfg1": "small_kernel<24, G=1, W=2, NS=2, MINB=4> (one launch per step)",
    "cfg2": "per variant: plan_kernel<w> + hash_kernel<w, varlen> (4 variants on 4 streams, one CUDA graph)",
    "cfg3": "tail_kernel<32, CPT=4, unmasked, NS=1, GP=4> (one launch per step)",
    "cfg4": "hash_kernel<40, fixed, W=2, NS=2, MINB=5, AL8> (one launch per step)",
    "cfg5": "hash_kernel<16, fixed, W=4, NS=2, MINB=4, AL8> (one launch per step)",
}
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_pkg():
    """The reference package (halftimehash 0.1.0) if installed in baseline/_ref."""
    if not os.path.isdir(os.path.join(REF_DIR, "halftimehash")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import halftimehash

        return halftimehash
    except Exception:
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(workload):
    """dram read+write bytes per launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(workload)
    except Exception:
        return None


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = [l for (t, l) in self.lines if (t0 is None or t >= t0 - 0.06) and (t1 is None or t <= t1 + 0.06)]
        if not rows:
            rows = [l for (_, l) in self.lines]
        for l in rows:
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU side
_CPU_SAMPLE = {}


def _cpu_task(arg):
    """Hash worker i's next `count` pre-generated strings (from `start`, cyclic)
    with the reference's batched engine (or its numpy restatement); the pool
    is inherited via fork."""
    i, start, count = arg
    n, pool = _CPU_SAMPLE["n"], _CPU_SAMPLE["words"][i]
    if start + count <= pool.shape[0]:
        words = pool[start:start + count]
    else:
        words = pool[(start + np.arange(count)) % pool.shape[0]]
    if _CPU_SAMPLE["ref"] is not None:
        R = _CPU_SAMPLE["ref"]
        R.hasher._hash_words_np(words, n, _CPU_SAMPLE["ref_seed"].words_np, _CPU_SAMPLE["ref_params"])
    else:
        from oracle import oracle_np as o

        o.hash_batch(_CPU_SAMPLE["v"], words, n, _CPU_SAMPLE["S"])
    return count * n


def _cpu_task_varlen(arg):
    """Config 2 on the CPU: the reference hashes each string with hash_bytes
    (lengths differ), all four variants; worker i takes strings
    i, i + cores, ... of its share of the batch."""
    i, cores = arg
    data, off, R = _CPU_SAMPLE["data"], _CPU_SAMPLE["off"], _CPU_SAMPLE["ref"]
    total = 0
    for w in (16, 24, 32, 40):
        if R is not None:
            p, seed = _CPU_SAMPLE["ref_params"][w], _CPU_SAMPLE["ref_seed"][w]
        for s in range(i, len(off) - 1, cores):
            b = data[int(off[s]):int(off[s + 1])]
            if R is not None:
                R.hash_bytes(b, seed, p)
            else:
                from oracle import oracle_np as o

                o.hash_bytes(_CPU_SAMPLE["v"][w], b, _CPU_SAMPLE["S"][w])
            total += len(b)
    return total


# strings per core per pass of the CPU arm (~4 MiB: the numpy port's best granularity)
CPU_PER_CORE = {"cfg1": 1024, "cfg3": 4096, "cfg4": 4, "cfg5": 1}

# per-core pool of distinct strings, larger than the last-level cache share,
# so every pass streams fresh data from DRAM as the reference would
CPU_POOL_BYTES = 64 << 20


class CpuBaseline:
    """The reference's CPU path on `cores` forked processes: the reference
    package's own ``_hash_words_np`` (hasher.py:331-413) when it is installed
    in baseline/_ref (kind "reference"), else its numpy restatement
    oracle/oracle_np.py (kind "port", bit-identical, ~1.3x faster).  Each
    process holds a pool of >= 64 MiB of distinct strings of the workload,
    generated before any timing; rate() times one pass in which every process
    hashes its next `per_core` strings (cyclic), so small samples are not
    served from cache.  Config 2: per-string hash_bytes over the batch, all
    four variants, strings dealt round-robin to the processes."""

    def __init__(self, workload: str, per_core: int, cores: int, use_reference: bool = True):
        from oracle import oracle_np as o

        R = _reference_pkg() if use_reference else None
        self.kind = "reference" if R is not None else "port"
        _CPU_SAMPLE.clear()
        _CPU_SAMPLE["ref"] = R
        self.workload = workload
        self.cores = cores
        self.next = 0
        if workload == "cfg2":
            lengths = wl.cfg2_lengths()
            off = wl.offsets_of(lengths)
            _CPU_SAMPLE.update(data=wl.host_bytes(0, int(off[-1])), off=off)
            mx = int(lengths.max())
            if R is not None:
                _CPU_SAMPLE["ref_params"] = {w: R.variant(w) for w in (16, 24, 32, 40)}
                _CPU_SAMPLE["ref_seed"] = {w: R.seed_for_input(wl.MASTER, R.variant(w), mx) for w in (16, 24, 32, 40)}
            else:
                _CPU_SAMPLE["v"] = {w: o.variant(w) for w in (16, 24, 32, 40)}
                _CPU_SAMPLE["S"] = {w: o.splitmix_words(o.master_fold(wl.MASTER), 0,
                                                        o.seed_words_needed(o.variant(w), mx)) for w in (16, 24, 32, 40)}
            self.n, self.w, self.per_core, self.per_pool = int(off[-1]), "16/24/32/40", 0, 0
        else:
            cfg = wl.CONFIGS[workload]
            w, n = cfg["variant"], cfg["n_bytes"]
            if workload == "cfg5":  # one huge string: time 16 MiB pieces of it
                n = 16 << 20
            v = o.variant(w)
            assert n % 8 == 0
            per_pool = max(per_core, -(-CPU_POOL_BYTES // n))
            _CPU_SAMPLE.update(v=v, n=n, S=o.splitmix_words(o.master_fold(wl.MASTER), 0, o.seed_words_needed(v, n)))
            if R is not None:
                _CPU_SAMPLE["ref_params"] = R.variant(w)
                _CPU_SAMPLE["ref_seed"] = R.seed_for_input(wl.MASTER, R.variant(w), n)
            _CPU_SAMPLE["words"] = [
                o.words_from_bytes(wl.host_bytes(i * per_pool * n, per_pool * n)).reshape(per_pool, -1)
                for i in range(cores)]
            self.per_core, self.n, self.w, self.per_pool = per_core, n, w, per_pool
        self.pool = mp.get_context("fork").Pool(cores) if cores > 1 else None

    def rate(self):
        if self.workload == "cfg2":
            fn, args = _cpu_task_varlen, [(i, self.cores) for i in range(self.cores)]
        else:
            fn, args = _cpu_task, [(i, self.next, self.per_core) for i in range(self.cores)]
            self.next = (self.next + self.per_core) % self.per_pool
        t0 = time.perf_counter()
        if self.pool is None:
            total = sum(fn(a) for a in args)
        else:
            total = sum(self.pool.map(fn, args, chunksize=1))
        dt = time.perf_counter() - t0
        return total / dt / 1e9, total, dt

    def sample(self):
        engine = ("the reference package itself (halftimehash 0.1.0 from baseline/_ref: _hash_words_np, "
                  "hasher.py:331-413)" if self.kind == "reference" else
                  "numpy restatement of hasher.py:331-413 (oracle/oracle_np.py, bit-identical to the reference, "
                  "~1.3x its single-core speed)")
        if self.workload == "cfg2":
            return (f"{self.cores} processes, the whole config-2 batch ({self.n} B, 16384 strings) per pass and "
                    f"variant, one hash_bytes per string (all 4 variants); {engine.replace('_hash_words_np', 'hash_bytes')}")
        return (f"{self.cores} processes x {self.per_core} strings of {self.n} B (v{self.w}) per pass, "
                f"each from its own pool of {self.per_pool} distinct pre-generated strings (cyclic, larger "
                f"than the caches); {engine}")

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


# ---------------------------------------------------------------- GPU side
def _algo_bytes(workload, n_strings, n_bytes, k):
    return n_strings * n_bytes + n_strings * k * 8


def _stream_strings(gidx, n):
    """Host bytes of global strings gidx (n bytes each, n % 8 == 0) of a config
    buffer: the data stream regenerated by the threaded C splitmix."""
    from oracle import c as coracle

    assert n % 8 == 0
    return np.concatenate([coracle.splitmix(wl.DATA_SEED, g * n // 8, n // 8).view(np.uint8) for g in gidx])


def setup_fixed(hh, torch, workload, rank=0, world=1):
    cfg = wl.CONFIGS[workload]
    w, n = cfg["variant"], cfg["n_bytes"]
    B = cfg["n_strings"]
    p = hh.variant(w)
    buf = torch.empty(B * n + 64, dtype=torch.uint8, device="cuda")
    # round-robin: local string i is global string rank + i * world (one launch)
    hh.fill_strings(B, n, rank, world, wl.DATA_SEED, out=buf)
    seed = hh.seed_for_input(wl.MASTER, p, n)
    st = seed.device_words()
    out = torch.empty((B, p.output_words), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    return dict(p=p, buf=buf, seed=seed, out=out, B=B, n=n, w=w)


def run_fixed(hh, torch, ctx, steps, warmup, flush=None, barrier=None):
    p, buf, seed, out, B, n = ctx["p"], ctx["buf"], ctx["seed"], ctx["out"], ctx["B"], ctx["n"]
    stream = torch.cuda.current_stream()

    def step():
        hh.hash_fixed(buf, n, seed, p, n_strings=B, stride=n, out=out)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if barrier:
        barrier()
        torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    t_start.record(stream)
    for i in range(steps):
        if flush is not None:
            flush()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    wall1 = time.time()
    per = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(per) if flush is not None else t_start.elapsed_time(t_end)
    return total_ms, per, (wall0, wall1)


def make_flush(torch):
    big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def flush():
        big.fill_(1)

    return flush


def measure_latency(hh, sizes=(64, 4096, 1 << 20, 64 << 20), variant=24, reps=20):
    """Single-string latency of the public one-shot API (hash_bytes on host
    bytes: seed expansion, H2D copy, hash, digest read-back),
    wall clock, median of 500 calls (inputs up to 64 KiB) or `reps` calls,
    beside the CPU port on one core."""
    from oracle import oracle_np as o

    p = hh.variant(variant)
    v = o.variant(variant)
    out = {"variant": variant, "api": "hash_bytes(bytes, SeedBuffer, params) -> Digest", "gpu_us": {}, "cpu_us": {}}
    for n in sizes:
        data = wl.host_bytes(0, n)
        seed = hh.seed_for_input(wl.MASTER, p, n)
        small = n <= 1 << 16
        for _ in range(1000 if small else 3):  # steady state (the first few hundred calls run ~15 % slower)
            d = hh.hash_bytes(data, seed, p)
        ts = []
        for _ in range(500 if small else reps):
            t0 = time.perf_counter()
            d = hh.hash_bytes(data, seed, p)
            ts.append(time.perf_counter() - t0)
        out["gpu_us"][str(n)] = round(statistics.median(ts) * 1e6, 1)
        if n <= 1 << 20:
            S = o.splitmix_words(o.master_fold(wl.MASTER), 0, o.seed_words_needed(v, n))
            words = o.words_from_bytes(data).reshape(1, -1)
            want = o.hash_batch(v, words, n, S)[0]
            assert tuple(int(x) for x in want) == tuple(d.words), "latency probe digest mismatch"
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                o.hash_batch(v, words, n, S)
                ts.append(time.perf_counter() - t0)
            out["cpu_us"][str(n)] = round(statistics.median(ts) * 1e6, 1)
    return out


def measure_workload(hh, torch, workload, steps, warmup, peak, barrier=None):
    """Measurement of one config on this GPU (the secondary configs at N=1;
    config 2's main line)."""
    res = {"desc": wl.CONFIGS[workload]["desc"]}
    if workload == "cfg2":
        # four variants over the same packed batch: independent pipelines (plan ->
        # scan -> scatter -> tail kernel -> hash kernel), forked onto four streams
        # and captured once as a CUDA graph; each step replays the graph
        lengths = wl.cfg2_lengths()
        off = wl.offsets_of(lengths)
        total = int(off[-1])
        buf = torch.empty(total + 64, dtype=torch.uint8, device="cuda")
        hh.fill_bytes(total, wl.DATA_SEED, 0, out=buf)
        d_off = torch.from_numpy(off.view(np.int64)).cuda()
        mx = int(lengths.max())
        widths = (16, 24, 32, 40)
        seeds = {w: hh.seed_for_input(wl.MASTER, hh.variant(w), mx) for w in widths}
        outs = {w: torch.empty((len(lengths), w // 8), dtype=torch.int64, device="cuda") for w in widths}
        from paper_2104_08865_b200 import batch as hb

        wss = {w: torch.zeros(hb.workspace_varlen(hh.variant(w), len(lengths), total), dtype=torch.uint8,
                              device="cuda") for w in widths}
        for w in widths:
            seeds[w].device_words()
        side = {w: torch.cuda.Stream() for w in widths}

        def step():
            cur = torch.cuda.current_stream()  # the capture stream while capturing
            ev = torch.cuda.Event()
            ev.record(cur)
            for w in widths:
                with torch.cuda.stream(side[w]):
                    side[w].wait_event(ev)
                    hh.hash_varlen(buf, d_off, seeds[w], hh.variant(w), max_n_bytes=mx, out=outs[w],
                                   workspace=wss[w], check=False)
            for w in widths:
                cur.wait_stream(side[w])

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        for w in widths:  # the device found no bound or offset violation
            hb.varlen_status(wss[w])
        # correctness of the concurrent path: compare with the serial result
        ref = {w: hh.hash_varlen(buf, d_off, seeds[w], hh.variant(w), max_n_bytes=mx).clone() for w in widths}
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for w in widths:
            outs[w].zero_()
        g.replay()
        torch.cuda.synchronize()
        same = all(bool(torch.equal(ref[w], outs[w])) for w in widths)
        flush = make_flush(torch)
        per = []
        stream = torch.cuda.current_stream()
        if barrier:
            barrier()
        for _ in range(steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            per.append(a.elapsed_time(b))
        ms = statistics.mean(per)
        res.update(value=4 * total / (ms / 1e3) / 1e9, ms_per_step=ms, bytes_per_step=4 * total,
                   l2="flushed (256 MB write) before every timed step",
                   execution="4 variants on 4 forked streams, captured as one CUDA graph, replayed per step",
                   graph_matches_serial=same,
                   bound=("latency: per variant two launches (plan kernel, which also hashes the ~10k strings "
                          "shorter than one instance, then the job kernel) and ~3 us per warp job (claim, "
                          "decode, finalize) against 2-3 us unaligned rounds; 98 MB per variant is 15 us of HBM "
                          "time (DESIGN.md section 5)"))
        del buf
        return res
    ctx = setup_fixed(hh, torch, workload)
    flush = make_flush(torch) if workload == "cfg1" else None
    k = ctx["p"].output_words
    total_ms, per, _ = run_fixed(hh, torch, ctx, steps, warmup, flush)
    ms = total_ms / steps
    algo = _algo_bytes(workload, ctx["B"], ctx["n"], k)
    gbs = ctx["B"] * ctx["n"] / (ms / 1e3) / 1e9
    rp = _read_peak(algo / (ms / 1e3) / 1e9)
    res.update(value=gbs, ms_per_step=ms, bytes_per_step=ctx["B"] * ctx["n"],
               roofline_frac=(algo / (ms / 1e3) / 1e9) / peak,
               frac_of_read_peak=rp["frac"] if rp else None,
               l2="flushed before every timed step" if flush else "inputs larger than L2 (126 MB)")
    if workload == "cfg1":
        res["bound"] = ("latency: one launch hashes 4 MiB (0.6 us of HBM time); each warp's critical path is "
                        "one stage's DRAM round trip after the flush + one two-instance leaf + finalize "
                        "(profiles/README.md)")
        floor = _cfg1_floor()
        if floor:
            res["floor"] = floor
            res["frac_of_floor"] = floor["us"] / (ms * 1e3)
    del ctx
    torch.cuda.empty_cache()
    return res


# exact NH multiplies per input byte (entropy_report of the
# reference's analysis.py:241-248 on each config)
MULT_PER_BYTE = {"cfg1": 0.2058, "cfg2": 0.300, "cfg3": 0.5039, "cfg4": 0.2676, "cfg5": 0.1667}


def _imad_bound(workload, achieved_gbs):
    """The north-star's other roofline: the 32x32->64 multiply pipe.  Rate =
    the measured IMAD.WIDE.U32 issue rate (tools/peaks.cu, profiles/peaks_r02.json)
    at the attribute clock; bound = rate / NH multiplies per byte."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_r02.json")) as fh:
            tops = json.load(fh)["imad_wide_tops"]
    except (OSError, KeyError, ValueError):
        return None
    mpb = MULT_PER_BYTE[workload]
    bound = tops * 1e12 / mpb / 1e9
    return {"mult_per_byte": mpb, "imad_wide_tops": tops, "bound_gbs": bound, "frac": achieved_gbs / bound,
            "note": "multiply-pipe roofline (measured IMAD.WIDE.U32 rate / multiplies per byte): never the "
                    "binding one here; the HBM figure is"}


def _cpu_model():
    """The host CPU the CPU baseline ran on (state the model)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _read_peak(achieved_gbs):
    """The kernels only read HBM (digests are ~0.01 % of the bytes), so beside
    the contract's copy peak (read + write) report the measured read-only
    streaming peak of their own load path: TMA bulk copies into a per-warp
    ring, best of a stage-size x warps/SM sweep (tools/peaks.cu)."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_r02.json")) as fh:
            rd = json.load(fh)["tma_read_gbs"]
    except (OSError, KeyError, ValueError):
        return None
    return {"gbs": rd, "frac": achieved_gbs / rd, "source": "profiles/peaks_r02.json tma_read_gbs (tools/peaks.cu)"}


def _cfg1_floor():
    """Config 1's measured floor (tools/peaks.cu, committed): 1024 warps each
    doing one 4 KiB bulk copy + one 24-byte store after the same 256 MB L2
    flush, CUDA events around the launch -- everything but the hash."""
    path = os.path.join(ROOT, "profiles", "peaks_r02.json")
    try:
        with open(path) as fh:
            f = json.load(fh)["cfg1_floor_us"]
    except (OSError, KeyError, ValueError):
        return None
    return {"us": f["bulk_copy_4KiB_per_warp"], "empty_launch_us": f["empty_launch"],
            "what": "512 CTAs x 2 warps: one 4 KiB cp.async.bulk + one 24-byte store per warp after the L2 flush, "
                    "event-timed like the step", "source": "profiles/peaks_r02.json (tools/peaks.cu)"}


def e2e_fixed(hh, torch, workload, steps, n_strings_cap=None, rank=0, world=1, local_rank=0, dist=None):
    """Public host-buffer API (hth_hash_fixed_host) from pinned memory on every
    rank at once: H2D + hash + D2H per step; value = all ranks' bytes / the
    slowest rank's wall time (barrier on both sides of each step)."""
    cfg = wl.CONFIGS[workload]
    w, n, B = cfg["variant"], cfg["n_bytes"], cfg["n_strings"]
    if n_strings_cap:
        B = min(B, n_strings_cap)
    p = hh.variant(w)
    ctx = setup_fixed(hh, torch, workload, rank, world) if not n_strings_cap else None
    if ctx is None:
        dev = torch.empty(B * n + 16, dtype=torch.uint8, device="cuda")
        hh.fill_bytes(B * n, wl.DATA_SEED, rank * B * n // 8, out=dev)
    else:
        dev = ctx["buf"]
    # every rank pins its buffer before any collective, and all ranks agree
    # on success, so a rank that cannot pin never leaves the others waiting
    try:
        host = torch.empty(B * n, dtype=torch.uint8, pin_memory=True)
        ok = 1
    except Exception:  # pragma: no cover
        host, ok = None, 0
    if dist:
        f = torch.tensor([ok], dtype=torch.int32, device="cuda")
        dist.all_reduce(f, op=dist.ReduceOp.MIN)
        ok = int(f.item())
    if not ok:
        raise RuntimeError("could not pin the e2e host buffer on every rank")
    host.copy_(dev[:B * n])
    del dev, ctx
    torch.cuda.empty_cache()
    hh.hash_fixed_host(host, B, n, wl.MASTER, p, device=local_rank)  # warm-up (allocates staging buffers)
    times = []
    for _ in range(steps):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        out = hh.hash_fixed_host(host, B, n, wl.MASTER, p, device=local_rank)
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        times.append(dt)
    dt = statistics.median(times)
    return {"value": world * B * n / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": world * B * n,
            "d2h_bytes_per_step": world * B * p.output_words * 8, "strings_per_step": world * B,
            "steps": steps, "api": "hth_hash_fixed_host (pinned host memory, 3-stream chunked H2D/hash, one D2H of the digests), "
                                   "all ranks concurrently, max-over-ranks wall time"}, out


# ---------------------------------------------------------------- arms
def arm_reference(args, rank, world):
    if rank != 0:
        return 0
    workload = args.workload
    cores = os.cpu_count() or 1
    per_core = CPU_PER_CORE.get(workload, 4)
    cpu = CpuBaseline(workload, per_core, cores)
    for _ in range(1 if workload == "cfg2" else args.warmup):
        cpu.rate()
    rates, dts, tot = [], [], 0
    for _ in range(args.steps):
        r, b, dt = cpu.rate()
        rates.append(r)
        dts.append(dt)
        tot = b
    cpu.close()
    value = statistics.median(rates)
    cfg = wl.CONFIGS[workload]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(dts) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (splitmix stream, seed 0)",
        "config": {"workload": workload, "desc": cfg["desc"], "variant": cfg["variant"],
                   "bytes_per_step": tot},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": cpu.kind, "sample": cpu.sample(),
                         "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _rank_report(dist, info):
    """Every rank's own record (device, busy time, clocks), gathered to all."""
    if dist is None:
        return [info]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, info)
    return out


def _comm(dist):
    if dist is None:
        return {"backend": None, "world_size": 1}
    return {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
            "note": "communicator of the barrier / max-over-ranks timing; the hash itself has no data-path collective"}


def arm_split(args, rank, world, local_rank, hh, torch, dist):
    """Config 5 on N > 1 GPUs: ONE 16 GiB string split at multiples of 8^c
    instances (hth_slice_plan); each rank generates and hashes its slice in
    place (hth_hash_slice_ex).  Exchange (--exchange):
      flags (default with one GPU per rank): in-stream -- the slice kernels
        store their subtree roots and partial digest into rank 0's memory
        over NVLink (CUDA-IPC peer pointers) and raise a per-rank arrival
        flag; rank 0's merge kernel waits on the flags in-stream; slots are
        double-buffered and handed back through a consumed flag.  No host
        synchronisation, barrier or collective inside the step.
      p2p: the same peer stores, then a host synchronize + barrier per string
        (the only safe form when ranks share a GPU).
      nccl: all_gather of roots/partials.
    A step = the whole string; total work is fixed as N grows (strong
    scaling)."""
    from paper_2104_08865_b200 import multi_gpu

    peak, peak_src = _peaks()
    cfg = wl.CONFIGS["cfg5"]
    w, n = cfg["variant"], cfg["n_bytes"]
    p = hh.variant(w)
    plan = multi_gpu.slice_plan(p, n, world)
    b0, b1 = plan.byte_range(rank)
    buf = torch.empty(b1 - b0 + 64, dtype=torch.uint8, device="cuda")
    hh.fill_bytes(b1 - b0, wl.DATA_SEED, b0 // 8, out=buf)
    seed = hh.seed_for_input(wl.MASTER, p, n)
    seed.device_words()
    dev = torch.device("cuda", torch.cuda.current_device())
    exchange = args.exchange
    ids = multi_gpu._device_ids(dev, None)
    distinct = len(set(ids)) == len(ids)
    if exchange == "auto":
        exchange = "flags" if distinct else "p2p"
    if exchange == "flags" and not distinct:
        raise SystemExit("--exchange flags needs one GPU per rank (kernels on one device must not wait on each other)")
    fx = multi_gpu.FlagExchange(plan, seed, dev) if exchange == "flags" else None
    stream = torch.cuda.current_stream()
    kern = []
    last = {}

    def step():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if fx is not None:
            last["d"] = fx.step(buf)
        elif exchange == "p2p":
            last["d"] = multi_gpu.hash_string_p2p(buf, plan, seed)
        else:
            last["d"] = multi_gpu.hash_string_distributed(buf, plan, seed)
        b.record(stream)
        kern.append((a, b))

    for _ in range(args.warmup):
        step()
    if fx is not None:
        fx.check()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    kern.clear()
    dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    wall1 = time.time()
    time.sleep(0.2)
    sampler.stop()
    if fx is not None:
        fx.check()
    mine_ms = t0.elapsed_time(t1)
    t = torch.tensor([mine_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    step_ms = statistics.mean(a.elapsed_time(b) for a, b in kern)
    ranks = _rank_report(dist, {"rank": rank, "device": ids[rank], "slice_bytes": b1 - b0,
                                "busy_ms_per_step": mine_ms / args.steps, "step_event_ms": step_ms,
                                "clocks": sampler.summary(wall0, wall1)})
    digest = None
    if rank == 0:
        d = last["d"]
        digest = d.cpu().numpy().view(np.uint64).copy() if hasattr(d, "cpu") else d
    check = None
    if rank == 0 and not args.no_check:
        from oracle import c as coracle

        host = coracle.splitmix(wl.DATA_SEED, 0, n // 8).view(np.uint8)
        want = coracle.hash_huge(w, host, seed.words_np(0, seed.capacity))
        check = bool(np.array_equal(digest, want))
    if rank == 0:
        ex_desc = {
            "flags": "in-stream: slice kernels store roots/partials into rank 0's memory (CUDA IPC over NVLink) and "
                     "raise per-rank arrival flags; rank 0's merge kernel waits on them; no host sync in the step",
            "p2p": "slice kernels store roots/partials into rank 0's memory (CUDA IPC) + host sync + barrier",
            "nccl": "all_gather of roots/partials",
        }[exchange]
        line = {
            "metric": METRIC, "value": n / (ms / 1e3) / 1e9, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (splitmix stream seed 0; seed array seed 1)",
            "config": {"workload": "cfg5", "desc": cfg["desc"], "n_bytes": n, "variant": w,
                       "sharding": f"one string split at multiples of 8^{plan.level} instances",
                       "slices_instances": list(plan.bounds), "frontier_roots": plan.n_frontier,
                       "l2": "inputs larger than L2 (126 MB); no flush needed",
                       "exchange": ex_desc, "parallelism": f"dp{world} slices + root exchange + merge on rank 0"},
            "roofline": {"bound": "hbm", "achieved": (b1 - b0) / (step_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": (b1 - b0) / (step_ms / 1e3) / 1e9 / peak, "traffic": None,
                         "kernel": "rank 0 step: hash_kernel<16> slice + exchange + merge_kernel",
                         "kernel_ms": step_ms, "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": None,
            "gpu_launches": (2 if exchange != "nccl" else 2) * args.steps,
            "clocks": sampler.summary(wall0, wall1),
            "ranks": ranks,
            "ranks_share_gpu": not distinct,
            "comm": _comm(dist),
            "oracle_check": check,
        }
        if not distinct:
            line["note"] = "ranks share one GPU (multi-rank code path exercised; timings are not a scaling number)"
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def measure_exchange_emulated(hh, torch, n_slices=8, steps=5):
    """Config 5's multi-GPU exchange, emulated on ONE GPU: the n_slices
    slices of the 16 GiB string run one after another on one stream (the
    FlagExchange protocol with every rank in this process: slice kernels that
    raise arrival flags, the merge kernel that waits on them -- already
    raised, since nothing runs concurrently -- and the consumed-flag slot
    hand-back), each launch timed with CUDA events.  On N GPUs the slices run
    concurrently, so a step costs max(slice) + merge; the merge (and the
    flag handling inside it) is the exchange's whole on-device cost."""
    from paper_2104_08865_b200 import multi_gpu

    cfg = wl.CONFIGS["cfg5"]
    w, n = cfg["variant"], cfg["n_bytes"]
    p = hh.variant(w)
    plan = multi_gpu.slice_plan(p, n, n_slices)
    buf = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    hh.fill_bytes(n, wl.DATA_SEED, 0, out=buf)
    seed = hh.seed_for_input(wl.MASTER, p, n)
    seed.device_words()
    stream = torch.cuda.current_stream()
    state, marks, epoch = None, [], 0

    def mark(tag):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        marks.append((tag, e))

    for it in range(steps + 2):
        epoch += 1
        if it == 2:
            marks.clear()
        d, state = multi_gpu.hash_string_emulated(buf, plan, seed, epoch, state, mark=mark)
    torch.cuda.synchronize()
    slices, merges = [], []
    for (ta, a), (tb, b) in zip(marks, marks[1:]):
        if ta.startswith("slice"):
            slices.append(a.elapsed_time(b))
        elif ta == "merge" and tb == "end":
            merges.append(a.elapsed_time(b))
    digest = d.cpu().numpy().view(np.uint64).copy()
    status = int(state["status"].item())
    from oracle import c as coracle

    host = coracle.splitmix(wl.DATA_SEED, 0, n // 8).view(np.uint8)
    want = coracle.hash_huge(w, host, seed.words_np(0, seed.capacity))
    per_step = np.array(slices).reshape(steps, n_slices)
    slice_max = float(per_step.max(axis=1).mean())
    merge = float(statistics.mean(merges))
    del buf
    torch.cuda.empty_cache()
    return {"desc": f"config 5 split into {n_slices} slices (the {n_slices}-GPU plan) on one GPU, sequentially",
            "frontier_level": plan.level, "frontier_roots": plan.n_frontier,
            "slice_ms_mean": float(per_step.mean()), "slice_ms_max": slice_max,
            "merge_ms": merge, "projected_step_ms": slice_max + merge,
            "exchange_frac_of_step": merge / (slice_max + merge),
            "projected_gbs": n / ((slice_max + merge) / 1e3) / 1e9,
            "digest_matches_oracle": bool(np.array_equal(digest, want)), "wait_status": status,
            "note": "exchange = merge kernel incl. its flag waits and slot hand-back; the slices' flag stores are "
                    "inside the slice kernels' times"}


def measure_sustained(hh, torch, workload, steps, local_rank):
    """The headline kernel over a long run (board power cap reached)."""
    ctx = setup_fixed(hh, torch, workload)
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.2)
    total_ms, per, (w0, w1) = run_fixed(hh, torch, ctx, steps, 5)
    time.sleep(0.1)
    sampler.stop()
    ms = total_ms / steps
    res = {"steps": steps, "value": ctx["B"] * ctx["n"] / (ms / 1e3) / 1e9, "ms_per_step": ms,
           "clocks": sampler.summary(w0, w1)}
    del ctx
    torch.cuda.empty_cache()
    return res


def arm_ours(args, rank, world, local_rank):
    import torch

    import paper_2104_08865_b200 as hh

    local_rank %= max(torch.cuda.device_count(), 1)  # HTH_BENCH_BACKEND=gloo runs share one GPU
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # HTH_BENCH_BACKEND=gloo: exercise the multi-rank code path with several
        # ranks on one GPU (no kernel waits on another rank; timing not meaningful)
        backend = os.environ.get("HTH_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    if args.workload == "cfg5" and world > 1:
        return arm_split(args, rank, world, local_rank, hh, torch, dist)
    peak, peak_src = _peaks()
    workload = args.workload
    dev_name = torch.cuda.get_device_name(local_rank)
    sampler = ClockSampler(local_rank)
    check = None
    if workload == "cfg2":
        # every rank hashes its own replica of the varlen batch (strings of
        # config 2 are not sharded by BASELINE; N > 1 = N independent replicas)
        sampler.start()
        time.sleep(0.3)
        w0 = time.time()
        r2 = measure_workload(hh, torch, "cfg2", args.steps, args.warmup, peak, barrier=dist.barrier if dist else None)
        w1 = time.time()
        time.sleep(0.2)
        sampler.stop()
        B, n, k = 16384, r2["bytes_per_step"], 0
        total_ms = r2["ms_per_step"] * args.steps
        kernel_ms = r2["ms_per_step"]
        algo = r2["bytes_per_step"] + 4 * 16384 * 28 * 8 // 7  # input bytes of 4 variants + their digests
        check = r2.get("graph_matches_serial")
        value_bytes = r2["bytes_per_step"]
    else:
        ctx = setup_fixed(hh, torch, workload, rank, world)
        k = ctx["p"].output_words
        sampler.start()
        time.sleep(0.3)
        # warm-up, then barrier + synchronize on both sides of exactly K timed steps
        small = ctx["B"] * ctx["n"] < (256 << 20)  # L2-sized input (config 1): flush L2 before every step
        total_ms, per, (w0, w1) = run_fixed(hh, torch, ctx, args.steps, args.warmup,
                                            flush=make_flush(torch) if small else None,
                                            barrier=dist.barrier if dist else None)
        time.sleep(0.2)
        sampler.stop()
        kernel_ms = statistics.mean(per)  # one kernel launch per step, events on its stream
        B, n = ctx["B"], ctx["n"]
        value_bytes = B * n
        algo = _algo_bytes(workload, B, n, k)
        # digests stay sharded; rank 0 checks a sample of its digests against the oracle
        if rank == 0 and not args.no_check:
            from oracle import c as coracle

            nchk = min(4, B)
            got = ctx["out"][:nchk].cpu().numpy().view(np.uint64)
            host = _stream_strings([rank + i * world for i in range(nchk)], n)
            S = ctx["seed"].words_np(0, ctx["seed"].capacity)
            want = coracle.hash_fixed(ctx["w"], host, nchk, n, n, S)
            check = bool(np.array_equal(got, want))
        del ctx
        torch.cuda.empty_cache()
    clocks = sampler.summary(w0, w1)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    value = world * value_bytes / (ms / 1e3) / 1e9
    achieved = algo / (kernel_ms / 1e3) / 1e9
    uuid = str(getattr(torch.cuda.get_device_properties(local_rank), "uuid", local_rank))
    ranks = _rank_report(dist, {"rank": rank, "device": dev_name, "uuid": uuid, "local_rank": local_rank,
                                "busy_ms_per_step": total_ms / args.steps, "kernel_ms": kernel_ms,
                                "clocks": clocks})
    shared = len({r["uuid"] for r in ranks}) < len(ranks)
    e2e = None
    if args.e2e_steps > 0 and workload != "cfg2":
        try:
            # N > 1: 2 GiB per rank (the e2e figure is a rate; 8 ranks x 8 GiB of
            # pinned host memory is more than a box need offer)
            e2e_cap = args.e2e_strings or (2048 if world > 1 and workload == "cfg4" else 0)
            e2e, e2e_out = e2e_fixed(hh, torch, workload, args.e2e_steps, e2e_cap, rank, world, local_rank, dist)
            if rank == 0 and not args.no_check:  # the host-path digests of 4 strings against the oracle
                from oracle import c as coracle

                cfg = wl.CONFIGS[workload]
                n_ = cfg["n_bytes"]
                # rank 0's strings: global i (capped batch) or i * world (round-robin shard)
                nchk = min(4, len(e2e_out))
                gidx = [i if e2e_cap else i * world for i in range(nchk)]
                host = _stream_strings(gidx, n_)
                seed_ = hh.seed_for_input(wl.MASTER, hh.variant(cfg["variant"]), n_)
                want = coracle.hash_fixed(cfg["variant"], host, nchk, n_, n_, seed_.words_np(0, seed_.capacity))
                e2e["oracle_check"] = bool(np.array_equal(np.asarray(e2e_out)[:nchk].view(np.uint64), want))
        except Exception as ex:  # pragma: no cover - report, do not hide
            e2e = {"value": None, "unit": UNIT, "error": repr(ex), "h2d_bytes_per_step": None,
                   "d2h_bytes_per_step": None}
    extra = {}
    cpu = None
    if rank == 0 and world == 1:
        if not args.no_extra:
            for wk in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "probe_tail1296"):
                if wk == workload:
                    continue
                try:
                    extra[wk] = measure_workload(hh, torch, wk, steps=max(5, min(args.steps, 50)), warmup=3,
                                                 peak=peak)
                except Exception as ex:  # pragma: no cover
                    extra[wk] = {"error": repr(ex)}
            for name, fn in (("cfg5_exchange_8gpu_emulated", lambda: measure_exchange_emulated(hh, torch)),
                             ("latency", lambda: measure_latency(hh))):
                try:
                    extra[name] = fn()
                except Exception as ex:  # pragma: no cover
                    extra[name] = {"error": repr(ex)}
            if workload != "cfg2":
                try:
                    extra["sustained"] = measure_sustained(hh, torch, workload, args.sustained_steps, local_rank)
                except Exception as ex:  # pragma: no cover
                    extra["sustained"] = {"error": repr(ex)}
        cores = os.cpu_count() or 1
        # the reference arm's granularity (small batches per pass), median of
        # several passes over fresh strings
        cb = CpuBaseline(workload, CPU_PER_CORE.get(workload, 4), cores)
        cb.rate()
        runs = [cb.rate() for _ in range(3 if workload == "cfg2" else 8)]
        cb.close()
        r = statistics.median(x[0] for x in runs)
        # the same algorithm in one process (single process and all cores)
        r1 = None
        if workload != "cfg2":
            c1 = CpuBaseline(workload, CPU_PER_CORE.get(workload, 4), 1)
            c1.rate()
            r1 = statistics.median(c1.rate()[0] for _ in range(3))
            c1.close()
        cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": cb.kind,
               "sample": cb.sample() + f"; median of {len(runs)} passes, {sum(x[2] for x in runs):.2f} s",
               "single_core_value": r1, "cpu_model": _cpu_model()}
    if rank == 0:
        cfg = wl.CONFIGS[workload]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (splitmix stream seed 0; seed array seed 1)",
            "config": {"workload": workload, "desc": cfg["desc"], "n_strings_per_gpu": B,
                       "n_bytes": n if workload != "cfg2" else "varlen", "variant": cfg["variant"],
                       "sharding": ("replica per GPU" if workload == "cfg2" else "round-robin by string"),
                       "l2": ("flushed (256 MB write) before every timed step"
                              if workload in ("cfg1", "cfg2") else "inputs larger than L2 (126 MB); no flush needed"),
                       "parallelism": f"dp{world} (independent strings, no collective)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(workload),
                         "kernel": KERNELS[workload], "kernel_ms": kernel_ms,
                         "algorithmic_bytes_per_launch": algo, "peak_source": peak_src,
                         "imad": _imad_bound(workload, achieved), "read_peak": _read_peak(achieved)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * (8 if workload == "cfg2" else 1),
            "clocks": clocks,
            "ranks": ranks,
            "ranks_share_gpu": shared,
            "comm": _comm(dist),
            "oracle_check": check,
            "workloads": extra,
        }
        if shared:
            line["note"] = "ranks share one GPU (multi-rank code path exercised; timings are not a scaling number)"
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def ctx_variant(workload):
    return wl.CONFIGS[workload]["variant"]


def _free_port():
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args):
    """--gpus N > 1 outside torchrun: run this script as N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary configs")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-strings", type=int, default=0, help="cap e2e batch (0 = full config)")
    ap.add_argument("--sustained-steps", type=int, default=300, help="long run of the headline kernel (N=1)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "flags", "p2p", "nccl"],
                    help="cfg5 on N > 1 GPUs: how the subtree roots reach rank 0 (auto: flags if one GPU per rank)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        return self_launch(args)
    world = int(env_world or 1)
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; launch {args.gpus} ranks "
              f"(or run without torchrun and let bench.py launch them)", file=sys.stderr, flush=True)
        return 2
    rank = int(os.environ.get("RANK", 0))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return arm_reference(args, rank, world)
    return arm_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
