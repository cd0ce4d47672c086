// HalftimeHash B200 engine: device-side building blocks.
//
// One kernel hashes a batch of strings.  Work is cut into warp JOBS: job
// (s, jq) covers instances [8^L jq, 8^L (jq + 1)) of string s, L = job_lvl
// (2 or 3): one level-L subtree of the reference's stack construction
// (tree.py:63-100).  The string's last job also covers its Toeplitz tail
// (hasher.py:407-412).
//
// Per warp: a ring of NS shared-memory stages fed by cp.async.bulk (TMA 1-D
// bulk copies completing on an mbarrier).  A stage holds one ROUND = 8
// instances = one level-1 group (plus the tail in the string's last round).
// Thread (q, j) of the warp (q = lane / 8, j = lane % 8) owns lane j of
// instances 8c + q and 8c + q + 4:
//   encode (GF(16) Cauchy / XOR parity, ehc.py:23-46) -> NH (ehc.py:49-72)
//   -> combine (ehc.py:75-99), all in registers.  For the Cauchy variants
// the two instances are packed plane-by-plane into shared 32-bit registers
// so every XOR of the encode advances 32 GF(16) elements.
// Level-1 nodes (nh.py:96-121) are reduced over the 4 threads sharing j
// with two shuffles and parked in shared memory; every 8th round the whole
// warp forms the level-2 node from the 8 parked blocks the same way; a
// level-3 node (job_lvl 3) accumulates in shared memory; levels >= job_lvl
// use a "last arriver" merge through a global scratch area.
//
// The reference's finalize (tree.py:103-134) is a plain sum of NH terms
// over leftover slots, zero slots and the length tag; the tail is a sum of
// NH terms too.  Every block that ends up a leftover therefore adds its
// finalize terms into the digest accumulator the moment it is produced;
// integer sums mod 2^64 are order-independent, so the result is bit-exact
// and deterministic however the warps interleave.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "encode_gen.cuh"
#include "variants.cuh"

namespace hth {

typedef uint64_t u64;
typedef uint32_t u32;

constexpr int ROUND_INST = 8;  // instances per stage: one level-1 group
constexpr int MAX_EW = 30;     // max e*w over the variants (v32: 10 * 3)

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(u64* bar, u32 phase) {
  u32 ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// 1-D bulk async copy global -> shared, completion counted on `bar`
// (SASS: UBLKCP).  dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar, u64 policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ u64 policy_evict_first() {
  u64 p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------ arithmetic
struct w2 {
  u32 lo, hi;
};
__device__ __forceinline__ w2 mk(u64 x) { return {(u32)x, (u32)(x >> 32)}; }
__device__ __forceinline__ w2 operator^(w2 a, w2 b) { return {a.lo ^ b.lo, a.hi ^ b.hi}; }

// NH(x, s) = ((x_lo + s_lo) mod 2^32) * ((x_hi + s_hi) mod 2^32)  (nh.py:48-67)
// acc + (u64)a*b lowers to one IMAD.WIDE.U32.
__device__ __forceinline__ u64 nh_acc(u64 acc, w2 x, u32 slo, u32 shi) { return acc + (u64)(x.lo + slo) * (x.hi + shi); }
__device__ __forceinline__ u64 nh_acc(u64 acc, w2 x, u64 s) { return nh_acc(acc, x, (u32)s, (u32)(s >> 32)); }
__device__ __forceinline__ u64 nh_acc(u64 acc, u64 x, u64 s) { return nh_acc(acc, mk(x), s); }

// acc += C * h (mod 2^64) for a small constant C.  Written as plain C++ so
// ptxas picks LEA + LEA.HI.X for powers of two and IMAD.WIDE.U32 (with the
// accumulator) + IMAD + IADD3 otherwise; an inline-PTX mad.wide/mad.lo pair
// was split by ptxas into four instructions per term.
template <int C>
__device__ __forceinline__ u64 mac_const(u64 acc, u64 h) {
  return acc + h * (u64)C;
}

// Arrival on a merge/completion counter: release publishes this warp's
// prior stores (ordered before lane 0 by __syncwarp), acquire makes the
// other warps' blocks visible to a last arriver.  Lowers to MEMBAR.ALL.GPU
// + ATOMG + CCTL.IVALL, cheaper than __threadfence()'s MEMBAR.SC.
__device__ __forceinline__ u32 atom_add_acq_rel(u32* p, u32 v) {
  u32 old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// System-scope release store / acquire load of a 64-bit flag (peer GPUs
// over NVLink read and write these).
__device__ __forceinline__ void st_release_sys(unsigned long long* p, u64 v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire_sys(const unsigned long long* p) {
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 global_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until *p >= v, or give up after timeout_ns (returns false): a wait on
// another GPU must never hang this one.
__device__ __forceinline__ bool wait_geq_sys(const unsigned long long* p, u64 v, u64 timeout_ns) {
  if (ld_acquire_sys(p) >= v) return true;
  const u64 t0 = global_ns();
  for (;;) {
    __nanosleep(128);
    if (ld_acquire_sys(p) >= v) return true;
    if (global_ns() - t0 > timeout_ns) return false;
  }
}

template <class T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// Sum v[0..K) over the 16 lanes of each half-warp; afterwards lane g holds
// the total of word (g & (KP-1)) for g < KP (KP = K rounded up to 2^n).
template <int K>
__device__ __forceinline__ u64 half_reduce_scatter(u64 (&v)[K], int g) {
  constexpr int KP = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
  u64 a[KP];
#pragma unroll
  for (int r = 0; r < KP; r++) a[r] = r < K ? v[r] : 0;
  // step with mask 8 (and 4 when KP == 8): halve the live words per lane
  int live = KP;
#pragma unroll
  for (int m = 8; m >= 1; m >>= 1) {
    if (live > 1) {
      const int half = live / 2;
      const bool upper = (g & m) != 0;  // keep upper half of the live words
#pragma unroll
      for (int r = 0; r < KP / 2; r++) {
        if (r < half) {
          const u64 send = upper ? a[r] : a[r + half];
          const u64 keep = upper ? a[r + half] : a[r];
          a[r] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
      }
      live = half;
    } else {
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], m);
    }
  }
  return a[0];
}

// lane g ends with the word index it holds after half_reduce_scatter
template <int K>
__device__ __forceinline__ int scatter_index(int g) {
  constexpr int KP = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
  int idx = 0, live = KP;
  for (int m = 8; m >= 1 && live > 1; m >>= 1) {
    const int half = live / 2;
    if (g & m) idx += half;
    live = half;
  }
  return idx;
}

// Sum NP values over all 32 lanes, scattered: afterwards every lane holds
// the total of value warp_scatter_index<NP>(lane) (lanes differing only in
// bits below 32 / NP hold the same one).  5 + NP - 2 shuffle rounds instead
// of 5 per value.
template <int NP>
__device__ __forceinline__ u64 warp_reduce_scatter(u64 (&a)[NP], int lane) {
  int live = NP;
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    if (live > 1) {
      const int half = live / 2;
      const bool upper = (lane & m) != 0;
#pragma unroll
      for (int r = 0; r < NP / 2; r++) {
        if (r < half) {
          const u64 send = upper ? a[r] : a[r + half];
          const u64 keep = upper ? a[r + half] : a[r];
          a[r] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
      }
      live = half;
    } else {
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], m);
    }
  }
  return a[0];
}
template <int NP>
__device__ __forceinline__ int warp_scatter_index(int lane) {
  int idx = 0, live = NP;
#pragma unroll
  for (int m = 16; m >= 1 && live > 1; m >>= 1) {
    const int half = live / 2;
    if (lane & m) idx += half;
    live = half;
  }
  return idx;
}

// Little-endian u64 word t of the string at byte `o0` of `data` (n bytes),
// straight from global memory at any alignment, the partial last word
// zero-padded (hasher.py:179-183); never reads past the string's last byte's
// aligned word.
__device__ __forceinline__ u64 gword(const uint8_t* data, u64 o0, u64 n, u64 t) {
  const u64 b = reinterpret_cast<u64>(data) + o0 + 8ull * t;
  const u64* p = reinterpret_cast<const u64*>(b & ~7ull);
  const u32 sh = (u32)(b & 7) * 8;
  const u64 rem = n - 8ull * t;
  u64 x = __ldg(p) >> sh;
  if (sh && rem > 8 - (b & 7)) x |= __ldg(p + 1) << (64 - sh);
  if (rem < 8) x &= (1ull << (8 * rem)) - 1;
  return x;
}

// splitmix seed word idx of a stream keyed by `fold` (hasher.py:55-58)
__host__ __device__ __forceinline__ u64 splitmix_word(u64 fold, u64 idx) {
  u64 z = fold + (idx + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Seed words of a job: the shared expanded array (one SeedBuffer for the
// batch), or -- PERSEED, the many-seeds seam of tests/test_hasher.py:254-310
// -- recomputed from the string's own fold.
template <bool PERSEED>
struct SeedSrc {
  const u64* S;
  u64 fold;
  __device__ __forceinline__ u64 operator()(u64 idx) const {
    if (PERSEED) return splitmix_word(fold, idx);
    return __ldg(S + idx);
  }
};

// ------------------------------------------------------------ per-string view
struct Str {
  const uint8_t* p;  // first byte (global)
  u64 n;             // bytes
  u64 n_inst;        // full instances
  u32 L;             // layout levels (>= 1)
  u32 J;             // warp jobs
  u64 scratch;       // base word of this string's scratch blocks
  u64 cnt;           // base index of this string's counters
  u64 s;             // string index
  u64 fold;          // PERSEED: this string's seed fold
};

// levels = 1 + floor(log8 n) for n >= 1 (tree.py:34-42)
__host__ __device__ __forceinline__ u32 level_count(u64 n) {
#ifdef __CUDA_ARCH__
  return 1 + (u32)(63 - __clzll((long long)(n | 1))) / 3;
#else
  u32 l = 1;
  while (n >= 8) {
    n >>= 3;
    l++;
  }
  return l;
#endif
}
__host__ __device__ __forceinline__ u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }

// jobs of a string: one per 8^job_lvl instances (at least one)
__host__ __device__ __forceinline__ u64 job_count(u64 n_inst, int job_lvl) {
  const u64 per = 1ull << (3 * job_lvl);
  return n_inst > per ? (n_inst + per - 1) >> (3 * job_lvl) : 1;  // per is a power of 8
}

// scratch words / counters a string needs for merges above the job level
// (levels below `upto` only: a slice whose subtree roots stop at frontier
// level c never merges at or above c)
__host__ __device__ __forceinline__ void scratch_need(u64 n_inst, int k, int job_lvl, u64* words, u64* cnts,
                                                     int upto = 64) {
  u64 w = 0, c = 0;
  for (int l = job_lvl; l < upto && (n_inst >> (3 * l)) >= 8; l++) {
    const u64 len = n_inst >> (3 * l);
    w += (len & ~7ull) * 8ull * k;
    c += len >> 3;
  }
  *words = w;
  *cnts = c;
}

// Completion events of a multi-job string: its last job, plus one per block
// at level >= job_lvl that ends as a leftover (each such block's producer
// is the last warp to touch anything beneath it).  When all have arrived,
// every finalize term is in the accumulator.
__host__ __device__ __forceinline__ u32 string_events(u64 n_inst, int job_lvl) {
  u32 e = 1;
  for (int l = job_lvl; (n_inst >> (3 * l)) > 0; l++) e += (u32)((n_inst >> (3 * l)) & 7);
  return e;
}

// Varlen jobs are bucketed by size class c = min(instances, 64) into queues
// of fixed capacity: a class-c job holds >= c instances, so at most
// q_inst / c of them exist.  Claim order is largest class first (LPT).
// Classes 1..PAIR_MAX hold single-job strings only (one level, c
// instances): the hash kernel takes them two per round.  A multi-job
// string's last job of <= PAIR_MAX instances goes to class PAIR_MAX + 1
// (at most one per 64 instances of the batch).
constexpr int NCLS = 65;
#ifndef HTH_PAIR_MAX
#define HTH_PAIR_MAX 4
#endif
constexpr int PAIR_MAX = HTH_PAIR_MAX;  // 0: no pair jobs (experiments)
static_assert(PAIR_MAX >= 0 && PAIR_MAX <= 4, "a pair's instances must fit one stage");
__host__ __device__ __forceinline__ u64 queue_cap(int c, u64 max_jobs, u64 q_inst) {
  if (c == 0) return 0;
  return min(max_jobs, q_inst / (u64)c + 1 + (c == PAIR_MAX + 1 ? q_inst / 64 + 1 : 0));
}

// Zero-slot finalize sums (tree.py:103-134): for a layout with L levels,
// level l and digit d = (n_inst >> 3l) & 7 the empty slots d..6 contribute
//   Z[L][l][d][r] = sum_{slot=d..6} sum_j NH(0, S[F_r(L) + 56 l + 8 slot + j]),
// stored for L = 1..lmax at ztab_base(L) + (l * 8 + d) * K + r.
__host__ __device__ __forceinline__ u64 ztab_base(u32 L, int K) { return 4ull * K * L * (L - 1); }

struct Params {
  const uint8_t* data;
  u64 n_strings;
  u64 stride;    // fixed mode
  u64 n_bytes;   // fixed mode: length; varlen: length clamp (host-checked bound)
  u64 J_fixed;   // fixed mode: jobs per string
  u64 n_inst_fixed;  // fixed mode: instances per string
  u32 L_fixed;       // fixed mode: layout levels per string
  u64 n_jobs;    // fixed mode: total jobs
  u64 scr_per;   // fixed mode: scratch words per string
  u64 cnt_per;   // fixed mode: counters per string
  const u64* offsets;  // varlen: n_strings + 1 byte offsets
  const u64* job_map;  // varlen: per-size-class job queues; each job a JOB_REC-word record
                       // {byte offset, length, string | job index << 32, merge bases} (plan_kernel)
  u32* cls_cnt;        // varlen: jobs per size class (plan_kernel; reset at exit)
  unsigned long long* totals;  // varlen: the plan's scratch/counter allocators (reset at exit)
  u64 var_total;       // varlen: data bytes (offset bound)
  const u64* ztab;     // varlen: zero-slot finalize sums per (levels, level, digit, row)
  u32 ztab_lmax;       // varlen: levels covered by ztab
  const u64* S;        // expanded seed words (SeedBuffer.words_np)
  const u64* folds;    // PERSEED: per-string seed folds
  u64* out;
  u64* scratch;   // level >= job_lvl blocks awaiting their group's merge
  u32* counters;  // per-group arrival counts (self-resetting)
  u64* acc;       // per multi-job string: k partial digest words (self-resetting)
  u32* events;    // per multi-job string: completion events seen (self-resetting)
  unsigned long long* job_ctr;  // dynamic job claiming (self-resetting)
  u32* exit_ctr;                 // warps finished (self-resetting)
  // fixed-length batches: the zero-slot and length-tag finalize terms
  // (tree.py:103-134) depend only on (n, seed), so the host sums them once
  int fin_const_ok;
  u64 fin_const[5];
  int job_lvl;    // a warp job is one level-`job_lvl` subtree
  // slice mode (one string split across GPUs, fixed mode with n_strings = 1):
  // jobs cover global instances [slice_inst0, ...); finished non-leftover
  // blocks at frontier_lvl go to `frontier` (index - frontier_base) instead
  // of merging further, and every finalize term accumulates into acc[0..k)
  // (no digest is written; hth_hash_merge completes it).
  int frontier_lvl;  // 0 = off
  u64 slice_job0;    // global jq of the slice's first job
  u64 frontier_base;
  u64* frontier;
  // slice mode, in-stream exchange: the last warp out stores done_value to
  // *done_flag (system-scope release; the flag may live on another GPU)
  // after every warp's frontier/partial stores are visible system-wide
  unsigned long long* done_flag;
  u64 done_value;
#ifdef HTH_DEBUG_TIMING
  unsigned long long* dbg;  // experiment builds: per-warp timing records (hth_debug_timing)
#endif
  // EHC seed words S[0..e*w), split into halves.  The kernel takes Params as
  // a __grid_constant__, so these are constant-bank operands of the NH adds.
  // Interleaved (lo, hi), word i at slot ehc_slot(i): the leaf's block-u pass
  // reads its e words from consecutive slots (16-byte constant loads).
  alignas(16) u32 ehc[2 * MAX_EW];
  // varlen: start of each size class's queue in job_map (host-computed; [NCLS] = end)
  u64 cls_qb[NCLS + 1];
};

// slot of EHC seed word idx = item * w + u in Params::ehc: u-major
__host__ __device__ constexpr int ehc_slot(int idx, int e, int w) { return (idx % w) * e + idx / w; }

template <int K>
__device__ __forceinline__ void layout_bases(u32 L, int ew, u64 (&T)[K], u64 (&F)[K], u64& R) {
#pragma unroll
  for (int r = 0; r < K; r++) {
    T[r] = (u64)ew + 7ull * L * r;
    F[r] = (u64)ew + 7ull * L * K + 64ull * L * r;
  }
  R = (u64)ew + 71ull * L * K;
}

constexpr int JOB_REC = 4;  // u64 words per varlen job record

// VARLEN: `rec` is the job's record (queue entry), resolved at claim time;
// fixed mode: `job` is the job index
template <bool VARLEN, int K, int M>
__device__ __forceinline__ void decode_job(const Params& P, u64 job, const u64* rec, Str& st, u32& jq) {
  u64 s;
  if (VARLEN) {
    s = rec[2] & 0xffffffffull;
    st.p = P.data + rec[0];
    st.n = rec[1];  // clamped to the host-checked bound by plan_kernel
    jq = (u32)(rec[2] >> 32);
  } else {
    // jq-major order: all strings' first jobs, then all second jobs, ...
    // Jobs of one jq have equal size, so static round-robin stays balanced.
    jq = (u32)(job / P.n_strings);
    s = job - (u64)jq * P.n_strings;
    st.p = P.data + s * P.stride;
    st.n = P.n_bytes;
    st.scratch = s * P.scr_per;
    st.cnt = s * P.cnt_per;
  }
  st.s = s;
  st.fold = P.folds ? P.folds[s] : 0;
  if (!VARLEN && P.frontier_lvl) {  // slice mode: P.n_bytes is the whole string
    jq += (u32)P.slice_job0;
  }
  if (VARLEN) {
    st.n_inst = ((st.n + 7) >> 3) / M;
    st.L = st.n_inst ? level_count(st.n_inst) : 1;
    st.J = (u32)job_count(st.n_inst, P.job_lvl);
  } else {  // launch constants (kept out of the per-round producer path)
    st.n_inst = P.n_inst_fixed;
    st.L = P.L_fixed;
    st.J = (u32)P.J_fixed;
  }
  if (VARLEN) {  // merge scratch and counters (multi-job strings): packed in the record
    st.scratch = rec[3] & ((1ull << 40) - 1);
    st.cnt = rec[3] >> 40;
  }
}

// bytes of job jq (its instances, plus the tail for the last job)
template <int M>
__device__ __forceinline__ void job_span(const Str& st, u32 jq, int job_lvl, u64& byte0, u64& nbytes, u32& ninst) {
  const u64 per = 1ull << (3 * job_lvl);
  const u64 i0 = (u64)jq * per;
  const u64 ni = st.n_inst > i0 ? min(per, st.n_inst - i0) : 0;
  ninst = (u32)ni;
  byte0 = i0 * (M * 8ull);
  nbytes = (jq + 1 == st.J) ? st.n - byte0 : ni * (M * 8ull);
}

}  // namespace hth
