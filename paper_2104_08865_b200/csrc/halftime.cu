// libhalftime_b200.so: C-ABI of the B200-native HalftimeHash engine.
// Declarations and error conventions: include/halftime_b200.h.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <omp.h>
#include <tuple>
#include <string>
#include <vector>


#include "../../include/halftime_b200.h"
#include "engine_api.cuh"

using namespace hth;

namespace {

// runtime helpers shared with the per-variant kernel units (rt.cuh)
}  // namespace
namespace hth {
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? HTH_ENOMEM : HTH_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}
int sm_count(int dev) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> g(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1, 0);
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev];
}

// Resident CTAs per SM of `kern` at (tpb, smem) on the current device; the
// dynamic shared-memory limit is raised once per (kernel, device, smem) and
// the answer cached, keeping the per-call host path to the launch itself.
int occupancy(const void* kern, int tpb, size_t smem, int* dev_out, int* occ_out) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  static std::map<std::pair<const void*, int>, size_t> limit;  // the attribute is per kernel: only raise it
  int dev = 0;
  CK(cudaGetDevice(&dev));
  *dev_out = dev;
  const auto key = std::make_tuple(kern, dev, smem, tpb);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *occ_out = it->second;
    return HTH_OK;
  }
  size_t& lim = limit[std::make_pair(kern, dev)];
  if (smem > lim) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    lim = smem;
  }
  int o = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, tpb, smem));
  cache[key] = *occ_out = std::max(o, 1);
  return HTH_OK;
}

}  // namespace hth
namespace {
u64 align_up(u64 x, u64 a) { return (x + a - 1) / a * a; }

struct Layout {
  u64 n_inst, levels, ew, tree_start, tree_per, fin_start, fin_per, rem_start, rem_words, total;
};
// seed_layout (hasher.py:126-153)
Layout make_layout(const VarInfo& v, u64 n_bytes) {
  Layout l;
  l.n_inst = ((n_bytes + 7) / 8) / (u64)v.m;
  l.levels = l.n_inst ? level_count(l.n_inst) : 1;
  l.ew = (u64)v.ew;
  l.tree_start = l.ew;
  l.tree_per = 7 * l.levels;
  l.fin_start = l.tree_start + l.tree_per * v.k;
  l.fin_per = 64 * l.levels;
  l.rem_start = l.fin_start + l.fin_per * v.k;
  l.rem_words = (u64)v.m + v.k - 1;
  l.total = l.rem_start + l.rem_words;
  return l;
}

int get_var(int out, VarInfo* v) {
  if (!var_info(out, v)) return fail(HTH_EINVAL, "unsupported output width %d; choose one of 16, 24, 32, 40", out);
  return HTH_OK;
}

// EHC seed words S[0..e*w) = mix(fold + (i+1) gamma) (hasher.py:55-58),
// passed to the kernel in its constant-bank parameters
u64 host_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
void fill_ehc(const VarInfo& v, u64 fold, Params& P) {
  for (int i = 0; i < v.ew; i++) {
    const u64 w = host_mix(fold + (u64)(i + 1) * 0x9E3779B97F4A7C15ull);
    const int slot = ehc_slot(i, v.e, v.w);
    P.ehc[2 * slot] = (u32)w;
    P.ehc[2 * slot + 1] = (u32)(w >> 32);
  }
}

#ifdef HTH_DEBUG_TIMING
unsigned long long* dbg_buf() {
  static unsigned long long* d = nullptr;
  if (!d && cudaMalloc(&d, 8192 * 12 * 8) == cudaSuccess) cudaMemset(d, 0, 8192 * 12 * 8);
  return d;
}
#endif

// dynamic job-claim counter and exit counter (zero-filled, self-resetting)
void set_ctl(Params& P, uint8_t* ctl) {
  P.job_ctr = reinterpret_cast<unsigned long long*>(ctl);
  P.exit_ctr = reinterpret_cast<u32*>(ctl + 8);
#ifdef HTH_DEBUG_TIMING
  P.dbg = dbg_buf();
#endif
}

// Zero-slot + length-tag finalize terms of one string length, summed on the
// host (tree.py:103-134, hasher.py:387-405): identical for every string of a
// fixed-length batch, so the kernel just adds them.
void fill_fin_const(const VarInfo& v, u64 fold, u64 n_bytes, Params& P) {
  const Layout l = make_layout(v, n_bytes);
  auto nh = [](u64 x, u64 s) { return (u64)((u32)x + (u32)s) * (u64)((u32)(x >> 32) + (u32)(s >> 32)); };
  auto S = [&](u64 i) { return host_mix(fold + (i + 1) * 0x9E3779B97F4A7C15ull); };
  for (int r = 0; r < v.k; r++) {
    const u64 F = l.fin_start + l.fin_per * r;
    u64 acc = 0;
    if (l.n_inst) {
      for (u64 lv = 0; lv < l.levels; lv++) {
        const u64 digit = (l.n_inst >> (3 * lv)) & 7;
        for (u64 slot = digit; slot < 7; slot++)
          for (u64 j = 0; j < 8; j++) acc += nh(0, S(F + 56 * lv + 8 * slot + j));
      }
      acc += nh(n_bytes, S(F + 56 * l.levels));
    } else {
      acc += nh(n_bytes, S(F));
    }
    P.fin_const[r] = acc;
  }
  P.fin_const_ok = 1;
}

u64 fold_of(const uint8_t* m) {
  u64 w[4];
  memcpy(w, m, 32);
  return w[0] ^ w[1] ^ w[2] ^ w[3];
}

// ------------------------------------------------------------ kernels (aux)
__device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void expand_seed_kernel(u64 fold, u64 start, u64 count, u64* out) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x)
    out[i] = mix64(fold + (start + i + 1) * 0x9E3779B97F4A7C15ull);
}

// hash_remainder (hasher.py:186-206): one CTA per output row r, the block
// sums NH(tail[i], keys[r + i]) over i.
__global__ void toeplitz_nh_kernel(const u64* tail, u64 n, const u64* keys, u64* out) {
  __shared__ u64 part[32];
  const u64 r = blockIdx.x;
  u64 acc = 0;
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) acc = nh_acc(acc, tail[i], keys[r + i]);
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += part[w];
    out[r] = t;
  }
}

// Publish / await one flag in-stream (system scope; see wait_geq_sys).
__global__ void signal_kernel(unsigned long long* flag, u64 value) {
  __threadfence_system();
  st_release_sys(flag, value);
}
__global__ void wait_kernel(const unsigned long long* flag, u64 value, u64 timeout_ns, int* status) {
  if (!wait_geq_sys(flag, value, timeout_ns)) atomicExch(status, 1);
  __threadfence_system();
}

// string i of a local buffer = global string first + i * step of a packed
// stream of `wps`-word strings (round-robin shards in one launch)
__global__ void fill_strings_kernel(u64 seed, u64 wps, u64 first, u64 step, u64 n_words, u64 dst_wstride, u64* dst) {
  for (u64 w = blockIdx.x * (u64)blockDim.x + threadIdx.x; w < n_words; w += (u64)gridDim.x * blockDim.x) {
    const u64 i = w / wps, t = w - i * wps;
    dst[i * dst_wstride + t] = mix64(seed + ((first + i * step) * wps + t + 1) * 0x9E3779B97F4A7C15ull);
  }
}

__global__ void fill_kernel(u64 seed, u64 woff, u64 n_words, u64 n_bytes, u64* dst) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n_words; i += (u64)gridDim.x * blockDim.x) {
    u64 v = mix64(seed + (woff + i + 1) * 0x9E3779B97F4A7C15ull);
    if (i * 8 + 8 > n_bytes) {  // partial last word: write only its bytes
      uint8_t* b = reinterpret_cast<uint8_t*>(dst + i);
      for (u64 t = 0; i * 8 + t < n_bytes; t++) b[t] = (uint8_t)(v >> (8 * t));
    } else {
      dst[i] = v;
    }
  }
}

// small_kernel applies: one level (1..7 instances), aligned strings packed
// closely, and the partial final word (if any) in the tail, not in an instance
bool small_ok(const VarInfo& v, u64 n_inst, u64 stride, u64 n_bytes, const void* data) {
  const u64 nw = (n_bytes + 7) / 8;
  return n_inst >= 1 && n_inst <= 7 && stride % 8 == 0 && (reinterpret_cast<uintptr_t>(data) & 7) == 0 &&
         stride <= n_bytes + 256 && ((n_bytes & 7) == 0 || nw > n_inst * (u64)v.m);
}

// kernel launches live in the per-variant units kv16/24/32/40.cu (launch.cuh)
template <template <int> class F, class... A>
int by_width(int out, A&&... a) {
  switch (out) {
    case 16: return F<16>::run(a...);
    case 24: return F<24>::run(a...);
    case 32: return F<32>::run(a...);
    case 40: return F<40>::run(a...);
  }
  return fail(HTH_EINVAL, "unsupported output width %d", out);
}
template <int OUT> struct HashF { static int run(const Params& P, u64 nj, int kind, cudaStream_t st) { return VarEngine<OUT>::hash(P, nj, kind, st); } };
template <int OUT> struct TailF { static int run(const TailParams& T, u64 nch, cudaStream_t st) { return VarEngine<OUT>::tail(T, nch, st); } };
template <int OUT> struct SmallF { static int run(const Params& P, cudaStream_t st) { return VarEngine<OUT>::small(P, st); } };
template <int OUT> struct PlanF { static int run(const PlanParams& Q, unsigned grid, cudaStream_t st) { return VarEngine<OUT>::plan(Q, grid, st); } };
template <int OUT> struct MergeF { static int run(const MergeParams& M, cudaStream_t st) { return VarEngine<OUT>::merge(M, st); } };
// fixed batches whose strings all start 8-byte aligned get the aligned-only kernel
template <bool VARLEN>
int dispatch(int out, const Params& P, u64 n_jobs_bound, cudaStream_t st) {
  int kind = HK_VARLEN;
  if (!VARLEN) kind = (reinterpret_cast<uintptr_t>(P.data) % 8) == 0 && P.stride % 8 == 0 ? HK_FIXED_AL8 : HK_FIXED;
  return by_width<HashF>(out, P, n_jobs_bound, kind, st);
}
// per-string seeds (many-seeds seam)
int dispatch_ps(int out, const Params& P, u64 n_jobs_bound, cudaStream_t st) {
  return by_width<HashF>(out, P, n_jobs_bound, (int)HK_PS, st);
}

// A failed launch must not leave a half-used workspace behind: its
// self-resetting counters would corrupt every later call.  Re-zero it
// (stream-ordered, best effort) and pass the error on.
int guard_ws(int rc, void* ws, u64 bytes, cudaStream_t st) {
  if (rc != HTH_OK && ws && bytes) {
    const std::string msg = g_err;
    cudaGetLastError();
    cudaMemsetAsync(ws, 0, bytes, st);
    g_err = msg;
  }
  return rc;
}

// Varlen workspaces: the hash kernel leaves its counters, accumulators and
// the plan's class counts zeroed, so a workspace reused with the same layout
// needs no clearing; a layout change (another batch shape) may leave an
// earlier call's T list / job records where this call's counters live, so
// the counter region is cleared once, on the first call with each layout.
struct WsSig {
  u64 v[8];
  bool operator==(const WsSig& o) const { return memcmp(v, o.v, sizeof v) == 0; }
};
std::mutex g_ws_mu;
std::map<const void*, WsSig> g_ws_sig;
bool ws_layout_known(const void* ws, const WsSig& sig) {
  std::lock_guard<std::mutex> g(g_ws_mu);
  auto it = g_ws_sig.find(ws);
  if (it != g_ws_sig.end() && it->second == sig) return true;
  g_ws_sig[ws] = sig;
  return false;
}
void ws_forget(const void* ws) {
  std::lock_guard<std::mutex> g(g_ws_mu);
  g_ws_sig.erase(ws);
}

int check_seed(const VarInfo& v, u64 n_bytes, u64 cap) {
  const Layout l = make_layout(v, n_bytes);
  if (cap < l.total)
    return fail(HTH_ESEEDSIZE,
                "seed buffer holds %llu words but this input needs %llu; expand with seed_words_needed()",
                (unsigned long long)cap, (unsigned long long)l.total);
  return HTH_OK;
}

// fixed-mode geometry
// warp job = one level-2 subtree (64 instances), or level-3 (512) for very
// long strings so the per-job merge traffic and fences stay negligible
int pick_job_lvl(u64 max_inst) { return max_inst >= 512 ? 3 : 2; }

struct FixedPlan {
  u64 n_inst, J, n_jobs, scr_per, cnt_per, ws_scratch, ws_acc, ws_cnt, ws_ev, ws_total;
  int job_lvl;
};
// frontier > 0: slice mode, merges stop below that level
// Few long strings (fewer than kLvl3Jobs level-3 jobs in the batch) use
// level-2 jobs instead, so a single 1 MiB string is 18 warps' work, not 3.
constexpr u64 kLvl3Jobs = 4096;
FixedPlan fixed_plan(const VarInfo& v, u64 n_strings, u64 n_bytes, int frontier = 0) {
  FixedPlan f;
  f.n_inst = ((n_bytes + 7) / 8) / (u64)v.m;
  f.job_lvl = pick_job_lvl(f.n_inst);
  if (frontier == 0 && f.job_lvl == 3 && n_strings * job_count(f.n_inst, 3) < kLvl3Jobs) f.job_lvl = 2;
  f.J = job_count(f.n_inst, f.job_lvl);
  f.n_jobs = n_strings * f.J;
  scratch_need(f.n_inst, v.k, f.job_lvl, &f.scr_per, &f.cnt_per, frontier > 0 ? frontier : 64);
  const bool multi = f.J > 1;
  f.ws_scratch = align_up(n_strings * f.scr_per * 8, 256);
  f.ws_acc = multi ? align_up(n_strings * v.k * 8, 256) : 0;
  f.ws_cnt = align_up(n_strings * f.cnt_per * 4, 256);
  f.ws_ev = multi ? align_up(n_strings * 4, 256) : 0;
  f.ws_total = f.ws_scratch + f.ws_acc + f.ws_cnt + f.ws_ev + 256;  // + job/exit counters
  return f;
}

// varlen workspace geometry
struct VarPlan {
  u64 off_err, off_cnt, off_acc, off_ev, off_ctl, off_pctl, off_clear, off_queue, off_scr, total,
      max_jobs, q_inst, scr_words, cnts, off_ztab, lmax;
  QueueTable Q;
};
// Workspace: the error flag (offset 0, hth_varlen_status), the self-resetting
// hash state and the plan counters first (cleared by one memset per call),
// then the per-string bases, class queues, merge scratch and zero-slot table.
int varlen_plan(const VarInfo& v, u64 n, u64 total_bytes, u64 max_n_bytes, VarPlan* p) {
  // a string's instances are ceil(len / 8) / m: a string of 8m-7..8m-1 bytes
  // already holds a full instance, so bound the batch's sum per string
  // rounding (up to 7 padding bytes each), not by total_bytes / 8m
  if (n > (~0ull - total_bytes) / 7) return fail(HTH_EINVAL, "n_strings too large");
  const u64 total_inst = (total_bytes + 7 * n) / (8ull * v.m);
  // no string has more levels than the longest allowed one, nor than the total
  const u64 max_inst = std::min(((max_n_bytes / 8) + 1) / (u64)v.m, total_inst);
  p->lmax = max_inst ? level_count(max_inst) : 1;
  p->max_jobs = n + total_inst / 64 + 1;
  p->q_inst = total_inst;
  p->scr_words = (total_inst / 56 + 1) * 8ull * v.k;
  p->cnts = total_inst / 448 + 1;
  // job records pack the merge bases as scratch word (40 bits) | counter << 40
  if (p->scr_words >= (1ull << 40) || p->cnts >= (1ull << 24)) return fail(HTH_EINVAL, "varlen batch too large");
  u64 qcap = 0;
  for (int c = 0; c < NCLS; c++) {
    p->Q.qb[c] = qcap;
    qcap += queue_cap(c, p->max_jobs, p->q_inst);
  }
  p->Q.qb[NCLS] = qcap;
  u64 o = 0;
  p->off_err = o; o += 256;
  p->off_cnt = o; o = align_up(o + p->cnts * 4, 256);
  p->off_acc = o; o = align_up(o + n * v.k * 8, 256);
  p->off_ev = o; o = align_up(o + n * 4, 256);
  p->off_ctl = o; o += 256;
  p->off_pctl = o; o += 512;  // class counts [NCLS] u32 @0, scratch/counter totals @384
  p->off_clear = o;
  p->off_queue = o; o = align_up(o + qcap * 8 * JOB_REC, 256);
  p->off_scr = o; o = align_up(o + p->scr_words * 8, 256);
  p->off_ztab = o; o = align_up(o + ztab_base(p->lmax + 1, v.k) * 8, 256);
  p->total = o;
  return HTH_OK;
}

// per-thread e2e context (device buffers reused across calls)
// host calls up to this many input bytes (and digest words) take the
// one-stream path through pinned staging: a single-string hash_bytes call is
// then one H2D DMA, one launch, one D2H DMA and one synchronize
constexpr u64 kSmallCall = 256 << 10, kSmallOut = 4096;
// calls up to this many input bytes skip both DMAs: the kernel reads the
// input straight out of mapped pinned host memory (over PCIe) and writes the
// digest words back into it, so a hash_bytes call is one launch and one
// synchronize (HTH_HOST_MAPPED=0 turns this off)
constexpr u64 kMappedCall = 64 << 10;
bool mapped_enabled() {
  static const bool on = [] {
    const char* e = getenv("HTH_HOST_MAPPED");
    return !(e && e[0] == '0');
  }();
  return on;
}
// larger calls move ~kChunk bytes per chunk; strings longer than kChunk are
// streamed through the same bounded buffers in slices (hth_hash_slice), so
// device memory stays at 3 chunks whatever the input size
constexpr u64 kChunk = 64ull << 20;
struct HostCtx {
  int dev = -1;
  cudaStream_t st[3] = {nullptr, nullptr, nullptr};
  void* buf[3] = {nullptr, nullptr, nullptr};  // allocated per slot, on first use
  u64 buf_bytes[3] = {0, 0, 0};
  u64* seeds = nullptr;
  u64 seed_bytes = 0;
  u64* out = nullptr;
  u64 out_bytes = 0;
  void* ws[3] = {nullptr, nullptr, nullptr};  // zero-filled, kept zero by the engine
  u64 ws_bytes[3] = {0, 0, 0};
  // small-call path: pinned staging both ways, and the fold whose first
  // `seeds_valid` words are already expanded in `seeds`
  uint8_t* hin = nullptr;  // pinned and mapped: din / dout are their device addresses
  u64* hout = nullptr;
  uint8_t* din = nullptr;
  u64* dout = nullptr;
  u64 seeds_fold = 0, seeds_valid = 0;
  // pageable sources: two pinned staging slots filled by parallel memcpy
  uint8_t* ring[2] = {nullptr, nullptr};
  cudaEvent_t ring_ev[2] = {nullptr, nullptr};
  cudaEvent_t ev = nullptr;  // cross-stream ordering (created once)
  // sliced long strings: subtree roots, per-slice partials, merge scratch
  u64* frontier = nullptr;
  u64 frontier_bytes = 0;
  u64* partials = nullptr;
  u64 partial_bytes = 0;
  void* mws = nullptr;
  u64 mws_bytes = 0;

  // Frees everything (errors ignored: at process exit the runtime may
  // already be unloading).  Called on device switch, hth_host_release and
  // thread exit.
  void release() {
    if (dev < 0) return;
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    for (int i = 0; i < 3; i++) {
      if (st[i]) cudaStreamSynchronize(st[i]);
    }
    for (int i = 0; i < 3; i++) {
      if (st[i]) cudaStreamDestroy(st[i]);
      if (buf[i]) cudaFree(buf[i]);
      if (ws[i]) cudaFree(ws[i]);
    }
    for (int i = 0; i < 2; i++) {
      if (ring[i]) cudaFreeHost(ring[i]);
      if (ring_ev[i]) cudaEventDestroy(ring_ev[i]);
    }
    if (ev) cudaEventDestroy(ev);
    if (seeds) cudaFree(seeds);
    if (out) cudaFree(out);
    if (frontier) cudaFree(frontier);
    if (partials) cudaFree(partials);
    if (mws) cudaFree(mws);
    if (hin) cudaFreeHost(hin);
    if (hout) cudaFreeHost(hout);
    if (cur >= 0 && cur != dev) cudaSetDevice(cur);
    cudaGetLastError();
    *this = HostCtx();
  }
  ~HostCtx() { release(); }
};
thread_local HostCtx g_host;

// grow-only device allocation
int grow(void** p, u64* have, u64 need, bool zero) {
  if (need <= *have) return HTH_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  CK(cudaMalloc(p, need));
  if (zero) CK(cudaMemset(*p, 0, need));  // legacy stream; callers synchronize below
  *have = need;
  return HTH_OK;
}

int host_ctx(int device, HostCtx** out) {
  HostCtx& c = g_host;
  if (c.dev >= 0 && c.dev != device) c.release();  // this thread moved to another device
  CK(cudaSetDevice(device));
  if (c.dev != device) {
    c = HostCtx();
    c.dev = device;
    for (int i = 0; i < 3; i++) CK(cudaStreamCreateWithFlags(&c.st[i], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c.ev, cudaEventDisableTiming));
  }
  if (!c.hin) {
    CK(cudaHostAlloc((void**)&c.hin, kSmallCall + 16, cudaHostAllocMapped));
    CK(cudaHostAlloc((void**)&c.hout, kSmallOut * 8, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void**)&c.din, c.hin, 0));
    CK(cudaHostGetDevicePointer((void**)&c.dout, c.hout, 0));
  }
  *out = &c;
  return HTH_OK;
}

// slots 0..nslots-1 of input buffer / workspace, plus seeds and digests
int host_reserve(HostCtx* c, int nslots, u64 buf_bytes, u64 ws_bytes, u64 seed_words, u64 out_words) {
  bool zeroed = false;
  for (int i = 0; i < nslots; i++) {
    if (int rc = grow(&c->buf[i], &c->buf_bytes[i], buf_bytes, false)) return rc;
    if (ws_bytes > c->ws_bytes[i]) zeroed = true;
    if (int rc = grow(&c->ws[i], &c->ws_bytes[i], ws_bytes, true)) return rc;
  }
  if (seed_words * 8 > c->seed_bytes) c->seeds_valid = 0;  // reallocated: nothing expanded yet
  if (int rc = grow((void**)&c->seeds, &c->seed_bytes, seed_words * 8, false)) return rc;
  if (int rc = grow((void**)&c->out, &c->out_bytes, out_words * 8, false)) return rc;
  // the memsets ran on the legacy stream; our streams are non-blocking
  if (zeroed) CK(cudaDeviceSynchronize());
  return HTH_OK;
}

}  // namespace
extern "C" int hth_expand_seed(uint64_t fold, uint64_t start, uint64_t count, uint64_t* d_words, void* stream);
namespace {
constexpr u64 kRing = 16ull << 20;  // bytes per pinned staging slot

// memcpy with several host threads (one thread reaches ~10 GB/s; the PCIe
// link takes ~55).  num_threads overrides OMP_NUM_THREADS=1 set by launchers.
void par_memcpy(void* dst, const void* src, u64 n) {
  const int T = (int)std::min<unsigned>(32, std::max(1u, std::thread::hardware_concurrency()));
#pragma omp parallel for num_threads(T) schedule(static)
  for (int t = 0; t < T; t++) {
    const u64 lo = (n * t / T) & ~63ull, hi = t + 1 == T ? n : (n * (t + 1) / T) & ~63ull;
    if (hi > lo) std::memcpy((uint8_t*)dst + lo, (const uint8_t*)src + lo, hi - lo);
  }
}

// host -> device copy on st.  Pinned sources (and small copies) go straight to
// the DMA engine; large pageable ones through the pinned staging slots:
// parallel memcpy of slice i+1 overlaps the DMA of slice i.
int h2d(HostCtx* c, void* dst, const void* src, u64 bytes, cudaStream_t st) {
  cudaPointerAttributes a{};
  const bool pinned = cudaPointerGetAttributes(&a, src) == cudaSuccess && a.type != cudaMemoryTypeUnregistered;
  cudaGetLastError();  // clear a sticky error from the attribute query on plain pointers
  static const u64 direct_below = [] {
    const char* e = getenv("HTH_PAGEABLE_DIRECT");  // experiments: pageable sizes left to the driver
    return e ? strtoull(e, nullptr, 10) : (256ull << 10);
  }();
  if (pinned || bytes < direct_below) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return HTH_OK;
  }
  for (int i = 0; i < 2; i++) {
    if (!c->ring[i]) {
      CK(cudaHostAlloc((void**)&c->ring[i], kRing, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&c->ring_ev[i], cudaEventDisableTiming));
    }
  }
  // slices of about a quarter of the copy (256 KiB .. one slot), so even a
  // few-MiB input overlaps its memcpy with its DMA
  static const u64 min_slice = [] {
    const char* e = getenv("HTH_RING_MIN_SLICE");  // experiments
    return e ? strtoull(e, nullptr, 10) : (256ull << 10);
  }();
  const u64 slice = std::min<u64>(kRing, std::max<u64>(min_slice, ((bytes / 4) + 63) & ~63ull));
  u64 i = 0;
  for (u64 off = 0; off < bytes; off += slice, i++) {
    const int slot = (int)(i & 1);
    const u64 len = std::min(slice, bytes - off);
    CK(cudaEventSynchronize(c->ring_ev[slot]));  // the slot's previous DMA has drained
    par_memcpy(c->ring[slot], (const uint8_t*)src + off, len);
    CK(cudaMemcpyAsync((uint8_t*)dst + off, c->ring[slot], len, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(c->ring_ev[slot], st));
  }
  return HTH_OK;
}

// seed words [0, total) of `fold` in c.seeds, expanded on st unless already there
int host_seeds(HostCtx* c, u64 fold, u64 total, cudaStream_t st) {
  if (c->seeds_valid >= total && c->seeds_fold == fold) return HTH_OK;
  if (int rc = hth_expand_seed(fold, 0, total, c->seeds, st)) return rc;
  c->seeds_fold = fold;
  c->seeds_valid = total;
  return HTH_OK;
}



}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* hth_last_error(void) { return g_err.c_str(); }

int hth_version(void) { return 100; }

int hth_variant_geometry(int output_bytes, int* k, int* e, int* d, int* w, int* instance_words) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (k) *k = v.k;
  if (e) *e = v.e;
  if (d) *d = v.d;
  if (w) *w = v.w;
  if (instance_words) *instance_words = v.m;
  return HTH_OK;
}

int hth_seed_words_needed(int output_bytes, uint64_t n_bytes, uint64_t* out_words) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (!out_words) return fail(HTH_EINVAL, "null output pointer");
  *out_words = make_layout(v, n_bytes).total;
  return HTH_OK;
}

int hth_seed_layout(int output_bytes, uint64_t n_bytes, uint64_t out10[10]) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (!out10) return fail(HTH_EINVAL, "null output pointer");
  const Layout l = make_layout(v, n_bytes);
  const u64 vals[10] = {l.levels, 0, l.ew, l.tree_start, l.tree_per, l.fin_start, l.fin_per, l.rem_start,
                        l.rem_words, l.total};
  memcpy(out10, vals, sizeof vals);
  return HTH_OK;
}

int hth_master_fold(const uint8_t master[32], uint64_t* fold) {
  if (!master || !fold) return fail(HTH_EINVAL, "master seed must be exactly 32 bytes");
  *fold = fold_of(master);
  return HTH_OK;
}

int hth_expand_seed(uint64_t fold, uint64_t start, uint64_t count, uint64_t* d_words, void* stream) {
  if (!count) return HTH_OK;
  if (!d_words) return fail(HTH_EINVAL, "null seed buffer");
  const u64 blocks = std::min<u64>(ceil_div(count, 256), 4096);
  expand_seed_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(fold, start, count, d_words);
  CK(cudaGetLastError());
  return HTH_OK;
}

int hth_toeplitz_nh(const uint64_t* d_tail, uint64_t n, const uint64_t* d_keys, uint64_t n_keys, int k,
                    uint64_t* d_out, void* stream) {
  if (k < 0) return fail(HTH_EINVAL, "k must be >= 0");
  if (n_keys + 1 < n + (u64)k) return fail(HTH_EINVAL, "remainder key region too short");
  if (!k) return HTH_OK;
  if (!d_out || (n && (!d_tail || !d_keys))) return fail(HTH_EINVAL, "null device pointer");
  toeplitz_nh_kernel<<<(unsigned)k, 256, 0, (cudaStream_t)stream>>>(d_tail, n, d_keys, d_out);
  CK(cudaGetLastError());
  return HTH_OK;
}

int hth_fill_splitmix(uint64_t fill_seed, uint64_t word_offset, uint64_t n_bytes, void* d_dst, void* stream) {
  if (!n_bytes) return HTH_OK;
  if (!d_dst || (reinterpret_cast<uintptr_t>(d_dst) & 7)) return fail(HTH_EINVAL, "destination must be 8-byte aligned");
  const u64 nw = (n_bytes + 7) / 8;
  const u64 blocks = std::min<u64>(ceil_div(nw, 256), 148 * 64);
  fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(fill_seed, word_offset, nw, n_bytes, (u64*)d_dst);
  CK(cudaGetLastError());
  return HTH_OK;
}

int hth_fill_splitmix_strings(uint64_t fill_seed, uint64_t n_strings, uint64_t n_bytes, uint64_t first_string,
                              uint64_t string_step, void* d_dst, uint64_t dst_stride, void* stream) {
  if (!n_strings || !n_bytes) return HTH_OK;
  if (n_bytes % 8 || dst_stride % 8 || dst_stride < n_bytes || !d_dst || (reinterpret_cast<uintptr_t>(d_dst) & 7))
    return fail(HTH_EINVAL, "strided fill needs n_bytes, dst_stride and d_dst 8-byte aligned, dst_stride >= n_bytes");
  const u64 nw = n_strings * (n_bytes / 8);
  const u64 blocks = std::min<u64>(ceil_div(nw, 256), 148 * 64);
  fill_strings_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(fill_seed, n_bytes / 8, first_string,
                                                                          string_step, nw, dst_stride / 8,
                                                                          (u64*)d_dst);
  CK(cudaGetLastError());
  return HTH_OK;
}

int hth_workspace_size_fixed(int output_bytes, uint64_t n_strings, uint64_t n_bytes, uint64_t* bytes) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (!bytes) return fail(HTH_EINVAL, "null output pointer");
  *bytes = fixed_plan(v, n_strings, n_bytes).ws_total;
  return HTH_OK;
}

int hth_hash_fixed(int output_bytes, const void* d_data, uint64_t n_strings, uint64_t stride_bytes, uint64_t n_bytes,
                   uint64_t seed_fold, const uint64_t* d_seed, uint64_t seed_capacity, uint64_t* d_out,
                   void* d_workspace, uint64_t workspace_bytes, void* stream) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (int rc = check_seed(v, n_bytes, seed_capacity)) return rc;
  if (!n_strings) return HTH_OK;
  if (!d_out || !d_seed) return fail(HTH_EINVAL, "null device pointer");
  if (n_bytes && !d_data) return fail(HTH_EINVAL, "null data pointer");
  if (n_strings > 1 && stride_bytes < n_bytes) return fail(HTH_EINVAL, "stride_bytes < n_bytes");
  // one string: the stride is meaningless; give every route the same
  // well-formed one (16-byte multiple covering the string)
  if (n_strings == 1) stride_bytes = align_up(n_bytes, 16);
  const FixedPlan f = fixed_plan(v, n_strings, n_bytes);
  if (workspace_bytes < f.ws_total)
    return fail(HTH_EINVAL, "workspace too small: %llu < %llu bytes", (unsigned long long)workspace_bytes,
                (unsigned long long)f.ws_total);
  cudaStream_t st = (cudaStream_t)stream;
  Params P{};
  P.data = (const uint8_t*)d_data;
  P.n_strings = n_strings;
  P.stride = stride_bytes;
  P.n_bytes = n_bytes;
  P.J_fixed = f.J;
  P.n_inst_fixed = f.n_inst;
  P.L_fixed = f.n_inst ? level_count(f.n_inst) : 1;
  P.n_jobs = f.n_jobs;
  P.scr_per = f.scr_per;
  P.cnt_per = f.cnt_per;
  P.S = d_seed;
  P.out = d_out;
  P.job_lvl = f.job_lvl;
  fill_ehc(v, seed_fold, P);
  fill_fin_const(v, seed_fold, n_bytes, P);
  if (f.n_inst == 0 && n_bytes > 0 && stride_bytes % 16 == 0 && stride_bytes <= 2048 &&
      (reinterpret_cast<uintptr_t>(d_data) & 15) == 0) {
    // strings shorter than one instance: dedicated half-warp-per-string kernel
    TailParams T{};
    T.data = (const uint8_t*)d_data;
    T.n_strings = n_strings;
    T.stride = stride_bytes;
    T.n_bytes = n_bytes;
    T.S = d_seed;
    T.R = (u64)v.ew + 71ull * v.k;
    T.out = d_out;
    for (int r = 0; r < v.k; r++) {  // finalize over the tag alone (hasher.py:400-405)
      const u64 sF = host_mix(seed_fold + ((u64)v.ew + 7ull * v.k + 64ull * r + 1) * 0x9E3779B97F4A7C15ull);
      const u32 a = (u32)n_bytes + (u32)sF, b = (u32)(n_bytes >> 32) + (u32)(sF >> 32);
      T.tag[r] = (u64)a * b;
    }
    const u64 nch = (n_bytes + 15) / 16;
    return by_width<TailF>(output_bytes, T, nch, st);
  }
  if (small_ok(v, f.n_inst, stride_bytes, n_bytes, d_data)) {
    return by_width<SmallF>(output_bytes, P, st);
  }
  uint8_t* ws = (uint8_t*)d_workspace;
  P.scratch = (u64*)ws;
  P.acc = (u64*)(ws + f.ws_scratch);
  P.counters = (u32*)(ws + f.ws_scratch + f.ws_acc);
  P.events = (u32*)(ws + f.ws_scratch + f.ws_acc + f.ws_cnt);
  set_ctl(P, ws + f.ws_total - 256);
  return guard_ws(dispatch<false>(output_bytes, P, f.n_jobs, st), d_workspace, f.ws_total, st);
}

int hth_hash_fixed_folds(int output_bytes, const void* d_data, uint64_t n_strings, uint64_t stride_bytes,
                         uint64_t n_bytes, const uint64_t* d_folds, uint64_t* d_out, void* d_workspace,
                         uint64_t workspace_bytes, void* stream) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (!n_strings) return HTH_OK;
  if (!d_out || !d_folds) return fail(HTH_EINVAL, "null device pointer");
  if (n_bytes && !d_data) return fail(HTH_EINVAL, "null data pointer");
  if (n_strings > 1 && stride_bytes && stride_bytes < n_bytes) return fail(HTH_EINVAL, "0 < stride_bytes < n_bytes");
  const FixedPlan f = fixed_plan(v, n_strings, n_bytes);
  if (workspace_bytes < f.ws_total) return fail(HTH_EINVAL, "workspace too small");
  Params P{};
  P.data = (const uint8_t*)d_data;
  P.n_strings = n_strings;
  P.stride = stride_bytes;
  P.n_bytes = n_bytes;
  P.J_fixed = f.J;
  P.n_inst_fixed = f.n_inst;
  P.L_fixed = f.n_inst ? level_count(f.n_inst) : 1;
  P.n_jobs = f.n_jobs;
  P.scr_per = f.scr_per;
  P.cnt_per = f.cnt_per;
  P.folds = d_folds;
  P.out = d_out;
  P.job_lvl = f.job_lvl;
  uint8_t* ws = (uint8_t*)d_workspace;
  P.scratch = (u64*)ws;
  P.acc = (u64*)(ws + f.ws_scratch);
  P.counters = (u32*)(ws + f.ws_scratch + f.ws_acc);
  P.events = (u32*)(ws + f.ws_scratch + f.ws_acc + f.ws_cnt);
  set_ctl(P, ws + f.ws_total - 256);
  return guard_ws(dispatch_ps(output_bytes, P, f.n_jobs, (cudaStream_t)stream), d_workspace, f.ws_total,
                  (cudaStream_t)stream);
}

int hth_workspace_size_varlen(int output_bytes, uint64_t n_strings, uint64_t total_bytes, uint64_t* bytes) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (!bytes) return fail(HTH_EINVAL, "null output pointer");
  VarPlan p;
  if (int rc = varlen_plan(v, n_strings, total_bytes, ~0ull, &p)) return rc;
  *bytes = p.total;
  return HTH_OK;
}

int hth_hash_varlen(int output_bytes, const void* d_data, const uint64_t* d_offsets, uint64_t n_strings,
                    uint64_t max_n_bytes, uint64_t total_bytes, uint64_t seed_fold, const uint64_t* d_seed,
                    uint64_t seed_capacity, uint64_t* d_out, void* d_workspace, uint64_t workspace_bytes,
                    void* stream) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (int rc = check_seed(v, max_n_bytes, seed_capacity)) return rc;
  if (!n_strings) return HTH_OK;
  if (!d_out || !d_seed || !d_offsets || !d_workspace) return fail(HTH_EINVAL, "null device pointer");
  if (total_bytes && !d_data) return fail(HTH_EINVAL, "null data pointer");
  if (n_strings >= (1ull << 32)) return fail(HTH_EINVAL, "at most 2^32-1 strings per call");
  VarPlan p;
  if (int rc = varlen_plan(v, n_strings, total_bytes, max_n_bytes, &p)) return rc;
  if (workspace_bytes < p.total)
    return fail(HTH_EINVAL, "workspace too small: %llu < %llu bytes", (unsigned long long)workspace_bytes,
                (unsigned long long)p.total);
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)d_workspace;
  int* err = (int*)(ws + p.off_err);
  u32* cls_cnt = (u32*)(ws + p.off_pctl);
  auto* totals = (unsigned long long*)(ws + p.off_pctl + 384);
  int cur_dev = 0;
  CK(cudaGetDevice(&cur_dev));
  const WsSig sig{{p.off_cnt, p.off_acc, p.off_ev, p.off_ctl, p.off_pctl, p.off_clear, (u64)v.k, (u64)cur_dev}};
  if (!ws_layout_known(ws, sig)) {
    const cudaError_t e = cudaMemsetAsync(ws, 0, p.off_clear, st);
    if (e != cudaSuccess) {
      ws_forget(ws);
      return cuda_fail(e, "cudaMemsetAsync(workspace)");
    }
  }
  const int job_lvl = pick_job_lvl(((max_n_bytes + 7) / 8) / (u64)v.m);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  PlanParams Q{};
  Q.off = d_offsets;
  Q.n = n_strings;
  Q.max_n = max_n_bytes;
  Q.total = total_bytes;
  Q.job_lvl = job_lvl;
  Q.lmax = (u32)p.lmax;
  Q.S = d_seed;
  Q.err = (int*)(ws + p.off_err);
  Q.cls_cnt = cls_cnt;
  Q.data = (const uint8_t*)d_data;
  Q.R = (u64)v.ew + 71ull * v.k;  // L' = 1 layout (hasher.py:130-153)
  Q.F0 = (u64)v.ew + 7ull * v.k;
  Q.out = d_out;
  Q.queues = (u64*)(ws + p.off_queue);
  Q.totals = totals;
  Q.ztab = (u64*)(ws + p.off_ztab);
  Q.Q = p.Q;
  // HTH_PLAN_SPW strings per warp, 8 warps per CTA (grid-stride beyond 8 CTAs per SM)
  const unsigned pb = (unsigned)std::max<u64>(1, std::min<u64>(ceil_div(n_strings, 8 * HTH_PLAN_SPW), (u64)sm_count(dev) * 8));
  if (int rc = by_width<PlanF>(output_bytes, Q, pb, st)) {
    ws_forget(ws);
    return rc;
  }
  Params P{};
  P.data = (const uint8_t*)d_data;
  P.n_strings = n_strings;
  P.offsets = d_offsets;
  P.job_map = Q.queues;
  P.cls_cnt = cls_cnt;
  P.totals = totals;
  P.var_total = total_bytes;
  P.ztab = (const u64*)(ws + p.off_ztab);
  P.ztab_lmax = (u32)p.lmax;
  P.n_jobs = p.max_jobs;  // varlen: queue sizing bound; the kernel counts the jobs itself
  memcpy(P.cls_qb, p.Q.qb, sizeof(P.cls_qb));
  P.n_bytes = max_n_bytes;  // varlen: clamp bound (matches plan_kernel)
  P.S = d_seed;
  P.out = d_out;
  P.job_lvl = job_lvl;
  fill_ehc(v, seed_fold, P);
  P.scratch = (u64*)(ws + p.off_scr);
  P.counters = (u32*)(ws + p.off_cnt);
  P.acc = (u64*)(ws + p.off_acc);
  P.events = (u32*)(ws + p.off_ev);
  set_ctl(P, ws + p.off_ctl);
  const int rc = dispatch<true>(output_bytes, P, p.max_jobs, st);
  if (rc != HTH_OK) ws_forget(ws);  // the next call clears the workspace
  return rc;
}

#ifdef HTH_DEBUG_TIMING
// experiment builds only: copy and clear the per-warp timing records
int hth_debug_timing(unsigned long long* host, int n_warps) {
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(host, dbg_buf(), (size_t)n_warps * 12 * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemset(dbg_buf(), 0, 8192 * 12 * 8));
  return HTH_OK;
}
#endif
int hth_varlen_status(void* d_workspace, void* stream) {
  if (!d_workspace) return fail(HTH_EINVAL, "null workspace");
  int h = 0;
  CK(cudaMemcpyAsync(&h, d_workspace, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  // the flag accumulates over calls until read: clear what was reported
  if (h) CK(cudaMemsetAsync(d_workspace, 0, 4, (cudaStream_t)stream));
  if (h & 1) return fail(HTH_ESEEDSIZE, "a string was longer than max_n_bytes; its digest is invalid");
  if (h & 4) return fail(HTH_EINVAL, "offsets decrease or run past total_bytes; digests are invalid");
  if (h & 2) return fail(HTH_EINVAL, "the strings hold more bytes than total_bytes declared; digests are invalid");
  return HTH_OK;
}

// ---- one string split across devices (config 5) ----------------------
int hth_slice_plan(int output_bytes, uint64_t n_bytes, uint64_t n_slices, uint64_t* inst_bounds,
                   int* frontier_level, uint64_t* frontier_counts) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (!n_slices || !inst_bounds || !frontier_level || !frontier_counts) return fail(HTH_EINVAL, "bad slice plan args");
  const u64 n_inst = ((n_bytes + 7) / 8) / (u64)v.m;
  const int jl = pick_job_lvl(n_inst);
  // frontier level: the largest c >= job level leaving >= 64 level-c subtrees
  // per slice (load balance within one subtree per 64)
  int c = jl;
  while ((n_inst >> (3 * (c + 1))) >= 64 * n_slices) c++;
  const u64 sub = 1ull << (3 * c), nsub = n_inst / sub;
  for (u64 i = 0; i <= n_slices; i++) inst_bounds[i] = (nsub * i / n_slices) * sub;
  inst_bounds[n_slices] = n_inst;  // the last slice also takes the ragged end and the tail
  const u64 keep = (n_inst >> (3 * c)) & ~7ull;  // non-leftover level-c blocks
  for (u64 i = 0; i < n_slices; i++) {
    const u64 a = inst_bounds[i] >> (3 * c), b = std::min(inst_bounds[i + 1] >> (3 * c), keep);
    frontier_counts[i] = b > a ? b - a : 0;
  }
  *frontier_level = c;
  return HTH_OK;
}

int hth_workspace_size_slice(int output_bytes, uint64_t n_bytes, uint64_t* bytes) {
  return hth_workspace_size_fixed(output_bytes, 1, n_bytes, bytes);
}

int hth_ipc_get_handle(const void* d_ptr, uint8_t handle_out[64], uint64_t* offset_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  if (!d_ptr || !handle_out || !offset_out) return fail(HTH_EINVAL, "null pointer");
  // the handle names the whole allocation (e.g. a caching-allocator segment):
  // report where d_ptr sits inside it
  typedef int (*AddrRange)(unsigned long long*, size_t*, unsigned long long);
  static std::mutex mu;
  static AddrRange range = nullptr;
  {
    std::lock_guard<std::mutex> g(mu);
    if (!range) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !fn) return fail(HTH_ECUDA, "cuMemGetAddressRange unavailable");
      range = (AddrRange)fn;
    }
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)(uintptr_t)d_ptr) != 0) return fail(HTH_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
  std::memcpy(handle_out, &h, 64);
  *offset_out = (uint64_t)((uintptr_t)d_ptr - base);
  return HTH_OK;
}

int hth_ipc_open_handle(const uint8_t handle[64], void** d_ptr_out) {
  if (!handle || !d_ptr_out) return fail(HTH_EINVAL, "null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  CK(cudaIpcOpenMemHandle(d_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return HTH_OK;
}

int hth_ipc_close_handle(void* d_ptr) {
  if (!d_ptr) return fail(HTH_EINVAL, "null pointer");
  CK(cudaIpcCloseMemHandle(d_ptr));
  return HTH_OK;
}

static int slice_impl(int output_bytes, const void* d_slice, uint64_t n_bytes, uint64_t inst_begin, uint64_t inst_end,
                      int frontier_level, uint64_t seed_fold, const uint64_t* d_seed, uint64_t seed_capacity,
                      uint64_t* d_frontier, uint64_t* d_partial, uint64_t* d_done_flag, uint64_t done_value,
                      int options, void* d_workspace, uint64_t workspace_bytes, void* stream) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (int rc = check_seed(v, n_bytes, seed_capacity)) return rc;
  if (options & ~HTH_SLICE_ACCUMULATE) return fail(HTH_EINVAL, "unknown slice options %d", options);
  const FixedPlan f = fixed_plan(v, 1, n_bytes, std::max(frontier_level, 1));
  const u64 per = 1ull << (3 * f.job_lvl), sub = 1ull << (3 * frontier_level);
  if (frontier_level < f.job_lvl || inst_begin % sub || inst_begin > inst_end || inst_end > f.n_inst ||
      (inst_end != f.n_inst && inst_end % sub))
    return fail(HTH_EINVAL, "slice bounds must be multiples of 8^frontier_level instances (frontier >= %d)", f.job_lvl);
  if (!d_partial || !d_seed) return fail(HTH_EINVAL, "null device pointer");
  if (workspace_bytes < f.ws_total) return fail(HTH_EINVAL, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  if (!(options & HTH_SLICE_ACCUMULATE)) CK(cudaMemsetAsync(d_partial, 0, v.k * 8, st));
  const bool last = inst_end == f.n_inst;
  const u64 j0 = inst_begin / per;
  const u64 j1 = last ? f.J : inst_end / per;
  if (j1 <= j0) {  // nothing to hash: still publish the (empty) slice
    if (d_done_flag) {
      signal_kernel<<<1, 1, 0, st>>>(reinterpret_cast<unsigned long long*>(d_done_flag), done_value);
      CK(cudaGetLastError());
    }
    return HTH_OK;
  }
  const u64 byte0 = inst_begin * (u64)v.m * 8;
  Params P{};
  P.data = (const uint8_t*)d_slice - byte0;  // global byte b of the string lives at d_slice[b - byte0]
  P.n_strings = 1;
  P.stride = 0;
  P.n_bytes = n_bytes;
  P.J_fixed = f.J;
  P.n_inst_fixed = f.n_inst;
  P.L_fixed = f.n_inst ? level_count(f.n_inst) : 1;
  P.n_jobs = j1 - j0;
  P.S = d_seed;
  P.out = d_partial;
  P.job_lvl = f.job_lvl;
  P.frontier_lvl = frontier_level;
  P.slice_job0 = j0;
  P.frontier_base = inst_begin >> (3 * frontier_level);
  P.frontier = d_frontier;
  P.done_flag = reinterpret_cast<unsigned long long*>(d_done_flag);
  P.done_value = done_value;
  fill_ehc(v, seed_fold, P);
  fill_fin_const(v, seed_fold, n_bytes, P);
  uint8_t* ws = (uint8_t*)d_workspace;
  P.scratch = (u64*)ws;
  P.acc = d_partial;
  P.counters = (u32*)(ws + f.ws_scratch + f.ws_acc);
  P.events = (u32*)(ws + f.ws_scratch + f.ws_acc + f.ws_cnt);
  set_ctl(P, ws + f.ws_total - 256);
  return guard_ws(dispatch<false>(output_bytes, P, P.n_jobs, st), d_workspace, f.ws_total, st);
}

int hth_hash_slice(int output_bytes, const void* d_slice, uint64_t n_bytes, uint64_t inst_begin, uint64_t inst_end,
                   int frontier_level, uint64_t seed_fold, const uint64_t* d_seed, uint64_t seed_capacity,
                   uint64_t* d_frontier, uint64_t* d_partial, void* d_workspace, uint64_t workspace_bytes,
                   void* stream) {
  return slice_impl(output_bytes, d_slice, n_bytes, inst_begin, inst_end, frontier_level, seed_fold, d_seed,
                    seed_capacity, d_frontier, d_partial, nullptr, 0, 0, d_workspace, workspace_bytes, stream);
}

int hth_hash_slice_ex(int output_bytes, const void* d_slice, uint64_t n_bytes, uint64_t inst_begin, uint64_t inst_end,
                      int frontier_level, uint64_t seed_fold, const uint64_t* d_seed, uint64_t seed_capacity,
                      uint64_t* d_frontier, uint64_t* d_partial, uint64_t* d_done_flag, uint64_t done_value,
                      int options, void* d_workspace, uint64_t workspace_bytes, void* stream) {
  return slice_impl(output_bytes, d_slice, n_bytes, inst_begin, inst_end, frontier_level, seed_fold, d_seed,
                    seed_capacity, d_frontier, d_partial, d_done_flag, done_value, options, d_workspace,
                    workspace_bytes, stream);
}

static int merge_impl(int output_bytes, uint64_t n_bytes, int frontier_level, const uint64_t* d_frontier,
                      uint64_t n_frontier, const uint64_t* d_partials, uint64_t n_partials, const uint64_t* d_seed,
                      uint64_t seed_capacity, uint64_t* d_out, const uint64_t* d_flags, uint64_t epoch,
                      uint64_t* d_consumed, uint64_t timeout_ns, int* d_status, void* d_workspace,
                      uint64_t workspace_bytes, void* stream) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (int rc = check_seed(v, n_bytes, seed_capacity)) return rc;
  const u64 n_inst = ((n_bytes + 7) / 8) / (u64)v.m;
  const u64 keep = (n_inst >> (3 * frontier_level)) & ~7ull;
  if (n_frontier != keep)
    return fail(HTH_EINVAL, "frontier holds %llu blocks, expected %llu", (unsigned long long)n_frontier,
                (unsigned long long)keep);
  const u64 need = 2 * (n_frontier / 8 + 8) * 8ull * v.k * 8;
  if (workspace_bytes < need) return fail(HTH_EINVAL, "merge workspace too small: need %llu", (unsigned long long)need);
  if (d_flags && (!d_consumed || !d_status)) return fail(HTH_EINVAL, "flags need a consumed flag and a status word");
  MergeParams M{};
  M.n_bytes = n_bytes;
  M.c = frontier_level;
  M.frontier = d_frontier;
  M.nf = n_frontier;
  M.partials = d_partials;
  M.np = n_partials;
  M.S = d_seed;
  M.tmp = (u64*)d_workspace;
  M.out = d_out;
  M.flags = reinterpret_cast<const unsigned long long*>(d_flags);
  M.nflags = d_flags ? n_partials : 0;
  M.epoch = epoch;
  M.timeout_ns = timeout_ns;
  M.consumed = reinterpret_cast<unsigned long long*>(d_consumed);
  M.partials_rw = d_flags ? const_cast<u64*>(d_partials) : nullptr;
  M.status = d_status;
  return by_width<MergeF>(output_bytes, M, (cudaStream_t)stream);
}

int hth_hash_merge(int output_bytes, uint64_t n_bytes, int frontier_level, const uint64_t* d_frontier,
                   uint64_t n_frontier, const uint64_t* d_partials, uint64_t n_partials, uint64_t seed_fold,
                   const uint64_t* d_seed, uint64_t seed_capacity, uint64_t* d_out, void* d_workspace,
                   uint64_t workspace_bytes, void* stream) {
  (void)seed_fold;
  return merge_impl(output_bytes, n_bytes, frontier_level, d_frontier, n_frontier, d_partials, n_partials, d_seed,
                    seed_capacity, d_out, nullptr, 0, nullptr, 0, nullptr, d_workspace, workspace_bytes, stream);
}

int hth_hash_merge_ex(int output_bytes, uint64_t n_bytes, int frontier_level, const uint64_t* d_frontier,
                      uint64_t n_frontier, uint64_t* d_partials, uint64_t n_partials, const uint64_t* d_seed,
                      uint64_t seed_capacity, uint64_t* d_out, const uint64_t* d_flags, uint64_t epoch,
                      uint64_t* d_consumed, uint64_t timeout_ns, int* d_status, void* d_workspace,
                      uint64_t workspace_bytes, void* stream) {
  if (!d_flags) return fail(HTH_EINVAL, "hth_hash_merge_ex needs flags (use hth_hash_merge)");
  return merge_impl(output_bytes, n_bytes, frontier_level, d_frontier, n_frontier, d_partials, n_partials, d_seed,
                    seed_capacity, d_out, d_flags, epoch, d_consumed, timeout_ns, d_status, d_workspace,
                    workspace_bytes, stream);
}

int hth_signal(uint64_t* d_flag, uint64_t value, void* stream) {
  if (!d_flag) return fail(HTH_EINVAL, "null flag");
  signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<unsigned long long*>(d_flag), value);
  CK(cudaGetLastError());
  return HTH_OK;
}

int hth_wait_flag(const uint64_t* d_flag, uint64_t value, uint64_t timeout_ns, int* d_status, void* stream) {
  if (!d_flag || !d_status) return fail(HTH_EINVAL, "null flag or status");
  wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<const unsigned long long*>(d_flag), value,
                                                 timeout_ns, d_status);
  CK(cudaGetLastError());
  return HTH_OK;
}

// Strings longer than kChunk from host memory: each is streamed in slices
// of whole level-c subtrees (c = the job level, 8^c instances) through the
// three bounded input buffers, one hth_hash_slice per slice on rotating
// streams (the H2D copy of slice i+1 overlaps the hash of slice i), then one
// hth_hash_merge finishes the tree (tree.py:63-134) and adds the tail.
static int host_hash_long(const VarInfo& v, int output_bytes, HostCtx* c, const uint8_t* h_data, u64 n_strings,
                          u64 stride_bytes, u64 n_bytes, u64 fold, u64 total) {
  const u64 n_inst = ((n_bytes + 7) / 8) / (u64)v.m;
  const int lvl = pick_job_lvl(n_inst);
  const u64 sub = 1ull << (3 * lvl), sub_bytes = sub * v.m * 8;
  const u64 ci = std::max<u64>(1, kChunk / sub_bytes) * sub;  // instances per slice
  const u64 nsl = ceil_div(n_inst, ci);
  const u64 keep = (n_inst >> (3 * lvl)) & ~7ull;  // non-leftover level-c roots
  const u64 k = (u64)v.k;
  const FixedPlan fp = fixed_plan(v, 1, n_bytes, lvl);
  const u64 slice_bytes = ci * v.m * 8 + v.m * 8 + 16;  // + the ragged tail of the last slice
  if (int rc = host_reserve(c, (int)std::min<u64>(nsl, 3), slice_bytes, fp.ws_total, total, n_strings * k)) return rc;
  if (int rc = grow((void**)&c->frontier, &c->frontier_bytes, std::max<u64>(keep, 1) * 8 * k * 8, false)) return rc;
  if (int rc = grow((void**)&c->partials, &c->partial_bytes, nsl * k * 8, false)) return rc;
  const u64 mneed = 2 * (keep / 8 + 8) * 8 * k * 8;
  if (int rc = grow(&c->mws, &c->mws_bytes, mneed, false)) return rc;
  if (int rc = host_seeds(c, fold, total, c->st[0])) return rc;
  for (u64 s = 0; s < n_strings; s++) {
    // slices of this string start after the seeds and the previous merge
    CK(cudaEventRecord(c->ev, c->st[0]));
    for (int i = 1; i < 3; i++) CK(cudaStreamWaitEvent(c->st[i], c->ev, 0));
    const uint8_t* src = h_data + s * stride_bytes;
    for (u64 i = 0; i < nsl; i++) {
      const int b = (int)(i % 3);
      const u64 ib = i * ci, ie = std::min(n_inst, ib + ci);
      const u64 b0 = ib * v.m * 8, b1 = ie == n_inst ? n_bytes : ie * v.m * 8;
      if (int rc = h2d(c, c->buf[b], src + b0, b1 - b0, c->st[b])) return rc;
      const u64 fa = ib >> (3 * lvl);
      if (int rc = hth_hash_slice(output_bytes, c->buf[b], n_bytes, ib, ie, lvl, fold, c->seeds, total,
                                  c->frontier + std::min(fa, keep) * 8 * k, c->partials + i * k, c->ws[b],
                                  c->ws_bytes[b], c->st[b]))
        return rc;
    }
    for (int i = 1; i < 3; i++) {
      CK(cudaEventRecord(c->ev, c->st[i]));
      CK(cudaStreamWaitEvent(c->st[0], c->ev, 0));
    }
    if (int rc = hth_hash_merge(output_bytes, n_bytes, lvl, c->frontier, keep, c->partials, nsl, fold, c->seeds,
                                total, c->out + s * k, c->mws, c->mws_bytes, c->st[0]))
      return rc;
  }
  return HTH_OK;
}

int hth_hash_host(int output_bytes, const void* h_data, uint64_t n_bytes, const uint8_t master[32],
                  uint64_t seed_capacity, uint64_t* h_out, int device) {
  return hth_hash_fixed_host(output_bytes, h_data, 1, n_bytes, n_bytes, master, seed_capacity, h_out, device);
}

int hth_hash_fixed_host(int output_bytes, const void* h_data, uint64_t n_strings, uint64_t stride_bytes,
                        uint64_t n_bytes, const uint8_t master[32], uint64_t seed_capacity, uint64_t* h_out,
                        int device) {
  VarInfo v;
  if (int rc = get_var(output_bytes, &v)) return rc;
  if (!master) return fail(HTH_EINVAL, "master seed must be exactly 32 bytes");
  const Layout lay = make_layout(v, n_bytes);
  // SeedBuffer.capacity semantics (hasher.py:209-214); HTH_SEED_AUTO sizes it
  if (seed_capacity != HTH_SEED_AUTO)
    if (int rc = check_seed(v, n_bytes, seed_capacity)) return rc;
  if (!n_strings) return HTH_OK;
  if (!h_out || (n_bytes && !h_data)) return fail(HTH_EINVAL, "null host pointer");
  if (n_strings > 1 && stride_bytes < n_bytes) return fail(HTH_EINVAL, "stride_bytes < n_bytes");
  if (n_strings == 1) stride_bytes = align_up(n_bytes, 16);
  HostCtx* c = nullptr;
  if (int rc = host_ctx(device, &c)) return rc;
  const u64 fold = fold_of(master);
  const u64 k = (u64)v.k;
  if (n_bytes > kChunk) {
    if (int rc = host_hash_long(v, output_bytes, c, (const uint8_t*)h_data, n_strings, stride_bytes, n_bytes, fold,
                                lay.total))
      return rc;
    CK(cudaMemcpyAsync(h_out, c->out, n_strings * k * 8, cudaMemcpyDeviceToHost, c->st[0]));
    CK(cudaStreamSynchronize(c->st[0]));
    return HTH_OK;
  }
  // chunking: whole strings per chunk, ~kChunk bytes per chunk, 3 buffers in
  // flight; strings keep their host stride on the device (the kernel handles
  // any start alignment)
  const u64 dstride = std::max<u64>(stride_bytes, 1);
  u64 per = std::max<u64>(1, kChunk / dstride);
  if (per > n_strings) per = n_strings;
  const u64 nchunks = ceil_div(n_strings, per);
  const FixedPlan fp = fixed_plan(v, per, n_bytes);
  const u64 in_bytes = n_bytes ? (n_strings - 1) * stride_bytes + n_bytes : 0;
  if (int rc = host_reserve(c, (int)std::min<u64>(nchunks, 3), per * dstride + 16, std::max<u64>(fp.ws_total, 256),
                            lay.total, n_strings * k))
    return rc;
  if (nchunks == 1 && in_bytes <= kSmallCall && n_strings * k <= kSmallOut) {
    cudaStream_t st = c->st[0];
    if (int rc = host_seeds(c, fold, lay.total, st)) return rc;
    if (in_bytes <= kMappedCall && mapped_enabled()) {
      if (in_bytes) std::memcpy(c->hin, h_data, in_bytes);
      if (int rc = hth_hash_fixed(output_bytes, c->din, n_strings, dstride, n_bytes, fold, c->seeds, lay.total,
                                  c->dout, c->ws[0], c->ws_bytes[0], st))
        return rc;
      CK(cudaStreamSynchronize(st));
      std::memcpy(h_out, c->hout, n_strings * k * 8);
      return HTH_OK;
    }
    if (in_bytes) {
      std::memcpy(c->hin, h_data, in_bytes);
      CK(cudaMemcpyAsync(c->buf[0], c->hin, in_bytes, cudaMemcpyHostToDevice, st));
    }
    if (int rc = hth_hash_fixed(output_bytes, c->buf[0], n_strings, dstride, n_bytes, fold, c->seeds, lay.total,
                                c->out, c->ws[0], c->ws_bytes[0], st))
      return rc;
    CK(cudaMemcpyAsync(c->hout, c->out, n_strings * k * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::memcpy(h_out, c->hout, n_strings * k * 8);
    return HTH_OK;
  }
  if (int rc = host_seeds(c, fold, lay.total, c->st[0])) return rc;
  CK(cudaEventRecord(c->ev, c->st[0]));
  for (int i = 1; i < 3; i++) CK(cudaStreamWaitEvent(c->st[i], c->ev, 0));
  for (u64 ch = 0; ch < nchunks; ch++) {
    const int b = (int)(ch % 3);
    cudaStream_t st = c->st[b];
    const u64 s0 = ch * per, ns = std::min(per, n_strings - s0);
    const uint8_t* src = (const uint8_t*)h_data + s0 * stride_bytes;
    if (n_bytes)
      if (int rc = h2d(c, c->buf[b], src, (ns - 1) * stride_bytes + n_bytes, st)) return rc;
    if (int rc = hth_hash_fixed(output_bytes, c->buf[b], ns, dstride, n_bytes, fold, c->seeds, lay.total,
                                c->out + s0 * k, c->ws[b], c->ws_bytes[b], st))
      return rc;
  }
  // digests stay on the device until every chunk is hashed: a per-chunk copy
  // into (pageable) h_out blocks this thread until that chunk's kernel ends,
  // which starves the copy engine of the next chunk (~0.1 ms gap per chunk)
  for (int i = 1; i < 3; i++) {
    CK(cudaEventRecord(c->ev, c->st[i]));
    CK(cudaStreamWaitEvent(c->st[0], c->ev, 0));
  }
  CK(cudaMemcpyAsync(h_out, c->out, n_strings * k * 8, cudaMemcpyDeviceToHost, c->st[0]));
  CK(cudaStreamSynchronize(c->st[0]));
  return HTH_OK;
}

int hth_host_release(void) {
  g_host.release();
  return HTH_OK;
}

int hth_workspace_reset(void* d_workspace, uint64_t workspace_bytes, void* stream) {
  if (!workspace_bytes) return HTH_OK;
  if (!d_workspace) return fail(HTH_EINVAL, "null workspace");
  ws_forget(d_workspace);
  CK(cudaMemsetAsync(d_workspace, 0, workspace_bytes, (cudaStream_t)stream));
  return HTH_OK;
}

}  // extern "C"
