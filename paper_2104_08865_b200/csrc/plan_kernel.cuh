// HalftimeHash B200 engine: the varlen planning kernel (also hashes the
// strings shorter than one instance).
#pragma once
#include "tail_kernel.cuh"

namespace hth {

// Varlen plan + the strings shorter than one instance (one kernel).  Each
// warp plans HTH_PLAN_SPW strings, one per lane: a string of >= 1 instance
// appends its jobs to the queue of their size class (min(instances, 64)),
// which the hash kernel claims largest class first (LPT scheduling with
// dynamic claiming); every queue position and scratch/counter base comes
// from one atomic per warp (warp scans and __match_any_sync groups) --
// digests are integer sums and do not depend on the order.  The warp then
// hashes its strings shorter than one instance, two at a time (one
// half-warp each, all words loaded before any is hashed):
//   D_r = NH(n, S[F_r]) + sum_i NH(W_i, S[R + r + i])   (hasher.py:400-412)
// with the Toeplitz keys staged in shared memory.  Few strings per warp keep
// the whole batch in flight at once, so the kernel costs a handful of
// memory round trips.  The grid's first threads also build the zero-slot
// table (ztab_base).  err bit 1: a string longer than max_n; bit 2: a class
// queue overflowed (the job is dropped); bit 4: offsets decreasing or past
// total_bytes (the string is hashed as empty).  Any set bit means the call's
// digests are invalid: hth_varlen_status reports (and clears) the bits.
#ifndef HTH_PLAN_SPW
#define HTH_PLAN_SPW 4
#endif
#ifndef HTH_PLAN_MINB
#define HTH_PLAN_MINB 4
#endif
#ifndef HTH_PLAN_TRIGGER_EARLY
#define HTH_PLAN_TRIGGER_EARLY 0
#endif
struct QueueTable {
  u64 qb[NCLS + 1];  // queue c occupies job_map[qb[c], qb[c+1])
};
struct PlanParams {
  const uint8_t* data;
  const u64* off;
  u64 n, max_n, total;
  int job_lvl;
  u32 lmax;
  const u64* S;
  u64 R, F0;  // L' = 1 layout: remainder start, finalize start of row 0 (row stride 64)
  u64* out;
  int* err;
  u32* cls_cnt;  // [NCLS] jobs per class
  u64* queues;
  unsigned long long* totals;  // scratch words, counters handed out so far
  u64* ztab;
  QueueTable Q;
};
// a job record {byte offset, length, string | job index << 32, merge bases}:
// merge bases = scratch word base (40 bits) | counter base << 40
__device__ __forceinline__ void put_job(const PlanParams& P, int cl, u64 pos, u64 o0, u64 n, u64 s, u64 q, u64 meta) {
  if (pos < P.Q.qb[cl + 1] - P.Q.qb[cl]) {
    u64* rec = P.queues + (P.Q.qb[cl] + pos) * JOB_REC;
    rec[0] = o0;
    rec[1] = n;
    rec[2] = s | (q << 32);
    rec[3] = meta;
  } else {
    atomicSub(P.cls_cnt + cl, 1u);
    atomicOr(P.err, 2);
  }
}
template <class T>
__device__ __forceinline__ T warp_incl_scan(T x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  return x;
}
template <int OUT>
__global__ void __launch_bounds__(256, HTH_PLAN_MINB) plan_kernel(const __grid_constant__ PlanParams P) {
  constexpr int K = Var<OUT>::k, M = Geo<Var<OUT>>::m, EW = Geo<Var<OUT>>::ew;
  constexpr int KP = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
  constexpr int SPW = HTH_PLAN_SPW;
  static_assert(SPW >= 1 && SPW <= 32, "strings per warp");
  __shared__ u64 key[M + K - 1];  // Toeplitz keys R .. R + m + k - 2 (the end of the L' = 1 layout)
  __shared__ u64 tagseed[K];
#if HTH_PLAN_TRIGGER_EARLY
  // let the hash kernel (a programmatic dependent) start its prologue now;
  // it waits for this grid's completion before reading the plan
  asm volatile("griddepcontrol.launch_dependents;");
#endif
  const int lane = threadIdx.x & 31;
  const u64 gwarp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  // this lane's first string bounds, loaded before the key staging so the
  // two latencies overlap
  const u64 s_first = gwarp * SPW + lane;
  const bool f_live = lane < SPW && s_first < P.n;
  const u64 f_o0 = f_live ? P.off[s_first] : 0;
  const u64 f_o1 = f_live ? P.off[s_first + 1] : 0;
  for (int i = threadIdx.x; i < M + K - 1; i += blockDim.x) key[i] = __ldg(P.S + P.R + i);
  if (threadIdx.x < K) tagseed[threadIdx.x] = __ldg(P.S + P.F0 + 64ull * threadIdx.x);
  // zero-slot table: one thread per (L, l, r) sums its 7 slots and writes the
  // suffix sums for digits 0..7
  const u64 nz = (u64)K * P.lmax * P.lmax;
  for (u64 x = (u64)blockIdx.x * blockDim.x + threadIdx.x; x < nz; x += (u64)gridDim.x * blockDim.x) {
    const u32 r = (u32)(x % K), l = (u32)(x / K % P.lmax), L = (u32)(x / K / P.lmax) + 1;
    if (l >= L) continue;
    const u64 F = (u64)EW + 7ull * L * K + 64ull * L * r + 56ull * l;  // seed_layout (hasher.py:130-153)
    u64* z = P.ztab + ztab_base(L, K) + (u64)l * 8 * K + r;
    u64 part[7];  // all 56 seed loads in flight at once
#pragma unroll
    for (int slot = 0; slot < 7; slot++) {
      part[slot] = 0;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const u64 sw = __ldg(P.S + F + 8 * slot + j);
        part[slot] += (u64)(u32)sw * (u64)(u32)(sw >> 32);  // NH(0, s)
      }
    }
    u64 acc = 0;
    z[7 * K] = 0;
#pragma unroll
    for (int slot = 6; slot >= 0; slot--) {
      acc += part[slot];
      z[slot * K] = acc;
    }
  }
  __syncthreads();
  const u32 lt = (1u << lane) - 1;
  const int g = lane & 15, half = lane >> 4;
  const int myidx = scatter_index<K>(g);
  const u64 per = 1ull << (3 * P.job_lvl);  // >= 64: every job but a string's last is class 64
  for (u64 base = gwarp * SPW; base < P.n; base += nwarps * SPW) {
    const u64 s = base + lane;
    const bool live = lane < SPW && s < P.n;
    const bool first = base == gwarp * SPW;
    u64 o0 = 0, o1 = 0;
    if (live) {
      o0 = first ? f_o0 : P.off[s];
      o1 = first ? f_o1 : P.off[s + 1];
    }
    u64 n = o1 - o0;
    if (live && (o1 < o0 || o1 > P.total)) {
      atomicOr(P.err, 4);
      n = 0;
    }
    if (n > P.max_n) {
      atomicOr(P.err, 1);
      n = P.max_n;
    }
    const u64 ni = ((n + 7) >> 3) / M;
    const bool tail = live && ni == 0;
    const u64 J = (live && ni) ? job_count(ni, P.job_lvl) : 0;
    if (__any_sync(0xffffffffu, J != 0)) {
    // merge scratch / counter bases of multi-job strings
    u64 w = 0, c = 0;
    if (J > 1) scratch_need(ni, K, P.job_lvl, &w, &c);
    const u64 wx = warp_incl_scan(w, lane), cx = warp_incl_scan(c, lane);
    u64 wb = 0, cb = 0;
    if (lane == 31) {
      if (wx) wb = atomicAdd(P.totals, (unsigned long long)wx);
      if (cx) cb = atomicAdd(P.totals + 1, (unsigned long long)cx);
    }
    wb = __shfl_sync(0xffffffffu, wb, 31) + wx - w;
    cb = __shfl_sync(0xffffffffu, cb, 31) + cx - c;
    const u64 meta = J > 1 ? (wb | (cb << 40)) : 0;
    // class-64 jobs: one atomic per warp
    const u64 last_ni = J ? ni - (J - 1) * per : 0;
    // (a multi-job string's small last job stays out of the pairable classes)
    const int cl_last = last_ni >= 64 ? 64 : (J > 1 && last_ni <= PAIR_MAX ? PAIR_MAX + 1 : (int)last_ni);
    const u64 n64 = J ? (J - 1) + (cl_last == 64 ? 1 : 0) : 0;
    const u64 x64 = warp_incl_scan(n64, lane);
    u64 b64 = 0;
    if (lane == 31 && x64) b64 = atomicAdd(P.cls_cnt + 64, (u32)x64);
    b64 = __shfl_sync(0xffffffffu, b64, 31) + x64 - n64;
    // last jobs of classes 1..63: one atomic per class present in the warp
    const bool small_last = J && cl_last < 64;
    const u32 grp = __match_any_sync(0xffffffffu, small_last ? cl_last : 0);
    if (small_last) {
      const int leader = __ffs(grp) - 1;
      u32 b = 0;
      if (lane == leader) b = atomicAdd(P.cls_cnt + cl_last, (u32)__popc(grp));
      b = __shfl_sync(grp, b, leader);
      put_job(P, cl_last, b + __popc(grp & lt), o0, n, s, J - 1, meta);
    }
    if (n64 <= 4) {
      for (u64 q = 0; q < n64; q++) put_job(P, 64, b64 + q, o0, n, s, q, meta);
    }
    // long strings: the whole warp writes their class-64 records
    u32 big = __ballot_sync(0xffffffffu, n64 > 4);
    while (big) {
      const int l = __ffs(big) - 1;
      big &= big - 1;
      const u64 cnt = __shfl_sync(0xffffffffu, n64, l), b = __shfl_sync(0xffffffffu, b64, l);
      const u64 lo0 = __shfl_sync(0xffffffffu, o0, l), ln = __shfl_sync(0xffffffffu, n, l);
      const u64 lm = __shfl_sync(0xffffffffu, meta, l);
      for (u64 q = lane; q < cnt; q += 32) put_job(P, 64, b + q, lo0, ln, base + l, q, lm);
    }
    }
    // this warp's strings shorter than one instance, two at a time
    constexpr int WPL = (M + 15) / 16;  // n < 8m: at most m words, 16 lanes
    u32 tb = __ballot_sync(0xffffffffu, tail);
    while (tb) {
      const int l0 = __ffs(tb) - 1;
      tb &= tb - 1;
      const int l1 = tb ? __ffs(tb) - 1 : -1;
      if (tb) tb &= tb - 1;
      const int my = half ? l1 : l0;
      const bool ok = my >= 0;
      const int src = ok ? my : 0;
      const u64 so0 = __shfl_sync(0xffffffffu, o0, src);
      const u64 sn_ = __shfl_sync(0xffffffffu, n, src);
      const u64 sn = ok ? sn_ : 0;
      const u64 nw = (sn + 7) >> 3;
      u64 x[WPL];
#pragma unroll
      for (int k = 0; k < WPL; k++) {
        const u64 t = g + 16 * k;
        x[k] = t < nw ? gword(P.data, so0, sn, t) : 0;
      }
      u64 acc[K];
#pragma unroll
      for (int r = 0; r < K; r++) acc[r] = 0;
#pragma unroll
      for (int k = 0; k < WPL; k++) {
        const u64 t = g + 16 * k;
        if (t < nw) {
#pragma unroll
          for (int r = 0; r < K; r++) acc[r] = nh_acc(acc[r], x[k], key[t + r]);
        }
      }
      if (g == 0 && ok) {
#pragma unroll
        for (int r = 0; r < K; r++) acc[r] = nh_acc(acc[r], sn, tagseed[r]);  // finalize over the tag
      }
      const u64 tot = half_reduce_scatter<K>(acc, g);
      if (ok && (g & (16 / KP - 1)) == 0 && myidx < K) P.out[(base + my) * K + myidx] = tot;
    }
  }
#if !HTH_PLAN_TRIGGER_EARLY
  // this CTA is done: once every CTA got here the hash kernel (a
  // programmatic dependent) may start its prologue; it waits for this
  // grid's completion and memory before reading the plan
  asm volatile("griddepcontrol.launch_dependents;");
#endif
}

}  // namespace hth
