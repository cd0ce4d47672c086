// HalftimeHash B200 engine: the varlen planning kernel (also hashes the
// strings shorter than one instance).
#pragma once
#include "tail_kernel.cuh"

namespace hth {

// Varlen plan + short strings (one kernel).  One half-warp per string: lane
// 0 plans it -- a string of >= 1 instance appends its jobs to the queue of
// their size class (min(instances, 64)), which the hash kernel claims largest
// class first (LPT scheduling with dynamic claiming) -- and a string shorter
// than one instance is hashed right here by its 16 lanes:
//   D_r = NH(n, S[F_r]) + sum_i NH(W_i, S[R + r + i])   (hasher.py:400-412)
// with the Toeplitz keys staged in shared memory.  Queue order inside a class
// and the scratch/counter bases of multi-job strings come from atomics:
// digests are integer sums and do not depend on them.  The grid's first
// threads also build the zero-slot table (ztab_base).  err bit 1: a string
// longer than max_n; bit 2: more instances than the declared total (the
// queues would overflow; the job is dropped); bit 4: offsets decreasing or
// past total_bytes (the string is hashed as empty).  Any set bit means the
// call's digests are invalid: hth_varlen_status reports it.
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
  u32* cls_cnt;
  u64* queues;
  u64* meta;
  unsigned long long* totals;
  u64* ztab;
  QueueTable Q;
};
template <int OUT>
__global__ void __launch_bounds__(256) plan_tail_kernel(const __grid_constant__ PlanParams P) {
  constexpr int K = Var<OUT>::k, M = Geo<Var<OUT>>::m, EW = Geo<Var<OUT>>::ew;
  constexpr int KP = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
  constexpr int NKEY = M + K;  // Toeplitz keys R .. R + m + k - 2, plus slack
  __shared__ u64 key[NKEY];
  __shared__ u64 tagseed[K];
  // this half-warp's first string bounds, loaded before the key staging so
  // the two latencies overlap
  const u64 s_first = (u64)blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4);
  const u64 f_o0 = s_first < P.n ? P.off[s_first] : 0;
  const u64 f_o1 = s_first < P.n ? P.off[s_first + 1] : 0;
  for (int i = threadIdx.x; i < NKEY; i += blockDim.x) key[i] = __ldg(P.S + P.R + i);
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
  const int lane = threadIdx.x & 31, g = lane & 15;
  const int myidx = scatter_index<K>(g);
  const u64 per = 1ull << (3 * P.job_lvl);
  const u64 halves = (u64)gridDim.x * (blockDim.x >> 4);
  // both halves of a warp iterate together (the reduction shuffles are warp-wide)
  for (u64 s = (u64)blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); s < ((P.n + 1) & ~1ull); s += halves) {
    const bool live = s < P.n;
    const bool first = s == s_first;
    const u64 o0 = live ? (first ? f_o0 : P.off[s]) : 0;
    const u64 o1 = live ? (first ? f_o1 : P.off[s + 1]) : 0;
    u64 n = o1 - o0;
    if (o1 < o0 || o1 > P.total) {
      if (g == 0) atomicOr(P.err, 4);
      n = 0;
    }
    if (n > P.max_n) {
      if (g == 0) atomicOr(P.err, 1);
      n = P.max_n;
    }
    const u64 ni = ((n + 7) >> 3) / M;
    const bool tail = live && ni == 0;
    if (live && !tail && g == 0) {
      const u64 J = job_count(ni, P.job_lvl);
      u64 w, c;
      scratch_need(ni, K, P.job_lvl, &w, &c);
      P.meta[2 * s] = w ? atomicAdd(P.totals, (unsigned long long)w) : 0;
      P.meta[2 * s + 1] = c ? atomicAdd(P.totals + 1, (unsigned long long)c) : 0;
      for (u64 q = 0; q < J; q++) {
        const u64 jn = min(per, ni - q * per);
        const int cl = jn > 64 ? 64 : (int)jn;
        const u32 pos = atomicAdd(P.cls_cnt + cl, 1u);
        if (pos < P.Q.qb[cl + 1] - P.Q.qb[cl]) {
          u64* rec = P.queues + (P.Q.qb[cl] + pos) * JOB_REC;  // the job's record (decode_job)
          rec[0] = o0;
          rec[1] = n;
          rec[2] = s | (q << 32);
          rec[3] = 0;
        } else {
          atomicSub(P.cls_cnt + cl, 1u);
          atomicOr(P.err, 2);
        }
      }
    }
    if (!__any_sync(0xffffffffu, tail)) continue;
    u64 acc[K];
#pragma unroll
    for (int r = 0; r < K; r++) acc[r] = 0;
    const u32 nw = tail ? (u32)((n + 7) >> 3) : 0;
    for (u32 t = g; t < nw; t += 16) {
      // absolute address: the buffer base itself may be unaligned
      const u64 b = reinterpret_cast<u64>(P.data) + o0 + 8ull * t;
      const u64* p = reinterpret_cast<const u64*>(b & ~7ull);
      const u32 sh = (u32)(b & 7) * 8;
      const u64 rem = n - 8ull * t;
      u64 x = __ldg(p) >> sh;
      // the next aligned word only if the string reaches into it (no over-read)
      if (sh && rem > 8 - (b & 7)) x |= __ldg(p + 1) << (64 - sh);
      if (rem < 8) x &= (1ull << (8 * rem)) - 1;  // zero-pad the partial last word (hasher.py:179-183)
#pragma unroll
      for (int r = 0; r < K; r++) acc[r] = nh_acc(acc[r], x, key[t + r]);
    }
    if (g == 0 && tail) {
#pragma unroll
      for (int r = 0; r < K; r++) acc[r] = nh_acc(acc[r], n, tagseed[r]);  // finalize over the tag
    }
    const u64 tot = half_reduce_scatter<K>(acc, g);
    if (tail && (g & (16 / KP - 1)) == 0 && myidx < K) P.out[s * K + myidx] = tot;
  }
}

}  // namespace hth
