// HalftimeHash B200 engine: top-of-tree merge for one string hashed in
// slices (config 5 across GPUs).  Each slice (hth_hash_slice) leaves its
// finished, non-leftover level-c subtree roots ("frontier") and a partial
// digest.  This kernel continues the reference's stack construction from
// level c over the gathered frontier (tree.py:63-100, level seeds
// tree.py:55-60), adds the finalize terms of the leftovers it produces
// (tree.py:103-134) and the slices' partials, and writes the digest.
#pragma once
#include "engine.cuh"

namespace hth {

struct MergeParams {
  u64 n_bytes;
  int c;                 // frontier level
  const u64* frontier;   // nf blocks [idx][r][lane] at level c, global order
  u64 nf;                // = (n_inst >> 3c) & ~7
  const u64* partials;   // np x k partial digests
  u64 np;
  const u64* S;
  u64* tmp;              // nf/8 * 8k words scratch (ping-pong half)
  u64* out;              // k words
  // in-stream exchange (optional): wait until flags[0..nflags) >= epoch
  // (stored by the slices' kernels, possibly on other GPUs), then merge,
  // re-zero the partials for the slot's next use and release *consumed =
  // epoch.  A wait longer than timeout_ns sets *status = 1 (no hang).
  const unsigned long long* flags;
  u64 nflags, epoch, timeout_ns;
  unsigned long long* consumed;
  u64* partials_rw;
  int* status;
};

// One CTA of MERGE_TPB threads; every level is one wave of independent
// 8-block nodes (8 loads in flight per thread).  Levels above the frontier
// stay in shared memory when they fit (ping-pong: the level above the
// frontier, then 1/8 of it), else in the global tmp buffer.
constexpr int MERGE_TPB = 1024;
constexpr size_t MERGE_SMEM_MAX = 96 * 1024;

template <int K>
__host__ __device__ __forceinline__ size_t merge_level_bytes(u64 nf) {
  return (size_t)(nf / 8) * 8 * K * 8;
}
template <int K>
__host__ __device__ __forceinline__ size_t merge_smem_bytes(u64 nf) {
  const size_t a = merge_level_bytes<K>(nf);
  return a + a / 8 + 8 * K * 8 <= MERGE_SMEM_MAX ? a + a / 8 + 8 * K * 8 : 0;
}

template <int OUT>
__global__ void __launch_bounds__(MERGE_TPB) merge_kernel(const __grid_constant__ MergeParams P) {
  constexpr int K = Var<OUT>::k, M = Geo<Var<OUT>>::m, EW = Geo<Var<OUT>>::ew;
  extern __shared__ __align__(16) u64 msm[];
  __shared__ unsigned long long red[K];
  const u64 n_inst = ((P.n_bytes + 7) >> 3) / M;
  const u64 L = n_inst ? level_count(n_inst) : 1;
  u64 fin[K];
#pragma unroll
  for (int r = 0; r < K; r++) fin[r] = 0;
  if (threadIdx.x < K) red[threadIdx.x] = 0;
  if (P.flags) {
    // acquire each slice's arrival; the barrier below orders every other
    // thread's reads after these acquires
    for (u64 i = threadIdx.x; i < P.nflags; i += blockDim.x)
      if (!wait_geq_sys(P.flags + i, P.epoch, P.timeout_ns)) atomicExch(P.status, 1);
  }
  const bool in_smem = merge_smem_bytes<K>(P.nf) != 0;
  const size_t first = merge_level_bytes<K>(P.nf) / 8 + 8 * K;  // words of the level above the frontier
  u64* bufs[2] = {in_smem ? msm : P.tmp, in_smem ? msm + first : P.tmp + (P.nf / 8 + 8) * 8 * K};
  const u64* cur = P.frontier;
  u64 nf = P.nf;
  int lvl = P.c, flip = 0;
  __syncthreads();
  while (nf >= 8) {
    const u64 nn = nf / 8, keep = nn & ~7ull;  // nodes at lvl+1; complete-group ones carry on
    u64* nxt = bufs[flip];
    const bool from_frontier = lvl == P.c;
    for (u64 it = threadIdx.x; it < nn * K * 8; it += blockDim.x) {
      const u64 g = it / (K * 8);
      const int r = (int)((it / 8) % K), j = (int)(it % 8);
      const u64* blk = cur + g * 8 * 8 * K + r * 8 + j;
      const u64* s = P.S + (u64)EW + 7ull * L * r + 7ull * lvl;
      u64 x[8];
      if (from_frontier) {  // may have arrived from peer GPUs: read through L2
#pragma unroll
        for (int q = 0; q < 8; q++) x[q] = __ldcg(blk + q * 8 * K);
      } else {
#pragma unroll
        for (int q = 0; q < 8; q++) x[q] = blk[q * 8 * K];
      }
      u64 v = x[7];
#pragma unroll
      for (int q = 0; q < 7; q++) v = nh_acc(v, x[q], __ldg(s + q));
      if (g >= keep) {  // leftover at level lvl+1 -> finalize slot
        const u64 F = (u64)EW + 7ull * L * K + 64ull * L * r;
#pragma unroll
        for (int rr = 0; rr < K; rr++)
          if (rr == r) fin[rr] = nh_acc(fin[rr], v, __ldg(P.S + F + 56ull * (lvl + 1) + (g & 7) * 8 + j));
      } else {
        nxt[g * 8 * K + r * 8 + j] = v;
      }
    }
    __syncthreads();
    cur = nxt;
    flip ^= 1;
    nf = keep;
    lvl++;
  }
#pragma unroll
  for (int r = 0; r < K; r++)
    if (fin[r]) atomicAdd(&red[r], (unsigned long long)fin[r]);
  __syncthreads();
  if (threadIdx.x < K) {
    u64 v = red[threadIdx.x];
    for (u64 p = 0; p < P.np; p++) v += __ldcg(P.partials + p * K + threadIdx.x);
    P.out[threadIdx.x] = v;
  }
  if (P.flags) {
    // the slot is consumed: zero its partials (the slices accumulate into
    // them next time), then hand it back to the producers
    __syncthreads();
    if (P.partials_rw)
      for (u64 i = threadIdx.x; i < P.np * K; i += blockDim.x) P.partials_rw[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(P.consumed, P.epoch);
    }
  }
}

}  // namespace hth
