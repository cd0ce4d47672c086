// HalftimeHash B200 engine: batch kernel for strings shorter than one
// instance (n_inst == 0; e.g. config 3, 1 KiB strings of the 32-byte
// variant).  For these the whole digest is
//   D_r = NH(n, S[F_r]) + sum_i NH(W_i, S[R + r + i])
// (hasher.py:400-412: finalize over the tag only, plus the Toeplitz tail).
//
// A half-warp hashes one string: lane g owns the 16-byte chunks g, g+16, ...
// (coalesced 128-bit loads, 256 contiguous bytes per half-warp per load).
// The Toeplitz key words a lane needs are the same for every string, so they
// are loaded once into registers; the tag term is a launch constant computed
// on the host.  Per string the lanes' k partial sums are combined with a
// reduce-scatter (fewer shuffles than k full butterflies) and lane r writes
// digest word r.
#pragma once
#include "engine.cuh"

namespace hth {

struct TailParams {
  const uint8_t* data;
  u64 n_strings;
  u64 stride;  // multiple of 16
  u64 n_bytes;
  const u64* S;
  u64 R;  // remainder-region start (layout with L' = 1)
  u64* out;
  u64 tag[5];  // NH(n, S[F_r]) per output word
};

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
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

template <int OUT, int CPT>
__global__ void __launch_bounds__(256, 2) tail_kernel(const __grid_constant__ TailParams P) {
  constexpr int K = Var<OUT>::k;
  const int lane = threadIdx.x & 31, g = lane & 15, half = lane >> 4;
  const u64 n = P.n_bytes;
  const u32 nw = (u32)((n + 7) >> 3);
  const u32 nch = (u32)((n + 15) >> 4);
  // Toeplitz keys for this lane's chunks: chunk c covers words 2c, 2c+1 and
  // needs S[R + 2c + r] for r <= K
  u32 klo[CPT][K + 1], khi[CPT][K + 1];
  u64 mask0[CPT], mask1[CPT];  // zero-padding / words past the end
#pragma unroll
  for (int i = 0; i < CPT; i++) {
    const u32 c = (u32)g + 16u * i;
#pragma unroll
    for (int r = 0; r <= K; r++) {
      const u64 s = c < nch ? __ldg(P.S + P.R + 2 * c + r) : 0;
      klo[i][r] = (u32)s;
      khi[i][r] = (u32)(s >> 32);
    }
    const u64 b0 = 16ull * c, b1 = b0 + 8;
    mask0[i] = b0 >= n ? 0 : (b0 + 8 <= n ? ~0ull : (1ull << (8 * (n - b0))) - 1);
    mask1[i] = b1 >= n ? 0 : (b1 + 8 <= n ? ~0ull : (1ull << (8 * (n - b1))) - 1);
  }
  const u64 warps = (u64)gridDim.x * (blockDim.x >> 5);
  const u64 w0 = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const u64 pairs = (P.n_strings + 1) >> 1;
  const int myidx = scatter_index<K>(g);

  uint4 cur[CPT], nxt[CPT];
  auto load = [&](u64 pr, uint4 (&dst)[CPT]) {
    const u64 s = 2 * pr + half;
    const uint8_t* base = P.data + s * P.stride;
#pragma unroll
    for (int i = 0; i < CPT; i++) {
      const u32 c = (u32)g + 16u * i;
      dst[i] = (s < P.n_strings && c < nch) ? ldg_stream(base + 16ull * c) : make_uint4(0, 0, 0, 0);
    }
  };
  if (w0 < pairs) load(w0, cur);
  for (u64 pr = w0; pr < pairs; pr += warps) {
    if (pr + warps < pairs) load(pr + warps, nxt);
    u64 acc[K];
#pragma unroll
    for (int r = 0; r < K; r++) acc[r] = 0;
#pragma unroll
    for (int i = 0; i < CPT; i++) {
      const u32 c = (u32)g + 16u * i;
      if (c < nch) {
        const u64 x0 = (((u64)cur[i].y << 32) | cur[i].x) & mask0[i];
        const u64 x1 = (((u64)cur[i].w << 32) | cur[i].z) & mask1[i];
        const bool w1 = 2 * c + 1 < nw;
#pragma unroll
        for (int r = 0; r < K; r++) {
          acc[r] = nh_acc(acc[r], mk(x0), klo[i][r], khi[i][r]);
          if (w1) acc[r] = nh_acc(acc[r], mk(x1), klo[i][r + 1], khi[i][r + 1]);
        }
      }
    }
    const u64 tot = half_reduce_scatter<K>(acc, g);
    const u64 s = 2 * pr + half;
    constexpr int KP = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
    if ((g & (16 / KP - 1)) == 0 && myidx < K && s < P.n_strings) P.out[s * K + myidx] = tot + P.tag[myidx];
#pragma unroll
    for (int i = 0; i < CPT; i++) cur[i] = nxt[i];
  }
}

}  // namespace hth
