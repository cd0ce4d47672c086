// HalftimeHash B200 engine: batch kernel for strings shorter than one
// instance (n_inst == 0; e.g. config 3, 1 KiB strings of the 32-byte
// variant).  For these the whole digest is
//   D_r = NH(n, S[F_r]) + sum_i NH(W_i, S[R + r + i])
// (hasher.py:400-412: finalize over the tag only, plus the Toeplitz tail).
//
// A half-warp hashes one string: lane g owns the 16-byte chunks g, g+16, ...
// staged through a per-warp cp.async.bulk ring (128-bit shared loads).
// The Toeplitz key words a lane needs are the same for every string, so they
// are loaded once into registers; the tag term is a launch constant computed
// on the host.  Per string the lanes' k partial sums are combined with a
// reduce-scatter (fewer shuffles than k full butterflies) and lane r writes
// digest word r.
#pragma once
#include "engine.cuh"

#ifndef HTH_TAIL_MINB
#define HTH_TAIL_MINB 2
#endif

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

// Per warp: a ring of NS stages, each one cp.async.bulk copy of GP PAIRS of
// consecutive strings (2 GP x stride bytes), so the loads stay deep in flight
// without holding registers and each copy is large enough to stream at full
// HBM rate.  MASKED: n % 16 != 0 (partial words / chunks).
template <int OUT, int CPT, bool MASKED, int NS, int GP>
__global__ void __launch_bounds__(256, HTH_TAIL_MINB) tail_kernel(const __grid_constant__ TailParams P) {
  constexpr int K = Var<OUT>::k;
  constexpr int KP = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane & 15, half = lane >> 4;
  const u64 n = P.n_bytes;
  const u32 nw = (u32)((n + 7) >> 3);
  const u32 nch = (u32)((n + 15) >> 4);
  const u32 pair_bytes = (u32)(2 * P.stride);
  const u32 SBY = (GP * pair_bytes + 127) & ~127u;
  uint8_t* ring = smem + (size_t)warp * NS * SBY;
  u64* bars = reinterpret_cast<u64*>(smem + (size_t)(blockDim.x >> 5) * NS * SBY) + warp * NS;
  if (lane == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
    fence_proxy_async();
  }
  __syncwarp();
  // Toeplitz keys for this lane's chunks: chunk c covers words 2c, 2c+1 and
  // needs S[R + 2c + r] for r <= K
  u32 klo[CPT][K + 1], khi[CPT][K + 1];
#pragma unroll
  for (int i = 0; i < CPT; i++) {
    const u32 c = (u32)g + 16u * i;
#pragma unroll
    for (int r = 0; r <= K; r++) {
      const u64 s = c < nch ? __ldg(P.S + P.R + 2 * c + r) : 0;
      klo[i][r] = (u32)s;
      khi[i][r] = (u32)(s >> 32);
    }
  }
  // MASKED: only the string's last chunk can be partial (chunks past it are
  // skipped), so two masks serve every lane: zero-padding of the final word
  // (hasher.py:179-183) and the word past the end
  const u64 lb0 = 16ull * (nch - 1), lb1 = lb0 + 8;
  const u64 lmask0 = lb0 + 8 <= n ? ~0ull : (1ull << (8 * (n - lb0))) - 1;
  const u64 lmask1 = lb1 >= n ? 0 : (lb1 + 8 <= n ? ~0ull : (1ull << (8 * (n - lb1))) - 1);
  const u64 NW = (u64)gridDim.x * (blockDim.x >> 5);
  const u64 w0 = (u64)blockIdx.x * (blockDim.x >> 5) + warp;
  const u64 pairs = (P.n_strings + 1) >> 1;
  const u64 groups = (pairs + GP - 1) / GP;
  const int myidx = scatter_index<K>(g);
  const u64 pol = policy_evict_first();
  const u64 total_bytes = (P.n_strings - 1) * P.stride + ((n + 15) & ~15ull);

  u64 pnext = w0;
  u32 pseq = 0;
  auto issue = [&]() {
    if (pnext >= groups) return;
    const u64 off = (u64)GP * pnext * pair_bytes;
    const u32 bytes = (u32)min((u64)GP * pair_bytes, total_bytes - off);
    const u32 slot = pseq % NS;
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[slot], bytes);
      bulk_g2s(ring + slot * SBY, P.data + off, bytes, &bars[slot], pol);
    }
    pseq++;
    pnext += NW;
  };
#pragma unroll
  for (int s = 0; s < NS; s++) issue();

  u32 cseq = 0;
  for (u64 gi = w0; gi < groups; gi += NW) {
    const u32 slot = cseq % NS;
    mbar_wait(&bars[slot], (cseq / NS) & 1);
#pragma unroll 1
    for (int gp = 0; gp < GP; gp++) {
      const u64 pr = gi * GP + gp;
      if (GP > 1 && pr >= pairs) break;
      const uint8_t* sb = ring + slot * SBY + (u32)gp * pair_bytes + (u32)half * (u32)P.stride;
      uint4 v[CPT];
#pragma unroll
      for (int i = 0; i < CPT; i++) {
        const u32 c = (u32)g + 16u * i;
        v[i] = (!MASKED || c < nch) ? *reinterpret_cast<const uint4*>(sb + 16u * c) : make_uint4(0, 0, 0, 0);
      }
      if (gp == GP - 1) {
        __syncwarp();
        issue();  // refill the slot just read
      }
      u64 acc[K];
#pragma unroll
      for (int r = 0; r < K; r++) acc[r] = 0;
#pragma unroll
      for (int i = 0; i < CPT; i++) {
        const u32 c = (u32)g + 16u * i;
        if (!MASKED || c < nch) {
          w2 x0 = {v[i].x, v[i].y}, x1 = {v[i].z, v[i].w};
          if (MASKED && c == nch - 1) {
            x0 = mk((((u64)v[i].y << 32) | v[i].x) & lmask0);
            x1 = mk((((u64)v[i].w << 32) | v[i].z) & lmask1);
          }
          const bool w1 = !MASKED || 2 * c + 1 < nw;
#pragma unroll
          for (int r = 0; r < K; r++) {
            acc[r] = nh_acc(acc[r], x0, klo[i][r], khi[i][r]);
            if (w1) acc[r] = nh_acc(acc[r], x1, klo[i][r + 1], khi[i][r + 1]);
          }
        }
      }
      const u64 tot = half_reduce_scatter<K>(acc, g);
      const u64 s = 2 * pr + half;
      if ((g & (16 / KP - 1)) == 0 && myidx < K && s < P.n_strings) P.out[s * K + myidx] = tot + P.tag[myidx];
    }
    cseq++;
  }
}

}  // namespace hth
