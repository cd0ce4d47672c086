// HalftimeHash B200 engine: the persistent warp-job hash kernel.
// See engine.cuh for the decomposition; reference citations inline.
#pragma once
#include "engine.cuh"

namespace hth {

// Little-endian u64 word `widx` of a stage whose first string byte sits at
// smem offset `delta` (0..15).  AL: delta % 8 == 0 (aligned LDS.64).
template <bool AL>
__device__ __forceinline__ u64 ld_word(const uint8_t* buf, u32 delta, u32 widx) {
  if (AL) return *reinterpret_cast<const u64*>(buf + delta + widx * 8u);
  u32 off = delta + widx * 8u;
  const u64* p = reinterpret_cast<const u64*>(buf + (off & ~7u));
  u32 sh = (off & 7u) * 8u;
  return (p[0] >> sh) | (p[1] << (64u - sh));
}

// Leaf of instance `q` of the stage, lane j -> C[r]   (hasher.py:356-364)
template <class V, bool AL>
__device__ __forceinline__ void stage_leaf(const uint8_t* buf, u32 delta, int q, int j, const u64* __restrict__ S,
                                           u64 (&C)[V::k]) {
  constexpr int M = Geo<V>::m;
  w2 X[V::d][V::w];
#pragma unroll
  for (int i = 0; i < V::d; i++)
#pragma unroll
    for (int u = 0; u < V::w; u++) X[i][u] = mk(ld_word<AL>(buf, delta, (u32)(q * M + (i * V::w + u) * 8 + j)));
  leaf<V>(X, S, C);
}

template <int K>
struct TreeCtx {
  u64 T[K], F[K], R;
};

// A finished block at level `lvl` >= 2, index `idx` (lanes 0-7 hold lane j
// of each row).  Either it is a leftover of its level -> finalize terms
// (tree.py:103-134), or it joins a complete group of 8 whose node the last
// arriving warp computes (nh.py:96-121 with level seeds, tree.py:55-60).
template <int K>
__device__ __forceinline__ u32 climb(const Params& P, const Str& st, const TreeCtx<K>& tc, int lvl, u64 idx,
                                      u64 (&B)[K], u64 (&fin)[K], int lane) {
  const int q = lane >> 3, j = lane & 7;
  const u64* __restrict__ S = P.S;
  for (;;) {
    const u64 len = st.n_inst >> (3 * lvl);
    if (idx >= (len & ~7ull)) {
      if (lane < 8) {
#pragma unroll
        for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], B[r], __ldg(S + tc.F[r] + 56ull * lvl + (idx & 7) * 8 + j));
      }
      return 1;
    }
    u64 woff = 0, coff = 0;
    for (int l = 2; l <= lvl; l++) {
      const u64 ln = st.n_inst >> (3 * l);
      if (l < lvl) woff += (ln & ~7ull) * 8ull * K;
      if (l >= 3) coff += ln;  // counters of levels 3..lvl precede level lvl+1's
    }
    u64* blk = P.scratch + st.scratch + woff;
    if (lane < 8) {
#pragma unroll
      for (int r = 0; r < K; r++) blk[idx * 8 * K + r * 8 + j] = B[r];
    }
    __threadfence();
    __syncwarp();
    u32 old = 0;
    u32* ctr = P.counters + st.cnt + coff + (idx >> 3);
    if (lane == 0) old = atomicAdd(ctr, 1u);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != 7) return 0;
    __threadfence();
    if (lane == 0) *ctr = 0;  // last arriver: leave the workspace zeroed
    u64* g = blk + (idx & ~7ull) * 8 * K;
#pragma unroll
    for (int r = 0; r < K; r++) {
      const u64 a = __ldcg(g + q * 8 * K + r * 8 + j);
      const u64 b = __ldcg(g + (q + 4) * 8 * K + r * 8 + j);
      g[q * 8 * K + r * 8 + j] = 0;  // consumed: leave the workspace zeroed
      g[(q + 4) * 8 * K + r * 8 + j] = 0;
      const u64* s = S + tc.T[r] + 7ull * lvl;
      u64 v = nh_acc(0, a, __ldg(s + q));
      v = (q < 3) ? nh_acc(v, b, __ldg(s + q + 4)) : v + b;
      v += shfl_xor(v, 8);
      v += shfl_xor(v, 16);
      B[r] = v;
    }
    lvl++;
    idx >>= 3;
  }
}

template <int OUT, bool VARLEN, int W, int NS>
__global__ void __launch_bounds__(W * 32) hash_kernel(const Params P) {
  using V = Var<OUT>;
  constexpr int K = V::k, M = Geo<V>::m;
  constexpr u32 CB = ROUND_INST * M * 8;  // stage payload bytes
  constexpr u32 SB = CB + 128;            // stage buffer (alignment + overread slack)
  extern __shared__ __align__(128) uint8_t smem[];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane >> 3, j = lane & 7;
  uint8_t* ring = smem + warp * NS * SB;
  u64* bars = reinterpret_cast<u64*>(smem + W * NS * SB) + warp * NS;
  if (lane == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
    fence_proxy_async();
  }
  __syncwarp();

  const u64 NW = (u64)gridDim.x * W;
  const u64 gw = (u64)blockIdx.x * W + warp;
  const u64 n_jobs = VARLEN ? P.meta[3 * P.n_strings] : P.n_jobs;
  const u64* __restrict__ S = P.S;
  const u64 pol = policy_evict_first();

  // ---- producer cursor (uniform across the warp; lane 0 issues) ----
  u64 pjob = gw;
  u32 pchunk = 0, pnchunks = 0, pseq = 0;
  const uint8_t* pbase = nullptr;
  u64 pbytes = 0;
  auto p_load = [&]() {
    Str st;
    u32 jq, ni;
    u64 b0;
    decode_job<VARLEN, K, M>(P, pjob, st, jq);
    job_span<M>(st, jq, b0, pbytes, ni);
    pbase = st.p + b0;
    pnchunks = (u32)ceil_div(pbytes, CB);
    pchunk = 0;
  };
  auto p_issue = [&]() {
    while (pjob < n_jobs && pchunk >= pnchunks) {
      pjob += NW;
      if (pjob < n_jobs) p_load();
    }
    if (pjob >= n_jobs) return;
    const u32 slot = pseq % NS;
    const uint8_t* src = pbase + (u64)pchunk * CB;
    const u64 len = min((u64)CB, pbytes - (u64)pchunk * CB);
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(src) + len + 15) & ~uintptr_t(15);
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[slot], (u32)(a1 - a0));
      bulk_g2s(ring + slot * SB, reinterpret_cast<const void*>(a0), (u32)(a1 - a0), &bars[slot], pol);
    }
    pseq++;
    pchunk++;
  };
  if (pjob < n_jobs) p_load();
  for (int s = 0; s < NS; s++) p_issue();

  // ---- consumer ----
  u32 cseq = 0;
  for (u64 job = gw; job < n_jobs; job += NW) {
    Str st;
    u32 jq, ninst;
    u64 byte0, nbytes;
    decode_job<VARLEN, K, M>(P, job, st, jq);
    job_span<M>(st, jq, byte0, nbytes, ninst);
    const u32 nchunks = (u32)ceil_div(nbytes, CB);
    const u32 delta = (u32)(reinterpret_cast<uintptr_t>(st.p) & 15);
    const bool last_job = (jq + 1 == st.J);
    TreeCtx<K> tc;
    layout_bases<K>(st.L, Geo<V>::ew, tc.T, tc.F, tc.R);

    u64 fin[K], n1[K], n2[K];
    u32 events = last_job ? 1u : 0u;
#pragma unroll
    for (int r = 0; r < K; r++) fin[r] = n1[r] = n2[r] = 0;
    const u64 inst0 = (u64)jq * JOB_INST;
    const u64 full0 = st.n_inst & ~7ull;      // level-0 blocks in complete groups
    const u64 len1 = st.n_inst >> 3;          // level-1 blocks
    const u64 full1 = len1 & ~7ull;

    for (u32 c = 0; c < nchunks; c++) {
      const u32 slot = cseq % NS;
      mbar_wait(&bars[slot], (cseq / NS) & 1);
      uint8_t* buf = ring + slot * SB;
      const bool tail_chunk = last_job && (c + 1 == nchunks);
      if (tail_chunk && (st.n & 7)) {
        // zero-pad the partial final word (hasher.py:179-183, 416-419)
        const u32 endpos = delta + (u32)(nbytes - (u64)c * CB);
        const u32 nz = 8 - (u32)(st.n & 7);
        if ((u32)lane < nz) buf[endpos + lane] = 0;
        fence_proxy_async();
        __syncwarp();
      }
      const u32 ri = c * ROUND_INST + q;
      if (ri < ninst) {
        u64 C[K];
        if (delta & 7)
          stage_leaf<V, false>(buf, delta, q, j, S, C);
        else
          stage_leaf<V, true>(buf, delta, q, j, S, C);
        const u64 g = inst0 + ri;
        const int pos = (int)(g & 7);
        if (g < full0) {
          // level-1 node term (nh_tree_node: last block added, not hashed)
#pragma unroll
          for (int r = 0; r < K; r++)
            n1[r] = (pos < 7) ? nh_acc(n1[r], C[r], __ldg(S + tc.T[r] + pos)) : n1[r] + C[r];
        } else {
          // level-0 leftover -> finalize slot (0, pos)
#pragma unroll
          for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], C[r], __ldg(S + tc.F[r] + pos * 8 + j));
        }
      }
      if (c & 1) {
        const u64 G1 = (inst0 >> 3) + (c >> 1);
        if (G1 < len1) {
          u64 B1[K];
#pragma unroll
          for (int r = 0; r < K; r++) {
            u64 v = n1[r];
            v += shfl_xor(v, 8);
            v += shfl_xor(v, 16);
            B1[r] = v;
            n1[r] = 0;
          }
          const int p1 = (int)(G1 & 7);
          if (G1 >= full1) {
            if (q == 0) {
#pragma unroll
              for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], B1[r], __ldg(S + tc.F[r] + 56 + p1 * 8 + j));
            }
          } else {
            if (q == 0) {
#pragma unroll
              for (int r = 0; r < K; r++)
                n2[r] = (p1 < 7) ? nh_acc(n2[r], B1[r], __ldg(S + tc.T[r] + 7 + p1)) : n2[r] + B1[r];
            }
            if (p1 == 7) {
              events += climb<K>(P, st, tc, 2, G1 >> 3, n2, fin, lane);
#pragma unroll
              for (int r = 0; r < K; r++) n2[r] = 0;
            }
          }
        }
      }
      if (tail_chunk) {
        // Toeplitz tail: Rem_r = sum_i NH(Y_i, S[R + r + i])  (hasher.py:407-412)
        const u64 tw0 = st.n_inst * M;
        const u64 nw = (st.n + 7) >> 3;
        const u32 cw0 = (u32)(tw0 - (inst0 * M + (u64)c * ROUND_INST * M));
        const u32 nt = (u32)(nw - tw0);
        for (u32 t = lane; t < nt; t += 32) {
          const u64 y = (delta & 7) ? ld_word<false>(buf, delta, cw0 + t) : ld_word<true>(buf, delta, cw0 + t);
#pragma unroll
          for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], y, __ldg(S + tc.R + r + t));
        }
      }
      __syncwarp();
      cseq++;
      p_issue();
    }

    if (last_job) {
      // zero slots and the length tag of the finalize NH (hasher.py:387-405)
      if (st.n_inst) {
        const u32 nz = 56u * st.L;
        for (u32 x = (u32)lane; x < nz; x += 32) {
          const u32 l = x / 56u, slot = (x % 56u) >> 3;
          if (slot >= (u32)((st.n_inst >> (3 * l)) & 7)) {
#pragma unroll
            for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], 0ull, __ldg(S + tc.F[r] + x));
          }
        }
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], st.n, __ldg(S + tc.F[r] + nz));
        }
      } else if (lane == 0) {
#pragma unroll
        for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], st.n, __ldg(S + tc.F[r]));
      }
    }
    u64 mine = 0;
#pragma unroll
    for (int r = 0; r < K; r++) {
      const u64 v = warp_sum(fin[r]);
      if (lane == r) mine = v;
    }
    if (st.J == 1) {
      if (lane < K) P.out[st.s * K + lane] = mine;
    } else if (events) {
      // multi-job string: add this job's finalize terms, then count its
      // events; the warp completing the count publishes the digest and
      // re-zeroes the accumulators (integer sums: order-independent).
      unsigned long long* a = reinterpret_cast<unsigned long long*>(P.acc + st.s * K);
      if (lane < K) atomicAdd(a + lane, (unsigned long long)mine);
      __threadfence();
      __syncwarp();
      u32 old = 0;
      if (lane == 0) old = atomicAdd(P.events + st.s, events);
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old + events == string_events(st.n_inst)) {
        __threadfence();
        if (lane < K) P.out[st.s * K + lane] = atomicExch(a + lane, 0ull);
        if (lane == 0) P.events[st.s] = 0;
      }
    }
  }
}

}  // namespace hth
