// HalftimeHash B200 engine: the persistent warp-job hash kernel.
// Decomposition and invariants: engine.cuh.  Reference citations inline.
#pragma once
#include <type_traits>
#include "engine.cuh"

#ifndef HTH_STATIC_FIRST
#define HTH_STATIC_FIRST 1
#endif
#ifndef HTH_S1_REGS
#define HTH_S1_REGS 1
#endif

namespace hth {

#ifdef HTH_DEBUG_TIMING
// experiment builds only: per warp {start, end, jobs, rounds, data-wait, valid, claim, decode, rounds, finish} (ns)
// into P.dbg (8192 warps x 10)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// Little-endian u64 word `widx` of a stage whose first string byte sits at
// smem offset `delta` (0..15).  AL: delta % 8 == 0 (aligned LDS.64).
// Unaligned: three 32-bit shared loads and two funnel shifts (SHF.R.W) for
// any byte offset (a shift of 0 passes the first operand through).
template <bool AL>
__device__ __forceinline__ u64 ld_word(const uint8_t* buf, u32 delta, u32 widx) {
  if (AL) return *reinterpret_cast<const u64*>(buf + delta + widx * 8u);
  const u32 off = delta + widx * 8u;
  const u32* p = reinterpret_cast<const u32*>(buf + (off & ~3u));
  const u32 sh = (off & 3u) * 8u;
  const u32 lo = __funnelshift_r(p[0], p[1], sh), hi = __funnelshift_r(p[1], p[2], sh);
  return ((u64)hi << 32) | lo;
}

template <int OUT>
__device__ __forceinline__ void enc_planes(const u32 (&x)[4 * Var<OUT>::d], u32 (&y)[4 * (Var<OUT>::e - Var<OUT>::d)]) {
  if constexpr (OUT == 24) enc_planes_24(x, y);
  if constexpr (OUT == 32) enc_planes_32(x, y);
  if constexpr (OUT == 40) enc_planes_40(x, y);
}

template <int C>
__device__ __forceinline__ u64 mac_sw(u64 acc, u64 h) {
  return mac_const<C>(acc, h);
}
// acc += c * h for a coefficient c known after unrolling (params.py:17-27
// shift/add forms; here two IMADs each)
__device__ __forceinline__ u64 mac_coef(int c, u64 acc, u64 h) {
  switch (c) {
    case 1: return mac_sw<1>(acc, h);
    case 2: return mac_sw<2>(acc, h);
    case 3: return mac_sw<3>(acc, h);
    case 4: return mac_sw<4>(acc, h);
    case 5: return mac_sw<5>(acc, h);
    case 7: return mac_sw<7>(acc, h);
    case 8: return mac_sw<8>(acc, h);
    case 9: return mac_sw<9>(acc, h);
    default: return acc;
  }
}

// EHC seed words: constant-bank kernel parameters (one seed for the launch)
// or, PERSEED, the job's words staged in shared memory.
template <bool PERSEED, int OUT>
struct EhcSrc {
  const Params& P;
  const u32* sm;
  static constexpr int E = Var<OUT>::e, WB = Var<OUT>::w;
  __device__ __forceinline__ u32 lo(int i) const {
    return PERSEED ? sm[2 * ehc_slot(i, E, WB)] : P.ehc[2 * ehc_slot(i, E, WB)];
  }
  __device__ __forceinline__ u32 hi(int i) const {
    return PERSEED ? sm[2 * ehc_slot(i, E, WB) + 1] : P.ehc[2 * ehc_slot(i, E, WB) + 1];
  }
};

// EHC leaf of two instances, lane j -> CA[r], CB[r] (hasher.py:356-364;
// ehc.py:102-118).  offA/offB: word offset of lane j's first word of each
// instance relative to its string's first byte, which sits at stage byte
// dA / dB (the two instances may belong to different strings).
template <int OUT, bool AL, class EH>
__device__ __forceinline__ void leaf2o(const uint8_t* buf, u32 dA, u32 offA, u32 dB, u32 offB, const EH& P,
                                       u64 (&CA)[Var<OUT>::k], u64 (&CB)[Var<OUT>::k]) {
  using V = Var<OUT>;
  constexpr int K = V::k, E = V::e, D = V::d, WB = V::w, NP = E - D;
  u64 HA[E], HB[E];
#pragma unroll
  for (int i = 0; i < E; i++) HA[i] = HB[i] = 0;
#pragma unroll
  for (int u = 0; u < WB; u++) {
    w2 xa[D], xb[D];
#pragma unroll
    for (int i = 0; i < D; i++) {
      xa[i] = mk(ld_word<AL>(buf, dA, offA + (i * WB + u) * 8));
      xb[i] = mk(ld_word<AL>(buf, dB, offB + (i * WB + u) * 8));
    }
    // hash the systematic items (ehc.py:49-72); seeds are constant-bank operands
#pragma unroll
    for (int i = 0; i < D; i++) {
      HA[i] = nh_acc(HA[i], xa[i], P.lo(i * WB + u), P.hi(i * WB + u));
      HB[i] = nh_acc(HB[i], xb[i], P.lo(i * WB + u), P.hi(i * WB + u));
    }
    if constexpr (OUT == 16) {
      // XOR parity code (params.py:105-112): one parity item = XOR of all inputs
      w2 pa = xa[0], pb = xb[0];
#pragma unroll
      for (int i = 1; i < D; i++) {
        pa = pa ^ xa[i];
        pb = pb ^ xb[i];
      }
      HA[D] = nh_acc(HA[D], pa, P.lo(D * WB + u), P.hi(D * WB + u));
      HB[D] = nh_acc(HB[D], pb, P.lo(D * WB + u), P.hi(D * WB + u));
    } else {
      // GF(16) Cauchy parity in bit-plane form: plane b of A | plane b of B << 16
      u32 x[4 * D], y[4 * NP];
#pragma unroll
      for (int i = 0; i < D; i++) {
        x[4 * i + 0] = __byte_perm(xa[i].lo, xb[i].lo, 0x5410);
        x[4 * i + 1] = __byte_perm(xa[i].lo, xb[i].lo, 0x7632);
        x[4 * i + 2] = __byte_perm(xa[i].hi, xb[i].hi, 0x5410);
        x[4 * i + 3] = __byte_perm(xa[i].hi, xb[i].hi, 0x7632);
      }
      enc_planes<OUT>(x, y);
#pragma unroll
      for (int p = 0; p < NP; p++) {
        const w2 pa = {__byte_perm(y[4 * p], y[4 * p + 1], 0x5410), __byte_perm(y[4 * p + 2], y[4 * p + 3], 0x5410)};
        const w2 pb = {__byte_perm(y[4 * p], y[4 * p + 1], 0x7632), __byte_perm(y[4 * p + 2], y[4 * p + 3], 0x7632)};
        HA[D + p] = nh_acc(HA[D + p], pa, P.lo((D + p) * WB + u), P.hi((D + p) * WB + u));
        HB[D + p] = nh_acc(HB[D + p], pb, P.lo((D + p) * WB + u), P.hi((D + p) * WB + u));
      }
    }
  }
  // combine (ehc.py:75-99): the coefficient-1 terms as one plain sum (3-input
  // IADD3 pairs), then the other coefficients as IMAD.WIDE/IMAD chains
#pragma unroll
  for (int r = 0; r < K; r++) {
    u64 a = 0, b = 0;
#pragma unroll
    for (int i = 0; i < E; i++) {
      if (V::mat(r, i) == 1) {
        a += HA[i];
        b += HB[i];
      }
    }
#pragma unroll
    for (int i = 0; i < E; i++) {
      if (V::mat(r, i) > 1) {
        a = mac_coef(V::mat(r, i), a, HA[i]);
        b = mac_coef(V::mat(r, i), b, HB[i]);
      }
    }
    CA[r] = a;
    CB[r] = b;
  }
}

template <int OUT, bool AL, class EH>
__device__ __forceinline__ void leaf2o(const uint8_t* buf, u32 delta, u32 offA, u32 offB, const EH& P,
                                       u64 (&CA)[Var<OUT>::k], u64 (&CB)[Var<OUT>::k]) {
  leaf2o<OUT, AL>(buf, delta, offA, delta, offB, P, CA, CB);
}

// instances q and q+4 of an 8-instance round
template <int OUT, bool AL, class EH>
__device__ __forceinline__ void leaf2(const uint8_t* buf, u32 delta, int q, int j, const EH& P,
                                      u64 (&CA)[Var<OUT>::k], u64 (&CB)[Var<OUT>::k]) {
  constexpr int M = Geo<Var<OUT>>::m;
  leaf2o<OUT, AL>(buf, delta, (u32)(q * M + j), (u32)((q + 4) * M + j), P, CA, CB);
}

// Seed-region bases of a layout with L levels (hasher.py:130-153), computed
// on demand rather than held in registers.
template <int K, int EW>
struct TreeCtx {
  u32 L;
  __device__ __forceinline__ u64 T(int r) const { return (u64)EW + 7ull * L * r; }
  __device__ __forceinline__ u64 F(int r) const { return (u64)EW + 7ull * L * K + 64ull * L * r; }
  __device__ __forceinline__ u64 R() const { return (u64)EW + 71ull * L * K; }
};

// A finished block at level `lvl` >= job_lvl, index `idx` (lanes 0-7 hold
// lane j of each row).  Either it is a leftover of its level -> finalize
// terms (tree.py:103-134), or it joins a complete group of 8 whose node the
// last arriving warp computes (nh.py:96-121 with level seeds,
// tree.py:55-60).  Returns the number of completion events (0 or 1).
template <int K, int EW, class SD>
__device__ __forceinline__ u32 climb(const Params& P, const Str& st, const TreeCtx<K, EW>& tc, int lvl, u64 idx,
                                     u64 (&B)[K], u64 (&fin)[K], int lane, const SD& sd) {
  const int q = lane >> 3, j = lane & 7;
  for (;;) {
    const u64 len = st.n_inst >> (3 * lvl);
    if (idx >= (len & ~7ull)) {
      if (lane < 8) {
#pragma unroll
        for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], B[r], sd(tc.F(r) + 56ull * lvl + (idx & 7) * 8 + j));
      }
      return 1;
    }
    if (P.frontier_lvl && lvl == P.frontier_lvl) {
      // slice mode: hand the subtree root to hth_hash_merge
      if (lane < 8) {
#pragma unroll
        for (int r = 0; r < K; r++) P.frontier[(idx - P.frontier_base) * 8 * K + r * 8 + j] = B[r];
      }
      return 0;
    }
    u64 woff = 0, coff = 0;
    for (int l = P.job_lvl; l <= lvl; l++) {
      const u64 ln = st.n_inst >> (3 * l);
      if (l < lvl) woff += (ln & ~7ull) * 8ull * K;
      if (l > P.job_lvl) coff += ln;  // counters of levels job_lvl+1..lvl precede level lvl+1's
    }
    u64* blk = P.scratch + st.scratch + woff;
    if (lane < 8) {
#pragma unroll
      for (int r = 0; r < K; r++) blk[idx * 8 * K + r * 8 + j] = B[r];
    }
    __syncwarp();
    u32 old = 0;
    u32* ctr = P.counters + st.cnt + coff + (idx >> 3);
    if (lane == 0) old = atom_add_acq_rel(ctr, 1u);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != 7) return 0;
    if (lane == 0) *ctr = 0;  // last arriver: leave the workspace zeroed
    u64* g = blk + (idx & ~7ull) * 8 * K;
#pragma unroll
    for (int r = 0; r < K; r++) {
      const u64 a = __ldcg(g + q * 8 * K + r * 8 + j);
      const u64 b = __ldcg(g + (q + 4) * 8 * K + r * 8 + j);
      g[q * 8 * K + r * 8 + j] = 0;  // consumed: leave the workspace zeroed
      g[(q + 4) * 8 * K + r * 8 + j] = 0;
      const u64 s = tc.T(r) + 7ull * lvl;
      u64 v = nh_acc(0, a, sd(s + q));
      v = (q < 3) ? nh_acc(v, b, sd(s + q + 4)) : v + b;
      v += shfl_xor(v, 8);
      v += shfl_xor(v, 16);
      B[r] = v;
    }
    lvl++;
    idx >>= 3;
  }
}

// AL8: every string starts 8-byte aligned (fixed batches with stride % 8 == 0),
// so only the aligned-word leaf is compiled in.
// PS: per-string seeds (Params.folds) instead of one shared seed array.
template <int OUT, bool VARLEN, int W, int NS, int MINB, bool AL8, bool PS>
__global__ void __launch_bounds__(W * 32, MINB) hash_kernel(const __grid_constant__ Params P) {
  using V = Var<OUT>;
  constexpr int K = V::k, M = Geo<V>::m;
  constexpr u32 CB = ROUND_INST * M * 8;  // stage payload bytes
  constexpr u32 SB = CB + 32;             // stage buffer: 16-B alignment superset + unaligned overread
  // varlen pair jobs: Y's instances start here (X's <= 4 instances + 16 bytes of alignment before it)
  constexpr u32 PAIR_OFF = 4 * M * 8 + 16;
  static_assert(PAIR_OFF + 4 * M * 8 + 16 <= SB, "a pair's instances fit one stage");
  // strings of <= 3 instances (< 4 m * 8 bytes with their tail) fit whole
  constexpr bool PAIR_FULL = PAIR_MAX <= 3;
  constexpr u32 PAIR_MARK = 0xffffffffu;  // prem of a claimed, not yet issued pair job
  constexpr u64 PAIR_BIT = 1ull << 63;    // record word 3 of a pair job (merge bases use < 64 bits)
  extern __shared__ __align__(128) uint8_t smem[];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane >> 3, j = lane & 7;
  uint8_t* ring = smem + warp * NS * SB;
  u64* bars = reinterpret_cast<u64*>(smem + W * NS * SB) + warp * NS;
  // per warp: the 8 level-1 blocks of the current level-2 group, [pos][r][lane],
  // then the level-3 node accumulator [r][lane] -- shared memory, not registers
  constexpr int NACC = 9 * K * 8;
  u64* nacc = reinterpret_cast<u64*>(smem + W * NS * SB + W * NS * 8) + warp * NACC;
  u64* n3acc = nacc + 8 * K * 8;
  if (lane == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
    fence_proxy_async();
  }
  __syncwarp();

  const int job_lvl = P.job_lvl;
  SeedSrc<PS> sd{P.S, 0};
  const u64 pol = policy_evict_first();

  // ---- producer: claims jobs dynamically (one atomic per job, lane 0) and
  // keeps the ring NS chunks ahead of the consumer; claimed job ids are
  // queued in shared memory so the consumer sees the same sequence.
  // Jobs are claimed in index order: fixed mode is jq-major (full jobs first),
  // so dynamic claiming also bounds the tail by one job.
  constexpr u32 QN = NS + 4;
  u64* jq_buf = reinterpret_cast<u64*>(smem + W * NS * SB + W * NS * 8) + W * NACC + warp * QN * JOB_REC;
  // PS: this warp's EHC seed words for the current job, (lo, hi) pairs
  u32* ehc_sm = reinterpret_cast<u32*>(jq_buf + (W - warp) * QN * JOB_REC) + warp * 2 * MAX_EW;
  const EhcSrc<PS, OUT> eh{P, ehc_sm};
  // varlen: per size class its first job id (largest class first);
  // cls_pre[0] = total jobs = end of class 1
  u32* cls_pre = reinterpret_cast<u32*>(smem + W * NS * SB + W * NS * 8 + W * NACC * 8 + W * QN * JOB_REC * 8 +
                                        (PS ? W * 2 * MAX_EW * 4 : 0));
  u32* cls_raw = cls_pre + NCLS + 1;  // varlen: raw string counts of the pair classes
  u64 n_jobs = P.n_jobs;
  if (VARLEN) {
    // launched as a programmatic dependent of the plan kernel: wait for its
    // completion (and memory) before reading what it planned
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // cls_pre[c] = jobs in classes > c (c >= 1), cls_pre[0] = all jobs: a
    // suffix scan of the 64 class counts by warp 0, two classes per lane
    static_assert(NCLS == 65, "two size classes per lane of one warp");
    if (warp == 0) {
      // classes 1..PAIR_MAX: jobs are pairs of strings (two per round)
      const int c1 = 2 * lane + 1, c2 = c1 + 1;
      const u32 ra = P.cls_cnt[c1], rb = P.cls_cnt[c2];
      if (c1 <= PAIR_MAX) cls_raw[c1] = ra;
      if (c2 <= PAIR_MAX) cls_raw[c2] = rb;
      const u32 a = c1 <= PAIR_MAX ? (ra + 1) >> 1 : ra, b = c2 <= PAIR_MAX ? (rb + 1) >> 1 : rb;
      u32 x = a + b;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_down_sync(0xffffffffu, x, d);
        if (lane + d < 32) x += t;
      }
      const u32 above = x - (a + b);  // classes > c2
      cls_pre[c2] = above;
      cls_pre[c1] = above + b;
      if (lane == 0) cls_pre[0] = x;
    }
    __syncthreads();
    n_jobs = cls_pre[0];
  }
  u32 qhead = 0, qtail = 0;        // queue: [qtail, qhead) claimed, not yet started
  bool pdone = false;
  // the first job of every warp is static (job = global warp index), so the
  // first bulk copy needs no atomic round trip; later claims start past it
  const u64 n_warps = (u64)gridDim.x * W;
  // small batches (one job per warp at most) never touch the counters
  const bool claims = n_jobs > n_warps;
  bool first = HTH_STATIC_FIRST || !claims;
  u32 pseq = 0, cseq = 0;
  u64 psrc = 0;  // next chunk's first byte (global address)
  u32 prem = 0;  // bytes of the current producer job not yet issued (a job is < 4 GiB)
  // cold path: claim the next job and set up its byte range (once per job)
#ifdef HTH_DEBUG_TIMING
  unsigned long long dbg_claim = 0;
#endif
  // varlen: job id -> its record in the class queues (one global load)
  u64 r1[JOB_REC];
  // the smallest class c with cls_pre[c] <= jc (cls_pre falls as c grows)
  auto v_class = [&](u64 jc) -> int {
    int lo = 1, hi = NCLS - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cls_pre[mid] <= jc) hi = mid;
      else lo = mid + 1;
    }
    return lo;
  };
  auto v_fetch = [&](u64 jc) {
    const int lo = v_class(jc);
    const u64 li = jc - cls_pre[lo];
    if (lo <= PAIR_MAX) {
      // a pair job: strings 2 li and 2 li + 1 of the class ->
      // {offset X, offset Y, sX | sY << 32, nX | nY << 32 | PAIR bit}
      const u64* q = P.job_map + (P.cls_qb[lo] + 2 * li) * JOB_REC;
      const bool hy = 2 * li + 1 < cls_raw[lo];
      const u64 x0 = __ldg(q), x1 = __ldg(q + 1), x2 = __ldg(q + 2);
      const u64 y0 = hy ? __ldg(q + JOB_REC) : 0, y1 = hy ? __ldg(q + JOB_REC + 1) : 0;
      const u64 y2 = hy ? __ldg(q + JOB_REC + 2) : 0xffffffffull;
      r1[0] = x0;
      r1[1] = y0;
      r1[2] = (x2 & 0xffffffffull) | (y2 << 32);
      r1[3] = x1 | (y1 << 32) | PAIR_BIT;
      return;
    }
    const u64* q = P.job_map + (P.cls_qb[lo] + li) * JOB_REC;
#pragma unroll
    for (int i = 0; i < JOB_REC; i++) r1[i] = __ldg(q + i);
  };
  auto p_claim_ = [&]() -> bool {
    if (pdone || qhead - qtail >= QN) return false;
    unsigned long long jc = (u64)blockIdx.x * W + warp;
    if (!first) {
      if (!claims) {
        pdone = true;
        return false;
      }
      if (lane == 0) jc = (HTH_STATIC_FIRST ? n_warps : 0) + atomicAdd(P.job_ctr, 1ull);
      jc = __shfl_sync(0xffffffffu, jc, 0);
    }
    first = false;
    if (jc >= n_jobs) {
      pdone = true;
      return false;
    }
    u64* e = jq_buf + (qhead % QN) * JOB_REC;
    if constexpr (VARLEN) {
      v_fetch(jc);
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < JOB_REC; i++) e[i] = r1[i];
      }
    } else if (lane == 0) {
      e[0] = jc;
    }
    qhead++;
    if (VARLEN && (r1[3] & PAIR_BIT)) {
      prem = PAIR_MARK;  // p_issue_one copies both strings' instances into one stage
      return true;
    }
    Str st;
    u32 jq, ni;
    u64 b0;
    decode_job<VARLEN, K, M>(P, jc, r1, st, jq);
    u64 jbytes;
    job_span<M>(st, jq, job_lvl, b0, jbytes, ni);
    prem = (u32)jbytes;
    psrc = reinterpret_cast<u64>(st.p) + b0;
    return true;
  };
#ifdef HTH_DEBUG_TIMING
  auto p_claim = [&]() -> bool {
    const unsigned long long t = gtimer();
    const bool r = p_claim_();
    dbg_claim += gtimer() - t;
    return r;
  };
#else
  auto& p_claim = p_claim_;
#endif
  // hot path: one bulk copy per round, address advanced incrementally
  auto p_issue_one = [&]() {
    if (VARLEN && prem == PAIR_MARK) {
      // pair job (just claimed, the newest queue entry): X's instances at
      // stage byte 0, Y's at PAIR_OFF, each as its 16-byte-aligned superset
      // (PAIR_FULL: the whole strings, tails included)
      const u32 slot = pseq % NS;
      if (lane == 0) {
        const u64* e = jq_buf + ((qhead - 1) % QN) * JOB_REC;
        const u64 base = reinterpret_cast<u64>(P.data);
        const u64 nX = e[3] & 0x7fffffffull, nY = (e[3] >> 32) & 0x7fffffffull;
        const u64 aX = base + e[0], aY = base + e[1];
        // PAIR_FULL: whole strings (instances + tail, < 4 m * 8 bytes each);
        // else instance bytes only; never past the string's last byte
        const u64 iX = PAIR_FULL ? nX : min(nX, (u64)((((nX + 7) >> 3) / M) * (M * 8ull)));
        const u64 iY = PAIR_FULL ? nY : min(nY, (u64)((((nY + 7) >> 3) / M) * (M * 8ull)));
        const u32 lX = (u32)(((aX + iX + 15) & ~15ull) - (aX & ~15ull));
        const u32 lY = nY ? (u32)(((aY + iY + 15) & ~15ull) - (aY & ~15ull)) : 0;
        mbar_arrive_expect_tx(&bars[slot], lX + lY);
        bulk_g2s(ring + slot * SB, reinterpret_cast<const void*>(aX & ~15ull), lX, &bars[slot], pol);
        if (lY) bulk_g2s(ring + slot * SB + PAIR_OFF, reinterpret_cast<const void*>(aY & ~15ull), lY, &bars[slot], pol);
      }
      pseq++;
      prem = 0;
      return;
    }
    const u32 len = min(CB, prem);
    const u64 a0 = psrc & ~15ull;
    const u32 bytes = (u32)(((psrc + len + 15) & ~15ull) - a0);
    const u32 slot = pseq % NS;
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[slot], bytes);
      bulk_g2s(ring + slot * SB, reinterpret_cast<const void*>(a0), bytes, &bars[slot], pol);
    }
    pseq++;
    psrc += CB;
    prem -= len;
  };
  auto p_issue = [&]() {
    while (pseq - cseq < (u32)NS) {
      if (prem == 0) {
        if (!p_claim()) return;
        continue;
      }
      p_issue_one();
    }
  };
  p_issue();

  // ---- consumer ----
  TreeCtx<K, Geo<V>::ew> tc;
#if HTH_S1_REGS
  u32 seedL = 0;
  u64 s1A[K], s1B[K];  // level-1 node seeds of this thread's two positions
#endif
#ifdef HTH_DEBUG_TIMING
  unsigned long long dbg_t0 = gtimer(), dbg_jobs = 0, dbg_rounds = 0, dbg_wait = 0, dbg_dec = 0, dbg_loop = 0,
                     dbg_fin = 0, dbg_m = 0;
#endif
  for (;;) {
    if (qtail == qhead) p_issue();
    if (qtail == qhead) break;  // no job left anywhere
#ifdef HTH_DEBUG_TIMING
    dbg_jobs++;
    dbg_m = gtimer();
#endif
    __syncwarp();
    const u64* jrec = jq_buf + (qtail % QN) * JOB_REC;
    qtail++;
    if constexpr (VARLEN) {
      if (jrec[3] & PAIR_BIT) {
        // Two one-level strings X, Y of <= 4 instances in one round: thread
        // (q, j) computes lane j of instance q of each.  Every instance is a
        // level-0 leftover (slot q, tree.py:103-134); the Toeplitz tails are
        // read from global memory (hasher.py:407-412).
        constexpr int EW = Geo<V>::ew;
        constexpr int NP = 2 * K <= 4 ? 4 : (2 * K <= 8 ? 8 : 16);
        const u64 oX = jrec[0], oY = jrec[1], sxy = jrec[2], nxy = jrec[3];
        const u64 nX = nxy & 0x7fffffffull, nY = (nxy >> 32) & 0x7fffffffull;
        const u64 sX = sxy & 0xffffffffull, sY = sxy >> 32;
        const bool hasY = sY != 0xffffffffull;
        const u32 cX = (u32)(((nX + 7) >> 3) / M), cY = hasY ? (u32)(((nY + 7) >> 3) / M) : 0;
        const u64 base = reinterpret_cast<u64>(P.data);
        const u32 dX = (u32)((base + oX) & 15), dY = (u32)((base + oY) & 15) + PAIR_OFF;
        const u32 slot = cseq % NS;
        mbar_wait(&bars[slot], (cseq / NS) & 1);
        // zero-pad a partial last word in the stage (hasher.py:179-183): the
        // string's last word (PAIR_FULL), else only one inside the instances
        const bool padX = PAIR_FULL ? (nX & 7) != 0 : nX < (u64)cX * M * 8;
        const bool padY = hasY && (PAIR_FULL ? (nY & 7) != 0 : nY < (u64)cY * M * 8);
        if (padX || padY) {
          uint8_t* b = ring + slot * SB;
          if (padX && (u32)lane < 8 - (u32)(nX & 7)) b[dX + nX + lane] = 0;
          if (padY && (u32)lane < 8 - (u32)(nY & 7)) b[dY + nY + lane] = 0;
          fence_proxy_async();
          __syncwarp();
        }
        u64 CA[K], CB_[K];
        const uint8_t* pbuf = ring + slot * SB;
        leaf2o<OUT, false>(pbuf, dX, (u32)(q * M + j), dY, (u32)(q * M + j), eh, CA, CB_);
        if (!PAIR_FULL) {  // the stage is consumed; the tails come from global memory
          __syncwarp();
          cseq++;
          if (prem != 0 && pseq - cseq == (u32)NS - 1)
            p_issue_one();
          else
            p_issue();
        }
        const u64 F1 = (u64)EW + 7ull * K, R1 = (u64)EW + 71ull * K;  // one-level layout (hasher.py:130-153)
        u64 a[NP];
#pragma unroll
        for (int r = 0; r < K; r++) {
          a[r] = (u32)q < cX ? nh_acc(0ull, CA[r], sd(F1 + 64ull * r + q * 8 + j)) : 0;
          a[K + r] = (u32)q < cY ? nh_acc(0ull, CB_[r], sd(F1 + 64ull * r + q * 8 + j)) : 0;
        }
#pragma unroll
        for (int r = 2 * K; r < NP; r++) a[r] = 0;
        const u64 tX = (u64)cX * M, tY = (u64)cY * M;
        const u64 nwX = (nX + 7) >> 3, nwY = hasY ? (nY + 7) >> 3 : 0;
        for (u64 t = tX + lane; t < nwX; t += 32) {
          const u64 y = PAIR_FULL ? ld_word<false>(pbuf, dX, (u32)t) : gword(P.data, oX, nX, t);
#pragma unroll
          for (int r = 0; r < K; r++) a[r] = nh_acc(a[r], y, sd(R1 + r + (t - tX)));
        }
        for (u64 t = tY + lane; t < nwY; t += 32) {
          const u64 y = PAIR_FULL ? ld_word<false>(pbuf, dY, (u32)t) : gword(P.data, oY, nY, t);
#pragma unroll
          for (int r = 0; r < K; r++) a[K + r] = nh_acc(a[K + r], y, sd(R1 + r + (t - tY)));
        }
        if (PAIR_FULL) {  // tails read: the stage is consumed
          __syncwarp();
          cseq++;
          if (prem != 0 && pseq - cseq == (u32)NS - 1)
            p_issue_one();
          else
            p_issue();
        }
        if (lane == 0) {
          // zero slots cX..6 and the length tag (tree.py:103-134)
#pragma unroll
          for (int r = 0; r < K; r++) {
            a[r] = nh_acc(a[r] + P.ztab[cX * K + r], nX, sd(F1 + 64ull * r + 56));
            if (hasY) a[K + r] = nh_acc(a[K + r] + P.ztab[cY * K + r], nY, sd(F1 + 64ull * r + 56));
          }
        }
        const u64 tot = warp_reduce_scatter<NP>(a, lane);
        const int idx = warp_scatter_index<NP>(lane);
        if ((lane & (32 / NP - 1)) == 0) {
          if (idx < K) P.out[sX * K + idx] = tot;
          else if (idx < 2 * K && hasY) P.out[sY * K + idx - K] = tot;
        }
        continue;
      }
    }
    Str st;
    u32 jq, ninst;
    u64 byte0, nbytes;
    decode_job<VARLEN, K, M>(P, jrec[0], jrec, st, jq);
    job_span<M>(st, jq, job_lvl, byte0, nbytes, ninst);
    const u32 nchunks = (u32)ceil_div(nbytes, CB);
    const u32 delta = (u32)(reinterpret_cast<uintptr_t>(st.p) & 15);
    const bool last_job = (jq + 1 == st.J);
    tc.L = st.L;  // tree seeds depend on the layout (hasher.py:130-153) via L only
    if (PS) {  // this string's own seed stream
      sd.fold = st.fold;
      __syncwarp();
      if (lane < Geo<V>::ew) {
        const u64 w = splitmix_word(st.fold, lane);
        const int slot = ehc_slot(lane, Var<OUT>::e, Var<OUT>::w);
        ehc_sm[2 * slot] = (u32)w;
        ehc_sm[2 * slot + 1] = (u32)(w >> 32);
      }
      __syncwarp();
    }
#if HTH_S1_REGS
    if (PS || st.L != seedL) {
#pragma unroll
      for (int r = 0; r < K; r++) {
        s1A[r] = sd(tc.T(r) + q);
        s1B[r] = q < 3 ? sd(tc.T(r) + q + 4) : 0;
      }
      seedL = st.L;
    }
#endif

#ifdef HTH_DEBUG_TIMING
    { const unsigned long long t = gtimer(); dbg_dec += t - dbg_m; dbg_m = t; }
#endif
    u64 fin[K];
    u32 events = last_job ? 1u : 0u;
#pragma unroll
    for (int r = 0; r < K; r++) fin[r] = 0;
    if (lane < 8) {
#pragma unroll
      for (int r = 0; r < K; r++) n3acc[r * 8 + lane] = 0;
    }
    const u64 inst0 = (u64)jq << (3 * job_lvl);
    const u64 full0 = st.n_inst & ~7ull;  // instances in complete level-1 groups
    const u64 len1 = st.n_inst >> 3, full1 = len1 & ~7ull;
    const u64 len2 = st.n_inst >> 6, full2 = len2 & ~7ull;

    // A full job (not the string's last, exactly 8^job_lvl instances) has no
    // tail, no partial round and no leftover groups below its root: its
    // round loop is instantiated without those checks (fixed batches; varlen
    // keeps one body for a small instruction footprint).
    auto rounds = [&](auto full_c) {
      constexpr bool FULL = decltype(full_c)::value;
      for (u32 c = 0; c < nchunks; c++) {
        const u32 slot = cseq % NS;
#ifdef HTH_DEBUG_TIMING
        const unsigned long long dbg_w = gtimer();
        mbar_wait(&bars[slot], (cseq / NS) & 1);
        dbg_wait += gtimer() - dbg_w;
        dbg_rounds++;
#else
        mbar_wait(&bars[slot], (cseq / NS) & 1);
#endif
        uint8_t* buf = ring + slot * SB;
        const bool tail_chunk = !FULL && last_job && (c + 1 == nchunks);
        if (tail_chunk && (st.n & 7)) {
          // zero-pad the partial final word (hasher.py:179-183, 416-419)
          const u32 endpos = delta + (u32)(nbytes - (u64)c * CB);
          const u32 nz = 8 - (u32)(st.n & 7);
          if ((u32)lane < nz) buf[endpos + lane] = 0;
          fence_proxy_async();
          __syncwarp();
        }
        const u32 r0 = c * ROUND_INST;  // first instance of the round (job-relative)
        if (FULL || r0 < ninst) {
          u64 CA[K], CB_[K];
          if (VARLEN || (!AL8 && (delta & 7)))
            leaf2<OUT, false>(buf, delta, q, j, eh, CA, CB_);
          else
            leaf2<OUT, true>(buf, delta, q, j, eh, CA, CB_);
          const u64 G1 = (inst0 >> 3) + c;  // level-1 group of this round
          if (FULL || G1 < len1) {
            // complete group -> level-1 node (nh_tree_node: last block added)
            u64 B1[K];
  #pragma unroll
            for (int r = 0; r < K; r++) {
              // level-0 seeds S[T_r + q] (tree.py:55-60); L1-resident
  #if HTH_S1_REGS
              u64 v = nh_acc(0, CA[r], s1A[r]);
              v = (q < 3) ? nh_acc(v, CB_[r], s1B[r]) : v + CB_[r];
  #else
              u64 v = nh_acc(0, CA[r], sd(tc.T(r) + q));
              v = (q < 3) ? nh_acc(v, CB_[r], sd(tc.T(r) + q + 4)) : v + CB_[r];
  #endif
              v += shfl_xor(v, 8);
              v += shfl_xor(v, 16);
              B1[r] = v;
            }
            const int p1 = (int)(G1 & 7);
            if (!FULL && G1 >= full1) {
              if (q == 0) {  // level-1 leftover -> finalize slot (1, p1)
  #pragma unroll
                for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], B1[r], sd(tc.F(r) + 56 + p1 * 8 + j));
              }
            } else {
              // park the level-1 block (lanes 0-7); every 8th round all 32 lanes
              // form the level-2 node from the parked group
              if (q == 0) {
  #pragma unroll
                for (int r = 0; r < K; r++) nacc[(p1 * K + r) * 8 + j] = B1[r];
              }
              if (p1 == 7) {
                __syncwarp();
                const u64 G2 = G1 >> 3;  // level-2 block complete (replicated in all lanes)
                u64 B2[K];
  #pragma unroll
                for (int r = 0; r < K; r++) {
                  const u64 a = nacc[(q * K + r) * 8 + j], b = nacc[((q + 4) * K + r) * 8 + j];
                  u64 v = nh_acc(0, a, sd(tc.T(r) + 7 + q));
                  v = (q < 3) ? nh_acc(v, b, sd(tc.T(r) + 11 + q)) : v + b;
                  v += shfl_xor(v, 8);
                  v += shfl_xor(v, 16);
                  B2[r] = v;
                }
                __syncwarp();
                if (job_lvl == 2) {
                  events += climb<K, Geo<V>::ew>(P, st, tc, 2, G2, B2, fin, lane, sd);
                } else {
                  const int p2 = (int)(G2 & 7);
                  if (lane < 8) {
                    if (!FULL && G2 >= full2) {
  #pragma unroll
                      for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], B2[r], sd(tc.F(r) + 112 + p2 * 8 + j));
                    } else {
  #pragma unroll
                      for (int r = 0; r < K; r++) {
                        const u64 a = n3acc[r * 8 + j];
                        n3acc[r * 8 + j] = (p2 < 7) ? nh_acc(a, B2[r], sd(tc.T(r) + 14 + p2)) : a + B2[r];
                      }
                    }
                  }
                  __syncwarp();
                  if ((FULL || G2 < full2) && p2 == 7) {
                    u64 B3[K];
  #pragma unroll
                    for (int r = 0; r < K; r++) {
                      B3[r] = lane < 8 ? n3acc[r * 8 + j] : 0;
                      if (lane < 8) n3acc[r * 8 + j] = 0;
                    }
                    events += climb<K, Geo<V>::ew>(P, st, tc, 3, G2 >> 3, B3, fin, lane, sd);
                  }
                }
              }
            }
          } else {
            // incomplete last group: level-0 leftovers -> finalize slot (0, pos)
            const u64 gA = inst0 + r0 + q, gB = gA + 4;
            const bool vA = r0 + q < ninst, vB = r0 + q + 4 < ninst;
  #pragma unroll
            for (int r = 0; r < K; r++) {
              if (vA) fin[r] = nh_acc(fin[r], CA[r], sd(tc.F(r) + (gA & 7) * 8 + j));
              if (vB) fin[r] = nh_acc(fin[r], CB_[r], sd(tc.F(r) + (gB & 7) * 8 + j));
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
            const u64 y = (VARLEN || (!AL8 && (delta & 7))) ? ld_word<false>(buf, delta, cw0 + t) : ld_word<true>(buf, delta, cw0 + t);
  #pragma unroll
            for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], y, sd(tc.R() + r + t));
          }
        }
        __syncwarp();
        cseq++;
        // the ring was full (or the producer is out of bytes): refill one slot
        if (prem != 0 && pseq - cseq == (u32)NS - 1)
          p_issue_one();
        else
          p_issue();
      }
    };
    if (!VARLEN && !last_job && ninst == (1u << (3 * job_lvl)))
      rounds(std::true_type{});
    else
      rounds(std::false_type{});

#ifdef HTH_DEBUG_TIMING
    { const unsigned long long t = gtimer(); dbg_loop += t - dbg_m; dbg_m = t; }
#endif
    if (last_job && P.fin_const_ok) {
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < K; r++) fin[r] += P.fin_const[r];
      }
    } else if (last_job && VARLEN && st.n_inst && st.L <= P.ztab_lmax) {
      // zero-slot sums from the plan's table (zero_slot_table), then the tag
      if (lane == 0) {
        const u64* z = P.ztab + ztab_base(st.L, K);
        for (u32 l = 0; l < st.L; l++) {
          const u64* zl = z + (l * 8 + ((st.n_inst >> (3 * l)) & 7)) * K;
#pragma unroll
          for (int r = 0; r < K; r++) fin[r] += zl[r];
        }
#pragma unroll
        for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], st.n, sd(tc.F(r) + 56u * st.L));
      }
    } else if (last_job) {
      // zero slots and the length tag of the finalize NH (hasher.py:387-405)
      if (st.n_inst) {
        const u32 nz = 56u * st.L;
        for (u32 x = (u32)lane; x < nz; x += 32) {
          const u32 l = x / 56u, slot = (x % 56u) >> 3;
          if (slot >= (u32)((st.n_inst >> (3 * l)) & 7)) {
#pragma unroll
            for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], 0ull, sd(tc.F(r) + x));
          }
        }
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], st.n, sd(tc.F(r) + nz));
        }
      } else if (lane == 0) {
#pragma unroll
        for (int r = 0; r < K; r++) fin[r] = nh_acc(fin[r], st.n, sd(tc.F(r)));
      }
    }
    // the k row sums over the warp, scattered (one 32-lane reduce-scatter:
    // 9 shuffles for k = 5 instead of 25): `own` lanes hold row `row`
    constexpr int NPK = K <= 2 ? 2 : (K <= 4 ? 4 : 8);
    u64 rs[NPK];
#pragma unroll
    for (int r = 0; r < NPK; r++) rs[r] = r < K ? fin[r] : 0;
    const u64 mine = warp_reduce_scatter<NPK>(rs, lane);
    const int row = warp_scatter_index<NPK>(lane);
    const bool own = (lane & (32 / NPK - 1)) == 0 && row < K;
    if (P.frontier_lvl) {
      // slice mode: accumulate only; the merge step publishes the digest
      if (own && mine) atomicAdd(reinterpret_cast<unsigned long long*>(P.acc) + row, (unsigned long long)mine);
    } else if (st.J == 1) {
      if (own) P.out[st.s * K + row] = mine;
    } else if (events) {
      // multi-job string: add this job's finalize terms, then count its
      // events; the warp completing the count publishes the digest and
      // re-zeroes the accumulators (integer sums: order-independent).
      unsigned long long* a = reinterpret_cast<unsigned long long*>(P.acc + st.s * K);
      if (own) atomicAdd(a + row, (unsigned long long)mine);
      __syncwarp();
      u32 old = 0;
      if (lane == 0) old = atom_add_acq_rel(P.events + st.s, events);
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old + events == string_events(st.n_inst, job_lvl)) {
        if (own) P.out[st.s * K + row] = atomicExch(a + row, 0ull);
        if (lane == 0) P.events[st.s] = 0;
      }
    }
#ifdef HTH_DEBUG_TIMING
    dbg_fin += gtimer() - dbg_m;
#endif
  }
#ifdef HTH_DEBUG_TIMING
  const unsigned long long dbg_jobs_end = gtimer();
#endif
#ifdef HTH_DEBUG_TIMING
  if (lane == 0) {
    const u64 gw = (u64)blockIdx.x * W + warp;
    if (gw < 8192) {
      unsigned long long* d = P.dbg + gw * 12;
      d[0] = dbg_t0; d[1] = gtimer(); d[2] = dbg_jobs; d[3] = dbg_rounds; d[4] = dbg_wait; d[5] = dbg_jobs_end;
      d[6] = dbg_claim; d[7] = dbg_dec; d[8] = dbg_loop; d[9] = dbg_fin;
    }
  }
#endif
  // slice mode: the frontier roots and partial digest may live in another
  // GPU's memory (peer stores over NVLink); make them visible system-wide
  if (P.frontier_lvl) __threadfence_system();
  __syncwarp();
  // every warp has stopped claiming; the last one out re-zeroes the counters
  // (relaxed is enough: each warp's last claim returned before it got here)
  // and, exchanging in-stream, publishes the slice: every warp fenced its
  // peer stores (fence.sc.sys above) before its arrival, so a fence and a
  // release store by the last arriver order them all before the flag
  if ((claims || P.done_flag || VARLEN) && lane == 0) {
    const u32 old = atomicAdd(P.exit_ctr, 1u);
    if (old + 1 == gridDim.x * (u32)W) {
      *P.job_ctr = 0;
      *P.exit_ctr = 0;
      if (VARLEN) {  // every CTA read the plan's counts at its start: leave them zeroed for the next call
        for (int c = 0; c < NCLS; c++) P.cls_cnt[c] = 0;
        P.totals[0] = 0;
        P.totals[1] = 0;
      }
      if (P.done_flag) {
        __threadfence_system();
        st_release_sys(P.done_flag, P.done_value);
      }
    }
  }
}

}  // namespace hth
