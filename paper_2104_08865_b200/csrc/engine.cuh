// HalftimeHash B200 engine: device side.
//
// One kernel hashes a batch of strings.  Work is cut into warp JOBS: job
// (s, jq) covers instances [64 jq, 64 jq + 64) of string s (one level-2
// subtree of the reference's stack construction, tree.py:63-100), and the
// string's last job also covers its Toeplitz tail (hasher.py:407-412).
//
// Per warp: a ring of NS shared-memory stages fed by cp.async.bulk (TMA 1-D
// bulk copies completing on an mbarrier).  A stage holds one ROUND = 4
// instances (plus the tail in the string's last round).  Thread (q, j) of
// the warp (q = lane / 8, j = lane % 8) owns lane j of instance 4c + q:
//   encode (GF(16) Cauchy / XOR parity, ehc.py:23-46) -> NH (ehc.py:49-72)
//   -> combine (ehc.py:75-99), all in registers.
// Level-1 nodes (nh.py:96-121) are reduced over the 4 threads sharing j
// with two shuffles; level-2 nodes accumulate serially in lanes 0-7.
// Levels >= 3 use a "last arriver" merge through a global scratch area.
//
// The reference's finalize (tree.py:103-134) is a plain sum of NH terms
// over leftover slots, zero slots and the length tag; the tail is a sum of
// NH terms too.  Every block that ends up a leftover therefore adds its
// finalize terms straight into the digest accumulator the moment it is
// produced; digests of multi-job strings are summed with 64-bit atomics
// (integer, mod 2^64: order-independent, so bit-exact and deterministic).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "variants.cuh"

namespace hth {

typedef uint64_t u64;
typedef uint32_t u32;

constexpr int JOB_INST = 64;   // instances per warp job (8^2)
constexpr int ROUND_INST = 4;  // instances per stage

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
__device__ __forceinline__ u64 cat(w2 a) { return ((u64)a.hi << 32) | a.lo; }
__device__ __forceinline__ w2 operator^(w2 a, w2 b) { return {a.lo ^ b.lo, a.hi ^ b.hi}; }

// NH(x, s) = ((x_lo + s_lo) mod 2^32) * ((x_hi + s_hi) mod 2^32)  (nh.py:48-67)
// acc + (u64)a*b lowers to one IMAD.WIDE.U32.
__device__ __forceinline__ u64 nh_acc(u64 acc, w2 x, u64 s) {
  u32 a = x.lo + (u32)s, b = x.hi + (u32)(s >> 32);
  return acc + (u64)a * b;
}
__device__ __forceinline__ u64 nh_acc(u64 acc, u64 x, u64 s) { return nh_acc(acc, mk(x), s); }

// x * v on 16 bit-sliced GF(16) elements (gf16.py:17-21), in 32-bit halves:
// lo = planes 0,1; hi = planes 2,3.  2 PRMT + 1 LOP3.
__device__ __forceinline__ w2 xtime(w2 v) {
  u32 nlo = __byte_perm(v.hi, v.lo, 0x5432);  // (lo << 16) | (hi >> 16)
  u32 nhi = __byte_perm(v.lo, v.hi, 0x5432);  // (hi << 16) | (lo >> 16)
  nlo ^= v.hi & 0xFFFF0000u;                  // reduction x^4 = x + 1
  return {nlo, nhi};
}

template <class T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}
__device__ __forceinline__ u64 warp_sum(u64 v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// ------------------------------------------------------------ EHC leaf
// X[i][u] = lane word of input item i, block u.  Returns C[r], r < k
// (hasher.py:356-364; ehc.py:102-118).  Encode uses the Horner form of
// gf16.scale: sum_i c_i * X_i = Q0 ^ x(Q1 ^ x(Q2 ^ x Q3)), Q_b = XOR of X_i
// whose coefficient has bit b set (xtime is GF(2)-linear).
template <class V>
__device__ __forceinline__ void leaf(const w2 (&X)[V::d][V::w], const u64* __restrict__ S, u64 (&C)[V::k]) {
#pragma unroll
  for (int r = 0; r < V::k; r++) C[r] = 0;
#pragma unroll
  for (int i = 0; i < V::e; i++) {
    u64 h = 0;
#pragma unroll
    for (int u = 0; u < V::w; u++) {
      w2 E;
      if (i < V::d) {
        E = X[i][u];
      } else {
        w2 q[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
#pragma unroll
        for (int t = 0; t < V::d; t++) {
          const int c = V::par(i - V::d, t);
#pragma unroll
          for (int b = 0; b < 4; b++)
            if ((c >> b) & 1) q[b] = q[b] ^ X[t][u];
        }
        E = q[0] ^ xtime(q[1] ^ xtime(q[2] ^ xtime(q[3])));
      }
      h = nh_acc(h, E, __ldg(S + i * V::w + u));
    }
#pragma unroll
    for (int r = 0; r < V::k; r++) {
      const int c = V::mat(r, i);
      if (c) C[r] += (u64)c * h;
    }
  }
}

// ------------------------------------------------------------ per-string view
struct Str {
  const uint8_t* p;  // first byte (global)
  u64 n;             // bytes
  u64 n_inst;        // full instances
  u32 L;             // leftover levels (layout levels, >= 1)
  u32 J;             // warp jobs
  u64 scratch;       // base word of this string's scratch blocks
  u64 cnt;           // base index of this string's counters
  u64 s;             // string index
};

__host__ __device__ __forceinline__ u32 level_count(u64 n) {
  u32 l = 1;
  while (n >= 8) {
    n >>= 3;
    l++;
  }
  return l;
}
__host__ __device__ __forceinline__ u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }

// scratch words / counters a string needs for merges above level 2
__host__ __device__ __forceinline__ void scratch_need(u64 n_inst, int k, u64* words, u64* cnts) {
  u64 w = 0, c = 0;
  for (int l = 2; (n_inst >> (3 * l)) >= 8; l++) {
    u64 len = n_inst >> (3 * l);
    w += (len & ~7ull) * 8ull * k;
    c += len >> 3;
  }
  *words = w;
  *cnts = c;
}
// offset of level `lvl` blocks inside the string's scratch, and of the
// counters of level `lvl` nodes (lvl >= 3) inside its counter area
__device__ __forceinline__ void scratch_off(u64 n_inst, int k, int lvl, u64* woff, u64* coff) {
  u64 w = 0, c = 0;
  for (int l = 2; l < lvl; l++) {
    u64 len = n_inst >> (3 * l);
    w += (len & ~7ull) * 8ull * k;
    if (l >= 3) c += len;
  }
  *woff = w;
  *coff = c;
}

struct Params {
  const uint8_t* data;
  u64 n_strings;
  u64 stride;      // fixed mode
  u64 n_bytes;     // fixed mode
  u64 J_fixed;     // fixed mode: jobs per string
  u64 n_jobs;      // fixed mode: total jobs
  u64 scr_per;     // fixed mode: scratch words per string
  u64 cnt_per;     // fixed mode: counters per string
  const u64* offsets;    // varlen: n_strings + 1 byte offsets
  const u32* job_str;    // varlen: job -> string
  const u64* meta;       // varlen: 3 u64 per string (job_first, scratch, cnt); entry n = totals
  const u64* S;
  u64* out;
  u64* scratch;   // level >= 2 blocks awaiting their group's merge
  u32* counters;  // per-group arrival counts (self-resetting)
  u64* acc;       // per multi-job string: k partial digest words (self-resetting)
  u32* events;    // per multi-job string: completion events seen (self-resetting)
};

// Completion events of a multi-job string: its last job, plus one per block
// at level >= 2 that ends as a leftover (each such block's producer is the
// last warp to touch anything beneath it).  When all have arrived, every
// finalize term is in `acc`.
__device__ __forceinline__ u32 string_events(u64 n_inst) {
  u32 e = 1;
  for (int l = 2; (n_inst >> (3 * l)) > 0; l++) e += (u32)((n_inst >> (3 * l)) & 7);
  return e;
}

template <int K>
__device__ __forceinline__ void layout_bases(u32 L, int ew, u64 (&T)[K], u64 (&F)[K], u64& R) {
#pragma unroll
  for (int r = 0; r < K; r++) {
    T[r] = (u64)ew + 7ull * L * r;
    F[r] = (u64)ew + 7ull * L * K + 64ull * L * r;
  }
  R = (u64)ew + 71ull * L * K;
}

template <bool VARLEN, int K, int M>
__device__ __forceinline__ void decode_job(const Params& P, u64 job, Str& st, u32& jq) {
  u64 s;
  if (VARLEN) {
    s = P.job_str[job];
    u64 o0 = P.offsets[s], o1 = P.offsets[s + 1];
    st.p = P.data + o0;
    st.n = min(o1 - o0, P.n_bytes);  // clamp to the host-checked bound (plan_count_kernel)
    const u64* mt = P.meta + 3 * s;
    jq = (u32)(job - mt[0]);
    st.scratch = mt[1];
    st.cnt = mt[2];
  } else {
    s = job / P.J_fixed;
    jq = (u32)(job - s * P.J_fixed);
    st.p = P.data + s * P.stride;
    st.n = P.n_bytes;
    st.scratch = s * P.scr_per;
    st.cnt = s * P.cnt_per;
  }
  st.s = s;
  st.n_inst = ((st.n + 7) >> 3) / M;
  st.L = st.n_inst ? level_count(st.n_inst) : 1;
  st.J = st.n_inst > (u64)JOB_INST ? (u32)ceil_div(st.n_inst, JOB_INST) : 1;
}

// bytes of job jq (its instances, plus the tail for the last job)
template <int M>
__device__ __forceinline__ void job_span(const Str& st, u32 jq, u64& byte0, u64& nbytes, u32& ninst) {
  u64 i0 = (u64)jq * JOB_INST;
  u64 ni = st.n_inst > i0 ? min((u64)JOB_INST, st.n_inst - i0) : 0;
  ninst = (u32)ni;
  byte0 = i0 * (M * 8ull);
  nbytes = (jq + 1 == st.J) ? st.n - byte0 : ni * (M * 8ull);
}

}  // namespace hth
