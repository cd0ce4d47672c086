// HalftimeHash B200 engine: launch configurations and the per-variant
// launchers (VarEngine<OUT> member definitions).  Included only by the
// per-variant units kv16/24/32/40.cu, which instantiate VarEngine<OUT>, so
// the kernels of the four variants compile in parallel.
#pragma once
#include "engine_api.cuh"

#ifndef HTH_VARLEN_PDL
#define HTH_VARLEN_PDL 1
#endif

namespace hth {

// ------------------------------------------------------------ launch config
template <int OUT> struct KCfg;
// W warps per CTA, NS ring stages per warp (one 8-instance round each),
// MINB CTAs per SM the register allocation must allow.
template <> struct KCfg<16> { static constexpr int W = 4, NS = 2, MINB = 4; };
#ifndef HTH_V2432_MINB
#define HTH_V2432_MINB 4
#endif
template <> struct KCfg<24> { static constexpr int W = 2, NS = 2, MINB = HTH_V2432_MINB; };
template <> struct KCfg<32> { static constexpr int W = 2, NS = 2, MINB = HTH_V2432_MINB; };
#ifndef HTH_V40_W
#define HTH_V40_W 2
#endif
#ifndef HTH_V40_NS
#define HTH_V40_NS 2
#endif
#ifndef HTH_V40_MINB
#define HTH_V40_MINB 5
#endif
template <> struct KCfg<40> { static constexpr int W = HTH_V40_W, NS = HTH_V40_NS, MINB = HTH_V40_MINB; };

template <int OUT, bool PS = false>
constexpr size_t smem_bytes() {
  constexpr int M = Geo<Var<OUT>>::m;
  constexpr size_t SB = ROUND_INST * M * 8 + 32;
  // ring + mbarriers + parked level-1 group and level-3 accumulator +
  // claimed-job queue (+ per-job EHC seeds in many-seeds mode), per warp
  return KCfg<OUT>::W * (KCfg<OUT>::NS * (SB + 8) + 9 * Var<OUT>::k * 8 * 8 + (KCfg<OUT>::NS + 4) * 8 * JOB_REC +
                         (PS ? 2 * MAX_EW * 4 : 0)) +
         (NCLS + 1) * 4 + NCLS * 8;  // + varlen class table (per CTA)
}
template <int OUT, bool VARLEN, bool AL8, bool PS = false>
int launch_hash(const Params& P, u64 n_jobs_bound, cudaStream_t st) {
  constexpr int W = KCfg<OUT>::W, NS = KCfg<OUT>::NS;
  auto kern = hash_kernel<OUT, VARLEN, W, NS, KCfg<OUT>::MINB, AL8, PS>;
  const size_t smem = smem_bytes<OUT, PS>();
  int dev = 0, occ = 1;
  if (int rc = occupancy((const void*)kern, W * 32, smem, &dev, &occ)) return rc;
  u64 grid = (u64)sm_count(dev) * occ;
  const u64 need = ceil_div(n_jobs_bound, W);
  if (need < grid) grid = need;
  if (grid == 0) grid = 1;
  if (VARLEN && HTH_VARLEN_PDL) {
    // programmatic dependent launch: the CTAs start (mbarrier setup) while
    // the plan kernel finishes and wait for its results in-kernel
    // (griddepcontrol.wait before the class counts are read)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, P));
    return HTH_OK;
  }
  kern<<<(unsigned)grid, W * 32, smem, st>>>(P);
  CK(cudaGetLastError());
  return HTH_OK;
}

#ifndef HTH_TAIL_NS
#define HTH_TAIL_NS 1
#endif
#ifndef HTH_TAIL_STAGE
#define HTH_TAIL_STAGE 8192
#endif
// NS stages of GP string pairs per warp; measured on config 3 (1 KiB strings):
// one 8 KiB stage per warp streams best (6.33 TB/s vs 6.21 for 2 x 4 KiB and
// 5.5 for 4 x 2 KiB), more than 64 KiB per 8-warp CTA costs occupancy
template <int OUT, int CPT, bool MASKED, int GP>
int launch_tail_g(const TailParams& P, cudaStream_t st) {
  constexpr int NS = HTH_TAIL_NS, TPB = 256;
  auto kern = tail_kernel<OUT, CPT, MASKED, NS, GP>;
  const u64 sby = (GP * 2 * P.stride + 127) & ~127ull;
  const size_t smem = (TPB / 32) * NS * (sby + 8);
  if (smem > 227 * 1024) return fail(HTH_EINVAL, "tail kernel stage too large");
  int dev = 0, occ = 1;
  if (int rc = occupancy((const void*)kern, TPB, smem, &dev, &occ)) return rc;
  const u64 groups = ceil_div((P.n_strings + 1) / 2, (u64)GP);
  u64 grid = (u64)sm_count(dev) * std::max(occ, 1);
  const u64 need = ceil_div(groups, TPB / 32);
  if (need < grid) grid = need;
  kern<<<(unsigned)std::max<u64>(grid, 1), TPB, smem, st>>>(P);
  CK(cudaGetLastError());
  return HTH_OK;
}
template <int OUT, int CPT, bool MASKED>
int launch_tail(const TailParams& P, cudaStream_t st) {
  const u64 pair = 2 * P.stride;
  if (4 * pair <= HTH_TAIL_STAGE) return launch_tail_g<OUT, CPT, MASKED, 4>(P, st);
  if (2 * pair <= HTH_TAIL_STAGE) return launch_tail_g<OUT, CPT, MASKED, 2>(P, st);
  return launch_tail_g<OUT, CPT, MASKED, 1>(P, st);
}

// chunks per lane of the instantiation that serves nch 16-byte chunks
inline int tail_cpt(u64 nch) {
  const u64 cpt = ceil_div(nch, 16);
  return cpt <= 1 ? 1 : (cpt <= 2 ? 2 : (cpt <= 4 ? 4 : 6));
}
template <int OUT, bool MASKED>
int dispatch_tail_m(const TailParams& P, u64 nch, cudaStream_t st) {
  // a string shorter than one instance has at most ceil((8m - 8) / 16)
  // chunks: 48 (v16), 84 (v24/v32), 60 (v40) -- only v24/v32 need CPT 6
  constexpr bool WIDE = Geo<Var<OUT>>::m * 8 - 8 > 16 * 16 * 4;
  switch (tail_cpt(nch)) {
    case 1: return launch_tail<OUT, 1, MASKED>(P, st);
    case 2: return launch_tail<OUT, 2, MASKED>(P, st);
    case 4: return launch_tail<OUT, 4, MASKED>(P, st);
  }
  if constexpr (WIDE) return launch_tail<OUT, 6, MASKED>(P, st);
  return fail(HTH_EINVAL, "tail kernel: %llu chunks exceed one instance", (unsigned long long)nch);
}
template <int OUT>
int dispatch_tail(const TailParams& P, u64 nch, cudaStream_t st) {
  // the unmasked body processes exactly 16 * CPT whole chunks per string:
  // anything else (a partial last chunk, or fewer chunks than the
  // instantiation covers, e.g. 80 chunks on the CPT = 6 body) is masked
  const bool masked = (P.n_bytes % 16) != 0 || nch != 16ull * tail_cpt(nch);
  return masked ? dispatch_tail_m<OUT, true>(P, nch, st) : dispatch_tail_m<OUT, false>(P, nch, st);
}

#ifndef HTH_SMALL_STAGE
#define HTH_SMALL_STAGE 8704
#endif
template <int OUT, int G>
int launch_small(const Params& P, cudaStream_t st) {
  constexpr int W = KCfg<OUT>::W, NS = 2;
  auto kern = small_kernel<OUT, G, W, NS, KCfg<OUT>::MINB>;
  const u64 sby = (G * P.stride + 16 + 127) & ~127ull;
  const size_t smem = W * NS * (sby + 8);
  int dev = 0, occ = 1;
  if (int rc = occupancy((const void*)kern, W * 32, smem, &dev, &occ)) return rc;
  u64 grid = (u64)sm_count(dev) * std::max(occ, 1);
  const u64 need = ceil_div(ceil_div(P.n_strings, (u64)G), (u64)W);
  if (need < grid) grid = need;
  kern<<<(unsigned)std::max<u64>(grid, 1), W * 32, smem, st>>>(P);
  CK(cudaGetLastError());
  return HTH_OK;
}
// strings per warp stage: about HTH_SMALL_STAGE bytes per contiguous copy,
// fewer when the batch would not give every resident warp two stages
template <int OUT>
int dispatch_small(const Params& P, cudaStream_t st) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const u64 slots = 2ull * sm_count(dev) * KCfg<OUT>::W * KCfg<OUT>::MINB;
  int g = 4 * P.stride <= HTH_SMALL_STAGE ? 4 : (2 * P.stride <= HTH_SMALL_STAGE ? 2 : 1);
  while (g > 1 && ceil_div(P.n_strings, (u64)g) < slots) g >>= 1;
  if (g == 4) return launch_small<OUT, 4>(P, st);
  if (g == 2) return launch_small<OUT, 2>(P, st);
  return launch_small<OUT, 1>(P, st);
}
template <int OUT>
int VarEngine<OUT>::hash(const Params& P, u64 n_jobs_bound, int kind, cudaStream_t st) {
  switch (kind) {
    case HK_VARLEN: return launch_hash<OUT, true, false>(P, n_jobs_bound, st);
    case HK_FIXED: return launch_hash<OUT, false, false>(P, n_jobs_bound, st);
    case HK_FIXED_AL8: return launch_hash<OUT, false, true>(P, n_jobs_bound, st);
    case HK_PS: return launch_hash<OUT, false, false, true>(P, n_jobs_bound, st);
  }
  return fail(HTH_EINVAL, "bad kernel kind %d", kind);
}
template <int OUT>
int VarEngine<OUT>::tail(const TailParams& T, u64 nch, cudaStream_t st) {
  return dispatch_tail<OUT>(T, nch, st);
}
template <int OUT>
int VarEngine<OUT>::small(const Params& P, cudaStream_t st) {
  return dispatch_small<OUT>(P, st);
}
template <int OUT>
int VarEngine<OUT>::plan(const PlanParams& Q, unsigned grid, cudaStream_t st) {
  plan_kernel<OUT><<<grid, 256, 0, st>>>(Q);
  CK(cudaGetLastError());
  return HTH_OK;
}
template <int OUT>
int VarEngine<OUT>::merge(const MergeParams& M, cudaStream_t st) {
  auto kern = merge_kernel<OUT>;
  const size_t smem = merge_smem_bytes<Var<OUT>::k>(M.nf);
  int dev = 0, occ = 1;
  if (int rc = occupancy((const void*)kern, MERGE_TPB, smem, &dev, &occ)) return rc;  // raises the smem limit
  kern<<<1, MERGE_TPB, smem, st>>>(M);
  CK(cudaGetLastError());
  return HTH_OK;
}

}  // namespace hth
