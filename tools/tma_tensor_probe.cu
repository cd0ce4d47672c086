// Probe (answered: NO): can a 1-D u8 tensor map (cp.async.bulk.tensor.1d, 256-byte boxes at
// ANY byte coordinate) stream HBM as fast as 1-D bulk copies, so that the
// varlen kernel could land every string 16-byte aligned in shared memory?
// Per warp: a 2-stage ring of 7680-byte stages (one v40 round); each stage is
// filled by 30 boxes issued by 30 lanes (tensor mode, start offset +5 bytes)
// or by one bulk copy (bulk mode, aligned).  Prints GB/s for both.
// Result on B200 (round 2): boxes at 16-byte-aligned coordinates stream at 6.8 TB/s (bulk: 7.15);
// any other start coordinate (TOFF=5) faults with an illegal instruction -- tensor TMA does not
// realign byte strings, so the varlen kernel keeps its funnel-shift word loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_tensor_probe tools/tma_tensor_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int STAGE = 7680, NS = 2, W = 2;
#ifndef TOFF
#define TOFF 5
#endif
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool TENSOR>
__global__ void __launch_bounds__(W * 32, 6) probe(const CUtensorMap* gtm, const uint8_t* base, uint64_t rounds,
                                                   uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * NS * STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + W * NS * STAGE) + warp * NS;
  if (lane == 0 && TENSOR) asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(gtm) : "memory");
  if (lane == 0) {
    for (int s = 0; s < NS; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncwarp();
  const uint64_t nw = (uint64_t)gridDim.x * W, gw = (uint64_t)blockIdx.x * W + warp;
  uint32_t acc = 0;
  const uint64_t desc = reinterpret_cast<uint64_t>(gtm);  // descriptor in global memory
  auto issue = [&](uint64_t r, int slot) {
    uint8_t* dst = ring + slot * STAGE;
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[slot])), "r"(STAGE));
    __syncwarp();
    if (TENSOR) {
      if (lane == 0) {
        for (int i = 0; i < STAGE / 256; i++) {
          const int c = (int)(TOFF + r * STAGE + i * 256);
          asm volatile("cp.async.bulk.tensor.1d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                       ::"r"(sa(dst + i * 256)), "l"(desc), "r"(c), "r"(sa(&bars[slot])) : "memory");
        }
      }
    } else if (lane == 0) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(dst)), "l"(base + r * STAGE), "r"(STAGE), "r"(sa(&bars[slot])) : "memory");
    }
  };
  uint32_t k = 0;
  uint64_t r = gw;
  for (int s = 0; s < NS && r + s * nw < rounds; s++) issue(r + s * nw, s);
  for (; r < rounds; r += nw, k++) {
    const int slot = k % NS;
    const uint32_t ph = (k / NS) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(&bars[slot])), "r"(ph));
    const uint32_t* v = reinterpret_cast<const uint32_t*>(ring + slot * STAGE);
    for (int i = lane; i < STAGE / 4; i += 32 * 8) acc ^= v[i];
    __syncwarp();
    if (r + NS * nw < rounds) issue(r + NS * nw, slot);
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const uint64_t bytes = 2000000000ull, rounds = (bytes - 64) / STAGE;
  uint8_t* d;
  uint32_t* sink;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(d, 1, bytes));
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t gdim[1] = {bytes};
  cuuint64_t gstr[1] = {bytes};
  cuuint32_t box[1] = {256}, es[1] = {1};
  CUresult cr = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f)(
      &tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
  CUtensorMap* dtm;
  CK(cudaMalloc(&dtm, sizeof(CUtensorMap)));
  CK(cudaMemcpy(dtm, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  const size_t smem = W * NS * (STAGE + 8) + 64;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int t = 0; t < 2; t++) {
    auto k = t ? probe<true> : probe<false>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, W * 32, smem));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int it = 0; it < 6; it++) {
      cudaEventRecord(a);
      k<<<sms * occ, W * 32, smem>>>(dtm, d, rounds, sink);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    printf("%s: occ %d CTAs/SM, %.1f GB/s\n", t ? "tensor 1-D u8, 30 x 256 B boxes at +5 B" : "bulk 1-D, one 7680 B copy",
           occ, rounds * (double)STAGE / best / 1e6);
  }
  return 0;
}
