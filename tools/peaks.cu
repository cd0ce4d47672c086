// Microbenchmarks for the roofline denominators of this path:
//   read   -- HBM read-only streaming (what the hash kernels do)
//   copy   -- HBM read + write (the MEASURED_PEAKS.json figure's kind)
//   imad   -- IMAD.WIDE.U32 issue rate (the NH multiply)
//   lop3   -- 3-input LOP3 issue rate (the GF(16) encode)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
// Run:   tools/peaks > profiles/peaks.json      (one GPU; prints one JSON object)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e = (x);                                                    \
    if (e != cudaSuccess) {                                                 \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));               \
      return 1;                                                             \
    }                                                                       \
  } while (0)

__global__ void read_kernel(const uint4* __restrict__ p, size_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;  // keep the loads alive
}

__global__ void copy_kernel(const uint4* __restrict__ p, uint4* __restrict__ q, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(q + i, __ldcs(p + i));
}

// 8 independent 64-bit accumulators per thread: acc += a * b (mad.wide.u32)
__global__ void imad_kernel(uint32_t a, uint32_t b, int iters, uint64_t* sink) {
  uint64_t acc[8];
#pragma unroll
  for (int k = 0; k < 8; k++) acc[k] = threadIdx.x + k;
  uint32_t x = a + threadIdx.x, y = b;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[k]) : "r"(x + k), "r"(y));
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s ^= acc[k];
  if (s == 1) sink[0] = s;
}

__global__ void lop3_kernel(uint32_t a, int iters, uint32_t* sink) {
  uint32_t r[8];
#pragma unroll
  for (int k = 0; k < 8; k++) r[k] = a + threadIdx.x * 8 + k;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[k]) : "r"(r[(k + 1) & 7]), "r"(r[(k + 3) & 7]));
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s ^= r[k];
  if (s == 1) sink[0] = s;
}

template <class F>
float time_ms(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < reps; r++) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  const size_t bytes = 8ull << 30;
  uint4 *a = nullptr, *b = nullptr;
  uint32_t* sink = nullptr;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes / 2));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(a, 1, bytes));
  const size_t n = bytes / 16;
  const int grid = sms * 8, tpb = 512;
  const float rd = time_ms([&] { read_kernel<<<grid, tpb>>>(a, n, sink); }, 10);
  const float cp = time_ms([&] { copy_kernel<<<grid, tpb>>>(a, b, n / 2); }, 10);
  const int iters = 4096;
  const float im = time_ms([&] { imad_kernel<<<sms * 16, 256>>>(3, 5, iters, (uint64_t*)sink); }, 5);
  const float lo = time_ms([&] { lop3_kernel<<<sms * 16, 256>>>(7, iters, sink); }, 5);
  CK(cudaGetLastError());
  const double ops = (double)sms * 16 * 256 * iters * 8;
  printf("{\"device_sms\": %d, \"clock_mhz_attr\": %d, \"read_gbs\": %.1f, \"copy_gbs\": %.1f, "
         "\"imad_wide_per_clk_per_sm_at_attr_clock\": %.1f, \"lop3_per_clk_per_sm_at_attr_clock\": %.1f, "
         "\"imad_wide_tops\": %.2f, \"lop3_tops\": %.2f, \"note\": \"read: ld.global.cs 16 B/thread over 8 GiB; "
         "copy: 4 GiB read + 4 GiB written, GB/s counts both; op rates are thread-instructions per second\"}\n",
         sms, clk / 1000, bytes / (rd * 1e6), bytes / (cp * 1e6), ops / (im * 1e-3) / sms / (clk * 1e3),
         ops / (lo * 1e-3) / sms / (clk * 1e3), ops / (im * 1e-3) / 1e12, ops / (lo * 1e-3) / 1e12);
  return 0;
}
