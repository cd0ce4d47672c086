// HalftimeHash B200 engine: what the host code (halftime.cu) sees of the
// kernels -- parameter blocks, the runtime helpers it shares with the kernel
// units, and VarEngine<OUT>, the per-variant launchers defined in launch.cuh
// and instantiated once per output width in kv16/24/32/40.cu.
#pragma once
#include <string>

#include "../../include/halftime_b200.h"
#include "merge_kernel.cuh"
#include "plan_kernel.cuh"
#include "small_kernel.cuh"
#include "tail_kernel.cuh"

namespace hth {

// runtime helpers (defined in halftime.cu)
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
#define CK(call)                                        \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)
int sm_count(int dev);
int occupancy(const void* kern, int tpb, size_t smem, int* dev_out, int* occ_out);

enum HashKind { HK_VARLEN = 0, HK_FIXED = 1, HK_FIXED_AL8 = 2, HK_PS = 3 };

template <int OUT>
struct VarEngine {
  static int hash(const Params& P, u64 n_jobs_bound, int kind, cudaStream_t st);
  static int tail(const TailParams& T, u64 nch, cudaStream_t st);
  static int small(const Params& P, cudaStream_t st);
  static int plan(const PlanParams& Q, unsigned grid, cudaStream_t st);
  static int merge(const MergeParams& M, cudaStream_t st);
};
extern template struct VarEngine<16>;
extern template struct VarEngine<24>;
extern template struct VarEngine<32>;
extern template struct VarEngine<40>;

}  // namespace hth
