// Compile-time HalftimeHash variant geometry and constants.
//
// Mirrors the reference's fixed parameter table (halftimehash 0.1.0,
// pkg/src/halftimehash/params.py:211-227) and the matrices/codes it uses
// (params.py:105-130, 185-209).  Everything is constexpr so the encode and
// combine loops unroll into straight-line LOP3/PRMT/IMAD code with the
// coefficients folded in.
#pragma once
#include <cstdint>

namespace hth {

// GF(16) with x^4 + x + 1 on single 4-bit elements (gf16.py:17-44).
__host__ __device__ constexpr int gf_xt4(int a) { return ((a << 1) & 0xF) ^ ((a >> 3) & 1) ^ (((a >> 3) & 1) << 1); }
__host__ __device__ constexpr int gf_mul4(int a, int b) {
  int acc = 0, t = b;
  for (int i = 0; i < 4; i++) {
    if ((a >> i) & 1) acc ^= t;
    t = gf_xt4(t);
  }
  return acc;
}
__host__ __device__ constexpr int gf_inv4(int a) {
  for (int b = 1; b < 16; b++)
    if (gf_mul4(a, b) == 1) return b;
  return 0;
}

// Cauchy parity coefficient (params.py:115-130): inv(j XOR (parities + i)).
__host__ __device__ constexpr int cauchy(int parities, int j, int i) { return gf_inv4(j ^ (parities + i)); }

template <int OUT> struct Var;

// bytes k e d w (b = f = 8)  -- params.py:217-227
template <> struct Var<16> {
  static constexpr int out = 16, k = 2, e = 7, d = 6, w = 2;
  __host__ __device__ static constexpr int par(int, int) { return 1; }  // XOR parity (params.py:105-112)
  __host__ __device__ static constexpr int mat(int r, int c) {
    constexpr int M[2][7] = {{1, 0, 1, 1, 2, 1, 4}, {0, 1, 1, 2, 1, 4, 1}};
    return M[r][c];
  }
};
template <> struct Var<24> {
  static constexpr int out = 24, k = 3, e = 9, d = 7, w = 3;
  __host__ __device__ static constexpr int par(int j, int i) { return cauchy(2, j, i); }
  __host__ __device__ static constexpr int mat(int r, int c) {
    constexpr int M[3][9] = {{0, 0, 1, 4, 1, 1, 2, 2, 1}, {1, 1, 0, 0, 1, 4, 1, 2, 2}, {1, 4, 1, 1, 0, 0, 2, 1, 2}};
    return M[r][c];
  }
};
template <> struct Var<32> {
  static constexpr int out = 32, k = 4, e = 10, d = 7, w = 3;
  __host__ __device__ static constexpr int par(int j, int i) { return cauchy(3, j, i); }
  __host__ __device__ static constexpr int mat(int r, int c) {
    constexpr int M[4][10] = {{0, 0, 0, 1, 1, 4, 2, 4, 1, 1},
                              {0, 1, 2, 0, 0, 1, 1, 2, 4, 1},
                              {2, 0, 1, 0, 4, 0, 1, 1, 1, 1},
                              {1, 1, 0, 1, 0, 0, 4, 1, 2, 8}};
    return M[r][c];
  }
};
template <> struct Var<40> {
  static constexpr int out = 40, k = 5, e = 9, d = 5, w = 3;
  __host__ __device__ static constexpr int par(int j, int i) { return cauchy(4, j, i); }
  __host__ __device__ static constexpr int mat(int r, int c) {
    constexpr int M[5][9] = {{1, 0, 0, 0, 0, 1, 1, 2, 4},
                             {0, 1, 0, 0, 0, 1, 2, 1, 7},
                             {0, 0, 1, 0, 0, 1, 3, 8, 5},
                             {0, 0, 0, 1, 0, 1, 4, 9, 8},
                             {0, 0, 0, 0, 1, 1, 5, 3, 9}};
    return M[r][c];
  }
};

// Derived geometry shared by host and device.
template <class V> struct Geo {
  static constexpr int b = 8, f = 8;
  static constexpr int m = V::d * V::w * 8;  // u64 words per instance (params.py:171-177)
  static constexpr int ew = V::e * V::w;     // EHC seed words (params.py:179-182)
  static constexpr int inst_bytes = m * 8;
};

// Host-side runtime view of the same table (for layout math in the C-ABI).
struct VarInfo {
  int out, k, e, d, w, m, ew;
};
inline bool var_info(int out, VarInfo* v) {
  switch (out) {
    case 16: *v = {16, 2, 7, 6, 2, 96, 14}; return true;
    case 24: *v = {24, 3, 9, 7, 3, 168, 27}; return true;
    case 32: *v = {32, 4, 10, 7, 3, 168, 30}; return true;
    case 40: *v = {40, 5, 9, 5, 3, 120, 27}; return true;
    default: return false;
  }
}

}  // namespace hth
