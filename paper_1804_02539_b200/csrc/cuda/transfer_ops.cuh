// Per-output device bodies of the two-scale transfers (restriction and
// prolongation outputs of one patch lattice), used by the fused transfer
// kernels of kernels_misc.cu.
#pragma once

#include "internal.cuh"

namespace pmgcu {

constexpr int kRowMaxP = 8;  // largest specialised degree

// Two-scale rows and columns have at most p+2 entries; the innermost sums
// below load all of theirs before multiplying (predicated, fixed bound).
constexpr int kTsMax = kRowMaxP + 2;

// Coarse output idx (patch-major lattice of level l-1) of the restriction
// (apply_along_axis_transpose(TwoScale), tensor.cpp:78-102, per patch as in
// restrict_patch, transfer.cpp:54-66): s0 over the fine rows of axis 0
// inner, then axis 1, then axis 2; Dirichlet coarse slots are 0.
__device__ __forceinline__ double restrict_out(const TsDev& ts, int d, int ext_f, int ext_c, long long Sc,
                                               long long Sf, const double* __restrict__ r, long long idx) {
  const long long k = idx / Sc;
  const long long rem = idx - k * Sc;
  const int j0 = int(rem % ext_c), j1 = int((rem / ext_c) % ext_c), j2 = d == 3 ? int(rem / ((long long)ext_c * ext_c)) : 0;
  const double* src = r + k * Sf;
  const int a0 = ts.col_off[j0], n0 = ts.col_off[j0 + 1] - a0;
  int c0[kTsMax];
  double w0[kTsMax];
#pragma unroll
  for (int q = 0; q < kTsMax; ++q) {
    c0[q] = q < n0 ? ts.col_row[a0 + q] : 0;
    w0[q] = q < n0 ? ts.col_val[a0 + q] : 0.0;
  }
  double s2 = 0.0;
  const int q2a = d == 3 ? ts.col_off[j2] : 0, q2b = d == 3 ? ts.col_off[j2 + 1] : 1;
  for (int q2 = q2a; q2 < q2b; ++q2) {
    const long long b2 = d == 3 ? (long long)ts.col_row[q2] * ext_f * ext_f : 0;
    double s1 = 0.0;
    for (int q1 = ts.col_off[j1]; q1 < ts.col_off[j1 + 1]; ++q1) {
      const double* row = src + b2 + (long long)ts.col_row[q1] * ext_f;
      double v[kTsMax];
#pragma unroll
      for (int q = 0; q < kTsMax; ++q) v[q] = q < n0 ? row[c0[q]] : 0.0;
      double s0 = 0.0;
#pragma unroll
      for (int q = 0; q < kTsMax; ++q)
        if (q < n0) s0 = fma(w0[q], v[q], s0);
      s1 = fma(ts.col_val[q1], s0, s1);
    }
    s2 = d == 3 ? fma(ts.col_val[q2], s1, s2) : s1;
  }
  return s2;
}

// Fine output idx of the prolongation P c (apply_along_axis(TwoScale),
// tensor.cpp:52-76, prolong_patch, transfer.cpp:21-38): the <= p+1 coarse
// parents per axis, axis 0 innermost.
__device__ __forceinline__ double prolong_out(const TsDev& ts, int d, int ext_f, int ext_c, long long Sc, long long Sf,
                                              const double* __restrict__ c, long long idx) {
  const long long k = idx / Sf;
  const long long rem = idx - k * Sf;
  const int i0 = int(rem % ext_f), i1 = int((rem / ext_f) % ext_f), i2 = d == 3 ? int(rem / ((long long)ext_f * ext_f)) : 0;
  const double* src = c + k * Sc;
  const int n0 = ts.row_len[i0], st0 = ts.row_start[i0];
  const double* v0 = ts.vals + ts.row_off[i0];
  double w0[kTsMax];
#pragma unroll
  for (int q = 0; q < kTsMax; ++q) w0[q] = q < n0 ? v0[q] : 0.0;
  const int n2 = d == 3 ? ts.row_len[i2] : 1;
  double s2 = 0.0;
  for (int q2 = 0; q2 < n2; ++q2) {
    const long long b2 = d == 3 ? (long long)(ts.row_start[i2] + q2) * ext_c * ext_c : 0;
    double s1 = 0.0;
    for (int q1 = 0; q1 < ts.row_len[i1]; ++q1) {
      const double* row = src + b2 + (long long)(ts.row_start[i1] + q1) * ext_c + st0;
      double v[kTsMax];
#pragma unroll
      for (int q = 0; q < kTsMax; ++q) v[q] = q < n0 ? row[q] : 0.0;
      double s0 = 0.0;
#pragma unroll
      for (int q = 0; q < kTsMax; ++q)
        if (q < n0) s0 = fma(w0[q], v[q], s0);
      s1 = fma(ts.vals[ts.row_off[i1] + q1], s0, s1);
    }
    s2 = d == 3 ? fma(ts.vals[ts.row_off[i2] + q2], s1, s2) : s1;
  }
  return s2;
}

}  // namespace pmgcu
