// Index-free tensor-band stiffness SpMV / residual.
//
// Replaces PatchOperator::apply_add (assembly.cpp:12-18) driven by
// MultiPatchOperator::apply (assembly.cpp:265-280) and
// ParallelBackend::apply_op/residual (parallel.cpp:281-304).  Vectors stay in
// the per-patch lattice form, so there is no gather/scatter through l2g: the
// distributed result y_k = A_k x_k is the patch's share.
//
// Roofline: HBM.  Algorithmic bytes per launch = 8 B per stored band entry
// (reference count, harness.cpp:274-282) + 8 B x read + 8 B f read + 8 B y
// write per lattice row.  One thread per row; for a fixed band offset a warp
// reads 32 consecutive rows = 256 contiguous bytes (band is offset-major).
// The row's sum runs over the offsets in the reference CSR column order
// (axis 0 fastest).
#include "internal.cuh"

namespace pmgcu {

namespace {

template <int D, int P>
__global__ void __launch_bounds__(kThreads) spmv_kernel(SpmvArgs a) {
  constexpr int W = 2 * P + 1;
  constexpr int O = D == 2 ? W * W : W * W * W;
  const long long S = a.S;
  const int ext = a.ext;
  const long long rows = S * a.K;
  const long long gid = (long long)blockIdx.x * kThreads + threadIdx.x;
  double prod = 0.0;
  if (gid < rows) {
    const long long k = gid / S;
    const long long r = gid - k * S;
    const int i0 = int(r % ext);
    const int i1 = int((r / ext) % ext);
    const int i2 = D == 3 ? int(r / ((long long)ext * ext)) : 0;
    const double* __restrict__ band = a.band + (size_t)k * O * S + r;
    const double* __restrict__ x = a.x + gid;
    const long long ext2 = (long long)ext * ext;
    double acc = 0.0;
#pragma unroll
    for (int d2 = (D == 3 ? -P : 0); d2 <= (D == 3 ? P : 0); ++d2) {
      const bool ok2 = D == 2 || (i2 + d2 >= 0 && i2 + d2 < ext);
#pragma unroll
      for (int d1 = -P; d1 <= P; ++d1) {
        const bool ok1 = ok2 && (i1 + d1 >= 0 && i1 + d1 < ext);
#pragma unroll
        for (int d0 = -P; d0 <= P; ++d0) {
          const int o = (d0 + P) + W * ((d1 + P) + W * (D == 3 ? d2 + P : 0));
          const long long off = d0 + (long long)ext * d1 + ext2 * d2;
          if (ok1 && i0 + d0 >= 0 && i0 + d0 < ext) acc = fma(__ldcs(band + (size_t)o * S), __ldg(x + off), acc);
        }
      }
    }
    const double y = a.f ? a.f[gid] - acc : acc;
    a.y[gid] = y;
    if (a.dot_partial) prod = y * x[0];
  }
  if (a.dot_partial) {
    __shared__ double red[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) prod += __shfl_down_sync(0xffffffffu, prod, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = prod;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) s += red[w];
      a.dot_partial[blockIdx.x] = s;
    }
  }
}

// Runtime-degree fallback (degrees without a specialisation).
__global__ void __launch_bounds__(kThreads) spmv_generic_kernel(SpmvArgs a) {
  const int D = a.dim, P = a.degree, W = 2 * P + 1;
  const int O = D == 2 ? W * W : W * W * W;
  const long long S = a.S;
  const int ext = a.ext;
  const long long rows = S * a.K;
  const long long gid = (long long)blockIdx.x * kThreads + threadIdx.x;
  double prod = 0.0;
  if (gid < rows) {
    const long long k = gid / S;
    const long long r = gid - k * S;
    const int i0 = int(r % ext), i1 = int((r / ext) % ext), i2 = D == 3 ? int(r / ((long long)ext * ext)) : 0;
    const double* band = a.band + (size_t)k * O * S + r;
    const double* x = a.x + gid;
    double acc = 0.0;
    for (int d2 = (D == 3 ? -P : 0); d2 <= (D == 3 ? P : 0); ++d2) {
      if (D == 3 && (i2 + d2 < 0 || i2 + d2 >= ext)) continue;
      for (int d1 = -P; d1 <= P; ++d1) {
        if (i1 + d1 < 0 || i1 + d1 >= ext) continue;
        for (int d0 = -P; d0 <= P; ++d0) {
          if (i0 + d0 < 0 || i0 + d0 >= ext) continue;
          const int o = (d0 + P) + W * ((d1 + P) + W * (D == 3 ? d2 + P : 0));
          acc = fma(band[(size_t)o * S], x[d0 + (long long)ext * d1 + (long long)ext * ext * d2], acc);
        }
      }
    }
    const double y = a.f ? a.f[gid] - acc : acc;
    a.y[gid] = y;
    if (a.dot_partial) prod = y * x[0];
  }
  if (a.dot_partial) {
    __shared__ double red[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) prod += __shfl_down_sync(0xffffffffu, prod, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = prod;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) s += red[w];
      a.dot_partial[blockIdx.x] = s;
    }
  }
}

}  // namespace

int spmv_blocks(long long rows) { return int((rows + kThreads - 1) / kThreads); }

void launch_spmv(cudaStream_t s, const SpmvArgs& a) {
  const int grid = spmv_blocks(a.S * a.K);
  if (grid == 0) return;
#define PMG_SPMV_CASE(D, P) \
  if (a.dim == D && a.degree == P) { spmv_kernel<D, P><<<grid, kThreads, 0, s>>>(a); return; }
  PMG_SPMV_CASE(2, 1) PMG_SPMV_CASE(2, 2) PMG_SPMV_CASE(2, 3) PMG_SPMV_CASE(2, 4)
  PMG_SPMV_CASE(2, 5) PMG_SPMV_CASE(2, 6) PMG_SPMV_CASE(2, 8)
  PMG_SPMV_CASE(3, 1) PMG_SPMV_CASE(3, 2) PMG_SPMV_CASE(3, 3) PMG_SPMV_CASE(3, 4)
#undef PMG_SPMV_CASE
  spmv_generic_kernel<<<grid, kThreads, 0, s>>>(a);
}

}  // namespace pmgcu
