// Fast-diagonalization mode products for the interior and face pieces.
//
// Replaces FastDiagonalSolver::solve (tensor.cpp:132-140) and its dense
// apply_along_axis(_transpose) calls (tensor.cpp:18-50): w = (x_a V_a^T) r,
// w /= diag, x = (x_a V_a) w, batched over every piece of a level.
//
// Each pass contracts the fastest axis of its input and writes the new axis
// slowest (a cyclic rotation), so every pass is the same panel GEMM
//   Y(r, n) = sum_k X(r, k) B(k, n),   X rows contiguous in k,
// with Y stored column-wise (r fastest).  After d forward passes the tensor is
// back in its original layout, where the diagonal division is applied in the
// epilogue; d backward passes follow.  The first pass reads the patch lattice
// box directly (gather fused), the last writes it (scatter, optionally
// u += tau z fused).
//
// Roofline: FP64 tensor cores.  The contraction runs on DMMA
// (mma.sync.m8n8k4.f64, measured 37.0 TFLOP/s on B200 against 33.6 for DFMA,
// profiles/fp64_peak_r01.txt).  CTA = 8 warps; warp w owns rows 8w..8w+7 of a
// 64-row panel and NTC n-tiles of 8 columns; K streams through shared memory
// in chunks of 16 with cp.async double buffering.  Flops per application =
// sum_pieces 4 prod(m_a) sum(m_a).
#include <cstdint>

#include "internal.cuh"

namespace pmgcu {

namespace {

constexpr int kBM = 64;        // rows per CTA
constexpr int kBK = 16;        // k per shared-memory stage
constexpr int kNTC = 9;        // n-tiles (of 8 columns) per CTA
constexpr int kBN = 8 * kNTC;  // 72 columns per CTA
constexpr int kXS = kBK + 4;   // X row stride (doubles): conflict-free A fragments
constexpr int kBS = 84;        // B row stride: round_up(72, 16) + 4, conflict-free B fragments

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src_size = pred ? 8 : 0;  // 0 bytes read -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all_but_one() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct PassCtx {
  const FdPiece* P;
  int naxes, in_mode, K, N, m0, m1;
  long long R, r0, ext, ext2;
  const double* B;
  const double* lat_in;
  const double* work_in;
};

__device__ __forceinline__ const double* row_ptr(const PassCtx& c, long long r) {
  if (c.in_mode == FD_IN_WORK) return c.work_in + c.P->work_off + r * c.K;
  const long long base = c.naxes == 3 ? c.ext * (r % c.m1) + c.ext2 * (r / c.m1) : c.ext * r;
  return c.lat_in + c.P->lat_base + base;
}

__device__ __forceinline__ void load_stage(const PassCtx& c, int k0, int n0, double* Xs, double* Bs) {
  // X: 64 rows x 16 k, 8-byte transfers, zero-filled outside [R) x [K)
  for (int idx = threadIdx.x; idx < kBM * kBK; idx += kThreads) {
    const int kk = idx % kBK, rr = idx / kBK;
    const long long r = c.r0 + rr;
    const int k = k0 + kk;
    const bool ok = r < c.R && k < c.K;
    cp_async8(Xs + rr * kXS + kk, ok ? row_ptr(c, r) + k : c.B, ok);
  }
  // B: 16 k x 72 n
  for (int idx = threadIdx.x; idx < kBK * kBN; idx += kThreads) {
    const int nn = idx % kBN, kk = idx / kBN;
    const int k = k0 + kk, n = n0 + nn;
    const bool ok = k < c.K && n < c.N;
    cp_async8(Bs + kk * kBS + nn, ok ? c.B + (long long)k * c.N + n : c.B, ok);
  }
}

__global__ void __launch_bounds__(kThreads) fd_pass_dmma_kernel(const FdPiece* __restrict__ pieces,
                                                                const int4* __restrict__ items, int pass,
                                                                int naxes, int in_mode, int out_mode,
                                                                const double* __restrict__ lat_in,
                                                                double* __restrict__ lat_out, double alpha,
                                                                const double* __restrict__ work_in,
                                                                double* __restrict__ work_out) {
  __shared__ __align__(16) double Xs[2][kBM * kXS];
  __shared__ __align__(16) double Bs[2][kBK * kBS];
  const int4 it = items[blockIdx.x];  // (piece, first row, first column, -)
  PassCtx c;
  c.P = pieces + it.x;
  c.naxes = naxes;
  c.in_mode = in_mode;
  const int axis = pass % naxes;
  const int dir = pass / naxes;
  c.K = c.P->dims[axis];
  c.N = c.K;
  c.R = c.P->total / c.K;
  c.r0 = it.y;
  c.m0 = c.P->dims[0];
  c.m1 = c.P->dims[1];
  c.ext = c.P->ext;
  c.ext2 = (long long)c.P->ext * c.P->ext;
  c.B = c.P->B[axis][dir];
  c.lat_in = lat_in;
  c.work_in = work_in;
  const int n0 = it.z;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double acc[kNTC][2];
#pragma unroll
  for (int j = 0; j < kNTC; ++j) acc[j][0] = acc[j][1] = 0.0;

  const int nstages = (c.K + kBK - 1) / kBK;
  load_stage(c, 0, n0, Xs[0], Bs[0]);
  cp_async_commit();
  for (int s = 0; s < nstages; ++s) {
    const int cur = s & 1;
    if (s + 1 < nstages) {
      load_stage(c, (s + 1) * kBK, n0, Xs[cur ^ 1], Bs[cur ^ 1]);
      cp_async_commit();
      cp_async_wait_all_but_one();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    const double* xs = Xs[cur] + (warp * 8 + g) * kXS + t;
    const double* bs = Bs[cur] + t * kBS + g;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const double a = xs[ks * 4];
#pragma unroll
      for (int j = 0; j < kNTC; ++j) dmma(acc[j][0], acc[j][1], a, bs[ks * 4 * kBS + j * 8]);
    }
    __syncthreads();
  }

  // epilogue: lane holds rows r0+8w+g, columns n0+8j+2t+{0,1}; Y(r,n) at r + R n
  const long long r = c.r0 + warp * 8 + g;
  if (r >= c.R) return;
  const FdPiece& P = *c.P;
  long long lat_row = 0;
  if (out_mode >= FD_OUT_LATTICE_SET)
    lat_row = P.lat_base + (naxes == 3 ? (r % c.m0) + c.ext * (r / c.m0) : r);
  const long long lat_stride = naxes == 3 ? c.ext2 : c.ext;
#pragma unroll
  for (int j = 0; j < kNTC; ++j) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int n = n0 + j * 8 + 2 * t + i;
      if (n >= c.N) continue;
      const double v = acc[j][i];
      const long long o = r + c.R * n;
      switch (out_mode) {
        case FD_OUT_WORK:
          work_out[P.work_off + o] = v;
          break;
        case FD_OUT_WORK_DIAG:
          work_out[P.work_off + o] = v / P.diag[o];
          break;
        case FD_OUT_LATTICE_SET:
          lat_out[lat_row + lat_stride * n] = alpha * v;
          break;
        default:
          lat_out[lat_row + lat_stride * n] += alpha * v;
      }
    }
  }
}

}  // namespace

void fd_configure() {}

int fd_rows_per_block() { return kBM; }
int fd_cols_per_block() { return kBN; }

void launch_fd_pass(cudaStream_t s, const FdPiece* pieces, const int4* items, int nitems, int pass, int naxes,
                    int in_mode, int out_mode, const double* lat_in, double* lat_out, double alpha,
                    const double* work_in, double* work_out) {
  if (nitems == 0) return;
  fd_pass_dmma_kernel<<<nitems, kThreads, 0, s>>>(pieces, items, pass, naxes, in_mode, out_mode, lat_in, lat_out,
                                                  alpha, work_in, work_out);
}

}  // namespace pmgcu
