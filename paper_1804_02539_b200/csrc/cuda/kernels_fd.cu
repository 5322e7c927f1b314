// Fast-diagonalization mode products for the interior and face pieces.
//
// Replaces FastDiagonalSolver::solve (tensor.cpp:132-140) and its dense
// apply_along_axis(_transpose) calls (tensor.cpp:18-50): w = (x_a V_a^T) r,
// w /= diag, x = (x_a V_a) w, batched over every piece of a level.
//
// Each pass contracts the fastest axis of its input and writes the new axis
// slowest (a cyclic rotation), so every pass is the same row-panel GEMM
// Y(r, n) = sum_k X(r, k) B(k, n) with X rows contiguous in k and Y written
// column-wise (r fastest).  After d forward passes the tensor is back in the
// original layout, where the diagonal division is applied in the epilogue;
// d backward passes follow.  The first pass reads the patch lattice box
// directly (gather fused), the last writes it (scatter, optionally
// u += tau z fused).
//
// Roofline: FP64 (DFMA).  Flops per application = sum_pieces 4 prod(m_a)
// sum(m_a).  CTA tile: BM rows x the whole N (BN >= N), K in
// chunks of 8 through shared memory, a RM x RN register tile per thread.
#include "internal.cuh"

namespace pmgcu {

namespace {

constexpr int kBK = 8;

template <int TX, int RM, int RN>
struct Tile {
  static constexpr int TY = kThreads / TX;
  static constexpr int BM = TY * RM;
  static constexpr int BN = TX * RN;
  static constexpr int SMEM_OPS = kBK * (BM + BN);
  static constexpr int SMEM_C = BN * (BM + 1);
  static constexpr int SMEM = SMEM_OPS > SMEM_C ? SMEM_OPS : SMEM_C;
};

template <int TX, int RM, int RN>
__global__ void __launch_bounds__(kThreads) fd_pass_kernel(const FdPiece* __restrict__ pieces,
                                                           const int2* __restrict__ items, int pass, int naxes,
                                                           int in_mode, int out_mode,
                                                           const double* __restrict__ lat_in,
                                                           double* __restrict__ lat_out, double alpha,
                                                           const double* __restrict__ work_in,
                                                           double* __restrict__ work_out) {
  using T = Tile<TX, RM, RN>;
  constexpr int BM = T::BM, BN = T::BN, TY = T::TY;
  extern __shared__ double smem[];
  double* Xs = smem;             // [kBK][BM]
  double* Bs = smem + kBK * BM;  // [kBK][BN]

  const int2 it = items[blockIdx.x];
  const FdPiece& P = pieces[it.x];
  const int axis = pass % naxes;
  const int dir = pass / naxes;
  const int K = P.dims[axis];
  const int N = K;
  const long long R = P.total / K;
  const long long r0 = it.y;
  const double* __restrict__ B = P.B[axis][dir];
  const int tx = threadIdx.x % TX;
  const int ty = threadIdx.x / TX;
  const int m0 = P.dims[0], m1 = P.dims[1];
  const long long ext = P.ext, ext2 = (long long)P.ext * P.ext;

  double acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) acc[i][j] = 0.0;

  for (int k0 = 0; k0 < K; k0 += kBK) {
    for (int idx = threadIdx.x; idx < BM * kBK; idx += kThreads) {
      const int kk = idx % kBK, rr = idx / kBK;
      const long long r = r0 + rr;
      const int k = k0 + kk;
      double v = 0.0;
      if (r < R && k < K) {
        if (in_mode == FD_IN_WORK) {
          v = work_in[P.work_off + r * K + k];
        } else {  // pass 0 on the lattice box: rows are (i1, i2), k = i0
          long long base;
          if (naxes == 3)
            base = ext * (r % m1) + ext2 * (r / m1);
          else
            base = ext * r;
          v = lat_in[P.lat_base + base + k];
        }
      }
      Xs[kk * BM + rr] = v;
    }
    for (int idx = threadIdx.x; idx < BN * kBK; idx += kThreads) {
      const int nn = idx % BN, kk = idx / BN;
      const int k = k0 + kk;
      Bs[kk * BN + nn] = (k < K && nn < N) ? B[(long long)k * N + nn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      double xv[RM], bv[RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) xv[i] = Xs[kk * BM + ty * RM + i];
#pragma unroll
      for (int j = 0; j < RN; ++j) bv[j] = Bs[kk * BN + tx + TX * j];
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = fma(xv[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  // stage the BM x BN tile n-major, then write columns with r fastest
  double* Cs = smem;
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) Cs[(tx + TX * j) * (BM + 1) + ty * RM + i] = acc[i][j];
  __syncthreads();
  const int rows = int(min((long long)BM, R - r0));
  for (int idx = threadIdx.x; idx < BM * N; idx += kThreads) {
    const int rr = idx % BM, n = idx / BM;
    if (rr >= rows) continue;
    const long long r = r0 + rr;
    double v = Cs[n * (BM + 1) + rr];
    const long long o = r + R * n;
    switch (out_mode) {
      case FD_OUT_WORK:
        work_out[P.work_off + o] = v;
        break;
      case FD_OUT_WORK_DIAG:
        work_out[P.work_off + o] = v / P.diag[o];
        break;
      default: {  // last pass: rows (j0, j1), n = j_last
        long long lat;
        if (naxes == 3)
          lat = P.lat_base + (r % m0) + ext * (r / m0) + ext2 * n;
        else
          lat = P.lat_base + r + ext * n;
        if (out_mode == FD_OUT_LATTICE_SET)
          lat_out[lat] = alpha * v;
        else
          lat_out[lat] += alpha * v;
      }
    }
  }
  (void)TY;
}

template <int TX, int RM, int RN>
void launch_tile(cudaStream_t s, const FdPiece* pieces, const int2* items, int nitems, int pass, int naxes, int in_mode,
                 int out_mode, const double* lat_in, double* lat_out, double alpha, const double* work_in,
                 double* work_out) {
  using T = Tile<TX, RM, RN>;
  const size_t smem = sizeof(double) * T::SMEM;
  fd_pass_kernel<TX, RM, RN><<<nitems, kThreads, smem, s>>>(pieces, items, pass, naxes, in_mode, out_mode, lat_in,
                                                            lat_out, alpha, work_in, work_out);
}

template <int TX, int RM, int RN>
void configure_tile() {
  cudaFuncSetAttribute(fd_pass_kernel<TX, RM, RN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(double) * Tile<TX, RM, RN>::SMEM));
}

}  // namespace

void fd_configure() {
  configure_tile<32, 4, 9>();
  configure_tile<8, 4, 9>();
}

// narrow tile: N <= 72, BM = 128 rows; wide tile: N <= 288, BM = 32 rows
int fd_rows_per_block(bool wide) { return wide ? Tile<32, 4, 9>::BM : Tile<8, 4, 9>::BM; }

void launch_fd_pass(cudaStream_t s, bool wide, const FdPiece* pieces, const int2* items, int nitems, int pass,
                    int naxes, int in_mode, int out_mode, const double* lat_in, double* lat_out, double alpha,
                    const double* work_in, double* work_out) {
  if (nitems == 0) return;
  if (wide)
    launch_tile<32, 4, 9>(s, pieces, items, nitems, pass, naxes, in_mode, out_mode, lat_in, lat_out, alpha, work_in,
                          work_out);
  else
    launch_tile<8, 4, 9>(s, pieces, items, nitems, pass, naxes, in_mode, out_mode, lat_in, lat_out, alpha, work_in,
                         work_out);
}

}  // namespace pmgcu
