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
// profiles/fp64_peak_r01.txt).  CTA = 4 warps; warp w owns rows 8w..8w+7 of a
// 32-row panel and the 9 n-tiles (72 columns) of the CTA; K streams through
// shared memory in chunks of 16 through a 3-stage cp.async ring.  Every
// thread's copy addresses are computed once per CTA.  Flops per application
// = sum_pieces 4 prod(m_a) sum(m_a).
#include <cstdint>

#include "internal.cuh"

namespace pmgcu {

namespace {

constexpr int kFdThreads = 128;
constexpr int kBM = 32;          // rows per CTA (4 warps x 8)
constexpr int kBK = 16;          // k per shared-memory stage
constexpr int kNTC = 9;          // n-tiles (of 8 columns) per CTA
constexpr int kBN = 8 * kNTC;    // 72 columns per CTA
constexpr int kXS = kBK + 4;     // X row stride (doubles): conflict-free A fragments
constexpr int kBS = 84;          // B row stride: round_up(72, 16) + 4, conflict-free B fragments
constexpr int kStagesFd = 3;
constexpr int kXPer = kBM * kBK / kFdThreads;  // 4 X copies per thread and stage
constexpr int kBPer = kBK * kBN / kFdThreads;  // 9 B copies per thread and stage

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kFdThreads) fd_pass_dmma_kernel(const FdPiece* __restrict__ pieces,
                                                                  const int4* __restrict__ items, int pass,
                                                                  int naxes, int in_mode, int out_mode,
                                                                  const double* __restrict__ lat_in,
                                                                  double* __restrict__ lat_out, double alpha,
                                                                  const double* __restrict__ work_in,
                                                                  double* __restrict__ work_out) {
  __shared__ __align__(16) double Xs[kStagesFd][kBM * kXS];
  __shared__ __align__(16) double Bs[kStagesFd][kBK * kBS];
  const int4 it = items[blockIdx.x];  // (piece, first row, first column, -)
  const FdPiece& P = pieces[it.x];
  const int axis = pass % naxes;
  const int dir = pass / naxes;
  const int K = P.dims[axis];
  const int N = K;
  const long long R = P.total / K;
  const long long r0 = it.y;
  const int n0 = it.z;
  const int m0 = P.dims[0], m1 = P.dims[1];
  const long long ext = P.ext, ext2 = (long long)P.ext * P.ext;
  const double* __restrict__ B = P.B[axis][dir];
  const int tid = threadIdx.x;

  // per-thread copy plan: X element (rr, kk) = (tid/16 + 8j, tid%16); B element
  // (kk, nn) of idx = tid + 128j
  const int xk = tid % kBK;
  const double* xsrc[kXPer];
  bool xrow_ok[kXPer];
#pragma unroll
  for (int j = 0; j < kXPer; ++j) {
    const long long r = r0 + tid / kBK + 8 * j;
    xrow_ok[j] = r < R;
    const long long rr = xrow_ok[j] ? r : 0;
    if (in_mode == FD_IN_WORK)
      xsrc[j] = work_in + P.work_off + rr * K + xk;
    else
      xsrc[j] = lat_in + P.lat_base + (naxes == 3 ? ext * (rr % m1) + ext2 * (rr / m1) : ext * rr) + xk;
  }
  int boff[kBPer], bkk[kBPer], bdst[kBPer];
  bool bn_ok[kBPer];
#pragma unroll
  for (int j = 0; j < kBPer; ++j) {
    const int idx = tid + kFdThreads * j;
    const int nn = idx % kBN, kk = idx / kBN;
    bn_ok[j] = n0 + nn < N;
    bkk[j] = kk;
    boff[j] = kk * N + n0 + nn;
    bdst[j] = kk * kBS + nn;
  }
  auto load = [&](int stage, int k0) {
    double* xs = Xs[stage];
    double* bs = Bs[stage];
#pragma unroll
    for (int j = 0; j < kXPer; ++j) {
      const bool ok = xrow_ok[j] && k0 + xk < K;
      cp_async8(xs + (tid / kBK + 8 * j) * kXS + xk, ok ? xsrc[j] + k0 : B, ok);
    }
#pragma unroll
    for (int j = 0; j < kBPer; ++j) {
      const bool ok = bn_ok[j] && k0 + bkk[j] < K;
      cp_async8(bs + bdst[j], ok ? B + boff[j] + (long long)k0 * N : B, ok);
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  double acc[kNTC][2];
#pragma unroll
  for (int j = 0; j < kNTC; ++j) acc[j][0] = acc[j][1] = 0.0;

  const int nst = (K + kBK - 1) / kBK;
#pragma unroll
  for (int s = 0; s < kStagesFd - 1; ++s) {
    if (s < nst) load(s, s * kBK);
    cp_async_commit();
  }
  for (int s = 0; s < nst; ++s) {
    const int cur = s % kStagesFd;
    cp_async_wait<kStagesFd - 2>();
    __syncthreads();
    {  // prefetch stage s + 2 into the slot freed at s - 1
      const int nxt = s + kStagesFd - 1;
      if (nxt < nst) load(nxt % kStagesFd, nxt * kBK);
      cp_async_commit();
    }
    const double* xs = Xs[cur] + (warp * 8 + g) * kXS + t;
    const double* bs = Bs[cur] + t * kBS + g;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const double a = xs[ks * 4];
#pragma unroll
      for (int j = 0; j < kNTC; ++j) dmma(acc[j][0], acc[j][1], a, bs[ks * 4 * kBS + j * 8]);
    }
  }

  // epilogue: lane holds rows r0+8w+g, columns n0+8j+2t+{0,1}; Y(r,n) at r + R n
  const long long r = r0 + warp * 8 + g;
  if (r >= R) return;
  long long lat_row = 0;
  if (out_mode >= FD_OUT_LATTICE_SET) lat_row = P.lat_base + (naxes == 3 ? (r % m0) + ext * (r / m0) : r);
  const long long lat_stride = naxes == 3 ? ext2 : ext;
#pragma unroll
  for (int j = 0; j < kNTC; ++j) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int n = n0 + j * 8 + 2 * t + i;
      if (n >= N) continue;
      const double v = acc[j][i];
      const long long o = r + R * n;
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

// ---------------------------------------------------------------- small pieces
// Pieces that fit in shared memory (coarse levels): one CTA runs the whole
// solve -- gather from the lattice (or a work buffer), d forward products,
// diagonal division, d backward products, scatter -- with no intermediate
// global traffic and one launch per smooth instead of 2d.  Same contraction
// order as FastDiagonalSolver::solve (ascending k per output).
constexpr int kSmallThreads = 256;

// out(t, j, o) = sum_k B[k*m + j] in(t, k, o) (layout axis 0 fastest) as a
// GEMM over rows (t, o): each warp owns 8 x 8 output tiles and runs DMMA over
// k in steps of 4; Bs is B staged in shared memory.
__device__ void small_axis(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ Bs,
                           int naxes, const int* dims, int axis) {
  int inner = 1, outer = 1;
  for (int a = 0; a < axis; ++a) inner *= dims[a];
  for (int a = axis + 1; a < naxes; ++a) outer *= dims[a];
  const int m = dims[axis];
  const int rows = inner * outer;
  const int tm_n = (rows + 7) / 8, tn_n = (m + 7) / 8, ks_n = (m + 3) / 4;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  for (int tile = warp; tile < tm_n * tn_n; tile += nwarps) {
    const int tm = tile % tm_n, tn = tile / tm_n;
    const int r = tm * 8 + g;  // A row of this lane
    const bool r_ok = r < rows;
    const int rt = r_ok ? r % inner : 0, ro = r_ok ? r / inner : 0;
    const double* arow = in + (long long)ro * inner * m + rt;
    const int n = tn * 8 + g;  // B column of this lane
    const bool n_ok = n < m;
    double d0 = 0.0, d1 = 0.0;
    for (int ks = 0; ks < ks_n; ++ks) {
      const int k = ks * 4 + t4;
      const double a = (r_ok && k < m) ? arow[(long long)k * inner] : 0.0;
      const double b = (n_ok && k < m) ? Bs[k * m + n] : 0.0;
      dmma(d0, d1, a, b);
    }
    const int orow = tm * 8 + g;
    if (orow < rows) {
      const int ot = orow % inner, oo = orow / inner;
      double* dst = out + (long long)oo * inner * m + ot;
      const int j0 = tn * 8 + 2 * t4;
      if (j0 < m) dst[(long long)j0 * inner] = d0;
      if (j0 + 1 < m) dst[(long long)(j0 + 1) * inner] = d1;
    }
  }
}

__device__ void stage_matrix(double* Bs, const double* __restrict__ B, int m) {
  for (int i = threadIdx.x; i < m * m; i += blockDim.x) Bs[i] = B[i];
}

__global__ void __launch_bounds__(kSmallThreads) fd_small_kernel(const FdPiece* __restrict__ pieces, int naxes,
                                                                 int in_mode, int out_mode,
                                                                 const double* __restrict__ lat_in,
                                                                 double* __restrict__ lat_out, double alpha,
                                                                 const double* __restrict__ work_in,
                                                                 double* __restrict__ work_out) {
  extern __shared__ double sm[];
  const FdPiece& P = pieces[blockIdx.x];
  const int dims[3] = {P.dims[0], P.dims[1], naxes == 3 ? P.dims[2] : 1};
  const int total = int(P.total);
  double* X = sm;
  double* Y = sm + total;
  double* Bs = sm + 2 * total;
  const long long ext = P.ext, ext2 = (long long)P.ext * P.ext;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    double v;
    if (in_mode == FD_IN_WORK) {
      v = work_in[P.work_off + idx];
    } else {
      const int i0 = idx % dims[0], i1 = (idx / dims[0]) % dims[1], i2 = idx / (dims[0] * dims[1]);
      v = lat_in[P.lat_base + i0 + ext * i1 + ext2 * i2];
    }
    X[idx] = v;
  }
  __syncthreads();
  for (int a = 0; a < naxes; ++a) {  // w = (x_a V_a^T) r
    stage_matrix(Bs, P.B[a][0], dims[a]);
    __syncthreads();
    small_axis(X, Y, Bs, naxes, dims, a);
    __syncthreads();
    double* tmp = X;
    X = Y;
    Y = tmp;
  }
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) X[idx] = X[idx] / P.diag[idx];
  __syncthreads();
  for (int a = 0; a < naxes; ++a) {  // x = (x_a V_a) w
    stage_matrix(Bs, P.B[a][1], dims[a]);
    __syncthreads();
    small_axis(X, Y, Bs, naxes, dims, a);
    __syncthreads();
    double* tmp = X;
    X = Y;
    Y = tmp;
  }
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const double v = X[idx];
    if (out_mode == FD_OUT_WORK || out_mode == FD_OUT_WORK_DIAG) {
      work_out[P.work_off + idx] = v;
    } else {
      const int i0 = idx % dims[0], i1 = (idx / dims[0]) % dims[1], i2 = idx / (dims[0] * dims[1]);
      const long long lat = P.lat_base + i0 + ext * i1 + ext2 * i2;
      if (out_mode == FD_OUT_LATTICE_SET)
        lat_out[lat] = alpha * v;
      else
        lat_out[lat] += alpha * v;
    }
  }
}

}  // namespace

size_t fd_small_smem(long long max_total, int max_dim) {
  return size_t(2 * max_total + (long long)max_dim * max_dim) * sizeof(double);
}

void launch_fd_small(cudaStream_t s, const FdPiece* pieces, int npieces, int naxes, long long max_total,
                     int max_dim, int in_mode, int out_mode, const double* lat_in, double* lat_out, double alpha,
                     const double* work_in, double* work_out) {
  if (npieces == 0) return;
  const size_t smem = fd_small_smem(max_total, max_dim);
  fd_small_kernel<<<npieces, kSmallThreads, smem, s>>>(pieces, naxes, in_mode, out_mode, lat_in, lat_out, alpha,
                                                       work_in, work_out);
}

void fd_configure() {
  cudaFuncSetAttribute(fd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

int fd_rows_per_block() { return kBM; }
int fd_cols_per_block() { return kBN; }

void launch_fd_pass(cudaStream_t s, const FdPiece* pieces, const int4* items, int nitems, int pass, int naxes,
                    int in_mode, int out_mode, const double* lat_in, double* lat_out, double alpha,
                    const double* work_in, double* work_out) {
  if (nitems == 0) return;
  fd_pass_dmma_kernel<<<nitems, kFdThreads, 0, s>>>(pieces, items, pass, naxes, in_mode, out_mode, lat_in, lat_out,
                                                    alpha, work_in, work_out);
}

}  // namespace pmgcu
