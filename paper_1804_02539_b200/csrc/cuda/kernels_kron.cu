// Matrix-free patch operator for axis-aligned affine patches (SURVEY.md 8(f)
// row 2).
//
// On a patch whose geometry map is x_a = c_a + h_a xi_a the stiffness the
// reference assembles by quadrature (assemble_patch_stiffness,
// assembly.cpp:127-248) is the exact Kronecker sum
//   A = sum_a g_a (x)_{b != a} M  (x) K   (K on axis a),
//   g_a = prod_{b != a} |h_b| / |h_a|,
// of the univariate mass M and stiffness K of the level's free-end spline space
// (the reference's own identity test: test_assembly.cpp:112-146).  M and K are
// (2p+1)-banded, so y = A x is d axis sweeps of 2p+1 terms instead of a
// (2p+1)^d band: 8 B x (x, f, y) + 4 B (l2g) per lattice row instead of
// 4 (2p+1)^d + 28 B (half band), and no band in HBM at all.
//
// Replaces PatchOperator::apply_add + the scatter of MultiPatchOperator::apply
// (assembly.cpp:12-18,265-280) on levels described as PMG_BAND_KRONECKER.
// Dirichlet rows and columns are removed as in the assembled band: x holds 0
// on Dirichlet slots (accumulated vectors), rows with l2g < 0 are written 0.
// The sum order differs from the reference's CSR order, so results agree to
// rounding (about 1e-15 relative), not bitwise.
//
// 2D: one kernel.  A CTA owns TL lattice lines of one patch: the x lines
// [L0-p, L0+TL+p) go to shared memory once, the axis-0 sweeps (M x, K x) of
// those lines stay in shared memory, the axis-1 sweep writes y.
// 3D: three sweeps through L2-resident scratch lattices.
#include <cstdint>

#include "internal.cuh"

namespace pmgcu {

namespace {

constexpr int kKronThreads = 256;

// block-wide deterministic sum -> partial[blockIdx.x]
__device__ __forceinline__ void block_partial(double v, double* __restrict__ partial) {
  __shared__ double wsum[kKronThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kKronThreads / 32; ++w) s += wsum[w];
    partial[blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------- 2D, fused
// shared memory (doubles): Ms, Ks [E][W]; xs [TL+2p][E+2p] (zero halo);
// tm, tk [TL+2p][E]
template <int P>
__global__ void __launch_bounds__(kKronThreads) kron2d_kernel(KronArgs a, int TL) {
  PMG_PDL_ENTRY();
  constexpr int W = 2 * P + 1;
  extern __shared__ __align__(16) double ksm[];
  const int E = a.ext;
  const int NL = TL + 2 * P;  // lines held
  const int XS = E + 2 * P;   // x line stride
  double* Ms = ksm;
  double* Ks = Ms + E * W;
  double* xs = Ks + E * W;
  double* tm = xs + NL * XS;
  double* tk = tm + NL * E;
  const int nseg = (E + TL - 1) / TL;
  const int k = blockIdx.x / nseg;
  const int L0 = (blockIdx.x % nseg) * TL;
  const long long base = (long long)k * a.S;
  const double* __restrict__ x = a.x + base;
  for (int i = threadIdx.x; i < E * W; i += kKronThreads) {
    Ms[i] = a.M[i];
    Ks[i] = a.Kst[i];
  }
  for (int i = threadIdx.x; i < NL * XS; i += kKronThreads) {
    const int l = i / XS, c = i % XS - P;
    const int line = L0 - P + l;
    xs[i] = (line >= 0 && line < E && c >= 0 && c < E) ? x[(long long)line * E + c] : 0.0;
  }
  __syncthreads();
  // axis 0: tm = M x, tk = K x on every held line (rows of M, K are zero
  // outside the lattice, the halo of xs is zero)
  for (int i = threadIdx.x; i < NL * E; i += kKronThreads) {
    const int l = i / E, c = i % E;
    const double* xr = xs + l * XS + c;  // xs column c - P
    const double* mr = Ms + c * W;
    const double* kr = Ks + c * W;
    double sm = 0.0, sk = 0.0;
#pragma unroll
    for (int d = 0; d < W; ++d) {
      const double v = xr[d];
      sm = fma(mr[d], v, sm);
      sk = fma(kr[d], v, sk);
    }
    tm[i] = sm;
    tk[i] = sk;
  }
  __syncthreads();
  // axis 1: y = g0 M1 (K0 x) + g1 K1 (M0 x)
  const double g0 = a.g[3 * k + 0], g1 = a.g[3 * k + 1];
  double dot = 0.0;
  const int lines = min(TL, E - L0);
  for (int i = threadIdx.x; i < lines * E; i += kKronThreads) {
    const int l = i / E, c = i % E;
    const int line = L0 + l;
    const double* mr = Ms + line * W;
    const double* kr = Ks + line * W;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int d = 0; d < W; ++d) {
      s0 = fma(mr[d], tk[(l + d) * E + c], s0);
      s1 = fma(kr[d], tm[(l + d) * E + c], s1);
    }
    const long long r = (long long)line * E + c;
    double v = fma(g0, s0, g1 * s1);
    if (a.l2g[base + r] < 0) v = 0.0;
    if (a.dot_partial) dot = fma(v, xs[(l + P) * XS + c + P], dot);
    a.y[base + r] = a.f ? a.f[base + r] - v : v;
  }
  if (a.dot_partial) block_partial(dot, a.dot_partial);
}

// ---------------------------------------------------------------- 3D, three sweeps
// sweep along `axis` (stride st, index i_axis) of one band matrix row
template <int P>
__device__ __forceinline__ double sweep(const double* __restrict__ T, int i, int E, const double* __restrict__ v,
                                        long long st) {
  constexpr int W = 2 * P + 1;
  const double* tr = T + i * W;
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < W; ++d) {
    const int j = i + d - P;
    if (j >= 0 && j < E) s = fma(tr[d], v[(long long)(d - P) * st], s);
  }
  return s;
}

// axis 0: t0 = M x, t1 = K x
template <int P>
__global__ void __launch_bounds__(kKronThreads) kron3d_axis0_kernel(KronArgs a, double* __restrict__ t0,
                                                                    double* __restrict__ t1) {
  PMG_PDL_ENTRY();
  const long long n = a.S * a.K;
  const long long idx = (long long)blockIdx.x * kKronThreads + threadIdx.x;
  if (idx >= n) return;
  const int i0 = int(idx % a.ext);
  t0[idx] = sweep<P>(a.M, i0, a.ext, a.x + idx, 1);
  t1[idx] = sweep<P>(a.Kst, i0, a.ext, a.x + idx, 1);
}

// axis 1: u0 = M1 t1 (K0 M1), u1 = K1 t0 (M0 K1), u2 = M1 t0 (M0 M1)
template <int P>
__global__ void __launch_bounds__(kKronThreads) kron3d_axis1_kernel(KronArgs a, const double* __restrict__ t0,
                                                                    const double* __restrict__ t1,
                                                                    double* __restrict__ u0, double* __restrict__ u1,
                                                                    double* __restrict__ u2) {
  PMG_PDL_ENTRY();
  const long long n = a.S * a.K;
  const long long idx = (long long)blockIdx.x * kKronThreads + threadIdx.x;
  if (idx >= n) return;
  const int E = a.ext;
  const int i1 = int((idx / E) % E);
  u0[idx] = sweep<P>(a.M, i1, E, t1 + idx, E);
  u1[idx] = sweep<P>(a.Kst, i1, E, t0 + idx, E);
  u2[idx] = sweep<P>(a.M, i1, E, t0 + idx, E);
}

// axis 2: y = g0 M2 u0 + g1 M2 u1 + g2 K2 u2
template <int P>
__global__ void __launch_bounds__(kKronThreads) kron3d_axis2_kernel(KronArgs a, const double* __restrict__ u0,
                                                                    const double* __restrict__ u1,
                                                                    const double* __restrict__ u2) {
  PMG_PDL_ENTRY();
  const long long n = a.S * a.K;
  const long long idx = (long long)blockIdx.x * kKronThreads + threadIdx.x;
  double dot = 0.0;
  if (idx < n) {
    const int E = a.ext;
    const long long E2 = (long long)E * E;
    const int k = int(idx / a.S);
    const int i2 = int((idx % a.S) / E2);
    double v = a.g[3 * k + 0] * sweep<P>(a.M, i2, E, u0 + idx, E2);
    v = fma(a.g[3 * k + 1], sweep<P>(a.M, i2, E, u1 + idx, E2), v);
    v = fma(a.g[3 * k + 2], sweep<P>(a.Kst, i2, E, u2 + idx, E2), v);
    if (a.l2g[idx] < 0) v = 0.0;
    if (a.dot_partial) dot = v * a.x[idx];
    a.y[idx] = a.f ? a.f[idx] - v : v;
  }
  if (a.dot_partial) block_partial(dot, a.dot_partial);
}

size_t kron2d_smem(int p, int E, int TL) {
  const int W = 2 * p + 1, NL = TL + 2 * p;
  return sizeof(double) * (size_t(2) * E * W + size_t(NL) * (E + 2 * p) + size_t(2) * NL * E);
}

}  // namespace

int kron2d_lines(int p, int ext, int K) {
  // lines per CTA: 32 (the axis-0 sweep of the 2p halo lines is recomputed by
  // the neighbouring CTA), 16 when that leaves most SMs without a CTA
  // (measured at c3p8, 16 patches of 136 lines: 25 us with 32 lines on 80 CTAs;
  // 8 lines on 272 CTAs with M, K through L1: 47 us); fewer if the tile
  // exceeds shared memory
  int tl = 32;
  if ((long long)K * ((ext + 31) / 32) < 120) tl = 16;
  while (tl > 1 && kron2d_smem(p, ext, tl) > 200 * 1024) tl /= 2;
  return kron2d_smem(p, ext, tl) <= 200 * 1024 ? tl : 0;
}

int kron_partials(int dim, int degree, int ext, long long S, int K) {
  if (dim == 2) {
    const int tl = kron2d_lines(degree, ext, K);
    return K * ((ext + tl - 1) / tl);
  }
  return int((S * K + kKronThreads - 1) / kKronThreads);
}

bool kron_supported(int dim, int degree, int ext) {
  if (degree < 1 || degree > 8) return false;
  return dim == 3 || (dim == 2 && kron2d_lines(degree, ext, 1 << 20) > 0);
}

void launch_kron_spmv(cudaStream_t s, const KronArgs& a, int* launches) {
  const long long n = a.S * a.K;
  const int blocks = int((n + kKronThreads - 1) / kKronThreads);
#define PMG_KRON_CASE(PP)                                                                                         \
  case PP:                                                                                                        \
    if (a.dim == 2) {                                                                                             \
      const int tl = kron2d_lines(PP, a.ext, a.K);                                                                     \
      const size_t smem = kron2d_smem(PP, a.ext, tl);                                                             \
      ensure_smem((const void*)kron2d_kernel<PP>, smem);                                                          \
      launch_k(kron2d_kernel<PP>, dim3(a.K * ((a.ext + tl - 1) / tl)), dim3(kKronThreads), smem, s, a, tl);       \
      *launches += 1;                                                                                             \
    } else {                                                                                                      \
      double* t = a.scratch;                                                                                      \
      launch_k(kron3d_axis0_kernel<PP>, dim3(blocks), dim3(kKronThreads), 0, s, a, t, t + n);                     \
      launch_k(kron3d_axis1_kernel<PP>, dim3(blocks), dim3(kKronThreads), 0, s, a, (const double*)t,              \
               (const double*)(t + n), t + 2 * n, t + 3 * n, t + 4 * n);                                          \
      launch_k(kron3d_axis2_kernel<PP>, dim3(blocks), dim3(kKronThreads), 0, s, a, (const double*)(t + 2 * n),    \
               (const double*)(t + 3 * n), (const double*)(t + 4 * n));                                           \
      *launches += 3;                                                                                             \
    }                                                                                                             \
    return;
  switch (a.degree) {
    PMG_KRON_CASE(1) PMG_KRON_CASE(2) PMG_KRON_CASE(3) PMG_KRON_CASE(4) PMG_KRON_CASE(5) PMG_KRON_CASE(6)
    PMG_KRON_CASE(7) PMG_KRON_CASE(8)
    default:
      throw LaunchError("Kronecker operator: degree outside 1..8");
  }
#undef PMG_KRON_CASE
}

}  // namespace pmgcu
