// Stiffness assembly on the device.
//
// Replaces assemble_patch_stiffness (/root/reference/proj/src/assembly.cpp:
// 127-248): A_ij = sum_elements sum_q w_q |det J| grad B_i^T J^-1 J^-T grad B_j
// with p+1 Gauss-Legendre points per element and direction.  The reference
// forms element matrices E = G H^T and scatters them; here the tensor-product
// structure is used instead (sum factorization).  With
//   C_ab(q) = w_q |det J(q)| (J^-1 J^-T)_ab          (d(d+1)/2 fields)
//   T^0 / T^1 = univariate basis value / derivative,
// every entry is a product of 1D factors per axis:
//   A[i, i+delta] = sum_ab sum_q C_ab(q) prod_x T^[a==x](i_x, q_x) T^[b==x](i_x+delta_x, q_x),
// so the quadrature axes are contracted one at a time, slowest first:
//   3D  C[ab][q2][q1][q0] -> Z1[ab][i2,d2][q1][q0] -> Z2[ab][i2,d2][i1,d1][q0] -> band[o][r]
//   2D  C[ab][q1][q0]     -> Z1[ab][i1,d1][q0]     -> band[o][r]
// Each output sums over the common support of its two basis functions along
// the contracted axis only (<= (p+1)^2 points).  The intermediates live in HBM
// (c4 finest level: 7 GB of scratch per patch); every stage is a plain
// thread-per-output kernel whose reads and writes are coalesced along the
// fastest index.  The result equals the host assembly up to rounding (a
// different summation order), checked by tests/test_gpu_assembly.py.
#include <cuda_runtime.h>

#include <chrono>
#include <string>
#include <vector>

#include "../host/numerics.hpp"
#include "internal.cuh"

namespace pmgcu {

namespace {

struct AsmDims {
  int d, p, n, q1, ext, W;
  long long Q;   // quadrature points per axis = n q1
  long long S;   // ext^d
  int ncomp;     // d (d + 1) / 2 coefficient fields
};

__device__ __forceinline__ int sym_index(int d, int a, int b) {
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
  // 2D: 00 01 11 -> 0 1 2; 3D: 00 01 02 11 12 22 -> 0..5
  return d == 2 ? a + b : (a == 0 ? b : (a == 1 ? 2 + b : 5));
}

// geometry Jacobian at quadrature point (k0,k1,k2) (GeometryMap::jacobian,
// geometry.cpp:62-79): J[i*d+j] = sum over the (gd+1)^d support of
// ctrl[flat][i] * prod_x (x == j ? dN_x : N_x); gtab[x] = [Q][2][gd_x+1]
__device__ void geo_jacobian(int d, const long long* q, const int* gdeg, const int* gncoef, const int* const* gfirst,
                             const double* const* gtab, const double* __restrict__ ctrl, double* J) {
  for (int i = 0; i < d * d; ++i) J[i] = 0.0;
  const int n0 = gdeg[0] + 1, n1 = gdeg[1] + 1, n2 = d == 3 ? gdeg[2] + 1 : 1;
  const double* t0 = gtab[0] + q[0] * 2 * n0;
  const double* t1 = gtab[1] + q[1] * 2 * n1;
  const double* t2 = d == 3 ? gtab[2] + q[2] * 2 * n2 : nullptr;
  const int f0 = gfirst[0][q[0]], f1 = gfirst[1][q[1]], f2 = d == 3 ? gfirst[2][q[2]] : 0;
  for (int j = 0; j < d; ++j)
    for (int c2 = 0; c2 < n2; ++c2)
      for (int c1 = 0; c1 < n1; ++c1)
        for (int c0 = 0; c0 < n0; ++c0) {
          double w = (j == 0 ? t0[n0 + c0] : t0[c0]) * (j == 1 ? t1[n1 + c1] : t1[c1]);
          if (d == 3) w *= j == 2 ? t2[n2 + c2] : t2[c2];
          const long long flat =
              (f0 + c0) + (long long)gncoef[0] * ((f1 + c1) + (long long)gncoef[1] * (d == 3 ? f2 + c2 : 0));
          for (int i = 0; i < d; ++i) J[i * d + j] += w * ctrl[flat * d + i];
        }
}

struct GeoArgs {
  int gdeg[3], gncoef[3];
  const int* gfirst[3];
  const double* gtab[3];
  const double* ctrl;
};

// C_ab at every quadrature point of one patch (assembly.cpp:161-182 semantics:
// w = prod_x weight_x / n, s = w |det J|, C_ab = s sum_k Ji_ak Ji_bk, and the
// folded / degenerate map check against the sign at the first point)
__global__ void asm_coeff_kernel(AsmDims A, GeoArgs G, const double* __restrict__ qw, double* __restrict__ coef,
                                 int* __restrict__ err) {
  PMG_PDL_ENTRY();
  const long long npts = A.d == 3 ? A.Q * A.Q * A.Q : A.Q * A.Q;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= npts) return;
  long long q[3] = {idx % A.Q, (idx / A.Q) % A.Q, A.d == 3 ? idx / (A.Q * A.Q) : 0};
  double J[9], Ji[9];
  const long long q00[3] = {0, 0, 0};
  geo_jacobian(A.d, q00, G.gdeg, G.gncoef, G.gfirst, G.gtab, G.ctrl, J);
  const double det00 = A.d == 2 ? J[0] * J[3] - J[1] * J[2]
                                : J[0] * (J[4] * J[8] - J[5] * J[7]) + J[1] * (J[5] * J[6] - J[3] * J[8]) +
                                      J[2] * (J[3] * J[7] - J[4] * J[6]);
  const double sgn = det00 > 0.0 ? 1.0 : -1.0;
  geo_jacobian(A.d, q, G.gdeg, G.gncoef, G.gfirst, G.gtab, G.ctrl, J);
  double w = 1.0;
  for (int a = 0; a < A.d; ++a) w *= qw[q[a] % A.q1] / A.n;
  double det;
  if (A.d == 2) {
    det = J[0] * J[3] - J[1] * J[2];
    Ji[0] = J[3] / det;
    Ji[1] = -J[1] / det;
    Ji[2] = -J[2] / det;
    Ji[3] = J[0] / det;
  } else {
    const double c00 = J[4] * J[8] - J[5] * J[7];
    const double c01 = J[5] * J[6] - J[3] * J[8];
    const double c02 = J[3] * J[7] - J[4] * J[6];
    det = J[0] * c00 + J[1] * c01 + J[2] * c02;
    Ji[0] = c00 / det;
    Ji[3] = c01 / det;
    Ji[6] = c02 / det;
    Ji[1] = (J[2] * J[7] - J[1] * J[8]) / det;
    Ji[4] = (J[0] * J[8] - J[2] * J[6]) / det;
    Ji[7] = (J[1] * J[6] - J[0] * J[7]) / det;
    Ji[2] = (J[1] * J[5] - J[2] * J[4]) / det;
    Ji[5] = (J[2] * J[3] - J[0] * J[5]) / det;
    Ji[8] = (J[0] * J[4] - J[1] * J[3]) / det;
  }
  if (!(det * sgn > 1e-14)) atomicOr(err, 1);
  const double s = w * fabs(det);
  for (int a = 0; a < A.d; ++a)
    for (int b = a; b < A.d; ++b) {
      double m = 0.0;
      for (int k = 0; k < A.d; ++k) m += Ji[a * A.d + k] * Ji[b * A.d + k];
      coef[(long long)sym_index(A.d, a, b) * npts + idx] = s * m;
    }
}

// sum over the common support of basis i and i+delta along one axis:
// sum_{e,k} T^al(e, i-e, k) T^be(e, i+delta-e, k) * src(e q1 + k)
struct Window {
  int lo, hi;
};
__device__ __forceinline__ Window common_support(int i, int delta, int p, int n) {
  const int j = i + delta;
  Window w;
  w.lo = max(max(0, i - p), j - p);
  w.hi = min(min(n - 1, i), j);
  return w;
}
__device__ __forceinline__ double tab(const double* __restrict__ T, const AsmDims& A, int al, int e, int l, int k) {
  return __ldg(T + (((long long)al * A.n + e) * (A.p + 1) + l) * A.q1 + k);
}

// 3D stage 1: Z1[ab][i2][w2][qq] (qq = q1 Q + q0) = sum_q2 P2 C[ab][q2][qq]
__global__ void asm_stage_slow_kernel(AsmDims A, const double* __restrict__ T, const double* __restrict__ coef,
                                      double* __restrict__ out) {
  PMG_PDL_ENTRY();
  const int naxes_rest = A.d - 1;  // the contracted axis is A.d - 1
  const long long plane = naxes_rest == 2 ? A.Q * A.Q : A.Q;
  const long long qq = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (qq >= plane) return;
  const int iw = blockIdx.y;  // i * W + w
  const int ab = blockIdx.z;  // a * d + b
  const int i = iw / A.W, delta = iw % A.W - A.p;
  const int a = ab / A.d, b = ab % A.d;
  const int x = A.d - 1;
  const int al = a == x, be = b == x;
  const double* __restrict__ src = coef + (long long)sym_index(A.d, a, b) * plane * A.Q;
  const Window win = common_support(i, delta, A.p, A.n);
  double acc = 0.0;
  for (int e = win.lo; e <= win.hi; ++e)
    for (int k = 0; k < A.q1; ++k)
      acc = fma(tab(T, A, al, e, i - e, k) * tab(T, A, be, e, i + delta - e, k),
                src[((long long)e * A.q1 + k) * plane + qq], acc);
  out[((long long)ab * A.ext * A.W + iw) * plane + qq] = acc;
}

// 3D stage 2: Z2[ab][iw2][i1][w1][q0] = sum_q1 P1 Z1[ab][iw2][q1][q0]
__global__ void asm_stage_mid_kernel(AsmDims A, const double* __restrict__ T, const double* __restrict__ z1,
                                     double* __restrict__ out) {
  PMG_PDL_ENTRY();
  const long long q0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q0 >= A.Q) return;
  const int iw1 = blockIdx.y;
  const long long z = blockIdx.z;  // ab * (ext W) + iw2
  const int nw = A.ext * A.W;
  const int ab = int(z / nw);
  const int a = ab / A.d, b = ab % A.d;
  const int al = a == 1, be = b == 1;
  const int i = iw1 / A.W, delta = iw1 % A.W - A.p;
  const double* __restrict__ src = z1 + z * A.Q * A.Q;
  const Window win = common_support(i, delta, A.p, A.n);
  double acc = 0.0;
  for (int e = win.lo; e <= win.hi; ++e)
    for (int k = 0; k < A.q1; ++k)
      acc = fma(tab(T, A, al, e, i - e, k) * tab(T, A, be, e, i + delta - e, k),
                src[((long long)e * A.q1 + k) * A.Q + q0], acc);
  out[(z * nw + iw1) * A.Q + q0] = acc;
}

// last stage: band[o][r] = sum_ab sum_q0 P0 Z[ab][(i_rest, w_rest)][q0]
__global__ void asm_stage_band_kernel(AsmDims A, const double* __restrict__ T, const double* __restrict__ zin,
                                      double* __restrict__ band, long long Sp, int Ob) {
  PMG_PDL_ENTRY();
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int o = blockIdx.y;
  if (r >= A.S || o >= Ob) return;
  const int i0 = int(r % A.ext), i1 = int((r / A.ext) % A.ext), i2 = A.d == 3 ? int(r / ((long long)A.ext * A.ext)) : 0;
  const int w0 = o % A.W, w1 = (o / A.W) % A.W, w2 = A.d == 3 ? o / (A.W * A.W) : 0;
  const int delta = w0 - A.p;
  const Window win = common_support(i0, delta, A.p, A.n);
  const int nw = A.ext * A.W;
  // row of the input block: 2D (i1, w1); 3D (i2, w2, i1, w1)
  const long long rest = A.d == 3 ? ((long long)(i2 * A.W + w2) * nw + (i1 * A.W + w1)) : (i1 * A.W + w1);
  const long long per_ab = A.d == 3 ? (long long)nw * nw : nw;
  double acc = 0.0;
  if (win.lo <= win.hi) {
    for (int ab = 0; ab < A.d * A.d; ++ab) {
      const int a = ab / A.d, b = ab % A.d;
      const int al = a == 0, be = b == 0;
      const double* __restrict__ src = zin + ((long long)ab * per_ab + rest) * A.Q;
      for (int e = win.lo; e <= win.hi; ++e)
        for (int k = 0; k < A.q1; ++k)
          acc = fma(tab(T, A, al, e, i0 - e, k) * tab(T, A, be, e, i0 + delta - e, k), src[(long long)e * A.q1 + k],
                    acc);
    }
  }
  band[(long long)o * Sp + r] = acc;
}

inline void ckA(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw AssemblyError(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

namespace {

// ---------------------------------------------------------------- load vector
// assemble_rhs (assembly.cpp:299-365) by sum factorization: the source term
// times w |det J| on the patch's tensor quadrature grid, then one contraction
// with the basis values per axis.  Source kinds as in pmg_host.h (PMGH_RHS_*).
__device__ __forceinline__ unsigned long long splitmix64_dev(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// node_uniform (hierarchy.cpp): uniform in [-1, 1) from (seed, index)
__device__ __forceinline__ double node_uniform_dev(unsigned long long seed, unsigned long long index) {
  const unsigned long long z = splitmix64_dev(seed ^ (index * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull));
  return 2.0 * (double(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}

// physical point of quadrature point q (GeometryMap::eval, geometry.cpp:50-60)
__device__ void geo_point(int d, const long long* q, const GeoArgs& G, double* x) {
  for (int i = 0; i < d; ++i) x[i] = 0.0;
  const int n0 = G.gdeg[0] + 1, n1 = G.gdeg[1] + 1, n2 = d == 3 ? G.gdeg[2] + 1 : 1;
  const double* t0 = G.gtab[0] + q[0] * 2 * n0;
  const double* t1 = G.gtab[1] + q[1] * 2 * n1;
  const double* t2 = d == 3 ? G.gtab[2] + q[2] * 2 * n2 : nullptr;
  const int f0 = G.gfirst[0][q[0]], f1 = G.gfirst[1][q[1]], f2 = d == 3 ? G.gfirst[2][q[2]] : 0;
  for (int c2 = 0; c2 < n2; ++c2)
    for (int c1 = 0; c1 < n1; ++c1)
      for (int c0 = 0; c0 < n0; ++c0) {
        double w = t0[c0] * t1[c1];
        if (d == 3) w *= t2[c2];
        const long long flat =
            (f0 + c0) + (long long)G.gncoef[0] * ((f1 + c1) + (long long)G.gncoef[1] * (d == 3 ? f2 + c2 : 0));
        for (int i = 0; i < d; ++i) x[i] += w * G.ctrl[flat * d + i];
      }
}

// c(q) = w |det J| f(q) at every quadrature point of one patch
__global__ void load_coeff_kernel(AsmDims A, GeoArgs G, const double* __restrict__ qw, int kind,
                                  unsigned long long seed, unsigned long long patch, double* __restrict__ coef,
                                  int* __restrict__ err) {
  PMG_PDL_ENTRY();
  const long long npts = A.d == 3 ? A.Q * A.Q * A.Q : A.Q * A.Q;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= npts) return;
  long long q[3] = {idx % A.Q, (idx / A.Q) % A.Q, A.d == 3 ? idx / (A.Q * A.Q) : 0};
  double J[9];
  const long long q00[3] = {0, 0, 0};
  auto det_of = [&](const double* M) {
    return A.d == 2 ? M[0] * M[3] - M[1] * M[2]
                    : M[0] * (M[4] * M[8] - M[5] * M[7]) + M[1] * (M[5] * M[6] - M[3] * M[8]) +
                          M[2] * (M[3] * M[7] - M[4] * M[6]);
  };
  geo_jacobian(A.d, q00, G.gdeg, G.gncoef, G.gfirst, G.gtab, G.ctrl, J);
  const double sgn = det_of(J) > 0.0 ? 1.0 : -1.0;
  geo_jacobian(A.d, q, G.gdeg, G.gncoef, G.gfirst, G.gtab, G.ctrl, J);
  const double det = det_of(J);
  if (!(det * sgn > 1e-14)) atomicOr(err, 1);
  double w = 1.0;
  for (int a = 0; a < A.d; ++a) w *= qw[q[a] % A.q1] / A.n;
  double f;
  if (kind == 5) {  // PMGH_RHS_RANDOM_NODES: index (patch, element, point) as the host loop numbers them
    unsigned long long e = 0, k = 0, ecount = 1, nq = 1;
    for (int a = A.d - 1; a >= 0; --a) {
      e = e * A.n + (unsigned long long)(q[a] / A.q1);
      k = k * A.q1 + (unsigned long long)(q[a] % A.q1);
      ecount *= A.n;
      nq *= A.q1;
    }
    f = node_uniform_dev(seed, (patch * ecount + e) * nq + k);
  } else if (kind == 1) {
    f = 1.0;
  } else if (kind == 6) {
    f = 0.0;
  } else {
    double x[3];
    geo_point(A.d, q, G, x);
    const double pi = 3.14159265358979323846;
    if (kind == 2)
      f = 50.0 * pi * pi * sin(5 * pi * x[0]) * sin(5 * pi * x[1]);
    else if (kind == 3)
      f = 75.0 * pi * pi * sin(5 * pi * x[0]) * sin(5 * pi * x[1]) * sin(5 * pi * x[2]);
    else
      f = 2.0 * pi * pi * sin(pi * x[0]) * sin(pi * x[1]);
  }
  coef[idx] = w * fabs(det) * f;
}

// contract the fastest quadrature axis of src [outer][Q] with the basis values:
// dst[i + ext o] = sum over the support of basis i (elements i-p..i, q1 points
// each).  transpose_out: the contracted axis becomes the slowest of dst
// ([i][outer] instead of [outer][i]), so three calls rotate the tensor back.
__global__ void load_contract_kernel(AsmDims A, const double* __restrict__ T, const double* __restrict__ src,
                                     long long outer, double* __restrict__ dst, const int* __restrict__ l2g) {
  PMG_PDL_ENTRY();
  const long long n = outer * A.ext;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= n) return;
  // consecutive threads walk `outer` (coalesced writes of the rotated layout)
  const long long o = idx % outer;
  const int i = int(idx / outer);
  const double* row = src + o * A.Q;
  double s = 0.0;
  for (int e = max(0, i - A.p); e <= min(A.n - 1, i); ++e)
    for (int k = 0; k < A.q1; ++k) s += tab(T, A, 0, e, i - e, k) * row[(long long)e * A.q1 + k];
  if (l2g) s = l2g[idx] >= 0 ? s : 0.0;
  dst[idx] = s;
}

}  // namespace

double assemble_level_device(cudaStream_t s, int dim, int degree, int elements, const pmg_patch_geometry* geo,
                             int patch_begin, int K, double* band, long long Sp, int Ob) {
  const auto t0 = std::chrono::steady_clock::now();
  AsmDims A;
  A.d = dim;
  A.p = degree;
  A.n = elements;
  A.q1 = degree + 1;
  A.ext = elements + degree;
  A.W = 2 * degree + 1;
  A.Q = (long long)elements * A.q1;
  A.S = 1;
  for (int a = 0; a < dim; ++a) A.S *= A.ext;
  A.ncomp = dim * (dim + 1) / 2;
  const pmg::QuadratureRule& rule = pmg::gauss_legendre(A.q1);

  // univariate basis tables at the Gauss points of every element, as the host
  // tabulates them (hierarchy.cpp tabulate): T[al][e][l][k]
  std::vector<double> T(size_t(2) * A.n * (A.p + 1) * A.q1);
  {
    pmg::UnivariateSpace space(degree, elements);
    for (int e = 0; e < A.n; ++e)
      for (int k = 0; k < A.q1; ++k) {
        const double x = (e + rule.nodes[k]) / elements;
        const pmg::BasisEval bv = pmg::eval_basis(space, x, 0);
        const pmg::BasisEval bd = pmg::eval_basis(space, x, 1);
        for (int l = 0; l <= A.p; ++l) {
          T[((size_t(0) * A.n + e) * (A.p + 1) + l) * A.q1 + k] = bv.values[l];
          T[((size_t(1) * A.n + e) * (A.p + 1) + l) * A.q1 + k] = bd.values[l];
        }
      }
  }
  // device scratch for this level, freed at the end
  const long long npts = dim == 3 ? A.Q * A.Q * A.Q : A.Q * A.Q;
  const long long nw = (long long)A.ext * A.W;
  const long long z1n = (long long)dim * dim * nw * (dim == 3 ? A.Q * A.Q : A.Q);
  const long long z2n = dim == 3 ? (long long)dim * dim * nw * nw * A.Q : 0;
  std::vector<void*> owned;
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    ckA(cudaMalloc(&p, bytes < 8 ? 8 : bytes), "assembly scratch");
    owned.push_back(p);
    return p;
  };
  struct Free {
    std::vector<void*>& v;
    ~Free() {
      for (void* p : v) cudaFree(p);
    }
  } freer{owned};
  double* dT = static_cast<double*>(dalloc(T.size() * sizeof(double)));
  double* dqw = static_cast<double*>(dalloc(A.q1 * sizeof(double)));
  double* dcoef = static_cast<double*>(dalloc(size_t(A.ncomp) * npts * sizeof(double)));
  double* dz1 = static_cast<double*>(dalloc(size_t(z1n) * sizeof(double)));
  double* dz2 = dim == 3 ? static_cast<double*>(dalloc(size_t(z2n) * sizeof(double))) : nullptr;
  int* derr = static_cast<int*>(dalloc(sizeof(int)));
  ckA(cudaMemcpyAsync(dT, T.data(), T.size() * sizeof(double), cudaMemcpyHostToDevice, s), "assembly tables");
  ckA(cudaMemcpyAsync(dqw, rule.weights.data(), A.q1 * sizeof(double), cudaMemcpyHostToDevice, s), "weights");
  ckA(cudaMemsetAsync(derr, 0, sizeof(int), s), "memset");

  for (int k = 0; k < K; ++k) {
    const pmg_patch_geometry& g = geo[patch_begin + k];
    GeoArgs G{};
    std::vector<int> first[3];
    std::vector<double> gt[3];
    long long nctrl = 1;
    for (int a = 0; a < dim; ++a) {
      if (g.degree[a] < 1 || g.degree[a] > pmg::kMaxDegree || g.elements[a] < 1)
        throw AssemblyError("assembly: bad patch geometry description");
      G.gdeg[a] = g.degree[a];
      G.gncoef[a] = g.elements[a] + g.degree[a];
      nctrl *= G.gncoef[a];
      pmg::UnivariateSpace gs(g.degree[a], g.elements[a]);
      const int ng = g.degree[a] + 1;
      first[a].resize(size_t(A.Q));
      gt[a].resize(size_t(A.Q) * 2 * ng);
      for (int e = 0; e < A.n; ++e)
        for (int kq = 0; kq < A.q1; ++kq) {
          const long long q = (long long)e * A.q1 + kq;
          const double x = (e + rule.nodes[kq]) / elements;
          const pmg::BasisEval bv = pmg::eval_basis(gs, x, 0);
          const pmg::BasisEval bd = pmg::eval_basis(gs, x, 1);
          if (bv.first_index != bd.first_index) throw AssemblyError("assembly: inconsistent geometry support");
          first[a][q] = bv.first_index;
          for (int c = 0; c < ng; ++c) {
            gt[a][size_t(q) * 2 * ng + c] = bv.values[c];
            gt[a][size_t(q) * 2 * ng + ng + c] = bd.values[c];
          }
        }
      int* df = static_cast<int*>(dalloc(first[a].size() * sizeof(int)));
      double* dg = static_cast<double*>(dalloc(gt[a].size() * sizeof(double)));
      ckA(cudaMemcpyAsync(df, first[a].data(), first[a].size() * sizeof(int), cudaMemcpyHostToDevice, s), "geo");
      ckA(cudaMemcpyAsync(dg, gt[a].data(), gt[a].size() * sizeof(double), cudaMemcpyHostToDevice, s), "geo");
      G.gfirst[a] = df;
      G.gtab[a] = dg;
    }
    double* dctrl = static_cast<double*>(dalloc(size_t(nctrl) * dim * sizeof(double)));
    ckA(cudaMemcpyAsync(dctrl, g.ctrl, size_t(nctrl) * dim * sizeof(double), cudaMemcpyHostToDevice, s), "ctrl");
    G.ctrl = dctrl;

    launch_k(asm_coeff_kernel, dim3(unsigned((npts + 255) / 256)), dim3(256), 0, s, A, G, (const double*)dqw, dcoef,
             derr);
    double* bk = band + size_t(k) * Ob * Sp;
    if (dim == 3) {
      launch_k(asm_stage_slow_kernel, dim3(unsigned((A.Q * A.Q + 255) / 256), unsigned(nw), 9u), dim3(256), 0, s, A,
               (const double*)dT, (const double*)dcoef, dz1);
      launch_k(asm_stage_mid_kernel, dim3(unsigned((A.Q + 127) / 128), unsigned(nw), unsigned(9 * nw)), dim3(128), 0,
               s, A, (const double*)dT, (const double*)dz1, dz2);
      launch_k(asm_stage_band_kernel, dim3(unsigned((A.S + 255) / 256), unsigned(Ob)), dim3(256), 0, s, A,
               (const double*)dT, (const double*)dz2, bk, Sp, Ob);
    } else {
      launch_k(asm_stage_slow_kernel, dim3(unsigned((A.Q + 255) / 256), unsigned(nw), 4u), dim3(256), 0, s, A,
               (const double*)dT, (const double*)dcoef, dz1);
      launch_k(asm_stage_band_kernel, dim3(unsigned((A.S + 255) / 256), unsigned(Ob)), dim3(256), 0, s, A,
               (const double*)dT, (const double*)dz1, bk, Sp, Ob);
    }
    ckA(cudaGetLastError(), "assembly launch");
    // the per-patch tables are freed with the scratch; keep the stream ordered
    ckA(cudaStreamSynchronize(s), "assembly");
  }
  int herr = 0;
  ckA(cudaMemcpy(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost), "assembly flag");
  if (herr) throw AssemblyError("assembly: degenerate or folded geometry map");
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Load vector of the local patches on the device: out = the distributed
// lattice vector [K][ext^d] (every patch's own share; Dirichlet slots 0).
// kind = PMGH_RHS_* resolved (1 one, 2 sine2d, 3 sine3d, 4 sine_pi,
// 5 random_nodes, 6 zero).  Returns wall seconds.
double assemble_load_device(cudaStream_t s, int dim, int degree, int elements, const pmg_patch_geometry* geo,
                            int patch_begin, int K, int kind, unsigned long long seed, const int* l2g,
                            double* out) {
  const auto t0 = std::chrono::steady_clock::now();
  if (kind < 1 || kind > 6) throw AssemblyError("load vector: unknown source kind");
  if ((kind == 2 || kind == 4) && dim != 2) throw AssemblyError("load vector: 2D source on a 3D domain");
  if (kind == 3 && dim != 3) throw AssemblyError("load vector: 3D source on a 2D domain");
  AsmDims A;
  A.d = dim;
  A.p = degree;
  A.n = elements;
  A.q1 = degree + 1;
  A.ext = elements + degree;
  A.W = 2 * degree + 1;
  A.Q = (long long)elements * A.q1;
  A.S = 1;
  for (int a = 0; a < dim; ++a) A.S *= A.ext;
  A.ncomp = 1;
  const pmg::QuadratureRule& rule = pmg::gauss_legendre(A.q1);
  std::vector<double> T(size_t(2) * A.n * (A.p + 1) * A.q1, 0.0);
  {
    pmg::UnivariateSpace space(degree, elements);
    for (int e = 0; e < A.n; ++e)
      for (int k = 0; k < A.q1; ++k) {
        const pmg::BasisEval bv = pmg::eval_basis(space, (e + rule.nodes[k]) / elements, 0);
        for (int l = 0; l <= A.p; ++l) T[((size_t(0) * A.n + e) * (A.p + 1) + l) * A.q1 + k] = bv.values[l];
      }
  }
  const long long npts = dim == 3 ? A.Q * A.Q * A.Q : A.Q * A.Q;
  std::vector<void*> owned;
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    ckA(cudaMalloc(&p, bytes < 8 ? 8 : bytes), "load vector scratch");
    owned.push_back(p);
    return p;
  };
  struct Free {
    std::vector<void*>& v;
    ~Free() {
      for (void* p : v) cudaFree(p);
    }
  } freer{owned};
  double* dT = static_cast<double*>(dalloc(T.size() * sizeof(double)));
  double* dqw = static_cast<double*>(dalloc(A.q1 * sizeof(double)));
  double* dcoef = static_cast<double*>(dalloc(size_t(npts) * sizeof(double)));
  const long long n1 = (dim == 3 ? A.Q * A.Q : A.Q) * A.ext;
  const long long n2 = dim == 3 ? A.Q * A.ext * A.ext : 0;
  double* dt1 = static_cast<double*>(dalloc(size_t(n1) * sizeof(double)));
  double* dt2 = dim == 3 ? static_cast<double*>(dalloc(size_t(n2) * sizeof(double))) : nullptr;
  int* derr = static_cast<int*>(dalloc(sizeof(int)));
  ckA(cudaMemcpyAsync(dT, T.data(), T.size() * sizeof(double), cudaMemcpyHostToDevice, s), "load vector tables");
  ckA(cudaMemcpyAsync(dqw, rule.weights.data(), A.q1 * sizeof(double), cudaMemcpyHostToDevice, s), "weights");
  ckA(cudaMemsetAsync(derr, 0, sizeof(int), s), "memset");
  auto blocks = [](long long n) { return dim3(unsigned((n + 255) / 256)); };
  for (int k = 0; k < K; ++k) {
    const pmg_patch_geometry& g = geo[patch_begin + k];
    GeoArgs G{};
    long long nctrl = 1;
    for (int a = 0; a < dim; ++a) {
      if (g.degree[a] < 1 || g.degree[a] > pmg::kMaxDegree || g.elements[a] < 1)
        throw AssemblyError("load vector: bad patch geometry description");
      G.gdeg[a] = g.degree[a];
      G.gncoef[a] = g.elements[a] + g.degree[a];
      nctrl *= G.gncoef[a];
      pmg::UnivariateSpace gs(g.degree[a], g.elements[a]);
      const int ng = g.degree[a] + 1;
      std::vector<int> first(size_t(A.Q));
      std::vector<double> gt(size_t(A.Q) * 2 * ng);
      for (int e = 0; e < A.n; ++e)
        for (int kq = 0; kq < A.q1; ++kq) {
          const long long q = (long long)e * A.q1 + kq;
          const double x = (e + rule.nodes[kq]) / elements;
          const pmg::BasisEval bv = pmg::eval_basis(gs, x, 0);
          const pmg::BasisEval bd = pmg::eval_basis(gs, x, 1);
          first[q] = bv.first_index;
          for (int c = 0; c < ng; ++c) {
            gt[size_t(q) * 2 * ng + c] = bv.values[c];
            gt[size_t(q) * 2 * ng + ng + c] = bd.values[c];
          }
        }
      int* df = static_cast<int*>(dalloc(first.size() * sizeof(int)));
      double* dg = static_cast<double*>(dalloc(gt.size() * sizeof(double)));
      // pageable sources: the copies return once staged
      ckA(cudaMemcpyAsync(df, first.data(), first.size() * sizeof(int), cudaMemcpyHostToDevice, s), "geo");
      ckA(cudaMemcpyAsync(dg, gt.data(), gt.size() * sizeof(double), cudaMemcpyHostToDevice, s), "geo");
      ckA(cudaStreamSynchronize(s), "geo");
      G.gfirst[a] = df;
      G.gtab[a] = dg;
    }
    double* dctrl = static_cast<double*>(dalloc(size_t(nctrl) * dim * sizeof(double)));
    ckA(cudaMemcpyAsync(dctrl, g.ctrl, size_t(nctrl) * dim * sizeof(double), cudaMemcpyHostToDevice, s), "ctrl");
    G.ctrl = dctrl;
    launch_k(load_coeff_kernel, blocks(npts), dim3(256), 0, s, A, G, (const double*)dqw, kind, seed,
             (unsigned long long)(patch_begin + k), dcoef, derr);
    double* ok = out + size_t(k) * A.S;
    const int* lk = l2g + size_t(k) * A.S;
    if (dim == 3) {
      launch_k(load_contract_kernel, blocks(n1), dim3(256), 0, s, A, (const double*)dT, (const double*)dcoef,
               A.Q * A.Q, dt1, (const int*)nullptr);
      launch_k(load_contract_kernel, blocks(n2), dim3(256), 0, s, A, (const double*)dT, (const double*)dt1,
               A.Q * A.ext, dt2, (const int*)nullptr);
      launch_k(load_contract_kernel, blocks(A.S), dim3(256), 0, s, A, (const double*)dT, (const double*)dt2,
               (long long)A.ext * A.ext, ok, lk);
    } else {
      launch_k(load_contract_kernel, blocks(n1), dim3(256), 0, s, A, (const double*)dT, (const double*)dcoef, A.Q,
               dt1, (const int*)nullptr);
      launch_k(load_contract_kernel, blocks(A.S), dim3(256), 0, s, A, (const double*)dT, (const double*)dt1,
               (long long)A.ext, ok, lk);
    }
    ckA(cudaGetLastError(), "load vector launch");
    ckA(cudaStreamSynchronize(s), "load vector");
  }
  int herr = 0;
  ckA(cudaMemcpy(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost), "load vector flag");
  if (herr) throw AssemblyError("assembly: degenerate or folded geometry map");
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace pmgcu
