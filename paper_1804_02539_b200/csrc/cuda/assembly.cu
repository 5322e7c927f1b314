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

}  // namespace pmgcu
