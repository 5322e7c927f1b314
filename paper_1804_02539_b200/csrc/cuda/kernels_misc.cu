// Vector algebra, deterministic reductions, interface sums, interface-piece
// solves, intergrid transfers and the coarse solve.
//
// All of these are HBM- or latency-bound.  Reductions use a fixed grid and a
// fixed-order final sum, so every result is bitwise reproducible run to run
// (the property the reference gets from ascending-rank sums, parallel.hpp:26-30).
#include <cstdlib>

#include "transfer_ops.cuh"
#include "internal.cuh"
#include "pieces.cuh"

namespace pmgcu {

namespace {

inline int grid_for(long long n, int per_thread = 1) {
  long long g = (n + (long long)kThreads * per_thread - 1) / ((long long)kThreads * per_thread);
  return int(g < 1 ? 1 : g);
}

__global__ void fill_kernel(double* x, long long n, double v) {
  PMG_PDL_ENTRY();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = v;
}

__global__ void copy_kernel(const double* __restrict__ x, double* __restrict__ y, long long n) {
  PMG_PDL_ENTRY();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = x[i];
}

// y += a x  (axpy_acc / axpy_dist, multigrid.hpp:108-109); a from device when given
__global__ void axpy_kernel(double a, const double* a_dev, double sign, const double* __restrict__ x,
                            double* __restrict__ y, long long n) {
  PMG_PDL_ENTRY();
  const double s = a_dev ? sign * a_dev[0] : a;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] += s * x[i];
}

// p = z + beta p  (xpay_acc, multigrid.hpp:110)
__global__ void xpay_kernel(const double* __restrict__ z, double beta, const double* beta_dev, double* __restrict__ p,
                            long long n) {
  PMG_PDL_ENTRY();
  const double b = beta_dev ? beta_dev[0] : beta;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + b * p[i];
}

__global__ void scale_set_kernel(double a, const double* __restrict__ x, double* __restrict__ y, long long n) {
  PMG_PDL_ENTRY();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x[i];
}

__device__ inline double block_sum(double v) {
  __shared__ double red[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  return s;
}

__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
                                   double* __restrict__ partial) {
  PMG_PDL_ENTRY();
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads)
    s += a[i] * b[i];
  s = block_sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int n, double* out) {
  PMG_PDL_ENTRY();
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads) s += partial[i];
  s = block_sum(s);
  if (threadIdx.x == 0) out[0] = s;
}

// Sigma over multi-replica dofs: ordered sum written to every replica
// (ParallelBackend::accumulate, parallel.cpp:306-337; serially the scatter-add
// of MultiPatchOperator::apply, assembly.cpp:276-277)
__global__ void group_sum_kernel(const int* __restrict__ goff, const int* __restrict__ gslot, int ngroups,
                                 const double* __restrict__ r, double* __restrict__ out) {
  PMG_PDL_ENTRY();
  const int g = blockIdx.x * kThreads + threadIdx.x;
  if (g >= ngroups) return;
  double s = 0.0;
  for (int q = goff[g]; q < goff[g + 1]; ++q) s += r[gslot[q]];
  for (int q = goff[g]; q < goff[g + 1]; ++q) out[gslot[q]] = s;
}

__global__ void gather_sum_kernel(const int* __restrict__ dof_g, long long ndof, const int* __restrict__ rep_off,
                                  const int* __restrict__ rep_slot, const double* __restrict__ r,
                                  double* __restrict__ buf) {
  PMG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (i >= ndof) return;
  const int g = dof_g[i];
  double s = 0.0;
  for (int q = rep_off[g]; q < rep_off[g + 1]; ++q) s += r[rep_slot[q]];
  buf[i] = s;
}

__global__ void scatter_kernel(const int* __restrict__ dof_g, long long ndof, const int* __restrict__ rep_off,
                               const int* __restrict__ rep_slot, const double* __restrict__ buf,
                               double* __restrict__ out, int add, double alpha) {
  PMG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (i >= ndof) return;
  const int g = dof_g[i];
  const double v = buf[i];
  for (int q = rep_off[g]; q < rep_off[g + 1]; ++q) {
    if (add)
      out[rep_slot[q]] += alpha * v;
    else
      out[rep_slot[q]] = alpha * v;
  }
}

// Edge and vertex pieces (bodies in pieces.cuh) on the interface totals t.
__global__ void __launch_bounds__(kThreads) edges_vertices_kernel(
    const EdgePiece* __restrict__ edges, const int2* __restrict__ items, int nitems,
    const int* __restrict__ edge_iface, const int* __restrict__ vert_iface, const double* __restrict__ vert_scalar,
    int nverts, const int* __restrict__ rep_off, const int* __restrict__ rep_slot, const double* __restrict__ t,
    double* __restrict__ out, int add, double alpha) {
  PMG_PDL_ENTRY();
  // t: interface totals (sum over every replica, all ranks); rep_off/rep_slot:
  // this rank's replicas of each interface dof
  if (blockIdx.x < nitems) {
    const int2 it = items[blockIdx.x];
    edge_item(edges[it.x], it.y, edge_iface, TotalsArray{t}, rep_off, rep_slot, out, add, alpha);
    return;
  }
  vertex_block(vert_iface, vert_scalar, nverts, TotalsArray{t}, rep_off, rep_slot, out, add, alpha);
}

__global__ void lattice_from_global_kernel(const int* __restrict__ l2g, const unsigned char* __restrict__ owner,
                                           long long n, int form, const double* __restrict__ g,
                                           double* __restrict__ lat) {
  PMG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (i >= n) return;
  const int d = l2g[i];
  double v = 0.0;
  if (d >= 0 && (form == 0 || owner[i])) v = g[d];
  lat[i] = v;
}

__global__ void global_from_lattice_kernel(const int* __restrict__ rep_off, const int* __restrict__ rep_slot,
                                           long long ndofs, int form, const double* __restrict__ lat,
                                           double* __restrict__ g) {
  PMG_PDL_ENTRY();
  const long long d = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (d >= ndofs) return;
  if (form == 0) {  // dofs without a replica on this rank read as 0
    g[d] = rep_off[d] < rep_off[d + 1] ? lat[rep_slot[rep_off[d]]] : 0.0;
  } else {
    double s = 0.0;
    for (int q = rep_off[d]; q < rep_off[d + 1]; ++q) s += lat[rep_slot[q]];
    g[d] = s;
  }
}

__global__ void coarse_gather_kernel(const int* __restrict__ rep_off, const int* __restrict__ rep_slot, int n0,
                                     const double* __restrict__ r, double* __restrict__ rhs) {
  PMG_PDL_ENTRY();
  const int d = blockIdx.x * kThreads + threadIdx.x;
  if (d >= n0) return;
  double s = 0.0;
  for (int q = rep_off[d]; q < rep_off[d + 1]; ++q) s += r[rep_slot[q]];
  rhs[d] = s;
}

// x = Ainv rhs, one warp per row, fixed lane-strided order + shuffle tree
__global__ void coarse_gemv_kernel(const double* __restrict__ Ainv, int n0, const double* __restrict__ rhs,
                                   double* __restrict__ x) {
  PMG_PDL_ENTRY();
  const int warp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n0) return;
  const double* row = Ainv + (long long)warp * n0;
  double s = 0.0;
  for (int j = lane; j < n0; j += 32) s = fma(row[j], rhs[j], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) x[warp] = s;
}

__global__ void coarse_scatter_kernel(const int* __restrict__ l2g, long long n, const double* __restrict__ x,
                                      double* __restrict__ out) {
  PMG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (i >= n) return;
  const int d = l2g[i];
  out[i] = d >= 0 ? x[d] : 0.0;
}

// One tensor axis of the two-scale kronecker product over K patches
// (apply_along_axis(TwoScale), tensor.cpp:52-102); each thread one output.
// mode 0: out = s; 1: out = s on non-Dirichlet slots, 0 elsewhere (last
// restriction pass); 2: out += coef s on non-Dirichlet slots (last
// prolongation pass, u += c P coarse).
// IDX = the index type of the element arithmetic: 32-bit whenever the
// vectors have < 2^31 entries (three 64-bit divisions per output made the
// pass instruction-bound: c5's finest transfers ran at 0.2 of their bytes).
template <typename IDX>
__global__ void ts_axis_kernel(TsDev ts, int transpose, int K, int d, int in0, int in1, int in2, int axis,
                               const double* __restrict__ in, double* __restrict__ out, int mode,
                               const int* __restrict__ l2g, double coef) {
  PMG_PDL_ENTRY();
  int dims_in[3] = {in0, in1, in2};
  int dims_out[3] = {in0, in1, in2};
  dims_out[axis] = transpose ? ts.coarse_dim : ts.fine_dim;
  IDX inner = 1, outer = 1;
  for (int a = 0; a < axis; ++a) inner *= dims_in[a];
  for (int a = axis + 1; a < d; ++a) outer *= dims_in[a];
  const int m_in = dims_in[axis], m_out = dims_out[axis];
  const IDX per_in = inner * m_in * outer, per_out = inner * m_out * outer;
  const IDX total = per_out * K;
  const IDX slab = inner * m_out;
  for (IDX idx = blockIdx.x * IDX(kThreads) + threadIdx.x; idx < total; idx += IDX(gridDim.x) * kThreads) {
    const IDX k = idx / per_out;
    const IDX rem = idx - k * per_out;
    const IDX o = rem / slab;
    const IDX rs = rem - o * slab;
    const int j = int(rs / inner);
    const IDX t = rs - IDX(j) * inner;
    const double* src = in + k * per_in + o * inner * m_in + t;
    double s = 0.0;
    if (!transpose) {
      const double* v = ts.vals + ts.row_off[j];
      const int st = ts.row_start[j];
      const int len = ts.row_len[j];
      for (int q = 0; q < len; ++q) s = fma(v[q], src[IDX(st + q) * inner], s);
    } else {
      const int q1 = ts.col_off[j + 1];
      for (int q = ts.col_off[j]; q < q1; ++q) s = fma(ts.col_val[q], src[IDX(ts.col_row[q]) * inner], s);
    }
    if (mode == 0)
      out[idx] = s;
    else if (mode == 1)
      out[idx] = l2g[idx] >= 0 ? s : 0.0;
    else if (l2g[idx] >= 0)
      out[idx] += coef * s;
  }
}

// ---------------------------------------------------------------- interface sums
// T_loc[i] = sum of this rank's replicas of interface dof i (ascending slot)
__global__ void iface_partial_kernel(int n, const int* __restrict__ rep_off, const int* __restrict__ rep_slot,
                                     const double* __restrict__ r, double* __restrict__ tloc) {
  PMG_PDL_ENTRY();
  const int i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int q = rep_off[i]; q < rep_off[i + 1]; ++q) s += r[rep_slot[q]];
  tloc[i] = s;
}

__global__ void iface_pack_kernel(int n, const int* __restrict__ idx, const double* __restrict__ tloc,
                                  double* __restrict__ send) {
  PMG_PDL_ENTRY();
  const int q = blockIdx.x * kThreads + threadIdx.x;
  if (q < n) send[q] = tloc[idx[q]];
}

// ascending-rank fold of the partials (ParallelBackend::accumulate order)
__global__ void iface_combine_kernel(int n, const int* __restrict__ comb_off, const int* __restrict__ comb_src,
                                     const double* __restrict__ tloc, const double* __restrict__ recv,
                                     double* __restrict__ t) {
  PMG_PDL_ENTRY();
  const int i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int q = comb_off[i]; q < comb_off[i + 1]; ++q) {
    const int src = comb_src[q];
    s += src < 0 ? tloc[i] : recv[src];
  }
  t[i] = s;
}

__global__ void iface_scatter_kernel(int n, const int* __restrict__ rep_off, const int* __restrict__ rep_slot,
                                     const double* __restrict__ t, double* __restrict__ out) {
  PMG_PDL_ENTRY();
  const int i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  const double v = t[i];
  for (int q = rep_off[i]; q < rep_off[i + 1]; ++q) out[rep_slot[q]] = v;
}

__global__ void gather_t_kernel(long long n, const int* __restrict__ map, const double* __restrict__ t,
                                double* __restrict__ buf) {
  PMG_PDL_ENTRY();
  const long long j = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (j < n) buf[j] = t[map[j]];
}

__global__ void scatter_iface_kernel(long long n, const int* __restrict__ map, const int* __restrict__ rep_off,
                                     const int* __restrict__ rep_slot, const double* __restrict__ buf,
                                     double* __restrict__ out, int add, double alpha) {
  PMG_PDL_ENTRY();
  const long long j = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (j >= n) return;
  const int i = map[j];
  const double v = buf[j];
  for (int q = rep_off[i]; q < rep_off[i + 1]; ++q) {
    if (add)
      out[rep_slot[q]] += alpha * v;
    else
      out[rep_slot[q]] = alpha * v;
  }
}

// ascending-rank sums: out[d] = sum_r parts[r * n + d]
__global__ void sum_ranks_kernel(const double* __restrict__ parts, int ranks, int n, double* __restrict__ out) {
  PMG_PDL_ENTRY();
  const int d = blockIdx.x * kThreads + threadIdx.x;
  if (d >= n) return;
  double s = 0.0;
  for (int r = 0; r < ranks; ++r) s += parts[(long long)r * n + d];
  out[d] = s;
}

// Whole tensor transfer in one pass, one output per thread; the nested sums run
// axis 0 innermost, i.e. in the order of the reference's successive
// apply_along_axis calls (restrict_patch / prolong_patch, transfer.cpp:21-66).
// Restriction (transpose): coarse(j) = sum_i2 P(i2,j2) sum_i1 P(i1,j1) sum_i0 P(i0,j0) r(i)
// with Dirichlet coarse slots zeroed; prolongation: u(i) += coef * sum over
// the <= p+1 parents per axis, on non-Dirichlet fine slots.
__global__ void restrict_fused_kernel(TsDev ts, int K, int d, int ext_f, int ext_c, const double* __restrict__ r,
                                      double* __restrict__ out, const int* __restrict__ l2g_c) {
  PMG_PDL_ENTRY();
  long long Sc = 1, Sf = 1;
  for (int a = 0; a < d; ++a) {
    Sc *= ext_c;
    Sf *= ext_f;
  }
  const long long total = Sc * K;
  for (long long idx = blockIdx.x * (long long)kThreads + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * kThreads)
    out[idx] = l2g_c[idx] < 0 ? 0.0 : restrict_out(ts, d, ext_f, ext_c, Sc, Sf, r, idx);
}

__global__ void prolong_fused_kernel(TsDev ts, int K, int d, int ext_f, int ext_c, const double* __restrict__ c,
                                     double coef, double* __restrict__ u, const int* __restrict__ l2g_f) {
  PMG_PDL_ENTRY();
  long long Sc = 1, Sf = 1;
  for (int a = 0; a < d; ++a) {
    Sc *= ext_c;
    Sf *= ext_f;
  }
  const long long total = Sf * K;
  for (long long idx = blockIdx.x * (long long)kThreads + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * kThreads)
    if (l2g_f[idx] >= 0) u[idx] += coef * prolong_out(ts, d, ext_f, ext_c, Sc, Sf, c, idx);
}

// 2D restriction of one coarse tile (kTileC x kTileC) per CTA: the fine
// window it reads is staged in shared memory, axis 0 is contracted into a
// second tile, then axis 1 -- per output the same sums in the same order as
// restrict_fused_kernel (s0 over q0 inner, s1 over q1).
__global__ void __launch_bounds__(kThreads) restrict_tile2d_kernel(TsDev ts, int K, int ext_f, int ext_c,
                                                                   const double* __restrict__ r,
                                                                   double* __restrict__ out,
                                                                   const int* __restrict__ l2g_c) {
  PMG_PDL_ENTRY();
  extern __shared__ __align__(16) double tsm[];
  const int tiles = (ext_c + kTileC - 1) / kTileC;
  const int k = blockIdx.x / (tiles * tiles);
  const int t = blockIdx.x % (tiles * tiles);
  const int a0 = (t % tiles) * kTileC, a1 = (t / tiles) * kTileC;
  const int b0 = min(ext_c, a0 + kTileC), b1 = min(ext_c, a1 + kTileC);
  const int span = ts.rspan;
  // fine windows of the tile's columns (monotone): first row of a, last of b-1
  const int f0 = ts.col_row[ts.col_off[a0]], f1 = ts.col_row[ts.col_off[a1]];
  const int n0 = ts.col_row[ts.col_off[b0] - 1] + 1 - f0, n1 = ts.col_row[ts.col_off[b1] - 1] + 1 - f1;
  double* R = tsm;                   // [n1][span]
  double* T = tsm + span * span;     // [n1][kTileC]
  const double* __restrict__ src = r + (long long)k * ext_f * ext_f;
  for (int idx = threadIdx.x; idx < n1 * n0; idx += blockDim.x) {
    const int y = idx / n0, x = idx % n0;
    R[y * span + x] = src[(long long)(f1 + y) * ext_f + f0 + x];
  }
  __syncthreads();
  const int w0 = b0 - a0;
  for (int idx = threadIdx.x; idx < n1 * w0; idx += blockDim.x) {
    const int y = idx / w0, j0 = a0 + idx % w0;
    double s0 = 0.0;
    for (int q0 = ts.col_off[j0]; q0 < ts.col_off[j0 + 1]; ++q0)
      s0 = fma(ts.col_val[q0], R[y * span + ts.col_row[q0] - f0], s0);
    T[y * kTileC + (j0 - a0)] = s0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < (b1 - a1) * w0; idx += blockDim.x) {
    const int j1 = a1 + idx / w0, j0 = a0 + idx % w0;
    const long long o = (long long)k * ext_c * ext_c + (long long)j1 * ext_c + j0;
    if (l2g_c[o] < 0) {
      out[o] = 0.0;
      continue;
    }
    double s1 = 0.0;
    for (int q1 = ts.col_off[j1]; q1 < ts.col_off[j1 + 1]; ++q1)
      s1 = fma(ts.col_val[q1], T[(ts.col_row[q1] - f1) * kTileC + (j0 - a0)], s1);
    out[o] = s1;
  }
}

// 2D prolongation u += coef P c of one fine tile (kTileF x kTileF) per CTA:
// the coarse window is staged in shared memory, axis 0 then axis 1, as
// prolong_fused_kernel per output.
__global__ void __launch_bounds__(kThreads) prolong_tile2d_kernel(TsDev ts, int K, int ext_f, int ext_c,
                                                                  const double* __restrict__ c, double coef,
                                                                  double* __restrict__ u,
                                                                  const int* __restrict__ l2g_f) {
  PMG_PDL_ENTRY();
  extern __shared__ __align__(16) double tsm[];
  const int tiles = (ext_f + kTileF - 1) / kTileF;
  const int k = blockIdx.x / (tiles * tiles);
  const int t = blockIdx.x % (tiles * tiles);
  const int a0 = (t % tiles) * kTileF, a1 = (t / tiles) * kTileF;
  const int b0 = min(ext_f, a0 + kTileF), b1 = min(ext_f, a1 + kTileF);
  const int span = ts.pspan;
  const int c0 = ts.row_start[a0], c1 = ts.row_start[a1];
  const int n0 = min(span, ext_c - c0), n1 = min(span, ext_c - c1);
  double* Cs = tsm;                // [n1][span]
  double* T = tsm + span * span;   // [n1][kTileF]
  const double* __restrict__ src = c + (long long)k * ext_c * ext_c;
  for (int idx = threadIdx.x; idx < n1 * n0; idx += blockDim.x) {
    const int y = idx / n0, x = idx % n0;
    Cs[y * span + x] = src[(long long)(c1 + y) * ext_c + c0 + x];
  }
  __syncthreads();
  const int w0 = b0 - a0;
  for (int idx = threadIdx.x; idx < n1 * w0; idx += blockDim.x) {
    const int y = idx / w0, i0 = a0 + idx % w0;
    const double* v0 = ts.vals + ts.row_off[i0];
    const int st = ts.row_start[i0] - c0;
    double s0 = 0.0;
    for (int q0 = 0; q0 < ts.row_len[i0]; ++q0) s0 = fma(v0[q0], Cs[y * span + st + q0], s0);
    T[y * kTileF + (i0 - a0)] = s0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < (b1 - a1) * w0; idx += blockDim.x) {
    const int i1 = a1 + idx / w0, i0 = a0 + idx % w0;
    const long long o = (long long)k * ext_f * ext_f + (long long)i1 * ext_f + i0;
    if (l2g_f[o] < 0) continue;
    const double* v1 = ts.vals + ts.row_off[i1];
    const int st = ts.row_start[i1] - c1;
    double s1 = 0.0;
    for (int q1 = 0; q1 < ts.row_len[i1]; ++q1) s1 = fma(v1[q1], T[(st + q1) * kTileF + (i0 - a0)], s1);
    u[o] += coef * s1;
  }
}

__global__ void masked_axpy_kernel(const int* __restrict__ l2g, long long n, double c, const double* __restrict__ val,
                                   double* __restrict__ u) {
  PMG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (i >= n) return;
  if (l2g[i] >= 0) u[i] += c * val[i];
}

__global__ void mask_dirichlet_kernel(const int* __restrict__ l2g, long long n, double* __restrict__ v) {
  PMG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
  if (i >= n) return;
  if (l2g[i] < 0) v[i] = 0.0;
}

// zero Dirichlet rows/columns and the columns leaving the lattice; padding
// rows r in [S, Sp) are zeroed too
__global__ void zero_dirichlet_band_kernel(int dim, int degree, int ext, long long S, long long Sp, int K, int O,
                                           const int* __restrict__ l2g, double* __restrict__ band) {
  PMG_PDL_ENTRY();
  const int W = 2 * degree + 1;
  const long long total = (long long)K * O * Sp;
  for (long long idx = blockIdx.x * (long long)kThreads + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * kThreads) {
    const long long k = idx / (O * Sp);
    const long long rem = idx - k * O * Sp;
    const int o = int(rem / Sp);
    const long long r = rem - (long long)o * Sp;
    if (r >= S) {
      band[idx] = 0.0;
      continue;
    }
    const int i0 = int(r % ext), i1 = int((r / ext) % ext), i2 = dim == 3 ? int(r / ((long long)ext * ext)) : 0;
    const int d0 = o % W - degree, d1 = (o / W) % W - degree, d2 = dim == 3 ? o / (W * W) - degree : 0;
    const int j0 = i0 + d0, j1 = i1 + d1, j2 = i2 + d2;
    bool live = j0 >= 0 && j0 < ext && j1 >= 0 && j1 < ext && (dim == 2 || (j2 >= 0 && j2 < ext));
    if (live) {
      const long long c = j0 + (long long)ext * j1 + (long long)ext * ext * j2;
      live = l2g[k * S + r] >= 0 && l2g[k * S + c] >= 0;
    }
    if (!live) band[idx] = 0.0;
  }
}

// PCG scalars kept on device: [0] rz [1] pAp [2] alpha [3] rz_next [4] beta [5] |r|^2 [6] |r| [7] flag
__global__ void pcg_scalars_kernel(int op, double* s) {
  PMG_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  switch (op) {
    case 0:  // alpha = rz / pAp; flag non-positive energy
      if (!(s[1] > 0.0)) s[7] = 1.0;
      s[2] = s[0] / s[1];
      break;
    case 1:  // beta = rz_next / rz; rz = rz_next
      s[4] = s[3] / s[0];
      s[0] = s[3];
      break;
    case 2:  // |r| = sqrt(|r|^2)
      s[6] = sqrt(s[5]);
      break;
  }
}

__global__ void pcg_check_kernel(int first, PcgLoopState* st, double* s, double* hist,
                                 cudaGraphConditionalHandle handle) {
  PMG_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  unsigned go = 0;
  if (first) {
    const double r0 = s[6];
    st->r0 = r0;
    st->k = 0;
    hist[0] = r0;
    st->status = r0 == 0.0 ? 1 : 0;  // pcg_generic returns at once on a zero residual
    s[0] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    go = r0 != 0.0;
  } else {
    const int k = ++st->k;
    const double rn = s[6];
    hist[k] = rn;
    if (s[7] != 0.0) {  // pAp <= 0 (DefinitenessError, multigrid.hpp:176)
      s[7] = 0.0;
      st->status = 2;
    } else if (rn <= st->tol * st->r0) {  // multigrid.hpp:182
      st->status = 1;
    } else if (k >= st->max_iter) {  // DivergenceError, multigrid.hpp:188
      st->status = 3;
    } else {
      go = 1;
    }
  }
  cudaGraphSetConditional(handle, go);
}

}  // namespace

void launch_pcg_check(cudaStream_t s, int first, PcgLoopState* st, double* scal, double* history,
                      cudaGraphConditionalHandle handle) {
  launch_k(pcg_check_kernel, dim3(1), dim3(32), 0, s, first, st, scal, history, handle);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PMG_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

void launch_fill(cudaStream_t s, double* x, long long n, double v) {
  if (n > 0) launch_k(fill_kernel, dim3(grid_for(n, 4)), dim3(kThreads), 0, s, x, n, v);
}
void launch_copy(cudaStream_t s, const double* x, double* y, long long n) {
  if (n > 0) launch_k(copy_kernel, dim3(grid_for(n, 4)), dim3(kThreads), 0, s, x, y, n);
}
void launch_axpy(cudaStream_t s, double a, const double* a_dev, double sign, const double* x, double* y, long long n) {
  if (n > 0) launch_k(axpy_kernel, dim3(grid_for(n, 4)), dim3(kThreads), 0, s, a, a_dev, sign, x, y, n);
}
void launch_xpay(cudaStream_t s, const double* z, double beta, const double* beta_dev, double* p, long long n) {
  if (n > 0) launch_k(xpay_kernel, dim3(grid_for(n, 4)), dim3(kThreads), 0, s, z, beta, beta_dev, p, n);
}
void launch_scale_set(cudaStream_t s, double a, const double* x, double* y, long long n) {
  if (n > 0) launch_k(scale_set_kernel, dim3(grid_for(n, 4)), dim3(kThreads), 0, s, a, x, y, n);
}
int dot_blocks(long long n) {
  long long g = (n + kThreads * 8 - 1) / (kThreads * 8);
  if (g > 1184) g = 1184;
  return int(g < 1 ? 1 : g);
}
void launch_dot_partial(cudaStream_t s, const double* a, const double* b, long long n, double* partial) {
  launch_k(dot_partial_kernel, dim3(dot_blocks(n)), dim3(kThreads), 0, s, a, b, n, partial);
}
void launch_sum_partials(cudaStream_t s, const double* partial, int nparts, double* out) {
  launch_k(sum_partials_kernel, dim3(1), dim3(kThreads), 0, s, partial, nparts, out);
}
void launch_group_sum(cudaStream_t s, const int* goff, const int* gslot, int ngroups, const double* r, double* out) {
  if (ngroups > 0) launch_k(group_sum_kernel, dim3(grid_for(ngroups)), dim3(kThreads), 0, s, goff, gslot, ngroups, r, out);
}
void launch_gather_sum(cudaStream_t s, const int* dof_g, long long ndof, const int* rep_off, const int* rep_slot,
                       const double* r, double* buf) {
  if (ndof > 0) launch_k(gather_sum_kernel, dim3(grid_for(ndof)), dim3(kThreads), 0, s, dof_g, ndof, rep_off, rep_slot, r, buf);
}
void launch_scatter(cudaStream_t s, const int* dof_g, long long ndof, const int* rep_off, const int* rep_slot,
                    const double* buf, double* out, int add, double alpha) {
  if (ndof > 0)
    launch_k(scatter_kernel, dim3(grid_for(ndof)), dim3(kThreads), 0, s, dof_g, ndof, rep_off, rep_slot, buf, out, add, alpha);
}
void launch_edges_vertices(cudaStream_t s, const EdgePiece* edges, const int2* items, int nitems,
                           const int* edge_dof_g, const int* vert_g, const double* vert_scalar, int nverts,
                           const int* rep_off, const int* rep_slot, const double* r, double* out, int add,
                           double alpha) {
  const int grid = nitems + (nverts > 0 ? 1 : 0);
  if (grid > 0)
    launch_k(edges_vertices_kernel, dim3(grid), dim3(kThreads), 0, s, edges, items, nitems, edge_dof_g, vert_g, vert_scalar, nverts,
                                                    rep_off, rep_slot, r, out, add, alpha);
}
void launch_lattice_from_global(cudaStream_t s, const int* l2g, const unsigned char* owner, long long n, int form,
                                const double* g, double* lat) {
  if (n > 0) launch_k(lattice_from_global_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, l2g, owner, n, form, g, lat);
}
void launch_global_from_lattice(cudaStream_t s, const int* rep_off, const int* rep_slot, long long ndofs, int form,
                                const double* lat, double* g) {
  if (ndofs > 0) launch_k(global_from_lattice_kernel, dim3(grid_for(ndofs)), dim3(kThreads), 0, s, rep_off, rep_slot, ndofs, form, lat, g);
}
void launch_coarse(cudaStream_t s, const int* rep_off, const int* rep_slot, const int* l2g, int n0, long long lat_n,
                   const double* Ainv, const double* r, double* rhs, double* x, double* out) {
  if (n0 > 0) {
    launch_k(coarse_gather_kernel, dim3(grid_for(n0)), dim3(kThreads), 0, s, rep_off, rep_slot, n0, r, rhs);
    launch_k(coarse_gemv_kernel, dim3(grid_for((long long)n0 * 32)), dim3(kThreads), 0, s, Ainv, n0, rhs, x);
  }
  launch_k(coarse_scatter_kernel, dim3(grid_for(lat_n)), dim3(kThreads), 0, s, l2g, lat_n, x, out);
}
void launch_coarse_gather(cudaStream_t s, const int* rep_off, const int* rep_slot, int n0, const double* r,
                          double* rhs) {
  if (n0 > 0) launch_k(coarse_gather_kernel, dim3(grid_for(n0)), dim3(kThreads), 0, s, rep_off, rep_slot, n0, r, rhs);
}
void launch_coarse_gemv(cudaStream_t s, const double* Ainv, int n0, const double* rhs, double* x) {
  if (n0 > 0) launch_k(coarse_gemv_kernel, dim3(grid_for((long long)n0 * 32)), dim3(kThreads), 0, s, Ainv, n0, rhs, x);
}
void launch_coarse_scatter(cudaStream_t s, const int* l2g, long long lat_n, const double* x, double* out) {
  launch_k(coarse_scatter_kernel, dim3(grid_for(lat_n)), dim3(kThreads), 0, s, l2g, lat_n, x, out);
}
void launch_ts_axis(cudaStream_t s, const TsDev& ts, bool transpose, int K, int d, const int* in_dims, int axis,
                    const double* in, double* out, int mode, const int* l2g, double coef) {
  long long per_out = 1;
  for (int a = 0; a < d; ++a) per_out *= (a == axis ? (transpose ? ts.coarse_dim : ts.fine_dim) : in_dims[a]);
  const long long total = per_out * K;
  long long g = (total + kThreads - 1) / kThreads;
  if (g > 148LL * 32) g = 148LL * 32;
  long long per_in = 1;
  for (int a = 0; a < d; ++a) per_in *= in_dims[a];
  const bool small = total < (1LL << 30) && per_in * K < (1LL << 30);
  if (small)
    launch_k(ts_axis_kernel<unsigned>, dim3(int(g < 1 ? 1 : g)), dim3(kThreads), 0, s, ts, transpose ? 1 : 0, K, d,
             in_dims[0], in_dims[1], d == 3 ? in_dims[2] : 1, axis, in, out, mode, l2g, coef);
  else
    launch_k(ts_axis_kernel<long long>, dim3(int(g < 1 ? 1 : g)), dim3(kThreads), 0, s, ts, transpose ? 1 : 0, K, d,
             in_dims[0], in_dims[1], d == 3 ? in_dims[2] : 1, axis, in, out, mode, l2g, coef);
}
void launch_iface_partial(cudaStream_t s, int n, const int* rep_off, const int* rep_slot, const double* r,
                          double* tloc) {
  if (n > 0) launch_k(iface_partial_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, n, rep_off, rep_slot, r, tloc);
}
void launch_iface_pack(cudaStream_t s, int n, const int* idx, const double* tloc, double* send) {
  if (n > 0) launch_k(iface_pack_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, n, idx, tloc, send);
}
void launch_iface_combine(cudaStream_t s, int n, const int* comb_off, const int* comb_src, const double* tloc,
                          const double* recv, double* t) {
  if (n > 0) launch_k(iface_combine_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, n, comb_off, comb_src, tloc, recv, t);
}
void launch_iface_scatter(cudaStream_t s, int n, const int* rep_off, const int* rep_slot, const double* t,
                          double* out) {
  if (n > 0) launch_k(iface_scatter_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, n, rep_off, rep_slot, t, out);
}
void launch_gather_t(cudaStream_t s, long long n, const int* map, const double* t, double* buf) {
  if (n > 0) launch_k(gather_t_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, n, map, t, buf);
}
void launch_scatter_iface(cudaStream_t s, long long n, const int* map, const int* rep_off, const int* rep_slot,
                          const double* buf, double* out, int add, double alpha) {
  if (n > 0)
    launch_k(scatter_iface_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, n, map, rep_off, rep_slot, buf, out, add, alpha);
}
void launch_sum_ranks(cudaStream_t s, const double* parts, int ranks, int n, double* out) {
  if (n > 0) launch_k(sum_ranks_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, parts, ranks, n, out);
}
void launch_restrict_fused(cudaStream_t s, const TsDev& ts, int K, int d, int ext_f, int ext_c, const double* r,
                           double* out, const int* l2g_c) {
  long long n = K;
  for (int a = 0; a < d; ++a) n *= ext_c;
  launch_k(restrict_fused_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, ts, K, d, ext_f, ext_c, r, out, l2g_c);
}
void launch_prolong_fused(cudaStream_t s, const TsDev& ts, int K, int d, int ext_f, int ext_c, const double* c,
                          double coef, double* u, const int* l2g_f) {
  long long n = K;
  for (int a = 0; a < d; ++a) n *= ext_f;
  launch_k(prolong_fused_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, ts, K, d, ext_f, ext_c, c, coef, u, l2g_f);
}
void launch_restrict_tile2d(cudaStream_t s, const TsDev& ts, int K, int ext_f, int ext_c, const double* r,
                            double* out, const int* l2g_c) {
  const int tiles = (ext_c + kTileC - 1) / kTileC;
  const size_t smem = sizeof(double) * (size_t(ts.rspan) * ts.rspan + size_t(ts.rspan) * kTileC);
  launch_k(restrict_tile2d_kernel, dim3(unsigned(K * tiles * tiles)), dim3(kThreads), smem, s, ts, K, ext_f, ext_c, r,
           out, l2g_c);
}
void launch_prolong_tile2d(cudaStream_t s, const TsDev& ts, int K, int ext_f, int ext_c, const double* c, double coef,
                           double* u, const int* l2g_f) {
  const int tiles = (ext_f + kTileF - 1) / kTileF;
  const size_t smem = sizeof(double) * (size_t(ts.pspan) * ts.pspan + size_t(ts.pspan) * kTileF);
  launch_k(prolong_tile2d_kernel, dim3(unsigned(K * tiles * tiles)), dim3(kThreads), smem, s, ts, K, ext_f, ext_c, c,
           coef, u, l2g_f);
}
void launch_masked_axpy(cudaStream_t s, const int* l2g, long long n, double c, const double* val, double* u) {
  if (n > 0) launch_k(masked_axpy_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, l2g, n, c, val, u);
}
void launch_mask_dirichlet(cudaStream_t s, const int* l2g, long long n, double* v) {
  if (n > 0) launch_k(mask_dirichlet_kernel, dim3(grid_for(n)), dim3(kThreads), 0, s, l2g, n, v);
}
void launch_zero_dirichlet_band(cudaStream_t s, int dim, int degree, int ext, long long S, long long Sp, int K,
                                int stored_offsets, const int* l2g, double* band) {
  launch_k(zero_dirichlet_band_kernel, dim3(148 * 32), dim3(kThreads), 0, s, dim, degree, ext, S, Sp, K, stored_offsets, l2g, band);
}
void launch_pcg_scalars(cudaStream_t s, int op, double* scal) { launch_k(pcg_scalars_kernel, dim3(1), dim3(32), 0, s, op, scal); }

}  // namespace pmgcu
