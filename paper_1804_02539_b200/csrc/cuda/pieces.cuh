// Device bodies of the interface piece solves, shared by the stand-alone
// edges/vertices kernel (interface totals read from t) and the fused
// small-level smoother (totals summed from the replicas on the fly).
//
// Edge pieces: z = L_T^-1 (sum of replica shares) with the explicit inverse of
// the banded operator (BandedCholesky::solve, banded.cpp:61-77).  One CTA per
// (edge, 32-row chunk): lane = row, the 8 warps split the columns, partial
// sums meet in shared memory in a fixed order.  Vertex pieces divide by the
// scalar (smoother.cpp:36-38).
#pragma once

#include "internal.cuh"

namespace pmgcu {

// the interface total of iface dof g as the reference's accumulate forms it:
// the replicas in ascending slot order (what iface_partial computes)
struct ReplicaSum {
  const int* __restrict__ rep_off;
  const int* __restrict__ rep_slot;
  const double* __restrict__ r;
  __device__ __forceinline__ double operator()(int g) const {
    double s = 0.0;
    for (int q = rep_off[g]; q < rep_off[g + 1]; ++q) s += r[rep_slot[q]];
    return s;
  }
};
struct TotalsArray {
  const double* __restrict__ t;
  __device__ __forceinline__ double operator()(int g) const { return t[g]; }
};

__device__ __forceinline__ void write_replicas(const int* __restrict__ rep_off, const int* __restrict__ rep_slot,
                                               int g, double v, double* __restrict__ out, int add) {
  for (int q = rep_off[g]; q < rep_off[g + 1]; ++q) {
    if (add)
      out[rep_slot[q]] += v;
    else
      out[rep_slot[q]] = v;
  }
}

// one (edge, 32-row) item; blockDim = kThreads
template <class Total>
__device__ void edge_item(const EdgePiece& e, int row0, const int* __restrict__ edge_iface, Total total,
                          const int* __restrict__ rep_off, const int* __restrict__ rep_slot, double* __restrict__ out,
                          int add, double alpha) {
  __shared__ double buf[512];
  __shared__ double part[kThreads / 32][32];
  const int* dofs = edge_iface + e.dof_off;
  for (int i = threadIdx.x; i < e.m; i += kThreads) buf[i] = total(dofs[i]);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = row0 + lane;
  const int per = (e.m + 7) / 8;
  const int j0 = warp * per, j1 = min(e.m, j0 + per);
  double z0 = 0.0, z1 = 0.0;
  if (i < e.m) {
    int j = j0;
    for (; j + 1 < j1; j += 2) {
      z0 = fma(e.Linv[(long long)j * e.m + i], buf[j], z0);
      z1 = fma(e.Linv[(long long)(j + 1) * e.m + i], buf[j + 1], z1);
    }
    if (j < j1) z0 = fma(e.Linv[(long long)j * e.m + i], buf[j], z0);
  }
  part[warp][lane] = z0 + z1;
  __syncthreads();
  if (warp == 0 && i < e.m) {
    double z = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) z += part[w][lane];
    write_replicas(rep_off, rep_slot, dofs[i], alpha * z, out, add);
  }
}

template <class Total>
__device__ void vertex_block(const int* __restrict__ vert_iface, const double* __restrict__ vert_scalar, int nverts,
                             Total total, const int* __restrict__ rep_off, const int* __restrict__ rep_slot,
                             double* __restrict__ out, int add, double alpha) {
  for (int v = threadIdx.x; v < nverts; v += blockDim.x) {
    const int g = vert_iface[v];
    const double z = total(g) / vert_scalar[v];
    write_replicas(rep_off, rep_slot, g, alpha * z, out, add);
  }
}

}  // namespace pmgcu
