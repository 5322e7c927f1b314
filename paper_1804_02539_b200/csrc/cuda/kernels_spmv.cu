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
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "internal.cuh"

namespace pmgcu {

namespace {

template <int D, int P>
__global__ void __launch_bounds__(kThreads) spmv_kernel(SpmvArgs a) {
  PMG_PDL_ENTRY();
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
    // Small levels are latency-bound: each d0-row's 2p+1 band values and x
    // values are loaded unconditionally first (x through a clamped address),
    // so they are all in flight together; the FMAs keep the reference's
    // per-entry predicate and column order.
#pragma unroll
    for (int d2 = (D == 3 ? -P : 0); d2 <= (D == 3 ? P : 0); ++d2) {
      const bool ok2 = D == 2 || (i2 + d2 >= 0 && i2 + d2 < ext);
#pragma unroll
      for (int d1 = -P; d1 <= P; ++d1) {
        const bool ok1 = ok2 && (i1 + d1 >= 0 && i1 + d1 < ext);
        double bv[W], xv[W];
#pragma unroll
        for (int d0 = -P; d0 <= P; ++d0) {
          const int o = (d0 + P) + W * ((d1 + P) + W * (D == 3 ? d2 + P : 0));
          const long long off = d0 + (long long)ext * d1 + ext2 * d2;
          const bool ok = ok1 && i0 + d0 >= 0 && i0 + d0 < ext;
          bv[d0 + P] = __ldg(band + (size_t)o * S);
          xv[d0 + P] = __ldg(ok ? x + off : x);
        }
#pragma unroll
        for (int d0 = -P; d0 <= P; ++d0)
          if (ok1 && i0 + d0 >= 0 && i0 + d0 < ext) acc = fma(bv[d0 + P], xv[d0 + P], acc);
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
  PMG_PDL_ENTRY();
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

// ---------------------------------------------------------------- TMA stream
// Large levels: the band is laid out [K][O][Sp] with the row stride Sp a
// multiple of 256 and >= S + halo (spmv_row_stride), so each (offset, 256-row
// chunk) is one aligned 2 KB segment and every offset row ends in zeros.  A producer
// warp streams the 2p+1 segments of one (d1, d2) offset row per stage with
// cp.async.bulk (TMA) into a kStages-deep shared-memory ring guarded by
// mbarriers; 8 consumer warps (one row per thread) run the FMAs.  The band
// never passes through registers ahead of use, so the loads in flight do not
// depend on register pressure.
constexpr int kStages = 4;
constexpr int kRowsTma = 256;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// "memory" clobbers: the ring's shared-memory reads must stay between the
// wait on full[s] and the arrive on empty[s] (the producer refills the stage
// once every consumer warp has arrived).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int D, int P>
__global__ void __launch_bounds__(kRowsTma + 32) spmv_tma_kernel(SpmvArgs a) {
  PMG_PDL_ENTRY();
  constexpr int W = 2 * P + 1;
  constexpr int O = D == 2 ? W * W : W * W * W;
  constexpr int NCHUNK = O / W;
  constexpr unsigned kStageBytes = W * kRowsTma * sizeof(double);
  extern __shared__ __align__(128) double ring[];  // [kStages][W][kRowsTma]
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ double red[kRowsTma / 32];

  const long long Sp = a.Sp;
  const long long blocks_per_patch = (a.S + kRowsTma - 1) / kRowsTma;
  const long long k = blockIdx.x / blocks_per_patch;
  const long long r0 = (blockIdx.x - k * blocks_per_patch) * kRowsTma;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRowsTma / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= kRowsTma) {  // producer warp
    if (tid == kRowsTma) {
      const double* base = a.band + (size_t)k * O * Sp + r0;
      for (int c = 0; c < NCHUNK; ++c) {
        const int s = c % kStages;
        if (c >= kStages) mbar_wait(&empty[s], ((c / kStages) - 1) & 1);
        mbar_expect_tx(&full[s], kStageBytes);
        double* dst = ring + (size_t)s * W * kRowsTma;
#pragma unroll
        for (int w = 0; w < W; ++w)
          tma_load_1d(dst + w * kRowsTma, base + (size_t)(c * W + w) * Sp, kRowsTma * sizeof(double), &full[s]);
      }
    }
    return;
  }

  const long long r = r0 + tid;
  const bool row_ok = r < a.S;
  const int ext = a.ext;
  const int i0 = int(r % ext);
  const int i1 = int((r / ext) % ext);
  const int i2 = D == 3 ? int(r / ((long long)ext * ext)) : 0;
  const double* __restrict__ x = a.x + k * a.S + r;
  const long long ext2 = (long long)ext * ext;
  double acc = 0.0;
  for (int c = 0; c < NCHUNK; ++c) {
    const int s = c % kStages;
    const int d1 = c % W - P;
    const int d2 = D == 3 ? c / W - P : 0;
    const bool ok1 = row_ok && i1 + d1 >= 0 && i1 + d1 < ext && (D == 2 || (i2 + d2 >= 0 && i2 + d2 < ext));
    mbar_wait(&full[s], (c / kStages) & 1);
    const double* seg = ring + (size_t)s * W * kRowsTma + tid;
    const long long off1 = (long long)ext * d1 + ext2 * d2;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int d0 = w - P;
      if (ok1 && i0 + d0 >= 0 && i0 + d0 < ext) acc = fma(seg[w * kRowsTma], __ldg(x + off1 + d0), acc);
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
  }
  double prod = 0.0;
  if (row_ok) {
    const long long gid = k * a.S + r;
    const double y = a.f ? a.f[gid] - acc : acc;
    a.y[gid] = y;
    if (a.dot_partial) prod = y * x[0];
  }
  if (a.dot_partial) {  // consumers only: named barrier 1
    for (int o = 16; o > 0; o >>= 1) prod += __shfl_down_sync(0xffffffffu, prod, o);
    if ((tid & 31) == 0) red[tid >> 5] = prod;
    asm volatile("bar.sync 1, %0;\n" ::"n"(kRowsTma) : "memory");
    if (tid == 0) {
      double sum = 0.0;
      for (int w = 0; w < kRowsTma / 32; ++w) sum += red[w];
      a.dot_partial[blockIdx.x] = sum;
    }
  }
}

// ---------------------------------------------------------------- half band
// The stiffness is symmetric, so large levels store only the offsets at or
// below the centre, o <= (O-1)/2, i.e. the (d2, d1, d0) <= 0 half in the
// lexicographic order of the CSR columns ([K][OB][Sp], OB = (O+1)/2).  The
// upper entry A(r, r+s) for s > 0 is the stored A(r+s, r) at the mirrored
// offset.  Every stage of the ring holds one d0-row of offsets; the sum still
// runs over o = 0..O-1 in the reference's column order:
//   chunks [0, RL)       d0-rows strictly below the centre (streamed from HBM)
//   chunk  RL            the centre row, d0 = -p..0 (ends with the diagonal)
//   chunk  RL+1          the centre row, d0 = 1..p   (mirrored)
//   chunks [RL+2, R+1)   d0-rows above the centre    (mirrored)
// A mirrored segment is the 256 rows [r0+s, r0+s+256) of the mirror offset: it
// belongs to a CTA a few hundred rows downstream that streams the same bytes
// at about the same time, so it is served by L2 and the HBM bytes per SpMV are
// the half band.  TMA needs 16-byte aligned sources, so a mirrored segment
// starts at the even row below r0+s and carries 258 rows; the consumer adds
// (s & 1).  Upper values are the lower triangle's: A is symmetric up to
// rounding in the reference's assembly (E = G H^T, assembly.cpp:218), and
// this reads each pair once, which is the textbook symmetric operator.
constexpr int kSeg = kRowsTma + 2;

// The x values one stage multiplies, x[g + off1 - p .. g + off1 + 255 + p]
// (g = the block's first lattice row), ride in the same stage as a 16-byte
// aligned window, so consumers read only shared memory.  At the two ends of
// the lattice the window is clamped (lattice vectors carry 64 B of slack, so
// the rounded-up end stays inside the allocation).
template <int P>
struct XWindow {
  static constexpr int kLen = kRowsTma + 2 * P + 2;
  __device__ __forceinline__ static long long start(long long g0, long long total) {
    long long st = g0 & ~1LL;
    st = st < 0 ? 0 : st;
    const long long hi = (total - kLen + 1) & ~1LL;
    return st > hi ? hi : st;
  }
};

// Stream order of the chunks.  2D: c = 0..R in the reference's column order
// (mirrored shifts are at most p ext + p rows, so the downstream CTA that
// streams the same bytes runs at the same time and L2 serves them).  3D: the
// mirror shifts reach p ext^2 rows (~50 CTAs downstream); visiting each lower
// row qm next to its mirrored row R-1-qm keeps the two reads of those bytes
// (this CTA's mirrored read and the downstream CTA's streamed read) at the
// same relative step of CTAs that run concurrently, so the second one hits
// L2.  In measured c4 traffic the ascending order re-read 70% of the mirrored
// half from HBM.  The 3D row sum is therefore taken in this pairwise order.
template <int D, int P>
__device__ __forceinline__ int chunk_of_step(int st) {
  constexpr int W = 2 * P + 1;
  constexpr int R = D == 2 ? W : W * W;
  constexpr int RL = (R - 1) / 2;
  if (D == 2) return st;
  if (st >= 2 * RL) return st - RL;  // centre row: lower half, then mirrored half
  return (st & 1) ? R - (st >> 1) : (st >> 1);
}

// (d1, d2) offset row a chunk of the half-band stream multiplies
template <int D, int P>
__device__ __forceinline__ int chunk_row(int c) {
  constexpr int W = 2 * P + 1;
  constexpr int RL = ((D == 2 ? W : W * W) - 1) / 2;
  return c <= RL ? c : (c == RL + 1 ? RL : c - 1);
}

// One stage of the half-band sum.  Guarded = false is the interior path: every
// column a row can name lies inside the lattice vector, and the band holds an
// exact 0 for each (row, column) pair outside the tensor stencil (wrapped
// lines, neighbouring patches, Dirichlet, padding rows -- zero_dirichlet_band
// and the Sp >= S + halo stride), so the pair adds fma(0, x, acc) == acc and
// the per-entry predicates of the reference loop are not needed.  Guarded =
// true (the blocks touching either end of the lattice) tests every column.
template <int D, int P, bool Guarded>
__device__ __forceinline__ double half_stage(int c, const double* seg, const double* xw, long long off1, bool ok1,
                                             bool row_ok, int i0, int ext, double acc) {
  constexpr int W = 2 * P + 1;
  constexpr int RL = ((D == 2 ? W : W * W) - 1) / 2;
  if (c < RL) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int d0 = w - P;
      if (!Guarded || (ok1 && i0 + d0 >= 0 && i0 + d0 < ext)) acc = fma(seg[w * kSeg], xw[d0], acc);
    }
  } else if (c == RL) {
#pragma unroll
    for (int w = 0; w <= P; ++w) {
      const int d0 = w - P;
      if (!Guarded || (ok1 && i0 + d0 >= 0)) acc = fma(seg[w * kSeg], xw[d0], acc);
    }
  } else if (c == RL + 1) {
#pragma unroll
    for (int w = 0; w < P; ++w) {
      const int d0 = w + 1;
      if (!Guarded || (row_ok && i0 + d0 < ext)) acc = fma(seg[w * kSeg + (d0 & 1)], xw[d0], acc);
    }
  } else {
    // mirrored segment w starts at the even row below r0 + off1 + d0
    const double* s0 = seg + int(off1 & 1);        // even d0
    const double* s1 = seg + int((off1 + 1) & 1);  // odd d0
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int d0 = w - P;
      const double* sw = (d0 & 1) ? s1 : s0;
      if (!Guarded || (ok1 && i0 + d0 >= 0 && i0 + d0 < ext)) acc = fma(sw[w * kSeg], xw[d0], acc);
    }
  }
  return acc;
}

// x source of the half-band kernel: false = __ldg through L1 (a block's x
// footprint is reused by all its offsets), true = a TMA window per stage.
constexpr bool kHalfXWindow = false;

template <int D, int P>
__global__ void __launch_bounds__(kRowsTma + 32) spmv_tma_half_kernel(SpmvArgs a) {
  PMG_PDL_ENTRY();
  constexpr int W = 2 * P + 1;
  constexpr int R = D == 2 ? W : W * W;  // d0-rows of offsets
  constexpr int RL = (R - 1) / 2;        // d0-rows strictly below the centre row
  constexpr int OB = RL * W + P + 1;     // stored offsets
  constexpr int NCH = R + 1;
  constexpr int kX = kHalfXWindow ? XWindow<P>::kLen : 0;
  constexpr int kStageDoubles = W * kSeg + kX;
  extern __shared__ __align__(128) double ring[];  // [kStages][W][kSeg] band + [kX] x
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ double red[kRowsTma / 32];

  const long long Sp = a.Sp;
  const long long blocks_per_patch = (a.S + kRowsTma - 1) / kRowsTma;
  const long long k = blockIdx.x / blocks_per_patch;
  const long long r0 = (blockIdx.x - k * blocks_per_patch) * kRowsTma;
  const int tid = threadIdx.x;
  const int ext = a.ext;
  const long long ext2 = (long long)ext * ext;
  const long long total = a.S * a.K;
  const long long g_r0 = k * a.S + r0;  // lattice index of the block's first row
  const long long halo = P * (1 + ext + (D == 3 ? ext2 : 0)) + 2;
  const bool guarded = g_r0 - halo < 0 || g_r0 + kRowsTma + halo > total;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRowsTma / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= kRowsTma) {  // producer warp
    if (tid == kRowsTma) {
      const double* base = a.band + (size_t)k * OB * Sp;
      for (int st = 0; st < NCH; ++st) {
        const int c = chunk_of_step<D, P>(st);
        const int s = st % kStages;
        if (st >= kStages) mbar_wait(&empty[s], ((st / kStages) - 1) & 1);
        double* dst = ring + (size_t)s * kStageDoubles;
        const int q = chunk_row<D, P>(c);
        const long long off1 = (long long)ext * (q % W - P) + (D == 3 ? ext2 * (q / W - P) : 0);
        const long long xs = XWindow<P>::start(g_r0 + off1 - P, total);
        if (c <= RL) {
          const int nw = c < RL ? W : P + 1;
          mbar_expect_tx(&full[s], unsigned((nw * kRowsTma + kX) * sizeof(double)));
          for (int w = 0; w < nw; ++w)
            tma_load_1d(dst + w * kSeg, base + (size_t)(c * W + w) * Sp + r0, kRowsTma * sizeof(double), &full[s]);
        } else if (c == RL + 1) {
          mbar_expect_tx(&full[s], unsigned((P * kSeg + kX) * sizeof(double)));
          for (int w = 0; w < P; ++w) {
            const int d0 = w + 1;
            const long long start = (r0 + d0) & ~1LL;
            tma_load_1d(dst + w * kSeg, base + (size_t)(RL * W + P - d0) * Sp + start, kSeg * sizeof(double),
                        &full[s]);
          }
        } else {
          const int qm = R - 1 - q;  // the mirror of offset row q
          mbar_expect_tx(&full[s], unsigned((W * kSeg + kX) * sizeof(double)));
          for (int w = 0; w < W; ++w) {
            const long long start = (r0 + off1 + (w - P)) & ~1LL;
            tma_load_1d(dst + w * kSeg, base + (size_t)(qm * W + (W - 1 - w)) * Sp + start,
                        kSeg * sizeof(double), &full[s]);
          }
        }
        if (kHalfXWindow) tma_load_1d(dst + W * kSeg, a.x + xs, kX * sizeof(double), &full[s]);
      }
    }
    return;
  }

  const long long r = r0 + tid;
  const bool row_ok = r < a.S;
  const int i0 = int(r % ext);
  const int i1 = int((r / ext) % ext);
  const int i2 = D == 3 ? int(r / ext2) : 0;
  const long long gid = g_r0 + tid;
  const double fv = (a.f && row_ok) ? a.f[gid] : 0.0;
  double acc = 0.0;
  for (int st = 0; st < NCH; ++st) {
    const int c = chunk_of_step<D, P>(st);
    const int s = st % kStages;
    const double* seg = ring + (size_t)s * kStageDoubles + tid;
    const int q = chunk_row<D, P>(c);
    const int d1 = q % W - P, d2 = D == 3 ? q / W - P : 0;
    const long long off1 = (long long)ext * d1 + ext2 * d2;
    // xw[d0] = x[gid + off1 + d0]
    const double* xw = kHalfXWindow ? seg + W * kSeg + int(g_r0 + off1 - XWindow<P>::start(g_r0 + off1 - P, total))
                                    : a.x + gid + off1;
    mbar_wait(&full[s], (st / kStages) & 1);
    if (guarded) {
      const bool ok1 = row_ok && i1 + d1 >= 0 && i1 + d1 < ext && (D == 2 || (i2 + d2 >= 0 && i2 + d2 < ext));
      acc = half_stage<D, P, true>(c, seg, xw, off1, ok1, row_ok, i0, ext, acc);
    } else {
      acc = half_stage<D, P, false>(c, seg, xw, off1, true, true, i0, ext, acc);
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
  }
  double prod = 0.0;
  if (row_ok) {
    const double y = a.f ? fv - acc : acc;
    a.y[gid] = y;
    if (a.dot_partial) prod = y * a.x[gid];
  }
  if (a.dot_partial) {
    for (int o = 16; o > 0; o >>= 1) prod += __shfl_down_sync(0xffffffffu, prod, o);
    if ((tid & 31) == 0) red[tid >> 5] = prod;
    asm volatile("bar.sync 1, %0;\n" ::"n"(kRowsTma) : "memory");
    if (tid == 0) {
      double sum = 0.0;
      for (int w = 0; w < kRowsTma / 32; ++w) sum += red[w];
      a.dot_partial[blockIdx.x] = sum;
    }
  }
}

// ---------------------------------------------------------------- 2D line sweep
// 2D half band, lattice lines of at most kSweepMaxExt rows.  These levels keep
// the band line-major: [K][line L][Ob offsets][tw], each offset row of a line
// holding its ext values at columns [PADL, PADL + ext) between zero pads
// (sweep_relayout_kernel builds it from the offset-major band once, at
// upload).  A CTA owns the output lines [L0, L1) of one patch and streams the
// band one lattice line at a time, as p+1 chunks: chunk q holds the offsets
// with d1 = q - p (2p+1 of them; p+1 with d0 <= 0 at d1 = 0), contiguous, so
// one bulk copy (TMA) fills one stage of a ring guarded by mbarriers.  Every
// band value is used twice from shared memory: as the lower entry A(r, r-s)
// of its own row (against x of lines L-p..L, held in a register window), and
// as the mirrored upper entry A(r-s, r) of the row r-s in line L-m, m = p-q
// (the accumulators of the last p+1 lines stay in registers).  A row of line
// L' therefore receives its terms in the reference's column order: chunks
// 0..p of line L' (lower rows, then the centre row), then chunk p-m of line
// L'+m for m = 1..p (mirrored rows).  Every band line crosses HBM and L2
// once.  Segment boundaries: the mirrored terms a segment's first p lines
// give to rows of the previous segment's last p lines ("carry", summed in the
// same line order) go to a scratch row per boundary, published early (after
// line L0+p-1) with a release flag; the previous segment's CTA waits for the
// flag when it reaches its end, which in practice has long been set, and adds
// the carry: y = f - (partial + carry).  Mirrored reads of columns outside the
// line land in the zero pads (in the band those pairs are wrapped and hold
// exact zeros as well).
constexpr int kSweepMaxExt = 288;
constexpr int kSweepMaxStages = 16;

struct SweepCfg {
  int segs, seglen;    // line segments per patch and their length
  int stages, tw, nc;  // ring depth (chunks), offset-row width, consumer threads
};

// offset-major [K][Ob][Sp] -> line-major [K][ext][Ob][tw] with zero pads
template <int P>
__global__ void sweep_relayout_kernel(const double* __restrict__ src, double* __restrict__ dst, int ext, int K,
                                      long long Sp, int tw) {
  constexpr int W = 2 * P + 1;
  constexpr int OB = P * W + P + 1;
  constexpr int PADL = (P + 1) & ~1;
  const long long n = (long long)K * ext * OB * tw;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = int(e % tw);
    const long long t = e / tw;
    const int o = int(t % OB);
    const long long kl = t / OB;
    const int L = int(kl % ext);
    const long long k = kl / ext;
    const int i = c - PADL;
    dst[e] = (i >= 0 && i < ext) ? src[((size_t)k * OB + o) * Sp + (size_t)L * ext + i] : 0.0;
  }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Consumer side of the sweep: one thread per column i of the line.  The
// register arrays are indexed by line modulo p+1 (acc[s], xw[s] belong to the
// line L with L - L0 = s mod p+1), and the line loop is unrolled p+1 times
// (line<PH>), so no value is moved between lines.  x and f reach shared
// memory through per-thread cp.async copies issued p lines ahead (x ring of
// p+2 lines, f ring of p+2 lines); one commit group per line.
template <int P>
struct SweepConsumer {
  static constexpr int W = 2 * P + 1;
  static constexpr int PADL = (P + 1) & ~1;
  static constexpr int NX = P + 2;  // x ring lines
  static constexpr int NF = P + 2;  // f ring lines
  const double* smem;  // band ring [stages][W][tw]
  double* xs;          // [NX][tw]
  double* fs;          // [NF][nc]
  uint64_t *full, *empty;
  const double* __restrict__ xk;
  const double* __restrict__ fk;
  double* __restrict__ yk;
  int i, ext, tw, stages, nc, L0, L1, Lend;
  bool col;
  double* carry_lo;         // mirrored terms this CTA computes for the previous segment's last p lines (or null)
  unsigned* flag_lo;       // set once carry_lo is written
  const double* carry_hi;  // the next segment's carry for this segment's last p lines (or null)
  unsigned* flag_hi;
  double cr[P];            // this column's carry, loaded p lines before it is added
  int st, ph;      // band ring: stage of the next chunk and its phase parity
  int xcur, fcur;  // ring slots of line L
  double acc[P + 1];
  double xw[P + 1][W];
  double prod;

  __device__ __forceinline__ void issue_x(int line, int slot) {
    if (col && line < Lend) cp_async8(xs + slot * tw + PADL + i, xk + (size_t)line * ext + i);
  }

  template <int PH>
  __device__ __forceinline__ void line(int L) {
    // this thread's copies of x(L) and f(L-p) (the group of line L-p) are done
    cp_async_wait<P - 1>();
    if (L < Lend) {
      // p lines before its end the CTA takes the next segment's carry rows
      // (published a few lines into that CTA's run, so the wait is short)
      const bool take = carry_hi && L == L1 - P;
      if (take && i == 0) {
        while (ld_acquire(flag_hi) == 0u) __nanosleep(32);
        *flag_hi = 0u;  // this CTA is its only reader: ready for the next launch
      }
      // every consumer has stored x(L) and finished line L-1
      asm volatile("bar.sync 1, %0;\n" ::"r"(nc) : "memory");
      if (take && col) {
#pragma unroll
        for (int q = 0; q < P; ++q) cr[q] = __ldcg(carry_hi + q * ext + i);
      }
      {
        int sx = xcur + P;
        sx -= sx >= NX ? NX : 0;
        issue_x(L + P, sx);
        if (col && fk && L < L1) cp_async8(fs + fcur * nc + i, fk + (size_t)L * ext + i);
      }
      cp_async_commit();
      const double* xl = xs + xcur * tw + PADL + (col ? i : 0);  // threads past the line read column 0
#pragma unroll
      for (int j = 0; j < W; ++j) xw[PH][j] = xl[j - P];
      const int nq = L < L1 ? P + 1 : P - (L - L1);
#pragma unroll
      for (int q = 0; q <= P; ++q) {
        if (q < nq) {
          mbar_wait(&full[st], ph);
          if (col) {
            const double* T = smem + (size_t)st * W * tw + PADL + i;
            if (L < L1) {  // lower entries of the rows of line L, d1 = q - p (d0 <= 0 at d1 = 0)
              const int sl = (PH + 1 + q) % (P + 1);  // slot of line L - (p - q)
#pragma unroll
              for (int w = 0; w < (q < P ? W : P + 1); ++w) acc[PH] = fma(T[w * tw], xw[sl][w], acc[PH]);
            }
            // mirrored entries A(r - s, r), s = (m, d0), m = p - q: row r of line L, offset -s
            const int m = P - q;
            if (L - m >= 0) {
              const int sa = (PH + 1 + q) % (P + 1);  // slot of line L - m
#pragma unroll
              for (int d0 = (m == 0 ? 1 : -P); d0 <= P; ++d0)
                acc[sa] = fma(T[(P - d0) * tw + d0], xw[PH][d0 + P], acc[sa]);
            }
          }
          __syncwarp();
          if ((i & 31) == 0) mbar_arrive(&empty[st]);
          if (++st == stages) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    } else {
      cp_async_commit();  // one group per line
    }
    constexpr int SW = (PH + 1) % (P + 1);  // slot of line L - p, complete now
    const int Lw = L - P;
    if (col && Lw >= 0) {
      if (Lw < L0) {  // mirrored terms of a row of the previous segment
        carry_lo[(L0 - 1 - Lw) * ext + i] = acc[SW];
      } else {
        // rows of the last p lines add the mirrored terms from the next segment's lines
        double s = acc[SW];
        if (carry_hi && Lw >= L1 - P) {
          const int t = L1 - 1 - Lw;
          double c = 0.0;
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (q == t) c = cr[q];
          s += c;
        }
        int sf = fcur + 2;  // slot of f(L - p)
        sf -= sf >= NF ? NF : 0;
        const double y = fk ? fs[sf * nc + i] - s : s;
        yk[(size_t)Lw * ext + i] = y;
        prod = fma(y, xw[SW][P], prod);
      }
    }
    if (L == L0 + P - 1 && carry_lo) {  // every carry row is written: publish them
      __threadfence();
      asm volatile("bar.sync 1, %0;\n" ::"r"(nc) : "memory");
      if (i == 0) st_release(flag_lo, 1u);
    }
    acc[SW] = 0.0;  // the accumulator of line L+1
    xcur = xcur + 1 == NX ? 0 : xcur + 1;
    fcur = fcur + 1 == NF ? 0 : fcur + 1;
  }
};

template <int P>
__global__ void __launch_bounds__(kSweepMaxExt + 32, 1) spmv_sweep2d_kernel(SpmvArgs a, SweepCfg g) {
  // no early launch_dependents: a CTA waits for the next segment's CTA, so
  // dependent grids must not take SMs before every CTA of this one runs
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  constexpr int W = 2 * P + 1;
  constexpr int OB = P * W + P + 1;  // stored offsets: d1 = -p..-1 (all d0), d1 = 0 (d0 <= 0)
  using C = SweepConsumer<P>;
  extern __shared__ __align__(128) double smem[];  // [stages][W][tw] band chunks, [NX][tw] x, [NF][nc] f
  __shared__ __align__(8) uint64_t full[kSweepMaxStages], empty[kSweepMaxStages];
  __shared__ double red[kSweepMaxExt / 32];

  __shared__ int s_seg;
  const int ext = a.ext;
  const int nc = g.nc;
  const int tw = g.tw;
  const int stages = g.stages;
  const int tid = threadIdx.x;
  // Segments are handed out in the order CTAs start (a ticket counter that
  // every launch advances by the grid size), last segment of a patch first:
  // a CTA only ever waits for the carry of the segment above it, which holds
  // an earlier ticket and so already runs.  No wait depends on how many CTAs
  // fit on the GPU at once.
  // (the ticket's round trip overlaps the pad zeroing and barrier setup)
  unsigned long long ticket = 0;
  if (tid == 0) ticket = atomicAdd(a.sweep_ticket, 1ull);
  double* xs = smem + (size_t)stages * W * tw;
  for (int q = tid; q < C::NX * tw; q += blockDim.x) xs[q] = 0.0;  // x pads
  if (tid == 0) {
    for (int st = 0; st < stages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], nc / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    const unsigned long long t = ticket % gridDim.x;
    s_seg = int(t / g.segs) * g.segs + (g.segs - 1 - int(t % g.segs));
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  const int seg = s_seg;  // k * segs + j
  const int k = seg / g.segs;
  const int jseg = seg - k * g.segs;
  const int L0 = jseg * g.seglen;
  const int L1 = min(ext, L0 + g.seglen);
  const int Lend = L1;  // streamed lines [L0, L1): each band line crosses HBM once
  const long long S = a.S;
  double* fs = xs + C::NX * tw;
  // segment boundaries: b_lo with segment j-1, b_hi with j+1
  const int b_lo = jseg > 0 ? seg : -1;
  const int b_hi = L1 < ext ? seg + 1 : -1;

  if (tid >= nc) {  // producer thread: one bulk copy per chunk
    if (tid == nc) {
      const double* base = a.band + (size_t)k * ext * OB * tw;
      int st = 0, ph = 0, step = 0;
      for (int L = L0; L < Lend; ++L) {
        // tail lines past L1 carry only the chunks q < p - (L - L1)
        const int nq = L < L1 ? P + 1 : P - (L - L1);
        for (int q = 0; q < nq; ++q, ++step) {
          if (step >= stages) mbar_wait(&empty[st], ph ^ 1);
          const unsigned bytes = unsigned((q < P ? W : P + 1) * tw * sizeof(double));
          mbar_expect_tx(&full[st], bytes);
          tma_load_1d(smem + (size_t)st * W * tw, base + ((size_t)L * OB + q * W) * tw, bytes, &full[st]);
          if (++st == stages) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }

  C c;
  c.smem = smem;
  c.xs = xs;
  c.fs = fs;
  c.full = full;
  c.empty = empty;
  c.i = tid;
  c.col = tid < ext;
  c.xk = a.x + (size_t)k * S;
  c.fk = a.f ? a.f + (size_t)k * S : nullptr;
  c.yk = a.y + (size_t)k * S;
  c.ext = ext;
  c.tw = tw;
  c.stages = stages;
  c.nc = nc;
  c.L0 = L0;
  c.L1 = L1;
  c.Lend = Lend;
  c.carry_lo = b_lo >= 0 ? a.sweep_scratch + (size_t)b_lo * P * ext : nullptr;
  c.flag_lo = b_lo >= 0 ? a.sweep_flags + b_lo : nullptr;
  c.carry_hi = b_hi >= 0 ? a.sweep_scratch + (size_t)b_hi * P * ext : nullptr;
  c.flag_hi = b_hi >= 0 ? a.sweep_flags + b_hi : nullptr;
  c.st = 0;
  c.ph = 0;
  c.xcur = 0;
  c.fcur = 0;
  c.prod = 0.0;
  // lines L0-m (slot p+1-m) straight from global memory; x(L0..L0+p-1) as p groups
#pragma unroll
  for (int m = 1; m <= P; ++m) {
    const int line = L0 - m;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const int cc = tid + j - P;
      c.xw[P + 1 - m][j] = (c.col && line >= 0 && cc >= 0 && cc < ext) ? __ldg(c.xk + (size_t)line * ext + cc) : 0.0;
    }
  }
#pragma unroll
  for (int j = 0; j < W; ++j) c.xw[0][j] = 0.0;
#pragma unroll
  for (int m = 0; m <= P; ++m) c.acc[m] = 0.0;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    c.issue_x(L0 + j, j);
    cp_async_commit();
  }
  for (int L = L0; L < L1 + P; L += P + 1) {
    c.template line<0>(L);
    if (L + 1 < L1 + P) c.template line<1 % (P + 1)>(L + 1);
    if (P >= 2 && L + 2 < L1 + P) c.template line<2 % (P + 1)>(L + 2);
    if (P >= 3 && L + 3 < L1 + P) c.template line<3 % (P + 1)>(L + 3);
    if (P >= 4 && L + 4 < L1 + P) c.template line<4 % (P + 1)>(L + 4);
  }
  cp_async_wait<0>();
  if (a.dot_partial) {
    double prod = c.prod;
    for (int o = 16; o > 0; o >>= 1) prod += __shfl_down_sync(0xffffffffu, prod, o);
    if ((tid & 31) == 0) red[tid >> 5] = prod;
    asm volatile("bar.sync 1, %0;\n" ::"r"(nc) : "memory");
    if (tid == 0) {
      double sum = 0.0;
      for (int w = 0; w < nc / 32; ++w) sum += red[w];
      a.dot_partial[seg] = sum;  // per segment: the same order of partials every run
    }
  }
}

// ---------------------------------------------------------------- 3D plane sweep
// 3D half band ([K][OB][Sp], offset-major).  A CTA owns the in-plane rows
// [ta, tb) of one patch (a tile of the ext^2 rows of a lattice plane) and the
// planes [Z0, Z1) of a segment, and sweeps them plane by plane.  For plane z
// it streams, offset by offset, the band rows of its tile (one bulk copy per
// offset: the rows (t, z) of the tile plus the |s_in| rows of halo the
// mirrored use needs, s_in = d0 + d1 ext being the in-plane part of the
// offset's shift s = s_in + d2 ext^2) and uses every value twice from shared
// memory:
//   lower     row (t, z):        += A(r, r + s) x(t + s_in, z + d2)
//   mirrored  row (t, z + d2):   += A(r', r' + s) x(r'),  r' = (t - s_in, z)
// (the mirrored term is the upper entry A(q, q - s) = A(q - s, q) of row q).
// x of planes z-p..z+1 sits in a ring of p+3 plane slots (each the tile plus
// p (1 + ext) rows of halo on both sides), filled one plane ahead.  Each
// output row keeps p+1 plane accumulators in registers: plane z-p is
// complete after plane z and is written then.  The mirrored terms a segment's
// rows receive from the next segment's first p planes are computed by
// streaming those planes as well (tail planes, only the offsets whose target
// plane lies inside the segment), so CTAs never wait for each other.  Every
// band value crosses HBM once; L2 serves the halo rows and the tail planes a
// second time (about |s_in| / T and 1.7 / (Z1 - Z0) of the band).  Pairs
// outside the tensor stencil hold exact zeros in the band (wrapped lines and
// planes, Dirichlet, padding) and shared-memory rows outside the vectors hold
// zeros, so no per-entry predicate is needed; offsets whose lower source
// plane is below the lattice (z + d2 < 0) are all-zero and skipped.
// Consumer thread i owns the rows ta + i + j NC, j < RPT (NC and RPT compile
// time, so every shared-memory read is one LDS with an immediate offset);
// rows past tb are computed on padding and not written.
// Swept levels keep the band plane-major: [K][plane z][offset o][e2p], the
// ext^2 rows of a (plane, offset) pair at [front, front + ext^2) between zero
// pads that cover every halo and padding read (sweep3_relayout_kernel builds
// it from the offset-major band once, at upload).  A CTA's stream of one
// plane is then one contiguous block (ob e2p doubles): a few DRAM pages and
// TLB entries per plane instead of one 2 MB offset row per stage.
constexpr int kSweep3MaxStages = 24;
constexpr int kSweep3Nc = 384;  // consumer threads (12 warps)
constexpr int kSweep3Pw = 4;    // producer warps: warp w issues the stages st with st % kSweep3Pw == w
constexpr int kSweep3MaxRpt = 4;

struct Sweep3Cfg {
  int tiles, T;     // in-plane tiles per plane, rows per tile
  int zsegs, zlen;  // plane segments per patch, planes per segment
  int rpt;          // rows per consumer thread (T <= rpt kSweep3Nc)
  int ns, sd, xd;   // band ring stages, doubles per stage, doubles per x plane slot
  int halo;         // p (1 + ext): the largest in-plane shift
  int front, e2p;   // plane-major band: zero rows before a (plane, offset) row, row stride
};

template <int P>
__device__ __forceinline__ int sweep3_shift(int o, int ext) {  // in-plane shift s_in of offset o
  constexpr int W = 2 * P + 1;
  const int q = o % (W * W);
  return (q % W - P) + ext * (q / W - P);
}

template <int P, int RPT>
struct Sweep3Consumer {
  static constexpr int W = 2 * P + 1;
  static constexpr int OB = (W * W * W + 1) / 2;
  static constexpr int NX = P + 3;  // x plane slots
  static constexpr int NA = P + 1;  // accumulator planes
  static constexpr int NC = kSweep3Nc;
  const SpmvArgs* a;
  const double* ring;
  const double* xs;
  uint64_t *full, *empty, *xfull, *xempty;
  long long E2, S;
  int ext, k, ta, tb, Z0, Z1, Zend, zfirst, tid, st, ph, ns, sd, xd, halo;
  double acc[NA][RPT];
  double prod;

  __device__ __forceinline__ const double* xp(int zz) const {  // xp(zz)[i] = x(i, zz) of patch k
    const int sl = (zz - zfirst) % NX;
    const long long g0 = (long long)k * S + (long long)zz * E2 + ta - halo;
    return xs + sl * xd + int(g0 & 1) + (halo - ta);
  }
  __device__ __forceinline__ void wait_x(int zz) {
    const int u = zz - zfirst;
    mbar_wait(&xfull[u % NX], (u / NX) & 1);
  }
  __device__ __forceinline__ void finish(int zo, double (&accz)[RPT]) {  // plane zo complete
    const double* xz = xp(zo);
    const long long base = (long long)k * S + (long long)zo * E2;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int t = ta + tid + j * NC;
      if (t < tb) {
        const double y = a->f ? a->f[base + t] - accz[j] : accz[j];
        a->y[base + t] = y;
        if (a->dot_partial) prod = fma(y, xz[t], prod);
      }
      accz[j] = 0.0;
    }
  }
  // the offsets [o_beg, o_end) of one d2 group (GI = d2 + p) at plane z
  template <int ZS, int GI, bool LOWER, bool MIRROR>
  __device__ __forceinline__ void offsets(int o_beg, int o_end, int base_par, const double* xl, const double* xz) {
    int d0 = (o_beg % W) - P;
    int s_in = sweep3_shift<P>(o_beg, ext);
    const double* xlt = xl + ta + tid;  // xlt[j NC] = x(ta + tid + j NC, z + d2)
    const double* xzt = xz + ta + tid;
    for (int o = o_beg; o < o_end; ++o) {
      const int sc = st;
      mbar_wait(&full[sc], ph);
      if (++st == ns) {
        st = 0;
        ph ^= 1;
      }
      const int lo_rel = min(0, -s_in);
      const int par = (base_par ^ lo_rel) & 1;  // parity of the stage's first in-plane index
      const double* bp = ring + sc * sd + par - lo_rel + tid;  // bp[j NC] = band row (ta + tid + j NC, z)
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        if (LOWER) acc[ZS][j] = fma(bp[j * NC], xlt[j * NC + s_in], acc[ZS][j]);
        // target slot (ZS + d2) mod (p+1) = (ZS + GI + 1) mod (p+1)
        if (MIRROR)
          acc[(ZS + GI + 1) % NA][j] = fma(bp[j * NC - s_in], xzt[j * NC - s_in], acc[(ZS + GI + 1) % NA][j]);
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[sc]);
      if (++d0 > P) {
        d0 = -P;
        s_in += ext - 2 * P;
      } else {
        s_in += 1;
      }
    }
  }
  template <int ZS, int GI>
  __device__ __forceinline__ void group(int z, int base_par, const double* xz) {
    const int zt = z + GI - P;  // mirrored target plane / lower source plane
    const bool in_seg = z < Z1;
    if ((!in_seg && zt >= Z1) || zt < 0) return;  // skipped by the producer as well
    const bool mirror = zt >= Z0 && zt < Z1;
    const double* xl = in_seg ? xp(zt) : xz;
    const int o_beg = GI * W * W;
    const int o_end = GI < P ? (GI + 1) * W * W : OB - 1;  // the centre (diagonal) separately
    if (in_seg && mirror)
      offsets<ZS, GI, true, true>(o_beg, o_end, base_par, xl, xz);
    else if (in_seg)
      offsets<ZS, GI, true, false>(o_beg, o_end, base_par, xl, xz);
    else
      offsets<ZS, GI, false, true>(o_beg, o_end, base_par, xl, xz);
    if (GI == P && in_seg) offsets<ZS, GI, true, false>(OB - 1, OB, base_par, xl, xz);
  }
  // one plane step; ZS = (z - Z0) mod (p+1) is the accumulator slot of plane z
  template <int ZS>
  __device__ __forceinline__ void plane(int z) {
    wait_x(z);
    const double* xz = xp(z);
    const int base_par = ta & 1;
    group<ZS, 0>(z, base_par, xz);
    if (P >= 1) group<ZS, 1 % (P + 1)>(z, base_par, xz);
    if (P >= 2) group<ZS, 2 % (P + 1)>(z, base_par, xz);
    if (P >= 3) group<ZS, 3 % (P + 1)>(z, base_par, xz);
    const int zo = z - P;  // complete now
    if (zo >= Z0 && zo < Z1) finish(zo, acc[(ZS + 1) % NA]);
    if (zo >= zfirst) {  // x plane zo is no longer read
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&xempty[(zo - zfirst) % NX]);
    }
  }
};

template <int P, int RPT>
__global__ void __launch_bounds__(kSweep3Nc + 32 * kSweep3Pw, 1) spmv_sweep3d_kernel(SpmvArgs a, Sweep3Cfg g) {
  PMG_PDL_ENTRY();
  using C = Sweep3Consumer<P, RPT>;
  constexpr int OB = C::OB;
  constexpr int NX = C::NX;
  constexpr int NA = C::NA;
  constexpr int NC = kSweep3Nc;
  extern __shared__ __align__(128) double smem[];  // [ns][sd] band ring, [NX][xd] x planes
  __shared__ __align__(8) uint64_t full[kSweep3MaxStages], empty[kSweep3MaxStages], xfull[NX], xempty[NX];
  __shared__ double red[NC / 32];

  const int ext = a.ext;
  const long long E2 = (long long)ext * ext;
  const long long S = a.S;
  const int tid = threadIdx.x;
  const int tile = blockIdx.x % g.tiles;
  const int zs = (blockIdx.x / g.tiles) % g.zsegs;
  const int k = blockIdx.x / (g.tiles * g.zsegs);
  const int ta = tile * g.T;
  const int tb = min(int(E2), ta + g.T);
  const int Z0 = zs * g.zlen;
  const int Z1 = min(ext, Z0 + g.zlen);
  const int Zend = min(ext, Z1 + P);
  const int zfirst = max(0, Z0 - P);
  double* xs = smem + (size_t)g.ns * g.sd;
  if (tid == 0) {
    for (int s = 0; s < g.ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NC / 32);
    }
    for (int s = 0; s < NX; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], NC / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= NC) {  // producers: one bulk copy per (plane, offset); x planes from warp 0
    const int pw = (tid - NC) >> 5;
    if (((tid - NC) & 31) == 0) {
      const long long total = S * a.K;
      const int H = g.halo;
      const int Tpad = RPT * NC;  // rows computed per tile (padding past tb included)
      auto load_x = [&](int zz) {
        const int u = zz - zfirst;
        const int sl = u % NX;
        if (u >= NX) mbar_wait(&xempty[sl], ((u / NX) - 1) & 1);
        double* dst = xs + (size_t)sl * g.xd;
        long long g0 = (long long)k * S + (long long)zz * E2 + ta - H;
        g0 -= g0 & 1;
        const long long n = g.xd;
        const long long lo = g0 < 0 ? 0 : g0;
        const long long hi = g0 + n > total ? total : g0 + n;
        const long long th = lo + ((hi - lo) & ~1LL);  // bulk part [lo, th), 16-byte sized
        for (long long e = g0; e < lo; ++e) dst[e - g0] = 0.0;  // before the vector
        for (long long e = th; e < g0 + n; ++e) dst[e - g0] = e < total ? a.x[e] : 0.0;  // odd end / past it
        mbar_expect_tx(&xfull[sl], unsigned((th - lo) * sizeof(double)));
        if (th > lo) tma_load_1d(dst + (lo - g0), a.x + lo, unsigned((th - lo) * sizeof(double)), &xfull[sl]);
      };
      if (pw == 0)
        for (int zz = zfirst; zz <= Z0; ++zz) load_x(zz);
      int s = 0, round = 0;  // ring slot and how many times the ring has been filled
      int seq = 0;           // stage sequence number
      for (int z = Z0; z < Zend; ++z) {
        if (pw == 0 && z + 1 < Zend) load_x(z + 1);
        for (int o = 0; o < OB; ++o) {
          constexpr int W = 2 * P + 1;
          const int zt = z + o / (W * W) - P;
          if ((z >= Z1 && zt >= Z1) || zt < 0) continue;  // no target in the segment / all-zero offset
          const int mine = (seq++ % kSweep3Pw) == pw;
          if (!mine) {
            if (++s == g.ns) {
              s = 0;
              ++round;
            }
            continue;
          }
          const int s_in = sweep3_shift<P>(o, ext);
          if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
          const int lo_in = ta + min(0, -s_in);
          const int hi_in = ta + Tpad + max(0, -s_in);
          const int r0 = lo_in - (lo_in & 1);  // in-plane index of the stage's first element (even)
          const int n = (hi_in - r0 + 1) & ~1;
          const double* src = a.band + (((size_t)k * ext + z) * OB + o) * g.e2p + g.front + r0;
          mbar_expect_tx(&full[s], unsigned(n * sizeof(double)));
          tma_load_1d(smem + (size_t)s * g.sd, src, unsigned(n * sizeof(double)), &full[s]);
          if (++s == g.ns) {
            s = 0;
            ++round;
          }
        }
      }
    }
    return;
  }

  C c;
  c.a = &a;
  c.ring = smem;
  c.xs = xs;
  c.full = full;
  c.empty = empty;
  c.xfull = xfull;
  c.xempty = xempty;
  c.E2 = E2;
  c.S = S;
  c.ext = ext;
  c.k = k;
  c.ta = ta;
  c.tb = tb;
  c.Z0 = Z0;
  c.Z1 = Z1;
  c.Zend = Zend;
  c.zfirst = zfirst;
  c.tid = tid;
  c.st = 0;
  c.ph = 0;
  c.ns = g.ns;
  c.sd = g.sd;
  c.xd = g.xd;
  c.halo = g.halo;
  c.prod = 0.0;
#pragma unroll
  for (int q = 0; q < NA; ++q)
#pragma unroll
    for (int j = 0; j < RPT; ++j) c.acc[q][j] = 0.0;
  for (int zz = zfirst; zz < Z0; ++zz) c.wait_x(zz);
  for (int zb = Z0; zb < Zend; zb += NA) {
    c.template plane<0>(zb);
    if (zb + 1 < Zend) c.template plane<1 % NA>(zb + 1);
    if (P >= 2 && zb + 2 < Zend) c.template plane<2 % NA>(zb + 2);
    if (P >= 3 && zb + 3 < Zend) c.template plane<3 % NA>(zb + 3);
  }
  // planes not written yet: the last segment of a patch has no tail planes
#pragma unroll
  for (int q = 0; q < NA; ++q)
    for (int zo = max(Z0, Zend - P); zo < Z1; ++zo)
      if ((zo - Z0) % NA == q) c.finish(zo, c.acc[q]);
  if (a.dot_partial) {
    double prod = c.prod;
    for (int o = 16; o > 0; o >>= 1) prod += __shfl_down_sync(0xffffffffu, prod, o);
    if ((tid & 31) == 0) red[tid >> 5] = prod;
    asm volatile("bar.sync 1, %0;\n" ::"n"(NC) : "memory");
    if (tid == 0) {
      double sum = 0.0;
      for (int w = 0; w < NC / 32; ++w) sum += red[w];
      a.dot_partial[blockIdx.x] = sum;
    }
  }
}

template <int D, int P>
void launch_tma(cudaStream_t s, const SpmvArgs& a) {
  constexpr int W = 2 * P + 1;
  const long long grid = (a.S + kRowsTma - 1) / kRowsTma * a.K;
  if (a.half) {
    const size_t smem = (size_t)kStages * (W * kSeg + (kHalfXWindow ? XWindow<P>::kLen : 0)) * sizeof(double);
    ensure_smem((const void*)spmv_tma_half_kernel<D, P>, smem);
    launch_k(spmv_tma_half_kernel<D, P>, dim3(unsigned(grid)), dim3(kRowsTma + 32), smem, s, a);
    return;
  }
  const size_t smem = (size_t)kStages * W * kRowsTma * sizeof(double);
  ensure_smem((const void*)spmv_tma_kernel<D, P>, smem);
  launch_k(spmv_tma_kernel<D, P>, dim3(unsigned(grid)), dim3(kRowsTma + 32), smem, s, a);
}

}  // namespace

static int sm_count() {
  static const int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}

static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// Line-sweep configuration of one 2D level: ring depth from the shared-memory
// budget, then enough line segments per patch to fill every SM
// (min_ext: the shortest line swept, from the context: PMG_SWEEP=0 disables
// the sweep, PMG_SWEEP_MIN_EXT sets the threshold, default 128 -- shorter
// lines are latency-bound and the 256-row kernel is faster there).
template <int P>
bool sweep_cfg_p(int ext, int K, int min_ext, SweepCfg* g, size_t* smem) {
  constexpr int W = 2 * P + 1;
  constexpr int PADL = (P + 1) & ~1;
  // shared memory per CTA: short lines run several CTAs per SM (their per-line
  // chain is latency-bound; measured at ext = 132: 33 -> 30 us per launch)
  static const int budget_env = env_int("PMG_SWEEP_SMEM", 0);
  const int budget = budget_env > 0 ? budget_env : (ext <= 160 ? 72 * 1024 : 200 * 1024);
  if (ext > kSweepMaxExt || ext < min_ext || ext < 2 * P + 2) return false;
  g->nc = (ext + 31) / 32 * 32;
  g->tw = (PADL + ext + P + 1) & ~1;  // columns PADL - p .. PADL + ext - 1 + p, even (16-byte rows)
  const size_t stage = size_t(W) * g->tw * sizeof(double);
  const size_t xbytes = size_t(P + 2) * (g->tw + g->nc) * sizeof(double);  // x and f rings
  const long long st = (budget - (long long)xbytes) / (long long)stage;
  if (st < 2) return false;
  g->stages = int(st < kSweepMaxStages ? st : kSweepMaxStages);
  *smem = g->stages * stage + xbytes;
  const int per_sm = std::max(1, int((227 * 1024) / (*smem + 2048)));
  const int target = sm_count() * per_sm;
  int segs = std::max(1, target / std::max(K, 1));
  segs = std::min(segs, std::max(1, ext / std::max(2 * P, 8)));
  g->seglen = (ext + segs - 1) / segs;
  g->segs = (ext + g->seglen - 1) / g->seglen;
  return true;
}

static bool sweep_cfg(int dim, int degree, int ext, long long S, int K, bool half, int sweep, SweepCfg* g,
                      size_t* smem) {
  if (sweep <= 0 || dim != 2 || !half || !spmv_tma_level(dim, degree, S)) return false;
  switch (degree) {
    case 1: return sweep_cfg_p<1>(ext, K, sweep, g, smem);
    case 2: return sweep_cfg_p<2>(ext, K, sweep, g, smem);
    case 3: return sweep_cfg_p<3>(ext, K, sweep, g, smem);
    case 4: return sweep_cfg_p<4>(ext, K, sweep, g, smem);
    default: return false;
  }
}

template <int P>
void launch_sweep(cudaStream_t s, const SpmvArgs& a, const SweepCfg& g, size_t smem) {
  ensure_smem((const void*)spmv_sweep2d_kernel<P>, smem);
  launch_k(spmv_sweep2d_kernel<P>, dim3(unsigned(g.segs * a.K)), dim3(g.nc + 32), smem, s, a, g);
}

// Every level of a specialised degree streams its band with TMA: on small
// levels the one-thread-per-row loop is latency-bound (each thread walks its
// (2p+1)^d entries with few loads in flight), while the staged stream keeps a
// whole block's band in flight.  PMG_TMA_MIN_ROWS raises the threshold.
static long long tma_min_rows() {
  static const long long v = [] {
    const char* e = std::getenv("PMG_TMA_MIN_ROWS");
    return e ? std::atoll(e) : 0LL;
  }();
  return v;
}

bool spmv_tma_level(int dim, int degree, long long S) {
  return S >= tma_min_rows() && ((dim == 2 && degree >= 1 && degree <= 8 && degree != 7) ||
                       (dim == 3 && degree >= 1 && degree <= 4));
}

long long spmv_row_stride(int dim, int degree, int ext, long long S) {
  if (!spmv_tma_level(dim, degree, S)) return S;
  // room for every mirrored read of a valid row to land in this offset's own
  // zero padding: S + halo, rounded to whole 256-row segments
  const long long halo = (long long)degree * (1 + ext + (dim == 3 ? (long long)ext * ext : 0)) + 2;
  return (S + halo + kRowsTma - 1) / kRowsTma * kRowsTma;
}

int spmv_stored_offsets(int dim, int degree, long long S, bool allow_half) {
  const int W = 2 * degree + 1;
  const int O = dim == 2 ? W * W : W * W * W;
  return allow_half && spmv_tma_level(dim, degree, S) ? (O + 1) / 2 : O;
}

int spmv_blocks(long long rows) { return int((rows + kThreads - 1) / kThreads); }

namespace {
__global__ void band_expand_kernel(const double* __restrict__ band, double* __restrict__ full, int dim, int p,
                                   int ext, long long S, int O, int Ob, long long Sp, int tw, int front, int e2p) {
  const int W = 2 * p + 1;
  const int padl = (p + 1) & ~1;
  const long long n = (long long)O * S;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int o = int(e / S);
    const long long r = e % S;
    int ob = o;
    long long row = r;
    if (o >= Ob) {  // upper half of a symmetric half band: mirror offset, shifted row
      long long shift = 0, mul = 1;
      int t = o;
      for (int a = 0; a < dim; ++a) {
        shift += (long long)(t % W - p) * mul;
        t /= W;
        mul *= ext;
      }
      ob = O - 1 - o;
      row = r + shift;
    }
    double v = 0.0;
    if (row >= 0 && row < S) {
      if (e2p > 0) {  // plane-major 3D sweep layout
        const long long E2 = (long long)ext * ext;
        v = band[((row / E2) * Ob + ob) * e2p + front + row % E2];
      } else if (tw > 0) {
        const long long L = row / ext;
        const int i = int(row % ext);
        v = band[(L * Ob + ob) * tw + padl + i];
      } else {
        v = band[(long long)ob * Sp + row];
      }
    }
    full[e] = v;
  }
}
}  // namespace

void launch_band_expand(cudaStream_t s, int dim, int degree, int ext, long long S, int Ob, long long Sp, int tw,
                        int front, int e2p, const double* band_patch, double* full) {
  const int W = 2 * degree + 1;
  const int O = dim == 2 ? W * W : W * W * W;
  band_expand_kernel<<<148 * 8, 256, 0, s>>>(band_patch, full, dim, degree, ext, S, O, Ob, Sp, tw, front, e2p);
}

long long spmv_sweep_band_doubles(int dim, int degree, int ext, long long S, int K, bool half, int sweep) {
  SweepCfg g;
  size_t smem;
  if (!sweep_cfg(dim, degree, ext, S, K, half, sweep, &g, &smem)) return 0;
  const int W = 2 * degree + 1;
  return (long long)K * ext * (degree * W + degree + 1) * g.tw;
}

void spmv_sweep_scratch(int dim, int degree, int ext, long long S, int K, bool half, int sweep, long long* doubles,
                        long long* flags) {
  SweepCfg g;
  size_t smem;
  *doubles = *flags = 0;
  if (!sweep_cfg(dim, degree, ext, S, K, half, sweep, &g, &smem)) return;
  *flags = (long long)g.segs * K;
  *doubles = *flags * degree * ext;
}

void launch_sweep_relayout(cudaStream_t s, int degree, int ext, long long S, int K, long long Sp, const double* src,
                           double* dst) {
  SweepCfg g;
  size_t smem;
  if (!sweep_cfg(2, degree, ext, S, K, true, 1, &g, &smem)) return;
  switch (degree) {
    case 1: sweep_relayout_kernel<1><<<1184, 256, 0, s>>>(src, dst, ext, K, Sp, g.tw); break;
    case 2: sweep_relayout_kernel<2><<<1184, 256, 0, s>>>(src, dst, ext, K, Sp, g.tw); break;
    case 3: sweep_relayout_kernel<3><<<1184, 256, 0, s>>>(src, dst, ext, K, Sp, g.tw); break;
    case 4: sweep_relayout_kernel<4><<<1184, 256, 0, s>>>(src, dst, ext, K, Sp, g.tw); break;
  }
}

// 3D plane-sweep configuration of one level: in-plane tiles and plane
// segments so that the CTAs fill the GPU in one wave (one CTA per SM: the
// consumers hold ~90 registers and a deep ring keeps enough band bytes in
// flight), with the least re-read band (halo rows |s_in| / T, tail planes
// ~1.7 / zlen); the ring depth from the shared-memory budget.  sweep3 = the
// shortest lattice axis swept (PMG_SWEEP3D at context creation; 0 disables).
static bool sweep3_cfg(int dim, int degree, int ext, long long S, int K, bool half, int sweep3, Sweep3Cfg* out,
                       size_t* smem_out) {
  if (sweep3 <= 0 || dim != 3 || !half || (degree != 2 && degree != 3) || ext < sweep3 || ext < 4 * degree)
    return false;
  (void)S;
  const long long E2 = (long long)ext * ext;
  const int H = degree * (1 + ext);
  const int sms = sm_count();
  const size_t budget = 227 * 1024 - 2048;
  double best = 1e30;
  bool found = false;
  // experiments: PMG_SWEEP3_TILES / PMG_SWEEP3_ZSEGS pin the in-plane tiles / plane segments
  // (levels with ext >= 48; PMG_SWEEP3_TILES_C / PMG_SWEEP3_ZSEGS_C the coarser ones)
  static const int pin_t = env_int("PMG_SWEEP3_TILES", 0), pin_z = env_int("PMG_SWEEP3_ZSEGS", 0);
  static const int pin_tc = env_int("PMG_SWEEP3_TILES_C", 0), pin_zc = env_int("PMG_SWEEP3_ZSEGS_C", 0);
  const int pin_tiles = ext >= 48 ? pin_t : pin_tc, pin_zsegs = ext >= 48 ? pin_z : pin_zc;
  for (int tiles = 1; tiles <= 32; ++tiles) {
    if (pin_tiles > 0 && tiles != pin_tiles) continue;
    const int T = int((E2 + tiles - 1) / tiles);
    if (T < 96) break;
    const int rpt = (T + kSweep3Nc - 1) / kSweep3Nc;
    if (rpt > kSweep3MaxRpt) continue;
    const int tpad = rpt * kSweep3Nc;
    const int sd = (tpad + H + 5) & ~1;
    const int xd = (tpad + 2 * H + 5) & ~1;
    const size_t xbytes = size_t(degree + 3) * xd * sizeof(double);
    if (xbytes + 4 * size_t(sd) * sizeof(double) > budget) continue;
    static const int ns_cap = env_int("PMG_SWEEP3_NS", kSweep3MaxStages);  // ring depth cap (experiments)
    const int ns = int(std::min<size_t>(std::min(kSweep3MaxStages, ns_cap),
                                        (budget - xbytes) / (size_t(sd) * sizeof(double))));
    for (int zsegs = 1; zsegs <= 16; ++zsegs) {
      if (pin_zsegs > 0 && zsegs != pin_zsegs) continue;
      const int zlen = (ext + zsegs - 1) / zsegs;
      if (zlen < 2 * degree) break;
      const int nz = (ext + zlen - 1) / zlen;
      const long long ctas = (long long)K * tiles * nz;
      if (ctas > sms) break;  // one wave: CTAs run start to end
      const double fill = std::min(1.0, double(ctas) / (0.9 * sms));
      // fitted to c4's finest level (K = 8, ext = 67; tiles x segments, ms per launch): 3 x 6 0.598,
      // 4 x 4 0.668, 6 x 3 0.849, 4 x 3 0.869, 9 x 2 1.183, 12 x 1 2.150 -- the in-plane halo costs about
      // twice its rows (band rows and x window re-read by the neighbouring tile, shorter bulk copies)
      const double cost = (double(tpad) / T + 2.0 * H / T) * (1.0 + (nz > 1 ? 1.7 / zlen : 0.0)) / fill;
      if (cost < best) {
        best = cost;
        found = true;
        out->tiles = tiles;
        out->T = T;
        out->zsegs = nz;
        out->zlen = zlen;
        out->rpt = rpt;
        out->ns = ns;
        out->sd = sd;
        out->xd = xd;
        out->halo = H;
        // zero pads: reads reach in-plane indices [-H - 1, ta + tpad + H], ta + tpad <= E2 + tiles + NC
        out->front = (H + 3) & ~1;
        out->e2p = (out->front + int(E2) + H + kSweep3Nc + tiles + 8) & ~1;
        *smem_out = size_t(ns) * sd * sizeof(double) + xbytes;
      }
    }
  }
  // a level whose best sweep still re-reads or idles this much (few patches
  // of a small lattice: c4 level 4 ran at 0.18 of HBM, c5 level 4 at 0.57) is
  // served as well or better by the 256-row half-band kernel (0.58 at c5 level 4)
  // (an explicit PMG_SWEEP3D threshold -- the parity tests -- sweeps every level that qualifies)
  static const int cost_cap = env_int("PMG_SWEEP3_COST_PCT", std::getenv("PMG_SWEEP3D") ? 1000000 : 170);
  return found && best <= 0.01 * cost_cap;
}

template <int P>
void launch_sweep3(cudaStream_t s, const SpmvArgs& a, const Sweep3Cfg& g, size_t smem) {
  const dim3 grid(unsigned(a.K * g.tiles * g.zsegs)), block(kSweep3Nc + 32 * kSweep3Pw);
#define PMG_SWEEP3_CASE(R)                                                      \
  if (g.rpt == R) {                                                             \
    ensure_smem((const void*)spmv_sweep3d_kernel<P, R>, smem);                  \
    launch_k(spmv_sweep3d_kernel<P, R>, grid, block, smem, s, a, g);            \
    return;                                                                     \
  }
  PMG_SWEEP3_CASE(1) PMG_SWEEP3_CASE(2) PMG_SWEEP3_CASE(3) PMG_SWEEP3_CASE(4)
#undef PMG_SWEEP3_CASE
}

namespace {
// offset-major [K][OB][Sp] -> plane-major [K][ext][OB][e2p] with zero pads
__global__ void sweep3_relayout_kernel(const double* __restrict__ src, double* __restrict__ dst, int ext, int K,
                                       int OB, long long Sp, int front, int e2p) {
  const long long E2 = (long long)ext * ext;
  const long long n = (long long)K * ext * OB * e2p;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = int(e % e2p);
    const long long t = e / e2p;
    const int o = int(t % OB);
    const long long kz = t / OB;
    const int z = int(kz % ext);
    const long long k = kz / ext;
    const long long i = c - front;
    dst[e] = (i >= 0 && i < E2) ? src[((size_t)k * OB + o) * Sp + (size_t)z * E2 + i] : 0.0;
  }
}
}  // namespace

long long spmv_sweep3_band_doubles(int dim, int degree, int ext, long long S, int K, bool half, int sweep3,
                                   int* front, int* e2p) {
  Sweep3Cfg g;
  size_t smem;
  if (!sweep3_cfg(dim, degree, ext, S, K, half, sweep3, &g, &smem)) return 0;
  const int W = 2 * degree + 1;
  *front = g.front;
  *e2p = g.e2p;
  return (long long)K * ext * ((W * W * W + 1) / 2) * g.e2p;
}

void launch_sweep3_relayout(cudaStream_t s, int degree, int ext, long long S, int K, long long Sp, const double* src,
                            double* dst) {
  Sweep3Cfg g;
  size_t smem;
  if (!sweep3_cfg(3, degree, ext, S, K, true, 1, &g, &smem)) return;
  const int W = 2 * degree + 1;
  sweep3_relayout_kernel<<<148 * 8, 256, 0, s>>>(src, dst, ext, K, (W * W * W + 1) / 2, Sp, g.front, g.e2p);
}

static int ext_of(int dim, long long S) {
  long long e = 1;
  if (dim == 2) {
    while (e * e < S) ++e;
  } else {
    while (e * e * e < S) ++e;
  }
  return int(e);
}

int spmv_partials(int dim, int degree, long long S, int K, bool half, int sweep, int sweep3) {
  SweepCfg g;
  size_t smem;
  if (dim == 2 && sweep_cfg(dim, degree, ext_of(dim, S), S, K, half, sweep, &g, &smem)) return g.segs * K;
  Sweep3Cfg g3;
  if (dim == 3 && sweep3_cfg(dim, degree, ext_of(dim, S), S, K, half, sweep3, &g3, &smem))
    return K * g3.tiles * g3.zsegs;
  if (spmv_tma_level(dim, degree, S)) return int((S + kRowsTma - 1) / kRowsTma * K);
  return spmv_blocks(S * K);
}

void launch_spmv(cudaStream_t s, const SpmvArgs& a) {
  SweepCfg g;
  size_t smem;
  if (sweep_cfg(a.dim, a.degree, a.ext, a.S, a.K, a.half != 0, a.sweep, &g, &smem)) {
    switch (a.degree) {
      case 1: launch_sweep<1>(s, a, g, smem); return;
      case 2: launch_sweep<2>(s, a, g, smem); return;
      case 3: launch_sweep<3>(s, a, g, smem); return;
      case 4: launch_sweep<4>(s, a, g, smem); return;
    }
  }
  Sweep3Cfg g3;
  if (sweep3_cfg(a.dim, a.degree, a.ext, a.S, a.K, a.half != 0, a.sweep3, &g3, &smem)) {
    switch (a.degree) {
      case 2: launch_sweep3<2>(s, a, g3, smem); return;
      case 3: launch_sweep3<3>(s, a, g3, smem); return;
    }
  }
  if (spmv_tma_level(a.dim, a.degree, a.S)) {
#define PMG_TMA_CASE(D, P) \
  if (a.dim == D && a.degree == P) { launch_tma<D, P>(s, a); return; }
    PMG_TMA_CASE(2, 1) PMG_TMA_CASE(2, 2) PMG_TMA_CASE(2, 3) PMG_TMA_CASE(2, 4)
    PMG_TMA_CASE(2, 5) PMG_TMA_CASE(2, 6) PMG_TMA_CASE(2, 8)
    PMG_TMA_CASE(3, 1) PMG_TMA_CASE(3, 2) PMG_TMA_CASE(3, 3) PMG_TMA_CASE(3, 4)
#undef PMG_TMA_CASE
  }
  const int grid = spmv_blocks(a.S * a.K);
  if (grid == 0) return;
#define PMG_SPMV_CASE(D, P) \
  if (a.dim == D && a.degree == P) { launch_k(spmv_kernel<D, P>, dim3(grid), dim3(kThreads), 0, s, a); return; }
  PMG_SPMV_CASE(2, 1) PMG_SPMV_CASE(2, 2) PMG_SPMV_CASE(2, 3) PMG_SPMV_CASE(2, 4)
  PMG_SPMV_CASE(2, 5) PMG_SPMV_CASE(2, 6) PMG_SPMV_CASE(2, 8)
  PMG_SPMV_CASE(3, 1) PMG_SPMV_CASE(3, 2) PMG_SPMV_CASE(3, 3) PMG_SPMV_CASE(3, 4)
#undef PMG_SPMV_CASE
  launch_k(spmv_generic_kernel, dim3(grid), dim3(kThreads), 0, s, a);
}

}  // namespace pmgcu
