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

template <int D, int P>
void launch_tma(cudaStream_t s, const SpmvArgs& a) {
  constexpr int W = 2 * P + 1;
  const long long grid = (a.S + kRowsTma - 1) / kRowsTma * a.K;
  if (a.half) {
    const size_t smem = (size_t)kStages * (W * kSeg + (kHalfXWindow ? XWindow<P>::kLen : 0)) * sizeof(double);
    static bool configured = false;  // per process; one device per context thread
    if (!configured) {
      cudaFuncSetAttribute(spmv_tma_half_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      configured = true;
    }
    launch_k(spmv_tma_half_kernel<D, P>, dim3(unsigned(grid)), dim3(kRowsTma + 32), smem, s, a);
    return;
  }
  const size_t smem = (size_t)kStages * W * kRowsTma * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(spmv_tma_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    configured = true;
  }
  launch_k(spmv_tma_kernel<D, P>, dim3(unsigned(grid)), dim3(kRowsTma + 32), smem, s, a);
}

}  // namespace

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

int spmv_partials(int dim, int degree, long long S, int K) {
  if (spmv_tma_level(dim, degree, S)) return int((S + kRowsTma - 1) / kRowsTma * K);
  return spmv_blocks(S * K);
}

void launch_spmv(cudaStream_t s, const SpmvArgs& a) {
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
