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

#include "internal.cuh"

namespace pmgcu {

namespace {

template <int D, int P>
__global__ void __launch_bounds__(kThreads) spmv_kernel(SpmvArgs a) {
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
#pragma unroll
    for (int d2 = (D == 3 ? -P : 0); d2 <= (D == 3 ? P : 0); ++d2) {
      const bool ok2 = D == 2 || (i2 + d2 >= 0 && i2 + d2 < ext);
#pragma unroll
      for (int d1 = -P; d1 <= P; ++d1) {
        const bool ok1 = ok2 && (i1 + d1 >= 0 && i1 + d1 < ext);
#pragma unroll
        for (int d0 = -P; d0 <= P; ++d0) {
          const int o = (d0 + P) + W * ((d1 + P) + W * (D == 3 ? d2 + P : 0));
          const long long off = d0 + (long long)ext * d1 + ext2 * d2;
          if (ok1 && i0 + d0 >= 0 && i0 + d0 < ext) acc = fma(__ldcs(band + (size_t)o * S), __ldg(x + off), acc);
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

// Runtime-degree fallback (degrees without a specialisation).
__global__ void __launch_bounds__(kThreads) spmv_generic_kernel(SpmvArgs a) {
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
// Large levels: the band is laid out [K][O][Sp] with Sp = S rounded up to 256,
// so each (offset, 256-row chunk) is one aligned 2 KB segment.  A producer
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
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int D, int P>
__global__ void __launch_bounds__(kRowsTma + 32) spmv_tma_kernel(SpmvArgs a, long long Sp) {
  constexpr int W = 2 * P + 1;
  constexpr int O = D == 2 ? W * W : W * W * W;
  constexpr int NCHUNK = O / W;
  constexpr unsigned kStageBytes = W * kRowsTma * sizeof(double);
  extern __shared__ __align__(128) double ring[];  // [kStages][W][kRowsTma]
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ double red[kRowsTma / 32];

  const long long chunks_per_patch = Sp / kRowsTma;
  const long long k = blockIdx.x / chunks_per_patch;
  const long long r0 = (blockIdx.x - k * chunks_per_patch) * kRowsTma;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRowsTma / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
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
    asm volatile("bar.sync 1, %0;\n" ::"n"(kRowsTma));
    if (tid == 0) {
      double sum = 0.0;
      for (int w = 0; w < kRowsTma / 32; ++w) sum += red[w];
      a.dot_partial[blockIdx.x] = sum;
    }
  }
}

template <int D, int P>
bool launch_tma(cudaStream_t s, const SpmvArgs& a, long long Sp) {
  constexpr int W = 2 * P + 1;
  const size_t smem = (size_t)kStages * W * kRowsTma * sizeof(double);
  static bool configured = false;  // per process; one device per context thread
  if (!configured) {
    cudaFuncSetAttribute(spmv_tma_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    configured = true;
  }
  const long long grid = (Sp / kRowsTma) * a.K;
  spmv_tma_kernel<D, P><<<unsigned(grid), kRowsTma + 32, smem, s>>>(a, Sp);
  return true;
}

}  // namespace

long long spmv_padded_rows(int dim, int degree, long long S) {
  const bool tma = S >= 1024 && ((dim == 2 && degree >= 1 && degree <= 8 && degree != 7) ||
                                 (dim == 3 && degree >= 1 && degree <= 4));
  return tma ? (S + kRowsTma - 1) / kRowsTma * kRowsTma : S;
}

int spmv_blocks(long long rows) { return int((rows + kThreads - 1) / kThreads); }

int spmv_partials(int dim, int degree, long long S, int K) {
  const long long Sp = spmv_padded_rows(dim, degree, S);
  if (Sp != S) return int((Sp / kRowsTma) * K);
  return spmv_blocks(S * K);
}

void launch_spmv(cudaStream_t s, const SpmvArgs& a) {
  const long long Sp = spmv_padded_rows(a.dim, a.degree, a.S);
  if (Sp != a.S) {
#define PMG_TMA_CASE(D, P) \
  if (a.dim == D && a.degree == P) { launch_tma<D, P>(s, a, Sp); return; }
    PMG_TMA_CASE(2, 1) PMG_TMA_CASE(2, 2) PMG_TMA_CASE(2, 3) PMG_TMA_CASE(2, 4)
    PMG_TMA_CASE(2, 5) PMG_TMA_CASE(2, 6) PMG_TMA_CASE(2, 8)
    PMG_TMA_CASE(3, 1) PMG_TMA_CASE(3, 2) PMG_TMA_CASE(3, 3) PMG_TMA_CASE(3, 4)
#undef PMG_TMA_CASE
  }
  const int grid = spmv_blocks(a.S * a.K);
  if (grid == 0) return;
#define PMG_SPMV_CASE(D, P) \
  if (a.dim == D && a.degree == P) { spmv_kernel<D, P><<<grid, kThreads, 0, s>>>(a); return; }
  PMG_SPMV_CASE(2, 1) PMG_SPMV_CASE(2, 2) PMG_SPMV_CASE(2, 3) PMG_SPMV_CASE(2, 4)
  PMG_SPMV_CASE(2, 5) PMG_SPMV_CASE(2, 6) PMG_SPMV_CASE(2, 8)
  PMG_SPMV_CASE(3, 1) PMG_SPMV_CASE(3, 2) PMG_SPMV_CASE(3, 3) PMG_SPMV_CASE(3, 4)
#undef PMG_SPMV_CASE
  spmv_generic_kernel<<<grid, kThreads, 0, s>>>(a);
}

}  // namespace pmgcu
