// DMMA + shared-memory fragment probe: what bounds the fast-diagonalization
// inner loop on a B200?  Every warp runs k-steps of (WM A-fragment LDS, NTC
// B-fragment LDS, WM x NTC DMMA) from a shared-memory tile that is never
// reloaded (no global traffic), for several shapes and occupancies.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fd_probe fd_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// MODE 0: A and B fragments from shared memory, double-buffered registers
// MODE 1: fragments from registers only (no LDS)
// MODE 2: like 0, fragments prefetched two k-steps ahead (3 register buffers)
template <int NTC, int WM, int MODE>
__global__ void probe(double* out, int ksteps, int iters) {
  extern __shared__ double sm[];
  constexpr int BS = (8 * NTC + 11) / 16 * 16 + 4;
  constexpr int XS = 68;
  const int KS = 16;  // k-steps held in shared memory (64 k)
  double* Bs = sm;                 // [64][BS]
  double* Xs = sm + 64 * BS;       // [warps * 8 * WM][XS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  for (int i = tid; i < 64 * BS; i += blockDim.x) Bs[i] = 1e-3 * (i % 7);
  for (int i = tid; i < (blockDim.x / 32) * 8 * WM * XS; i += blockDim.x) Xs[i] = 1e-3 * (i % 5);
  __syncthreads();
  double acc[WM][NTC][2];
#pragma unroll
  for (int u = 0; u < WM; ++u)
#pragma unroll
    for (int j = 0; j < NTC; ++j) acc[u][j][0] = acc[u][j][1] = 0.0;
  const double* xs = Xs + (warp * 8 * WM + g) * XS + t;
  const double* bs = Bs + t * BS + g;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1) {
      double a = 1e-3 * lane, b = 1.0 - 1e-3 * lane;
      for (int ks = 0; ks < ksteps; ++ks)
#pragma unroll
        for (int j = 0; j < NTC; ++j)
#pragma unroll
          for (int u = 0; u < WM; ++u) dmma(acc[u][j][0], acc[u][j][1], a, b);
    } else if (MODE == 0) {
      double af[2][WM], bf[2][NTC];
#pragma unroll
      for (int u = 0; u < WM; ++u) af[0][u] = xs[u * 8 * XS];
#pragma unroll
      for (int j = 0; j < NTC; ++j) bf[0][j] = bs[j * 8];
#pragma unroll 2
      for (int ks = 0; ks < ksteps; ++ks) {
        const int c = ks & 1;
        const int kn = (ks + 1) % KS;
#pragma unroll
        for (int u = 0; u < WM; ++u) af[c ^ 1][u] = xs[u * 8 * XS + kn * 4];
#pragma unroll
        for (int j = 0; j < NTC; ++j) bf[c ^ 1][j] = bs[kn * 4 * BS + j * 8];
#pragma unroll
        for (int j = 0; j < NTC; ++j)
#pragma unroll
          for (int u = 0; u < WM; ++u) dmma(acc[u][j][0], acc[u][j][1], af[c][u], bf[c][j]);
      }
    } else {
      double af[3][WM], bf[3][NTC];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
#pragma unroll
        for (int u = 0; u < WM; ++u) af[q][u] = xs[u * 8 * XS + q * 4];
#pragma unroll
        for (int j = 0; j < NTC; ++j) bf[q][j] = bs[q * 4 * BS + j * 8];
      }
#pragma unroll 3
      for (int ks = 0; ks < ksteps; ++ks) {
        const int c = ks % 3, cn = (ks + 2) % 3;
        const int kn = (ks + 2) % KS;
#pragma unroll
        for (int u = 0; u < WM; ++u) af[cn][u] = xs[u * 8 * XS + kn * 4];
#pragma unroll
        for (int j = 0; j < NTC; ++j) bf[cn][j] = bs[kn * 4 * BS + j * 8];
#pragma unroll
        for (int j = 0; j < NTC; ++j)
#pragma unroll
          for (int u = 0; u < WM; ++u) dmma(acc[u][j][0], acc[u][j][1], af[c][u], bf[c][j]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < WM; ++u)
#pragma unroll
    for (int j = 0; j < NTC; ++j) s += acc[u][j][0] + acc[u][j][1];
  if (s == 12345.678) out[0] = s;
}

template <int NTC, int WM, int MODE>
void run(const char* name, int warps, int ctas_per_sm, double* d, int sms) {
  constexpr int BS = (8 * NTC + 11) / 16 * 16 + 4;
  const size_t smem = sizeof(double) * (64 * BS + size_t(warps) * 8 * WM * 68);
  cudaFuncSetAttribute(probe<NTC, WM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe<NTC, WM, MODE>, warps * 32, smem);
  if (occ < ctas_per_sm) {
    printf("%-10s NTC=%2d WM=%d warps=%2d ctas/SM=%d  (occupancy %d, skipped)\n", name, NTC, WM, warps, ctas_per_sm, occ);
    return;
  }
  const int ksteps = 64, iters = 200;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dim3 grid(sms * ctas_per_sm), block(warps * 32);
  probe<NTC, WM, MODE><<<grid, block, smem>>>(d, ksteps, 2);
  cudaEventRecord(e0);
  probe<NTC, WM, MODE><<<grid, block, smem>>>(d, ksteps, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 512.0 * NTC * WM * double(ksteps) * iters * grid.x * warps;
  printf("%-10s NTC=%2d WM=%d warps=%2d ctas/SM=%d  %6.2f TFLOP/s  %s\n", name, NTC, WM, warps, ctas_per_sm,
         flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
#define ROW(NTC, WM)                                             \
  run<NTC, WM, 1>("regs", 4, 4, d, sms);                         \
  run<NTC, WM, 1>("regs", 8, 1, d, sms);                         \
  run<NTC, WM, 0>("lds", 4, 1, d, sms);                          \
  run<NTC, WM, 0>("lds", 4, 2, d, sms);                          \
  run<NTC, WM, 0>("lds", 4, 4, d, sms);                          \
  run<NTC, WM, 0>("lds", 8, 1, d, sms);                          \
  run<NTC, WM, 0>("lds", 8, 2, d, sms);                          \
  run<NTC, WM, 0>("lds", 12, 1, d, sms);                         \
  run<NTC, WM, 0>("lds", 16, 1, d, sms);                         \
  run<NTC, WM, 2>("lds-pf2", 4, 4, d, sms);                      \
  run<NTC, WM, 2>("lds-pf2", 8, 1, d, sms);                      \
  run<NTC, WM, 2>("lds-pf2", 12, 1, d, sms);                     \
  run<NTC, WM, 2>("lds-pf2", 16, 1, d, sms);
  ROW(9, 1)
  ROW(11, 1)
  ROW(5, 1)
  ROW(9, 2)
  ROW(5, 2)
  ROW(3, 4)
  return 0;
}
