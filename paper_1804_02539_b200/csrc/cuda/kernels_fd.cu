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
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#include "internal.cuh"
#include "pieces.cuh"

namespace pmgcu {

namespace {

constexpr int kBK = 16;        // k per shared-memory stage
constexpr int kXS = kBK + 4;   // X row stride (doubles): conflict-free A fragments

// CTA = NW warps, warp w owns the 8 rows 8w..8w+7 of an 8 NW-row panel and all
// NTC n-tiles (8 columns each) of the CTA's column panel; K streams through a
// STAGES-deep cp.async ring.  B row stride = 4 mod 16 doubles so the 4 x 8
// B-fragment reads of a half-warp hit distinct banks.
//   <NTC, 4, 3>, 4 CTAs per SM: 32 x 8 NTC tiles, many CTAs (small levels, 3D)
//   <NTC, 8, 4>, 2 CTAs per SM: 64 x 8 NTC tiles
//   <NTC, 11, 5>, 1 CTA per SM: 88 x 8 NTC tiles -- at c2's finest level
//       (4128 rows x 258 columns per pass) 47 x 3 = 141 equal CTAs on 148 SMs,
//       264 padded columns instead of 288, and 0.39x the L2 -> SM operand bytes
//       per flop of the 32 x 72 tile
template <int NTC, int NW, int STAGES>
struct FdTile {
  static constexpr int Threads = 32 * NW;
  static constexpr int BM = 8 * NW;
  static constexpr int XPer = BM * kBK / Threads;  // = 4
  static constexpr int XRowStep = Threads / kBK;   // X rows covered by one copy round
  static constexpr int BN = 8 * NTC;
  static constexpr int BS = (BN + 11) / 16 * 16 + 4;
  static constexpr int BPer = (kBK * BN + Threads - 1) / Threads;
  static constexpr size_t smem = sizeof(double) * STAGES * (BM * kXS + kBK * BS);
};

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

// store of one 8-row fragment row set (see the kernel's epilogue comment)
template <int NTC>
__device__ __forceinline__ void fd_epilogue(const FdPiece& P, long long rl, const double (&acc)[NTC][2], int n0, int N,
                                            int t, int naxes, int m0, long long ext, long long ext2, long long R,
                                            int out_mode, double alpha, double* __restrict__ lat_out,
                                            double* __restrict__ work_out) {
  long long lat_row = 0;
  if (out_mode >= FD_OUT_LATTICE_SET) lat_row = P.lat_base + (naxes == 3 ? (rl % m0) + ext * (rl / m0) : rl);
  const long long lat_stride = naxes == 3 ? ext2 : ext;
  double* __restrict__ wout = work_out + P.work_off;
  const double* __restrict__ diag = P.diag;
  // epilogues that read global data issue all their loads first, so the
  // lane's 2 NTC reads are in flight together (one round trip, not 2 NTC)
  if (out_mode == FD_OUT_WORK_DIAG || out_mode == FD_OUT_LATTICE_ADD) {
    double ld[NTC][2];
#pragma unroll
    for (int j = 0; j < NTC; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int n = n0 + j * 8 + 2 * t + i;
        const int nn = n < N ? n : N - 1;
        ld[j][i] = out_mode == FD_OUT_WORK_DIAG ? diag[rl + R * nn] : lat_out[lat_row + lat_stride * nn];
      }
#pragma unroll
    for (int j = 0; j < NTC; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int n = n0 + j * 8 + 2 * t + i;
        if (n >= N) continue;
        if (out_mode == FD_OUT_WORK_DIAG)
          wout[rl + R * n] = acc[j][i] / ld[j][i];
        else
          lat_out[lat_row + lat_stride * n] = ld[j][i] + alpha * acc[j][i];
      }
    return;
  }
#pragma unroll
  for (int j = 0; j < NTC; ++j) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int n = n0 + j * 8 + 2 * t + i;
      if (n >= N) continue;
      const double v = acc[j][i];
      if (out_mode == FD_OUT_WORK)
        wout[rl + R * n] = v;
      else
        lat_out[lat_row + lat_stride * n] = alpha * v;
    }
  }
}

// One pass over a group of pieces with the same dims and the same factor B
// (pieces are independent; a group's rows are concatenated so the M
// dimension has no per-piece padding).  item = (first piece of the group,
// first row of the panel within the group, first column, rows of the group).
template <int NTC, int NW, int STAGES, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB) fd_pass_dmma_kernel(const FdPiece* __restrict__ pieces,
                                                                     const int4* __restrict__ items, int pass,
                                                                     int naxes, int in_mode, int out_mode,
                                                                     const double* __restrict__ lat_in,
                                                                     double* __restrict__ lat_out, double alpha,
                                                                     const double* __restrict__ work_in,
                                                                     double* __restrict__ work_out) {
  PMG_PDL_ENTRY();
  using T = FdTile<NTC, NW, STAGES>;
  extern __shared__ __align__(16) double fd_smem[];  // Xs[STAGES][BM * kXS], Bs[STAGES][kBK * BS]
  auto Xs = reinterpret_cast<double(*)[T::BM * kXS]>(fd_smem);
  auto Bs = reinterpret_cast<double(*)[kBK * T::BS]>(fd_smem + STAGES * T::BM * kXS);
  const int4 it = items[blockIdx.x];
  const FdPiece& P0 = pieces[it.x];
  const int axis = pass % naxes;
  const int dir = pass / naxes;
  const int K = P0.dims[axis];
  const int N = K;
  const long long R = P0.total / K;  // rows per piece
  const long long rows = it.w;       // rows of the group
  const long long r0 = it.y;
  const int n0 = it.z;
  const int m0 = P0.dims[0], m1 = P0.dims[1];
  const long long ext = P0.ext, ext2 = (long long)P0.ext * P0.ext;
  const double* __restrict__ B = P0.B[axis][dir];
  const int tid = threadIdx.x;

  // per-thread copy plan: X element (rr, kk) = (tid/16 + XRowStep j, tid%16); B
  // element (kk, nn) of idx = tid + Threads j
  const int xk = tid % kBK;
  const double* xsrc[T::XPer];
  bool xrow_ok[T::XPer];
#pragma unroll
  for (int j = 0; j < T::XPer; ++j) {
    const long long r = r0 + tid / kBK + T::XRowStep * j;
    xrow_ok[j] = r < rows;
    const long long rg = xrow_ok[j] ? r : 0;
    const FdPiece& P = pieces[it.x + int(rg / R)];
    const long long rr = rg % R;
    if (in_mode == FD_IN_WORK)
      xsrc[j] = work_in + P.work_off + rr * K + xk;
    else
      xsrc[j] = lat_in + P.lat_base + (naxes == 3 ? ext * (rr % m1) + ext2 * (rr / m1) : ext * rr) + xk;
  }
  int boff[T::BPer], bkk[T::BPer], bdst[T::BPer];
  bool bn_ok[T::BPer];
#pragma unroll
  for (int j = 0; j < T::BPer; ++j) {
    const int idx = tid + T::Threads * j;
    const int nn = idx % T::BN, kk = idx / T::BN;
    bn_ok[j] = n0 + nn < N && kk < kBK;
    bkk[j] = kk;
    boff[j] = kk * N + n0 + nn;
    bdst[j] = kk * T::BS + nn;
  }
  auto load = [&](int stage, int k0) {
    double* xs = Xs[stage];
    double* bs = Bs[stage];
#pragma unroll
    for (int j = 0; j < T::XPer; ++j) {
      const bool ok = xrow_ok[j] && k0 + xk < K;
      cp_async8(xs + (tid / kBK + T::XRowStep * j) * kXS + xk, ok ? xsrc[j] + k0 : B, ok);
    }
#pragma unroll
    for (int j = 0; j < T::BPer; ++j) {
      if (bkk[j] >= kBK) continue;
      const bool ok = bn_ok[j] && k0 + bkk[j] < K;
      cp_async8(bs + bdst[j], ok ? B + boff[j] + (long long)k0 * N : B, ok);
    }
  };

  // epilogues that read global data (the diagonal, or u for u += tau z) pull
  // their lines into L2 now, so the reads after the main loop hit L2: per
  // column, the panel's BM rows are 8 BM contiguous bytes (within one piece)
  if (out_mode == FD_OUT_WORK_DIAG || out_mode == FD_OUT_LATTICE_ADD) {
    constexpr int LPC = T::BM / 16 + 1;  // 128-byte lines per column
    const long long rl0 = r0 % R;
    const FdPiece& Pf = pieces[it.x + int(r0 / R)];
    for (int idx = tid; idx < LPC * T::BN; idx += T::Threads) {
      const int n = n0 + idx / LPC;
      const long long dr = min((long long)16 * (idx % LPC), R - 1 - rl0);  // stay inside the piece
      if (n >= N) continue;
      const double* a;
      if (out_mode == FD_OUT_WORK_DIAG) {
        a = Pf.diag + rl0 + dr + R * n;
      } else {
        const long long rl = rl0 + dr;
        const long long lr = naxes == 3 ? (rl % m0) + ext * (rl / m0) : rl;
        a = lat_out + Pf.lat_base + lr + (naxes == 3 ? ext2 : ext) * n;
      }
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a));
    }
  }

  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  double acc[NTC][2];
#pragma unroll
  for (int j = 0; j < NTC; ++j) acc[j][0] = acc[j][1] = 0.0;

  const int nst = (K + kBK - 1) / kBK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nst) load(s, s * kBK);
    cp_async_commit();
  }
  for (int s = 0; s < nst; ++s) {
    const int cur = s % STAGES;
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch stage s + STAGES - 1 into the slot freed at s - 1
      const int nxt = s + STAGES - 1;
      if (nxt < nst) load(nxt % STAGES, nxt * kBK);
      cp_async_commit();
    }
    // warp w owns rows 8 w .. 8 w + 7 of the panel
    const double* xs = Xs[cur] + (warp * 8 + g) * kXS + t;
    const double* bs = Bs[cur] + t * T::BS + g;
    // fragments of k-step ks + 1 are read while k-step ks multiplies
    double af[2], bf[2][NTC];
    af[0] = xs[0];
#pragma unroll
    for (int j = 0; j < NTC; ++j) bf[0][j] = bs[j * 8];
    // k-steps of 4 that hold rows of B (the last stage of a pass is short)
    const int nks = min(kBK / 4, (K - s * kBK + 3) / 4);
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      if (ks >= nks) break;
      const int c = ks & 1;
      if (ks + 1 < kBK / 4) {
        af[c ^ 1] = xs[(ks + 1) * 4];
#pragma unroll
        for (int j = 0; j < NTC; ++j) bf[c ^ 1][j] = bs[(ks + 1) * 4 * T::BS + j * 8];
      }
#pragma unroll
      for (int j = 0; j < NTC; ++j) dmma(acc[j][0], acc[j][1], af[c], bf[c][j]);
    }
  }

  // epilogue: lane holds row r0 + 8 w + g of the group, columns
  // n0+8j+2t+{0,1}; within its piece, Y(rl, n) at rl + R n
  const long long r = r0 + warp * 8 + g;
  if (r < rows)
    fd_epilogue<NTC>(pieces[it.x + int(r / R)], r % R, acc, n0, N, t, naxes, m0, ext, ext2, R, out_mode, alpha,
                     lat_out, work_out);
}

// ---------------------------------------------------------------- short contractions
// Passes with K = N <= 8 NTC (the 3D levels: c4/c5 contract 65-67 entries):
// the factor stays resident.  One persistent CTA per SM loads B once; each of
// its NW warps then works alone -- it takes the next 8-row strip of its
// group from a global counter (so every CTA of a group ends together: with
// static ranges the slowest SM ran 20% behind the average), copies the
// strip's X rows into its own double buffer with cp.async while the previous
// strip multiplies, runs ceil(K / 4) k-steps of NTC DMMAs from shared memory,
// and stores.  No CTA-wide barrier after the prologue, no per-tile pipeline
// fill.  item = (first piece of the group, group index, number of groups,
// rows of the group); queue = one strip counter per group, then the count of
// finished CTAs: the last CTA to finish zeroes the counters for the next
// launch (fd_resident_items shares the SMs out over the groups).
constexpr int kResWarps = 12;  // the strip threshold of fd_pick_cfg

// Row of a group as a warp lane sees it: the piece it lies in, its row there,
// and where that row's input starts / its output goes.  All patch-local
// indices fit 32 bits (a rank's lattice has < 2^31 slots), so the per-strip
// index arithmetic is 32-bit: with 64-bit divisions the strip's ~150 DMMAs
// were outnumbered 10:1 by integer instructions and the pass was issue-bound.
struct ResRow {
  const double* src;  // first input element of the row
  double* dst;        // output element (row, column 0)
  const double* aux;  // reciprocal diagonal of the row (FD_OUT_WORK_DIAG)
};

template <int NTC, int NW>
__global__ void __launch_bounds__(32 * NW, 1) fd_pass_resident_kernel(
    const FdPiece* __restrict__ pieces, const int4* __restrict__ items, unsigned* __restrict__ queue, int pass,
    int naxes, int in_mode, int out_mode, const double* __restrict__ lat_in, double* __restrict__ lat_out,
    double alpha, const double* __restrict__ work_in, double* __restrict__ work_out) {
  PMG_PDL_ENTRY();
  constexpr int BN = 8 * NTC;
  constexpr int BS = (BN + 11) / 16 * 16 + 4;  // = 4 mod 16: conflict-free B fragments
  extern __shared__ __align__(16) double fd_smem[];
  const int4 it = items[blockIdx.x];
  const FdPiece& P0 = pieces[it.x];
  unsigned* const next_strip = queue + it.y;
  const int axis = pass % naxes, dir = pass / naxes;
  const int K = P0.dims[axis];
  const int N = K;
  const int nks = (K + 3) / 4;
  const int Kp = 4 * nks;
  const int XS = (Kp & 7) == 4 ? Kp : Kp + 4;  // = 4 mod 8: conflict-free A fragments
  const int R = int(P0.total / K);             // rows per piece
  const int rows = it.w;
  const int nstrips = (rows + 7) / 8;
  const int m0 = P0.dims[0], m1 = P0.dims[1];
  const int ext = P0.ext, ext2 = P0.ext * P0.ext;
  const int ostride = out_mode >= FD_OUT_LATTICE_SET ? (naxes == 3 ? ext2 : ext) : R;  // output column stride
  const double* __restrict__ B = P0.B[axis][dir];
  double* Bs = fd_smem;                 // [Kp][BS], zero outside K x N
  double* Xall = Bs + (size_t)Kp * BS;  // [NW][2][8][XS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;

  for (int idx = tid; idx < Kp * BS; idx += 32 * NW) {
    const int kk = idx / BS, nn = idx - kk * BS;
    const bool ok = kk < K && nn < N;
    cp_async8(Bs + idx, ok ? B + kk * N + nn : B, ok);
  }
  cp_async_commit();
  double* Xw = Xall + (size_t)warp * 2 * 8 * XS;
  for (int idx = lane; idx < 2 * 8 * XS; idx += 32) Xw[idx] = 0.0;  // the columns >= K stay zero
  __syncthreads();

  // lane (g, t) owns row g of a strip: it copies the row's elements t, t + 4,
  // ... and stores the row's outputs of columns 8 j + 2 t + {0, 1}
  auto locate = [&](int strip) {
    int r = strip * 8 + g;
    if (r >= rows) r = rows - 1;  // a short last strip repeats its last row (never stored)
    const int pi = r / R, rl = r - pi * R;
    const FdPiece& P = pieces[it.x + pi];
    ResRow w;
    if (in_mode == FD_IN_WORK) {
      w.src = work_in + P.work_off + (long long)rl * K;
    } else {
      const int i2 = naxes == 3 ? rl / m1 : 0, i1 = naxes == 3 ? rl - i2 * m1 : rl;
      w.src = lat_in + P.lat_base + (ext * i1 + ext2 * i2);
    }
    if (out_mode >= FD_OUT_LATTICE_SET) {
      const int j1 = naxes == 3 ? rl / m0 : 0, j0 = naxes == 3 ? rl - j1 * m0 : rl;
      w.dst = lat_out + P.lat_base + (j0 + ext * j1);
    } else {
      w.dst = work_out + P.work_off + rl;
    }
    w.aux = P.rdiag + rl;
    return w;
  };
  auto issue = [&](const ResRow& w, double* xb) {
    double* dst = xb + g * XS + t;
    const double* src = w.src + t;
    int k = t;
#pragma unroll 1
    for (; k + 12 < K; k += 16, dst += 16, src += 16) {
      cp_async8(dst, src, true);
      cp_async8(dst + 4, src + 4, true);
      cp_async8(dst + 8, src + 8, true);
      cp_async8(dst + 12, src + 12, true);
    }
    for (; k < K; k += 4, dst += 4, src += 4) cp_async8(dst, src, true);
  };
  // lane 0 takes strips from the group's counter two ahead: the atomic's
  // round trip (about 1 us) is over before its result is broadcast
  unsigned pending = 0;
  auto request = [&]() {
    if (lane == 0) pending = atomicAdd(next_strip, 1u);
  };
  auto take = [&]() {
    const unsigned s = __shfl_sync(0xffffffffu, pending, 0);
    return s < unsigned(nstrips) ? int(s) : nstrips;
  };

  request();
  int cur = take();
  request();
  ResRow wc = locate(cur < nstrips ? cur : 0);
  if (cur < nstrips) issue(wc, Xw);
  cp_async_commit();
  int buf = 0;
  while (cur < nstrips) {
    const int nxt = take();
    request();
    ResRow wn = wc;
    if (nxt < nstrips) {
      wn = locate(nxt);
      issue(wn, Xw + (buf ^ 1) * 8 * XS);
    }
    cp_async_commit();
    // epilogues that read global data pull their lines into L2 during the
    // products: per column the strip's 8 rows are 64 contiguous bytes
    if (out_mode == FD_OUT_WORK_DIAG || out_mode == FD_OUT_LATTICE_ADD) {
      const double* a0 = out_mode == FD_OUT_WORK_DIAG ? wc.aux : wc.dst;
      if (g == 0 || g == 7)  // first and last row: both lines a misaligned strip touches
        for (int n = t; n < N; n += 4) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a0 + (long long)ostride * n));
    }
    cp_async_wait<1>();  // the current strip (and, the first time, B) has landed
    __syncwarp();
    const double* xs = Xw + buf * 8 * XS + g * XS + t;
    const double* bs = Bs + t * BS + g;
    double acc[NTC][2];
#pragma unroll
    for (int j = 0; j < NTC; ++j) acc[j][0] = acc[j][1] = 0.0;
    // k-steps in pairs over two named fragment sets (static register names:
    // a [2][NTC] array indexed by ks & 1 lands in local memory); the fragments
    // of the next k-step are read while the current one multiplies
    double a0 = xs[0], a1 = 0.0, b0[NTC], b1[NTC];
#pragma unroll
    for (int j = 0; j < NTC; ++j) b0[j] = bs[j * 8];
    int ks = 0;
    for (; ks + 1 < nks; ks += 2) {
      a1 = xs[(ks + 1) * 4];
#pragma unroll
      for (int j = 0; j < NTC; ++j) b1[j] = bs[(ks + 1) * 4 * BS + j * 8];
#pragma unroll
      for (int j = 0; j < NTC; ++j) dmma(acc[j][0], acc[j][1], a0, b0[j]);
      if (ks + 2 < nks) {
        a0 = xs[(ks + 2) * 4];
#pragma unroll
        for (int j = 0; j < NTC; ++j) b0[j] = bs[(ks + 2) * 4 * BS + j * 8];
      }
#pragma unroll
      for (int j = 0; j < NTC; ++j) dmma(acc[j][0], acc[j][1], a1, b1[j]);
    }
    if (ks < nks) {
#pragma unroll
      for (int j = 0; j < NTC; ++j) dmma(acc[j][0], acc[j][1], a0, b0[j]);
    }
    if (cur * 8 + g < rows) {
      // Y(row, n) at dst + ostride n, n = 8 j + 2 t + i: two running pointers
      // (columns n and n + 1) stepped by 8 columns, so the per-element address
      // arithmetic is two 64-bit adds per j
      const long long step = (long long)ostride * 8;
      double* o0 = wc.dst + (long long)ostride * (2 * t);
      double* o1 = o0 + ostride;
      const int nrem = N - 2 * t;  // column n = 8 j + 2 t is valid iff 8 j < nrem
      if (out_mode == FD_OUT_WORK) {
#pragma unroll
        for (int j = 0; j < NTC; ++j, o0 += step, o1 += step) {
          if (8 * j < nrem) *o0 = acc[j][0];
          if (8 * j + 1 < nrem) *o1 = acc[j][1];
        }
      } else if (out_mode == FD_OUT_LATTICE_SET) {
#pragma unroll
        for (int j = 0; j < NTC; ++j, o0 += step, o1 += step) {
          if (8 * j < nrem) *o0 = alpha * acc[j][0];
          if (8 * j + 1 < nrem) *o1 = alpha * acc[j][1];
        }
      } else {
        // all loads first (one round trip), then the stores
        const double* q0 = (out_mode == FD_OUT_WORK_DIAG ? wc.aux : wc.dst) + (long long)ostride * (2 * t);
        const double* q1 = q0 + ostride;
        double ld[NTC][2];
#pragma unroll
        for (int j = 0; j < NTC; ++j, q0 += step, q1 += step) {
          ld[j][0] = 8 * j < nrem ? *q0 : 1.0;
          ld[j][1] = 8 * j + 1 < nrem ? *q1 : 1.0;
        }
        if (out_mode == FD_OUT_WORK_DIAG) {  // ld = 1 / diag
#pragma unroll
          for (int j = 0; j < NTC; ++j, o0 += step, o1 += step) {
            if (8 * j < nrem) *o0 = acc[j][0] * ld[j][0];
            if (8 * j + 1 < nrem) *o1 = acc[j][1] * ld[j][1];
          }
        } else {
#pragma unroll
          for (int j = 0; j < NTC; ++j, o0 += step, o1 += step) {
            if (8 * j < nrem) *o0 = fma(alpha, acc[j][0], ld[j][0]);
            if (8 * j + 1 < nrem) *o1 = fma(alpha, acc[j][1], ld[j][1]);
          }
        }
      }
    }
    __syncwarp();  // every lane is done with this buffer before the next copy into it
    cur = nxt;
    wc = wn;
    buf ^= 1;
  }
  cp_async_wait<0>();
  // every warp of this CTA has taken its last strip: the last CTA of the
  // launch re-arms the counters (the next launch is ordered after this grid)
  __syncthreads();
  if (tid == 0) {
    const unsigned ngroups = unsigned(it.z);
    if (atomicInc(queue + ngroups, gridDim.x - 1) == gridDim.x - 1)
      for (unsigned q = 0; q < ngroups; ++q) queue[q] = 0u;
  }
}

template <int NTC, int NW>
size_t fd_resident_smem(int K) {
  const int Kp = (K + 3) / 4 * 4;
  const int XS = (Kp & 7) == 4 ? Kp : Kp + 4;
  const int BS = (8 * NTC + 11) / 16 * 16 + 4;
  return sizeof(double) * (size_t(Kp) * BS + size_t(NW) * 2 * 8 * XS);
}
// warps per CTA: 16 with the 72-column panel (203 KB), 12 with 88 columns
// (8 for passes with few strips per warp: c4's finest level has 4290 strips)
constexpr int kResWarps9 = 16, kResWarps9s = 8, kResWarps11 = 12;

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
  const int ntiles = tm_n * tn_n;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  // a warp runs two tiles' accumulator chains interleaved (DMMA latency)
  for (int tile = warp; tile < ntiles; tile += 2 * nwarps) {
    const int tiles[2] = {tile, tile + nwarps};
    const double* arow[2];
    bool r_ok[2], n_ok[2];
    int n[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int tl = tiles[u] < ntiles ? tiles[u] : tile;
      const int tm = tl % tm_n, tn = tl / tm_n;
      const int r = tm * 8 + g;
      r_ok[u] = r < rows && tiles[u] < ntiles;
      const int rt = r < rows ? r % inner : 0, ro = r < rows ? r / inner : 0;
      arow[u] = in + (long long)ro * inner * m + rt;
      n[u] = tn * 8 + g;
      n_ok[u] = n[u] < m && tiles[u] < ntiles;
    }
    double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int ks = 0; ks < ks_n; ++ks) {
      const int k = ks * 4 + t4;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double a = (r_ok[u] && k < m) ? arow[u][(long long)k * inner] : 0.0;
        const double b = (n_ok[u] && k < m) ? Bs[k * m + n[u]] : 0.0;
        dmma(d[u][0], d[u][1], a, b);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (tiles[u] >= ntiles) continue;
      const int tm = tiles[u] % tm_n, tn = tiles[u] / tm_n;
      const int orow = tm * 8 + g;
      if (orow < rows) {
        const int ot = orow % inner, oo = orow / inner;
        double* dst = out + (long long)oo * inner * m + ot;
        const int j0 = tn * 8 + 2 * t4;
        if (j0 < m) dst[(long long)j0 * inner] = d[u][0];
        if (j0 + 1 < m) dst[(long long)(j0 + 1) * inner] = d[u][1];
      }
    }
  }
}

// The whole solve of one piece in one CTA.  Every factor (2 per axis) and the
// diagonal are fetched with cp.async at entry, overlapping the input gather,
// so the 2d products run back to back from shared memory.
// smem: X, Y, diag (total each), then B[a][dir] (m_a^2 each).
template <class In, class Out>
__device__ void fd_small_body(const FdPiece& P, int naxes, In in, Out out, double* sm) {
  const int dims[3] = {P.dims[0], P.dims[1], naxes == 3 ? P.dims[2] : 1};
  const int total = int(P.total);
  double* X = sm;
  double* Y = sm + total;
  double* D = sm + 2 * total;
  double* Bs[3][2];
  {
    double* q = sm + 3 * total;
    for (int a = 0; a < naxes; ++a)
      for (int dir = 0; dir < 2; ++dir) {
        Bs[a][dir] = q;
        const int mm = dims[a] * dims[a];
        const double* src = P.B[a][dir];
        for (int i = threadIdx.x; i < mm; i += blockDim.x) cp_async8(q + i, src + i, true);
        q += mm;
      }
    for (int i = threadIdx.x; i < total; i += blockDim.x) cp_async8(D + i, P.diag + i, true);
    cp_async_commit();
  }
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) X[idx] = in(idx);
  cp_async_wait<0>();
  __syncthreads();
  for (int a = 0; a < naxes; ++a) {  // w = (x_a V_a^T) r
    small_axis(X, Y, Bs[a][0], naxes, dims, a);
    __syncthreads();
    double* tmp = X;
    X = Y;
    Y = tmp;
  }
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) X[idx] = X[idx] / D[idx];
  __syncthreads();
  for (int a = 0; a < naxes; ++a) {  // x = (x_a V_a) w
    small_axis(X, Y, Bs[a][1], naxes, dims, a);
    __syncthreads();
    double* tmp = X;
    X = Y;
    Y = tmp;
  }
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) out(idx, X[idx]);
}

// lattice box of an interior piece: box index -> lattice slot
struct LatticeBox {
  long long base, ext, ext2;
  int m0, m1;
  __device__ __forceinline__ long long operator()(int idx) const {
    const int i0 = idx % m0, i1 = (idx / m0) % m1, i2 = idx / (m0 * m1);
    return base + i0 + ext * i1 + ext2 * i2;
  }
};

__global__ void __launch_bounds__(kSmallThreads) fd_small_kernel(const FdPiece* __restrict__ pieces, int naxes,
                                                                 int in_mode, int out_mode,
                                                                 const double* __restrict__ lat_in,
                                                                 double* __restrict__ lat_out, double alpha,
                                                                 const double* __restrict__ work_in,
                                                                 double* __restrict__ work_out) {
  PMG_PDL_ENTRY();
  extern __shared__ __align__(16) double sm[];
  const FdPiece& P = pieces[blockIdx.x];
  const LatticeBox box{P.lat_base, P.ext, (long long)P.ext * P.ext, P.dims[0], P.dims[1]};
  const long long woff = P.work_off;
  auto in = [&](int idx) { return in_mode == FD_IN_WORK ? work_in[woff + idx] : lat_in[box(idx)]; };
  auto out = [&](int idx, double v) {
    if (out_mode == FD_OUT_WORK || out_mode == FD_OUT_WORK_DIAG)
      work_out[woff + idx] = v;
    else if (out_mode == FD_OUT_LATTICE_SET)
      lat_out[box(idx)] = alpha * v;
    else
      lat_out[box(idx)] += alpha * v;
  };
  fd_small_body(P, naxes, in, out, sm);
}

// The whole smoother of a small level on one rank, one launch
// (HybridSmoother::apply, smoother.cpp:110-115): CTAs [0, n_int) solve the
// interior pieces on the lattice; then the face pieces (3D), the edge items
// and one vertex CTA act on interface totals that each CTA sums from the
// replicas itself (the order iface_partial uses), and write every replica.
// Pieces are disjoint, so the CTAs are independent.
__global__ void __launch_bounds__(kSmallThreads) smooth_small_kernel(SmoothSmallArgs a) {
  PMG_PDL_ENTRY();
  extern __shared__ __align__(16) double sm[];
  const ReplicaSum total{a.rep_off, a.rep_slot, a.r};
  int b = blockIdx.x;
  if (b < a.n_int) {
    const FdPiece& P = a.ints[b];
    const LatticeBox box{P.lat_base, P.ext, (long long)P.ext * P.ext, P.dims[0], P.dims[1]};
    const double* __restrict__ r = a.r;
    double* __restrict__ o = a.out;
    const double alpha = a.alpha;
    if (a.add)
      fd_small_body(P, a.d, [&](int idx) { return r[box(idx)]; }, [&](int idx, double v) { o[box(idx)] += alpha * v; },
                    sm);
    else
      fd_small_body(P, a.d, [&](int idx) { return r[box(idx)]; }, [&](int idx, double v) { o[box(idx)] = alpha * v; },
                    sm);
    return;
  }
  b -= a.n_int;
  if (b < a.n_face) {
    const FdPiece& P = a.faces[b];
    const int* __restrict__ g = a.face_iface + P.work_off;
    fd_small_body(
        P, 2, [&](int idx) { return total(g[idx]); },
        [&](int idx, double v) { write_replicas(a.rep_off, a.rep_slot, g[idx], a.alpha * v, a.out, a.add); }, sm);
    return;
  }
  b -= a.n_face;
  if (b < a.n_edge_items) {
    const int2 it = a.edge_items[b];
    edge_item(a.edges[it.x], it.y, a.edge_iface, total, a.rep_off, a.rep_slot, a.out, a.add, a.alpha);
    return;
  }
  vertex_block(a.vert_iface, a.vert_scalar, a.nverts, total, a.rep_off, a.rep_slot, a.out, a.add, a.alpha);
}

}  // namespace

size_t fd_small_smem(long long max_total, int max_dim, int naxes) {
  return size_t(3 * max_total + 2LL * naxes * max_dim * max_dim) * sizeof(double);
}

void launch_fd_small(cudaStream_t s, const FdPiece* pieces, int npieces, int naxes, long long max_total,
                     int max_dim, int in_mode, int out_mode, const double* lat_in, double* lat_out, double alpha,
                     const double* work_in, double* work_out) {
  if (npieces == 0) return;
  const size_t smem = fd_small_smem(max_total, max_dim, naxes);
  launch_k(fd_small_kernel, dim3(npieces), dim3(kSmallThreads), smem, s, pieces, naxes, in_mode, out_mode, lat_in,
           lat_out, alpha, work_in, work_out);
}

void launch_smooth_small(cudaStream_t s, const SmoothSmallArgs& a, size_t smem) {
  const int grid = a.n_int + a.n_face + a.n_edge_items + (a.nverts > 0 ? 1 : 0);
  if (grid == 0) return;
  launch_k(smooth_small_kernel, dim3(grid), dim3(kSmallThreads), smem, s, a);
}

// kernel configurations: cfg = NTC | NW << 8
#define PMG_FD_CONFIGS(X)                                                                                   \
  X(3, 4, 3, 4) X(5, 4, 3, 4) X(9, 4, 3, 4) X(11, 4, 3, 4) X(9, 8, 4, 2) X(11, 8, 4, 2) X(9, 11, 5, 1) \
  X(11, 11, 5, 1)

void fd_configure() {
  ensure_smem((const void*)fd_small_kernel, 200 * 1024);
  ensure_smem((const void*)smooth_small_kernel, 200 * 1024);
#define PMG_FD_ATTR(NT, NW, ST, MB) \
  ensure_smem((const void*)fd_pass_dmma_kernel<NT, NW, ST, MB>, FdTile<NT, NW, ST>::smem);
  PMG_FD_CONFIGS(PMG_FD_ATTR)
#undef PMG_FD_ATTR
  ensure_smem((const void*)fd_pass_resident_kernel<9, kResWarps9>, fd_resident_smem<9, kResWarps9>(72));
  ensure_smem((const void*)fd_pass_resident_kernel<9, kResWarps9s>, fd_resident_smem<9, kResWarps9s>(72));
  ensure_smem((const void*)fd_pass_resident_kernel<11, kResWarps11>, fd_resident_smem<11, kResWarps11>(88));
}

// CTA items of the resident-factor kernel: the SMs are shared out over the
// groups in proportion to their strips (every group at least one CTA), and a
// group's CTAs split its strips evenly.  groups: (first piece, rows).
void fd_resident_items(const std::vector<std::pair<int, long long>>& groups, std::vector<int4>& items) {
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long total = 0;
  for (const auto& gr : groups) total += (gr.second + 7) / 8;
  int left = sms - int(groups.size());
  std::vector<int> ctas(groups.size(), 1);
  std::vector<double> want(groups.size());
  for (size_t i = 0; i < groups.size(); ++i) {
    want[i] = double((groups[i].second + 7) / 8) * sms / double(total);
    const int extra = std::max(0, std::min(left, int(want[i]) - 1));
    ctas[i] += extra;
    left -= extra;
  }
  // the SMs left by rounding go to the groups with the most strips per CTA
  while (left > 0) {
    size_t b = 0;
    double worst = -1.0;
    for (size_t i = 0; i < groups.size(); ++i) {
      const double load = double((groups[i].second + 7) / 8) / ctas[i];
      if (load > worst) worst = load, b = i;
    }
    ctas[b]++;
    left--;
  }
  for (size_t i = 0; i < groups.size(); ++i) {
    const long long strips = (groups[i].second + 7) / 8;
    const int nc = int(std::min<long long>(ctas[i], strips));
    for (int j = 0; j < nc; ++j)
      items.push_back(make_int4(groups[i].first, int(i), int(groups.size()), int(groups[i].second)));
  }
}

// cfg with kFdResident set: fd_pass_resident_kernel<NTC> (persistent CTAs, resident factor)
bool fd_cfg_resident(int cfg) { return (cfg & kFdResident) != 0; }
int fd_cfg_rows(int cfg) { return 8 * ((cfg >> 8) & 255); }
int fd_cfg_cols(int cfg) { return 8 * (cfg & 255); }

bool fd_cfg_valid(int cfg) {
  if (fd_cfg_resident(cfg)) {  // NTC | warps << 8 | kFdResident
    const int ntc = cfg & 255, nw = (cfg >> 8) & 255;
    return (ntc == 9 && (nw == kResWarps9 || nw == kResWarps9s)) || (ntc == 11 && nw == kResWarps11);
  }
#define PMG_FD_VALID(NT, NW, ST, MB) \
  if (cfg == (NT | NW << 8)) return true;
  PMG_FD_CONFIGS(PMG_FD_VALID)
#undef PMG_FD_VALID
  return false;
}

int fd_pick_cfg(const long long* cols, const long long* weight, int n) {
  // PMG_FD_CFG="ntc,nw" forces one configuration; PMG_FD_NTC forces the
  // column panel of the 4-warp kernel
  if (const char* e = std::getenv("PMG_FD_CFG")) {
    int ntc = 0, nw = 0;
    if (std::sscanf(e, "%d,%d", &ntc, &nw) == 2) {
      if (nw != 0) return ntc | nw << 8;
      // "ntc,0": the resident-factor kernel where the contraction fits, else the default
      int kmax = 0;
      long long strips = 0;
      for (int i = 0; i < n; ++i) {
        kmax = std::max<long long>(kmax, cols[i]);
        strips += (weight[i] + 7) / 8;
      }
      if (kmax <= 8 * ntc && n <= 148 && (ntc == 9 || ntc == 11)) {
        const int rw = ntc == 11 ? kResWarps11 : strips >= 4LL * 148 * kResWarps ? kResWarps9 : kResWarps9s;
        return ntc | rw << 8 | kFdResident;
      }
    }
  }
  if (const char* e = std::getenv("PMG_FD_NTC")) return std::atoi(e) | 4 << 8;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // short contractions with many rows (3D levels): the resident-factor kernel
  {
    static const bool res_ok = [] {
      const char* e = std::getenv("PMG_FD_RESIDENT");
      return !(e && e[0] == '0');
    }();
    int kmax = 0;
    long long strips = 0;
    for (int i = 0; i < n; ++i) {
      kmax = std::max<long long>(kmax, cols[i]);
      strips += (weight[i] + 7) / 8;
    }
    static const int small_ok = [] {  // experiments: PMG_FD_RES_SMALL=1 takes the 8-warp variant from 2 strips per warp
      const char* e = std::getenv("PMG_FD_RES_SMALL");
      return e && e[0] == '1';
    }();
    if (res_ok && kmax <= 88 && kmax >= 24 && n <= sms) {
      if (strips >= 4LL * sms * kResWarps)
        return kmax <= 72 ? (9 | kResWarps9 << 8 | kFdResident) : (11 | kResWarps11 << 8 | kFdResident);
      if (small_ok && kmax <= 72 && strips >= 2LL * sms * kResWarps9s) return 9 | kResWarps9s << 8 | kFdResident;
    }
  }
  // large passes (every SM gets a full 88-row tile and the contraction is
  // long enough to amortise the tile's fill and drain): one 11-warp CTA per
  // SM, with the column panel (72 or 88) that pads N less
  {
    static const bool wide_ok = [] {
      const char* e = std::getenv("PMG_FD_WIDE");
      return !(e && e[0] == '0');
    }();
    long long ctas[2] = {0, 0};
    double pad[2] = {0.0, 0.0};
    int kmin = 1 << 30;
    for (int i = 0; i < n; ++i) {
      kmin = std::min<long long>(kmin, cols[i]);
      for (int ci = 0; ci < 2; ++ci) {
        const int bn = ci ? 88 : 72;
        const long long cp = (cols[i] + bn - 1) / bn;
        ctas[ci] += (weight[i] + 87) / 88 * cp;
        pad[ci] += double((weight[i] + 87) / 88 * 88) * double(cp * bn) * double(cols[i]);
      }
    }
    const int ci = pad[1] <= pad[0] ? 1 : 0;
    if (wide_ok && kmin >= 192 && ctas[ci] >= (3 * sms) / 4) return (ci ? 11 : 9) | 11 << 8;
  }
  // the 4-warp kernel: the column-panel width (in n-tiles) with the least
  // padding over the groups; 11 (88 columns) is measured slower than 9 at the
  // c2 finest level (fewer, larger CTAs per wave) and is only used when forced
  // (PMG_FD_NTC).  weight = rows of each group.
  static const int cands[3] = {3, 5, 9};
  // narrow panels reload A fragments more often per DMMA: measured 0.92x the
  // 72-column rate on c2's finest level for 40 columns
  static const double rate[3] = {1.2, 1.09, 1.0};
  double cost[3] = {0.0, 0.0, 0.0}, pad[3] = {0.0, 0.0, 0.0};
  long long ctas[3] = {0, 0, 0};
  double work = 0.0;
  for (int ci = 0; ci < 3; ++ci) {
    const int c = cands[ci];
    for (int i = 0; i < n; ++i) {
      const double w = double((cols[i] + 8 * c - 1) / (8 * c) * (8 * c));
      cost[ci] += rate[ci] * double(weight[i]) * w;
      pad[ci] += double(weight[i]) * w;
      ctas[ci] += (weight[i] + 31) / 32 * ((cols[i] + 8 * c - 1) / (8 * c));
      if (ci == 0) work += double(weight[i]) * double(cols[i]);
    }
  }
  int best = 2;  // 5 and 9 by cost (3 only for parallelism, below)
  if (cost[1] < cost[2]) best = 1;
  // a pass that fills fewer than two CTAs per SM is latency-bound: take the
  // panel with the most CTAs among those padding <= 25% (c2 levels 5-6:
  // 8.4 -> 7.3 and 15.5 -> 14 us per pass with 40-column panels, measured)
  if (ctas[best] < 2LL * sms)
    for (int ci = 0; ci < 3; ++ci)
      if (pad[ci] <= 1.25 * work && ctas[ci] > ctas[best]) best = ci;
  return cands[best] | 4 << 8;
}

void launch_fd_pass(cudaStream_t s, const FdPiece* pieces, const int4* items, int nitems, int cfg, int pass,
                    int naxes, int in_mode, int out_mode, const double* lat_in, double* lat_out, double alpha,
                    const double* work_in, double* work_out, unsigned* queue) {
  if (nitems == 0) return;
  if (fd_cfg_resident(cfg)) {
    // one smem size per launch: the largest contraction the kernel may see is 8 NTC
    if (!queue) throw std::runtime_error("FD pass: the resident-factor kernel needs its strip counters");
    if ((cfg & 255) == 9 && ((cfg >> 8) & 255) == kResWarps9s) {
      launch_k(fd_pass_resident_kernel<9, kResWarps9s>, dim3(nitems), dim3(32 * kResWarps9s),
               fd_resident_smem<9, kResWarps9s>(72), s, pieces, items, queue, pass, naxes, in_mode, out_mode, lat_in,
               lat_out, alpha, work_in, work_out);
    } else if ((cfg & 255) == 9) {
      launch_k(fd_pass_resident_kernel<9, kResWarps9>, dim3(nitems), dim3(32 * kResWarps9),
               fd_resident_smem<9, kResWarps9>(72), s, pieces, items, queue, pass, naxes, in_mode, out_mode, lat_in,
               lat_out, alpha, work_in, work_out);
    } else {
      launch_k(fd_pass_resident_kernel<11, kResWarps11>, dim3(nitems), dim3(32 * kResWarps11),
               fd_resident_smem<11, kResWarps11>(88), s, pieces, items, queue, pass, naxes, in_mode, out_mode, lat_in,
               lat_out, alpha, work_in, work_out);
    }
    return;
  }
#define PMG_FD_CASE(NT, NW, ST, MB)                                                                             \
  if (cfg == (NT | NW << 8)) {                                                                                  \
    launch_k(fd_pass_dmma_kernel<NT, NW, ST, MB>, dim3(nitems), dim3(32 * NW), FdTile<NT, NW, ST>::smem, s, pieces, \
             items, pass, naxes, in_mode, out_mode, lat_in, lat_out, alpha, work_in, work_out);                 \
    return;                                                                                                     \
  }
  PMG_FD_CONFIGS(PMG_FD_CASE)
#undef PMG_FD_CASE
  throw std::runtime_error("FD pass: no kernel for this configuration (PMG_FD_NTC must be 3, 5, 9 or 11)");
}

}  // namespace pmgcu
