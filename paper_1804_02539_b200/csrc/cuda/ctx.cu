// libpmg_cuda: context creation (host-side layout planning + uploads), the C
// ABI of include/pmg_cuda.h, and the device-resident V-cycle / PCG drivers.
//
// The drivers restate, on device-resident lattice vectors:
//   mg_cycle_generic / mg_precondition / pcg_generic  multigrid.hpp:120-189
// with the Backend operations of SerialBackend (multigrid.hpp:80-114) /
// ParallelBackend (parallel.cpp:247-468) implemented by the kernels in
// kernels_*.cu.  Two reference operations are restated exactly and cheaper:
//   * the first residual of a cycle from a zero start is f itself
//     (f - A*0 == f bitwise), so that SpMV is skipped;
//   * restriction runs on the distributed per-patch shares directly; the
//     owner masking of restrict_full (transfer.cpp:68-91) only picks one split
//     of the same sum, and P^T is linear.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/pmg_cuda.h"
#include "../common/rank_plan.hpp"
#include "../host/numerics.hpp"
#include "comm.cuh"
#include "internal.cuh"

using namespace pmgcu;

namespace {

struct PmgError : std::runtime_error {
  int code;
  PmgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw PmgError(PMG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevLevel {
  int n = 0, ext = 0, O = 0, K = 0;
  int Ob = 0;  // stored offsets per patch: O, or (O+1)/2 for the symmetric half band
  int sweep_tw = 0;  // > 0: the band is line-major [K][ext][Ob][tw] (2D line-sweep level)
  int sweep3_front = 0, sweep3_e2p = 0;  // e2p > 0: plane-major [K][ext][Ob][e2p] (3D plane-sweep level)
  long long S = 0, Sp = 0, lat_n = 0, N = 0;
  double* band = nullptr;
  // PMG_BAND_KRONECKER level (kernels_kron.cu): no band; univariate mass and
  // stiffness as full bands [ext][2p+1], per-patch geometry factors [K][3]
  bool kron = false;
  double *kron_M = nullptr, *kron_K = nullptr, *kron_g = nullptr, *kron_scratch = nullptr;
  double* sweep_scratch = nullptr;  // line sweep: segment-boundary rows
  unsigned* sweep_flags = nullptr;
  unsigned long long* sweep_ticket = nullptr;
  int* l2g = nullptr;
  unsigned char* owner = nullptr;
  int* rep_off = nullptr;
  int* rep_slot = nullptr;
  // interface dofs of this rank (pmgplan::RankPlan): local replicas, fold
  // sources, exchange buffers, partial and total sums
  int n_iface = 0;
  int *if_rep_off = nullptr, *if_rep_slot = nullptr, *if_comb_off = nullptr, *if_comb_src = nullptr;
  double *if_tloc = nullptr, *if_t = nullptr;
  const double* if_total = nullptr;  // the totals: if_t, or if_tloc itself on one rank
  int* if_send_idx = nullptr;
  int n_send = 0, n_recv = 0;
  double *if_send = nullptr, *if_recv = nullptr;
  std::vector<Peer> peers;
  // interior FD
  FdPiece* d_int = nullptr;
  int n_int = 0;
  int4* int_items[6] = {};
  unsigned* int_queue[6] = {};  // resident-factor passes: strip counters (kernels_fd.cu)
  int n_int_items[6] = {};
  int int_ntc[6] = {};  // kernel configuration per pass (fd_pick_cfg)
  std::vector<std::array<int, 3>> int_dims;  // host copy for flop counts
  bool int_small = false, face_small = false;  // whole solve per CTA in shared memory
  long long int_max_total = 0, face_max_total = 0;
  int int_max_dim = 0, face_max_dim = 0;
  // faces
  FdPiece* d_face = nullptr;
  int n_face = 0;
  int* face_iface = nullptr;  // face piece dofs as interface indices
  long long face_ndof = 0;
  int4* face_items[4] = {};
  unsigned* face_queue[4] = {};
  int n_face_items[4] = {};
  int face_ntc[4] = {};
  // edges / vertices
  EdgePiece* d_edges = nullptr;
  int n_edges = 0;
  int2* edge_items = nullptr;
  int n_edge_items = 0;
  int* edge_iface = nullptr;
  int* vert_iface = nullptr;
  double* vert_scalar = nullptr;
  int n_verts = 0;
  // two-scale factor from level-1 (level >= 1)
  TsDev ts{};
  // V-cycle workspace
  double* f = nullptr;
  double* u = nullptr;
  double* r = nullptr;
};

}  // namespace

struct pmg_hub {
  explicit pmg_hub(int r) : hub(r) {}
  Hub hub;
};

struct pmg_ctx {
  int device = 0;
  int dim = 0, degree = 0, K_global = 0, pb = 0, pe = 0, nl = 0;
  int rank = 0, size = 1;
  // null on a single-GPU context; an NCCL job creates it at any size, so a
  // world-1 job runs every collective (exchange, all-gathers, coarse
  // gather / broadcast) through NCCL exactly as a multi-GPU job does
  std::unique_ptr<Transport> comm;
  bool multi() const { return comm != nullptr; }
  double* rank_buf = nullptr;       // size doubles (scalar all-gathers)
  double* coarse_parts = nullptr;   // size x n0 (coarse gather on rank 0)
  pmg_cycle_params prm{};
  std::vector<DevLevel> lv;
  double* work[2] = {nullptr, nullptr};
  double* tbuf[2] = {nullptr, nullptr};
  double* face_buf[2] = {nullptr, nullptr};
  double* Ainv = nullptr;
  int n0 = 0;
  double* coarse_rhs = nullptr;
  double* coarse_x = nullptr;
  double* partial = nullptr;
  int partial_n = 0;
  int sweep = 128;  // 2D line-sweep SpMV on lines of >= sweep rows; 0: off (PMG_SWEEP, PMG_SWEEP_MIN_EXT at creation)
  int sweep3 = 30;  // 3D plane-sweep SpMV on lattices of >= sweep3 rows per axis; 0: off (PMG_SWEEP3D)
  double* scal = nullptr;     // device scalars
  double* h_scal = nullptr;   // pinned mirror
  double* staging = nullptr;  // device global-vector staging (finest num_dofs)
  long long staging_n = 0;
  // PCG vectors on the finest level
  double *pcg_r = nullptr, *pcg_z = nullptr, *pcg_p = nullptr, *pcg_Ap = nullptr, *pcg_acc = nullptr,
         *pcg_u = nullptr, *pcg_f = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  // the interface pieces of a smooth run on side_stream, concurrent with the
  // interior FD (they write disjoint slots); fork/join by events, so the
  // overlap is captured into the CUDA graphs too.  PMG_NO_OVERLAP=1 disables.
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool overlap = true;
  std::vector<void*> allocs;
  size_t bytes = 0;
  long long launches = 0, spmv_launches = 0;
  double assembly_seconds = 0.0;  // device stiffness assembly (PMG_BAND_ASSEMBLE levels)
  double load_seconds = 0.0;      // device load-vector assembly (pmg_assemble_load)
  // the patch geometry, copied when the descriptor carries it (pmg_assemble_load)
  std::vector<pmg_patch_geometry> geo;
  std::vector<std::vector<double>> geo_ctrl;
  std::string err;
  // live event timing (pmg_profile)
  bool profiling = false;
  struct Timed {
    int cls, level;
    double work;
    cudaEvent_t a, b;
  };
  std::vector<Timed> timed;
  std::vector<cudaEvent_t> event_pool;
  // CUDA graphs of the PCG iteration (captured on own_stream, launched on stream)
  bool use_graphs = true;
  cudaGraphExec_t graph_front = nullptr, graph_back = nullptr;
  long long graph_front_launches = 0, graph_back_launches = 0;
  const double* graph_u = nullptr;
  cudaEvent_t ev_norm = nullptr;
  // device-resident PCG loop: the whole solve is one graph launch, its
  // iteration body under a WHILE conditional node (one GPU; PMG_HOST_LOOP=1
  // keeps the host-driven front/back graphs).  Two cached graphs, keyed by
  // the (f, u) device pointers they were captured on.
  struct LoopGraph {
    const double* f = nullptr;
    const double* u = nullptr;
    cudaGraphExec_t exec = nullptr;
    long long head = 0, body = 0;  // kernel launches of the head and of one iteration
  };
  LoopGraph loop[2];
  int loop_next = 0;
  bool device_loop = true;
  PcgLoopState* loop_state = nullptr;  // device
  PcgLoopState* h_loop = nullptr;      // pinned mirror
  double* loop_hist = nullptr;         // device residual history
  int loop_hist_cap = 0;
  // graph-replayed mg_precondition (pmg_precondition), keyed by (r, z)
  cudaGraphExec_t graph_pre = nullptr;
  long long graph_pre_launches = 0;
  const double *graph_pre_r = nullptr, *graph_pre_z = nullptr;

  template <class F>
  void capture(cudaGraphExec_t& exec, long long& nlaunch, F&& body) {
    if (exec) {
      cudaGraphExecDestroy(exec);
      exec = nullptr;
    }
    cudaStream_t saved = stream;
    stream = own_stream;
    const long long before = launches;
    ck(cudaStreamBeginCapture(own_stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    cudaGraph_t g = nullptr;
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(own_stream, &g);
      if (g) cudaGraphDestroy(g);
      stream = saved;
      launches = before;
      throw;
    }
    stream = saved;
    ck(cudaStreamEndCapture(own_stream, &g), "cudaStreamEndCapture");
    ck(cudaGraphInstantiate(&exec, g, 0), "cudaGraphInstantiate");
    cudaGraphDestroy(g);
    nlaunch = launches - before;
    launches = before;
  }
  void launch_graph(cudaGraphExec_t exec, long long n) {
    ck(cudaGraphLaunch(exec, stream), "cudaGraphLaunch");
    launches += n;
  }
  cudaEvent_t get_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
  }

  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    // 64 B of slack: TMA windows over a lattice vector round its end up to 16 B
    ck(cudaMalloc(&p, count * sizeof(T) + 64), "cudaMalloc");
    allocs.push_back(p);
    bytes += count * sizeof(T);
    return static_cast<T*>(p);
  }
  template <class T>
  void release(T* p, size_t count) {
    for (auto it = allocs.begin(); it != allocs.end(); ++it)
      if (*it == static_cast<void*>(p)) {
        cudaFree(p);
        allocs.erase(it);
        bytes -= count * sizeof(T);
        return;
      }
  }
  template <class T>
  T* upload(const T* h, size_t count) {
    T* d = alloc<T>(count);
    if (count) ck(cudaMemcpyAsync(d, h, count * sizeof(T), cudaMemcpyHostToDevice, stream), "cudaMemcpy H2D");
    return d;
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    return upload(v.data(), v.size());
  }
  ~pmg_ctx() {
    cudaSetDevice(device);
    if (graph_front) cudaGraphExecDestroy(graph_front);
    if (graph_back) cudaGraphExecDestroy(graph_back);
    if (graph_pre) cudaGraphExecDestroy(graph_pre);
    for (auto& g : loop)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (h_loop) cudaFreeHost(h_loop);
    if (ev_norm) cudaEventDestroy(ev_norm);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side_stream) cudaStreamDestroy(side_stream);
    for (auto& t : timed) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
    for (void* p : allocs) cudaFree(p);
    if (h_scal) cudaFreeHost(h_scal);
    if (own_stream) cudaStreamDestroy(own_stream);
  }
};

struct pmg_vec {
  pmg_ctx* ctx;
  int level;
  double* d;
  long long n;
};

namespace {

thread_local std::string g_create_error;

// Explicit inverse of the banded Cholesky operator: column j is the
// reference BandedCholesky::solve (banded.cpp:61-77) of e_j; stored
// column-major so a warp's rows read consecutive addresses.
std::vector<double> banded_inverse(int n, int bw, const double* l) {
  const int w = bw + 1;
  std::vector<double> inv(size_t(n) * n), y(n);
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < n; ++i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = std::max(0, i - bw); k < i; ++k) s -= l[size_t(i) * w + (i - k)] * y[k];
      y[i] = s / l[size_t(i) * w];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < std::min(n, i + bw + 1); ++k) s -= l[size_t(k) * w + (k - i)] * y[k];
      y[i] = s / l[size_t(i) * w];
    }
    for (int i = 0; i < n; ++i) inv[size_t(j) * n + i] = y[i];
  }
  return inv;
}

// A0^-1 = L^-T L^-1 from the lower Cholesky factor (column-major); row-major out
std::vector<double> spd_inverse(int n, const double* L) {
  std::vector<double> Li(size_t(n) * n, 0.0);  // column-major lower inverse
  for (int j = 0; j < n; ++j) {
    Li[size_t(j) * n + j] = 1.0 / L[size_t(j) * n + j];
    for (int i = j + 1; i < n; ++i) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s += L[size_t(k) * n + i] * Li[size_t(j) * n + k];
      Li[size_t(j) * n + i] = -s / L[size_t(i) * n + i];
    }
  }
  std::vector<double> inv(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0.0;
      for (int k = i; k < n; ++k) s += Li[size_t(i) * n + k] * Li[size_t(j) * n + k];
      inv[size_t(i) * n + j] = inv[size_t(j) * n + i] = s;
    }
  return inv;
}

int level_spmv_partials(const pmg_ctx& c, const DevLevel& L);
void build_kron_level(pmg_ctx& c, const pmg_hierarchy_desc& D, int l, const int* l2g);
void build_band_level(pmg_ctx& c, const pmg_hierarchy_desc& D, int l, const int* l2g);
void build_level_rest(pmg_ctx& c, const pmg_hierarchy_desc& D, int l);

void build_level(pmg_ctx& c, const pmg_hierarchy_desc& D, int l) {
  const pmg_level_desc& ld = D.levels[l];
  DevLevel& L = c.lv[l];
  const int d = D.dim, p = D.degree;
  L.n = ld.elements;
  L.ext = ld.elements + p;
  L.O = 1;
  L.S = 1;
  for (int a = 0; a < d; ++a) {
    L.O *= 2 * p + 1;
    L.S *= L.ext;
  }
  L.K = c.pe - c.pb;
  L.lat_n = L.S * L.K;
  L.N = ld.num_dofs;
  const long long S = L.S;
  const int* l2g_all = ld.l2g;
  const int* l2g = l2g_all + (size_t)c.pb * S;

  if (ld.band_format == PMG_BAND_KRONECKER) {
    build_kron_level(c, D, l, l2g);
  } else {
    build_band_level(c, D, l, l2g);
  }
  build_level_rest(c, D, l);
}

// Matrix-free level (PMG_BAND_KRONECKER): the univariate matrices of the
// level's free-end space (univariate_mass / univariate_stiffness,
// spline.cpp:86-110,141-145) and the geometry factors of every local patch.
void build_kron_level(pmg_ctx& c, const pmg_hierarchy_desc& D, int l, const int* l2g) {
  const pmg_level_desc& ld = D.levels[l];
  DevLevel& L = c.lv[l];
  const int d = D.dim, p = D.degree;
  if (!D.geometry) throw PmgError(PMG_ERR_CONFIG, "the Kronecker operator needs the patch geometry (desc.geometry)");
  if (!kron_supported(d, p, L.ext))
    throw PmgError(PMG_ERR_CONFIG, "the Kronecker operator supports degrees 1..8 (2D lines must fit shared memory)");
  std::vector<double> g(size_t(L.K) * 3, 0.0);
  for (int k = 0; k < L.K; ++k) {
    const pmg_patch_geometry& pg = D.geometry[c.pb + k];
    // x_a = c_a + h_a xi_a  <=>  the control net sits on the Greville abscissae of every axis
    std::vector<std::vector<double>> grev(d);
    long long npts = 1;
    for (int a = 0; a < d; ++a) {
      const pmg::UnivariateSpace sp(pg.degree[a], pg.elements[a]);
      const std::vector<double> kn = sp.knots();
      const int q = pg.degree[a], m = pg.elements[a] + q;
      grev[a].resize(m);
      for (int i = 0; i < m; ++i) {
        double sum = 0.0;
        for (int j = 1; j <= q; ++j) sum += kn[i + j];
        grev[a][i] = sum / q;
      }
      npts *= m;
    }
    double h[3] = {1.0, 1.0, 1.0}, c0[3] = {0.0, 0.0, 0.0}, scale = 0.0;
    {
      long long stride = 1;
      for (int a = 0; a < d; ++a) {
        const int m = pg.elements[a] + pg.degree[a];
        c0[a] = pg.ctrl[a];
        h[a] = pg.ctrl[size_t(stride * (m - 1)) * d + a] - c0[a];
        scale = std::max(scale, std::fabs(h[a]));
        stride *= m;
      }
    }
    for (long long f = 0; f < npts; ++f) {
      long long r = f;
      for (int a = 0; a < d; ++a) {
        const int m = pg.elements[a] + pg.degree[a];
        const int ia = int(r % m);
        r /= m;
        if (std::fabs(pg.ctrl[size_t(f) * d + a] - (c0[a] + h[a] * grev[a][ia])) > 1e-13 * scale)
          throw PmgError(PMG_ERR_CONFIG, "the Kronecker operator needs axis-aligned affine patch maps");
      }
    }
    for (int a = 0; a < d; ++a) {
      if (!(std::fabs(h[a]) > 1e-14 * scale))
        throw PmgError(PMG_ERR_GEOMETRY, "the Kronecker operator: degenerate patch map");
      double v = 1.0 / std::fabs(h[a]);
      for (int b = 0; b < d; ++b)
        if (b != a) v *= std::fabs(h[b]);
      g[size_t(k) * 3 + a] = v;
    }
  }
  const pmg::UnivariateSpace sp(p, ld.elements);
  const pmg::BandedSymMatrix Mb = pmg::univariate_mass(sp), Kb = pmg::univariate_stiffness(sp);
  const int W = 2 * p + 1;
  std::vector<double> M(size_t(L.ext) * W, 0.0), Kst(size_t(L.ext) * W, 0.0);
  for (int i = 0; i < L.ext; ++i)
    for (int dl = -p; dl <= p; ++dl) {
      const int j = i + dl;
      if (j < 0 || j >= L.ext) continue;
      M[size_t(i) * W + dl + p] = Mb(i, j);
      Kst[size_t(i) * W + dl + p] = Kb(i, j);
    }
  L.kron = true;
  L.kron_M = c.upload(M);
  L.kron_K = c.upload(Kst);
  L.kron_g = c.upload(g);
  if (d == 3) L.kron_scratch = c.alloc<double>(size_t(5) * L.lat_n);
  L.Sp = L.S;
  L.Ob = L.O;
  L.l2g = c.upload(l2g, size_t(L.lat_n));
  {
    const char* e = std::getenv("PMG_SWEEP");
    const char* m = std::getenv("PMG_SWEEP_MIN_EXT");
    c.sweep = (e && e[0] == '0') ? 0 : std::max(1, m ? std::atoi(m) : 128);
    const char* e3 = std::getenv("PMG_SWEEP3D");
    c.sweep3 = (e && e[0] == '0') ? 0 : (e3 ? std::atoi(e3) : 30);
  }
}

void build_band_level(pmg_ctx& c, const pmg_hierarchy_desc& D, int l, const int* l2g) {
  const pmg_level_desc& ld = D.levels[l];
  DevLevel& L = c.lv[l];
  const int d = D.dim, p = D.degree;
  const long long S = L.S;
  // ---- band: rows of one (patch, offset) pair at stride Sp (>= S, see spmv_row_stride)
  L.Sp = spmv_row_stride(d, p, L.ext, S);
  const long long Sp = L.Sp;
  // the symmetric half band (kernels_spmv.cu) on TMA levels; PMG_FULL_BAND=1 keeps all O offsets
  const char* fb = std::getenv("PMG_FULL_BAND");
  L.Ob = spmv_stored_offsets(d, p, S, !(fb && fb[0] == '1'));
  // slack past the last patch: mirrored segments read up to Sp + 2 rows beyond a patch's rows
  const size_t band_n = size_t(L.K) * L.Ob * Sp + size_t(Sp) + 256;
  L.band = c.alloc<double>(band_n);
  ck(cudaMemsetAsync(L.band, 0, band_n * sizeof(double), c.stream), "band clear");
  if (ld.band_format == PMG_BAND_TENSOR) {
    for (int k = 0; k < L.K; ++k)
      ck(cudaMemcpy2DAsync(L.band + size_t(k) * L.Ob * Sp, sizeof(double) * Sp,
                           ld.band + (size_t)(c.pb + k) * L.O * S, sizeof(double) * S, sizeof(double) * S,
                           size_t(L.Ob), cudaMemcpyHostToDevice, c.stream),
         "band upload");
  } else if (ld.band_format == PMG_BAND_CSR) {
    // place every CSR entry at its tensor offset (PatchOperator, assembly.hpp:16-25)
    std::vector<double> hb(size_t(L.O) * S);
    const int W = 2 * p + 1;
    for (int k = 0; k < L.K; ++k) {
      std::fill(hb.begin(), hb.end(), 0.0);
      const int64_t* rp = ld.csr_row_ptr[c.pb + k];
      const int32_t* cols = ld.csr_cols[c.pb + k];
      const double* vals = ld.csr_vals[c.pb + k];
      for (long long r = 0; r < S; ++r)
        for (int64_t q = rp[r]; q < rp[r + 1]; ++q) {
          long long rr = r, cc = cols[q];
          int o = 0, mul = 1;
          for (int a = 0; a < d; ++a) {
            const int delta = int(cc % L.ext) - int(rr % L.ext);
            if (delta < -p || delta > p) throw PmgError(PMG_ERR_DOMAIN, "CSR column outside the tensor band");
            o += (delta + p) * mul;
            mul *= W;
            rr /= L.ext;
            cc /= L.ext;
          }
          hb[size_t(o) * S + r] += vals[q];
        }
      // pageable source: the call returns once hb is staged, so hb is reusable
      ck(cudaMemcpy2DAsync(L.band + size_t(k) * L.Ob * Sp, sizeof(double) * Sp, hb.data(), sizeof(double) * S,
                           sizeof(double) * S, size_t(L.Ob), cudaMemcpyHostToDevice, c.stream),
         "band upload");
    }
  } else if (ld.band_format == PMG_BAND_ASSEMBLE) {
    if (!D.geometry) throw PmgError(PMG_ERR_CONFIG, "device assembly needs the patch geometry (desc.geometry)");
    try {
      c.assembly_seconds +=
          assemble_level_device(c.stream, d, p, ld.elements, D.geometry, c.pb, L.K, L.band, Sp, L.Ob);
    } catch (const AssemblyError& e) {
      throw PmgError(PMG_ERR_GEOMETRY, e.what());
    }
  } else {
    throw PmgError(PMG_ERR_CONFIG, "unknown band format");
  }
  L.l2g = c.upload(l2g, size_t(L.lat_n));
  launch_zero_dirichlet_band(c.stream, d, p, L.ext, S, Sp, L.K, L.Ob, L.l2g, L.band);
  {
    const char* e = std::getenv("PMG_SWEEP");
    const char* m = std::getenv("PMG_SWEEP_MIN_EXT");
    c.sweep = (e && e[0] == '0') ? 0 : std::max(1, m ? std::atoi(m) : 128);
    // 3D plane sweep on lattices with >= PMG_SWEEP3D rows per axis (default 30; 0 disables)
    const char* e3 = std::getenv("PMG_SWEEP3D");
    c.sweep3 = (e && e[0] == '0') ? 0 : (e3 ? std::atoi(e3) : 30);
  }
  if (const long long lm = spmv_sweep_band_doubles(d, p, L.ext, S, L.K, L.Ob != L.O, c.sweep)) {
    double* nb = c.alloc<double>(size_t(lm));
    launch_sweep_relayout(c.stream, p, L.ext, S, L.K, Sp, L.band, nb);
    ck(cudaGetLastError(), "sweep relayout");
    ck(cudaStreamSynchronize(c.stream), "sweep relayout");
    c.release(L.band, band_n);
    L.band = nb;
    L.sweep_tw = int(lm / ((long long)L.K * L.ext * L.Ob));
  }
  {
    int front = 0, e2p = 0;
    if (const long long lm = spmv_sweep3_band_doubles(d, p, L.ext, S, L.K, L.Ob != L.O, c.sweep3, &front, &e2p)) {
      double* nb = c.alloc<double>(size_t(lm));
      launch_sweep3_relayout(c.stream, p, L.ext, S, L.K, Sp, L.band, nb);
      ck(cudaGetLastError(), "sweep3 relayout");
      ck(cudaStreamSynchronize(c.stream), "sweep3 relayout");
      c.release(L.band, band_n);
      L.band = nb;
      L.sweep3_front = front;
      L.sweep3_e2p = e2p;
    }
  }
  {
    long long nd = 0, nf = 0;
    spmv_sweep_scratch(d, p, L.ext, S, L.K, L.Ob != L.O, c.sweep, &nd, &nf);
    if (nf > 0) {
      L.sweep_scratch = c.alloc<double>(size_t(nd));
      // one flag per segment boundary, then the 64-bit segment ticket counter
      // at the next even word (cudaMalloc memory is 256-byte aligned)
      const long long tk = (nf + 1) & ~1LL;
      L.sweep_flags = c.alloc<unsigned>(size_t(tk + 2));
      ck(cudaMemsetAsync(L.sweep_flags, 0, sizeof(unsigned) * (tk + 2), c.stream), "memset");
      L.sweep_ticket = reinterpret_cast<unsigned long long*>(L.sweep_flags + tk);
    }
  }

}

void build_level_rest(pmg_ctx& c, const pmg_hierarchy_desc& D, int l) {
  const pmg_level_desc& ld = D.levels[l];
  DevLevel& L = c.lv[l];
  const int d = D.dim, p = D.degree;
  const long long S = L.S;
  const int* l2g_all = ld.l2g;
  const int* l2g = l2g_all + (size_t)c.pb * S;
  (void)p;
  // ---- replicas: global owner patch over all patches; local replica CSR
  std::vector<int> owner_patch(size_t(L.N), -1);
  for (int k = 0; k < D.num_patches; ++k)
    for (long long f = 0; f < S; ++f) {
      const int g = l2g_all[size_t(k) * S + f];
      if (g >= 0 && owner_patch[g] < 0) owner_patch[g] = k;
    }
  std::vector<int> rep_off(size_t(L.N) + 1, 0);
  for (long long s = 0; s < L.lat_n; ++s)
    if (l2g[s] >= 0) rep_off[l2g[s] + 1]++;
  for (long long g = 0; g < L.N; ++g) rep_off[g + 1] += rep_off[g];
  std::vector<int> rep_slot(rep_off.back()), cur(rep_off.begin(), rep_off.end() - 1);
  std::vector<unsigned char> owner(size_t(L.lat_n), 0);
  for (long long s = 0; s < L.lat_n; ++s) {
    const int g = l2g[s];
    if (g < 0) continue;
    rep_slot[cur[g]++] = int(s);
    if (owner_patch[g] == c.pb + int(s / S)) owner[s] = 1;
  }
  L.rep_off = c.upload(rep_off);
  L.rep_slot = c.upload(rep_slot);
  L.owner = c.upload(owner);
  // ---- interface dofs and the exchange plan of this rank (RankLayout, parallel.cpp:200-237)
  const pmgplan::Partition part = pmgplan::contiguous(D.num_patches, c.size);
  const pmgplan::RankPlan plan = pmgplan::build(l2g_all, D.num_patches, S, L.N, part, c.rank);
  L.n_iface = int(plan.iface_g.size());
  L.if_rep_off = c.upload(plan.rep_off);
  L.if_rep_slot = c.upload(plan.rep_slot);
  L.if_comb_off = c.upload(plan.comb_off);
  L.if_comb_src = c.upload(plan.comb_src);
  L.if_tloc = c.alloc<double>(size_t(L.n_iface));
  L.if_t = c.alloc<double>(size_t(L.n_iface));
  L.if_total = c.multi() ? L.if_t : L.if_tloc;
  std::vector<int> send_idx;
  for (const auto& nb : plan.neighbors) send_idx.insert(send_idx.end(), nb.iface.begin(), nb.iface.end());
  L.n_send = L.n_recv = int(send_idx.size());
  L.if_send_idx = c.upload(send_idx);
  L.if_send = c.alloc<double>(size_t(L.n_send));
  L.if_recv = c.alloc<double>(size_t(L.n_recv));
  {
    size_t off = 0;
    for (const auto& nb : plan.neighbors) {
      L.peers.push_back(Peer{nb.rank, L.if_send + off, nb.iface.size(), L.if_recv + off, nb.iface.size()});
      off += nb.iface.size();
    }
  }
  auto iface_of = [&](int g) {
    const int i = plan.iface_of_g[g];
    if (i < 0) throw PmgError(PMG_ERR_DOMAIN, "interface piece dof is not shared");
    return i;
  };

  // ---- pieces
  std::map<const double*, std::pair<const double*, const double*>> vmats;  // V -> (Bfwd, Bbwd)
  auto mats_of = [&](const double* V, int m) {
    auto it = vmats.find(V);
    if (it != vmats.end()) return it->second;
    std::vector<double> bf(size_t(m) * m);
    for (int k = 0; k < m; ++k)
      for (int n = 0; n < m; ++n) bf[size_t(k) * m + n] = V[size_t(n) * m + k];
    const double* dbf = c.upload(bf);
    const double* dbb = c.upload(V, size_t(m) * m);
    return vmats[V] = {dbf, dbb};
  };
  std::map<const double*, const double*> diags;
  auto diag_of = [&](const double* h, long long n) {
    auto it = diags.find(h);
    if (it != diags.end()) return it->second;
    return diags[h] = c.upload(h, size_t(n));
  };
  // reciprocals for the resident-factor FD kernel: x * (1 / d) instead of x / d
  // (an fp64 division is ~40 instructions, 18 per lane and strip in the
  // diagonal pass: 99 us against 63 us for the other passes at c5); at most
  // one ulp from the quotient
  std::map<const double*, const double*> rdiags;
  auto rdiag_of = [&](const double* h, long long n) {
    auto it = rdiags.find(h);
    if (it != rdiags.end()) return it->second;
    std::vector<double> r(static_cast<size_t>(n));
    for (long long i = 0; i < n; ++i) r[size_t(i)] = 1.0 / h[i];
    return rdiags[h] = c.upload(r);
  };
  std::map<std::vector<double>, const double*> linvs;
  std::vector<FdPiece> h_int, h_face;
  std::vector<int> face_dofs, edge_dofs, vert_g;
  std::vector<double> vert_scalar;
  std::vector<EdgePiece> h_edges;
  long long work_int = 0, work_face = 0;
  int maxdim_int = 0, maxdim_face = 0;
  for (int i = 0; i < ld.num_pieces; ++i) {
    const pmg_piece_desc& pc = ld.pieces[i];
    // pieces of other ranks' patches are skipped; interface pieces touching
    // this rank are kept (every replica here takes part in the sum)
    bool mine = false;
    for (int64_t q = 0; q < pc.ndofs && !mine; ++q) {
      const int g = pc.dofs[q];
      if (rep_off[g + 1] > rep_off[g]) mine = true;
    }
    if (!mine) continue;
    if (pc.kind == PMG_PIECE_INTERIOR) {
      if (pc.naxes != d) throw PmgError(PMG_ERR_DOMAIN, "interior piece: axis count mismatch");
      const int k = pc.patch - c.pb;
      // locate the box: the first dof's lattice position is the corner
      const int g0 = pc.dofs[0];
      int slot0 = -1;
      for (int q = rep_off[g0]; q < rep_off[g0 + 1]; ++q)
        if (rep_slot[q] / S == k) slot0 = rep_slot[q];
      if (slot0 < 0) throw PmgError(PMG_ERR_DOMAIN, "interior piece: corner dof not on its patch");
      const long long local0 = slot0 - (long long)k * S;
      int lo[3] = {0, 0, 0};
      long long rem = local0;
      for (int a = 0; a < d; ++a) {
        lo[a] = int(rem % L.ext);
        rem /= L.ext;
      }
      FdPiece fp{};
      fp.naxes = d;
      fp.total = 1;
      for (int a = 0; a < d; ++a) {
        fp.dims[a] = pc.dims[a];
        fp.total *= pc.dims[a];
        if (lo[a] + pc.dims[a] > L.ext) throw PmgError(PMG_ERR_DOMAIN, "interior piece box leaves the lattice");
        maxdim_int = std::max(maxdim_int, pc.dims[a]);
      }
      if (fp.total != pc.ndofs) throw PmgError(PMG_ERR_DOMAIN, "piece smoother: local vector size mismatch");
      // every dof of the box must be the lattice slot in box order (classify_dofs, topology.cpp:408-436)
      {
        int idx[3] = {0, 0, 0};
        for (long long q = 0; q < fp.total; ++q) {
          long long loc = 0;
          for (int a = d - 1; a >= 0; --a) loc = loc * L.ext + (lo[a] + idx[a]);
          if (l2g[(long long)k * S + loc] != pc.dofs[q])
            throw PmgError(PMG_ERR_DOMAIN, "interior piece is not a lattice box");
          for (int a = 0; a < d; ++a) {
            if (++idx[a] < pc.dims[a]) break;
            idx[a] = 0;
          }
        }
      }
      fp.ext = L.ext;
      fp.lat_base = slot0;
      fp.work_off = work_int;
      work_int += fp.total;
      for (int a = 0; a < d; ++a) {
        auto m = mats_of(pc.V[a], pc.dims[a]);
        fp.B[a][0] = m.first;
        fp.B[a][1] = m.second;
      }
      fp.diag = diag_of(pc.diag, fp.total);
      fp.rdiag = rdiag_of(pc.diag, fp.total);
      h_int.push_back(fp);
      L.int_dims.push_back({fp.dims[0], fp.dims[1], fp.dims[2]});
    } else if (pc.kind == PMG_PIECE_FACE) {
      FdPiece fp{};
      fp.naxes = 2;
      fp.total = 1;
      for (int a = 0; a < 2; ++a) {
        fp.dims[a] = pc.dims[a];
        fp.total *= pc.dims[a];
        maxdim_face = std::max(maxdim_face, pc.dims[a]);
        auto m = mats_of(pc.V[a], pc.dims[a]);
        fp.B[a][0] = m.first;
        fp.B[a][1] = m.second;
      }
      if (fp.total != pc.ndofs) throw PmgError(PMG_ERR_DOMAIN, "piece smoother: local vector size mismatch");
      fp.dims[2] = 1;
      fp.work_off = work_face;
      work_face += fp.total;
      fp.diag = diag_of(pc.diag, fp.total);
      fp.rdiag = rdiag_of(pc.diag, fp.total);
      for (int64_t q = 0; q < pc.ndofs; ++q) face_dofs.push_back(iface_of(pc.dofs[q]));
      h_face.push_back(fp);
    } else if (pc.kind == PMG_PIECE_EDGE) {
      if (pc.chol_dim != pc.ndofs) throw PmgError(PMG_ERR_DOMAIN, "piece smoother: local vector size mismatch");
      if (pc.ndofs > 512) throw PmgError(PMG_ERR_CONFIG, "edge pieces longer than 512 dofs are not supported");
      std::vector<double> key(pc.chol_l, pc.chol_l + size_t(pc.chol_dim) * (pc.chol_bw + 1));
      key.push_back(pc.chol_dim);
      key.push_back(pc.chol_bw);
      auto it = linvs.find(key);
      const double* dinv;
      if (it != linvs.end()) {
        dinv = it->second;
      } else {
        dinv = c.upload(banded_inverse(pc.chol_dim, pc.chol_bw, pc.chol_l));
        linvs[key] = dinv;
      }
      h_edges.push_back(EdgePiece{int(pc.ndofs), (long long)edge_dofs.size(), dinv});
      for (int64_t q = 0; q < pc.ndofs; ++q) edge_dofs.push_back(iface_of(pc.dofs[q]));
    } else {
      vert_g.push_back(iface_of(pc.dofs[0]));
      vert_scalar.push_back(pc.scalar);
    }
  }
  for (const auto& fp : h_int) L.int_max_total = std::max(L.int_max_total, fp.total);
  for (const auto& fp : h_face) L.face_max_total = std::max(L.face_max_total, fp.total);
  L.int_max_dim = maxdim_int;
  L.face_max_dim = maxdim_face;
  // one CTA per piece only while the piece is small enough that the pass
  // kernels (many CTAs per piece) would not be faster
  const char* fsm = std::getenv("PMG_FD_SMALL_MAX");
  const long long small_max = fsm ? std::atoll(fsm) : 2048;
  L.int_small = fd_small_smem(L.int_max_total, maxdim_int, d) <= kFdSmallDoubles * sizeof(double) &&
                L.int_max_total <= small_max;
  L.face_small = fd_small_smem(L.face_max_total, maxdim_face, 2) <= kFdSmallDoubles * sizeof(double) &&
                 L.face_max_total <= small_max;
  // pieces ordered so that equal (dims, factors) are adjacent
  auto piece_key = [&](const FdPiece& a) {
    return std::make_tuple(a.dims[0], a.dims[1], a.dims[2], a.B[0][0], a.B[1][0], a.B[2][0]);
  };
  auto by_key = [&](const FdPiece& a, const FdPiece& b) { return piece_key(a) < piece_key(b); };
  std::stable_sort(h_int.begin(), h_int.end(), by_key);
  std::stable_sort(h_face.begin(), h_face.end(), by_key);
  L.n_int = int(h_int.size());
  L.d_int = c.upload(h_int);
  L.n_face = int(h_face.size());
  L.d_face = c.upload(h_face);
  L.face_iface = c.upload(face_dofs);
  L.face_ndof = (long long)face_dofs.size();
  L.n_edges = int(h_edges.size());
  L.d_edges = c.upload(h_edges);
  {
    std::vector<int2> ei;
    for (int e = 0; e < L.n_edges; ++e)
      for (int r0 = 0; r0 < h_edges[e].m; r0 += 32) ei.push_back(make_int2(e, r0));
    L.n_edge_items = int(ei.size());
    L.edge_items = c.upload(ei);
  }
  L.edge_iface = c.upload(edge_dofs);
  L.n_verts = int(vert_g.size());
  L.vert_iface = c.upload(vert_g);
  L.vert_scalar = c.upload(vert_scalar);
  // CTA work items of every pass.  Pieces with the same dims and the same
  // factor for the pass form a group whose rows are concatenated (no per-piece
  // row padding); items = (first piece, row panel, column panel, group rows).
  auto make_items = [&](const std::vector<FdPiece>& ps, int naxes, int4** items, int* counts, int* ntcs,
                        unsigned** queues) {
    for (int pass = 0; pass < 2 * naxes; ++pass) {
      const int axis = pass % naxes, dir = pass / naxes;
      std::vector<std::pair<int, int>> groups;  // (first, count)
      static const bool group_pieces = [] {
        const char* e = std::getenv("PMG_FD_GROUP");
        return !(e && e[0] == '0');
      }();
      for (int i = 0; i < int(ps.size()); ++i) {
        bool same = group_pieces && !groups.empty();
        if (same) {
          const FdPiece& a = ps[groups.back().first];
          const FdPiece& b = ps[i];
          for (int x = 0; x < naxes; ++x) same = same && a.dims[x] == b.dims[x];
          same = same && a.B[axis][dir] == b.B[axis][dir];
        }
        if (same)
          groups.back().second++;
        else
          groups.push_back({i, 1});
      }
      std::vector<long long> cols, weight;
      for (const auto& gr : groups) {
        cols.push_back(ps[gr.first].dims[axis]);
        weight.push_back(ps[gr.first].total * gr.second / ps[gr.first].dims[axis]);
      }
      const int cfg = fd_pick_cfg(cols.data(), weight.data(), int(groups.size()));
      if (!fd_cfg_valid(cfg))
        throw PmgError(PMG_ERR_CONFIG, "no FD kernel for this configuration (PMG_FD_NTC must be 3, 5, 9 or 11)");
      const int BM = fd_cfg_rows(cfg), BN = fd_cfg_cols(cfg);
      std::vector<int4> it;
      if (fd_cfg_resident(cfg)) {
        std::vector<std::pair<int, long long>> gl;
        for (const auto& gr : groups) {
          const long long rows = ps[gr.first].total / ps[gr.first].dims[axis] * gr.second;
          if (rows > INT32_MAX) throw PmgError(PMG_ERR_CONFIG, "FD piece group too large");
          gl.push_back({gr.first, rows});
        }
        fd_resident_items(gl, it);
        queues[pass] = c.alloc<unsigned>(gl.size() + 1);
        ck(cudaMemsetAsync(queues[pass], 0, sizeof(unsigned) * (gl.size() + 1), c.stream), "memset");
      }
      for (const auto& gr : groups) {
        if (fd_cfg_resident(cfg)) break;
        const int K = ps[gr.first].dims[axis];
        const long long rows = ps[gr.first].total / K * gr.second;
        if (rows > INT32_MAX) throw PmgError(PMG_ERR_CONFIG, "FD piece group too large");
        for (long long r0 = 0; r0 < rows; r0 += BM)
          for (int n0 = 0; n0 < K; n0 += BN) it.push_back(make_int4(gr.first, int(r0), n0, int(rows)));
      }
      counts[pass] = int(it.size());
      items[pass] = c.upload(it);
      ntcs[pass] = cfg;
    }
  };
  make_items(h_int, d, L.int_items, L.n_int_items, L.int_ntc, L.int_queue);
  if (d == 3) make_items(h_face, 2, L.face_items, L.n_face_items, L.face_ntc, L.face_queue);

  // ---- two-scale factor (TransferOperator ctor, transfer.cpp:10-19)
  if (l >= 1) {
    const int nf = ld.ts_fine_dim, ncd = ld.ts_coarse_dim;
    int nnz = 0;
    for (int i = 0; i < nf; ++i) nnz = std::max(nnz, ld.ts_row_off[i] + ld.ts_row_len[i]);
    L.ts.fine_dim = nf;
    L.ts.coarse_dim = ncd;
    L.ts.row_start = c.upload(ld.ts_row_start, nf);
    L.ts.row_len = c.upload(ld.ts_row_len, nf);
    L.ts.row_off = c.upload(ld.ts_row_off, nf);
    L.ts.vals = c.upload(ld.ts_vals, size_t(nnz));
    std::vector<int> col_off(size_t(ncd) + 1, 0), col_row;
    std::vector<double> col_val;
    std::vector<std::vector<std::pair<int, double>>> cols(ncd);
    for (int i = 0; i < nf; ++i)
      for (int q = 0; q < ld.ts_row_len[i]; ++q)
        cols[ld.ts_row_start[i] + q].push_back({i, ld.ts_vals[ld.ts_row_off[i] + q]});
    for (int j = 0; j < ncd; ++j) {
      for (auto& e : cols[j]) {
        col_row.push_back(e.first);
        col_val.push_back(e.second);
      }
      col_off[j + 1] = int(col_row.size());
    }
    L.ts.col_off = c.upload(col_off);
    L.ts.col_row = c.upload(col_row);
    L.ts.col_val = c.upload(col_val);
    {  // tile spans (rows and columns of the two-scale matrix are monotone windows)
      bool mono = true;
      for (int i = 1; i < nf; ++i) mono = mono && ld.ts_row_start[i] >= ld.ts_row_start[i - 1];
      int ps = 0, rs = 0;
      for (int i0 = 0; i0 < nf && mono; i0 += 1) {
        const int i1 = std::min(nf, i0 + kTileF);
        int lo = INT32_MAX, hi = 0;
        for (int i = i0; i < i1; ++i) {
          lo = std::min(lo, ld.ts_row_start[i]);
          hi = std::max(hi, ld.ts_row_start[i] + ld.ts_row_len[i]);
        }
        ps = std::max(ps, hi - lo);
      }
      for (int j0 = 0; j0 < ncd && mono; ++j0) {
        const int j1 = std::min(ncd, j0 + kTileC);
        int lo = INT32_MAX, hi = 0;
        for (int j = j0; j < j1; ++j)
          for (int q = col_off[j]; q < col_off[j + 1]; ++q) {
            lo = std::min(lo, col_row[q]);
            hi = std::max(hi, col_row[q] + 1);
          }
        rs = std::max(rs, hi - lo);
      }
      L.ts.pspan = mono ? ps : 0;
      L.ts.rspan = mono ? rs : 0;
    }
    if (nf != L.ext) throw PmgError(PMG_ERR_DOMAIN, "transfer: fine level must have twice the elements");
  }
  L.f = c.alloc<double>(size_t(L.lat_n));
  L.u = c.alloc<double>(size_t(L.lat_n));
  L.r = c.alloc<double>(size_t(L.lat_n));
  ck(cudaMemsetAsync(L.f, 0, sizeof(double) * L.lat_n, c.stream), "memset");
  ck(cudaMemsetAsync(L.u, 0, sizeof(double) * L.lat_n, c.stream), "memset");
  ck(cudaMemsetAsync(L.r, 0, sizeof(double) * L.lat_n, c.stream), "memset");
}

void build_ctx(pmg_ctx& c, const pmg_hierarchy_desc& D) {
  c.dim = D.dim;
  c.degree = D.degree;
  c.K_global = D.num_patches;
  c.nl = D.num_levels;
  c.prm = D.params;
  if (D.dim < 2 || D.dim > 3) throw PmgError(PMG_ERR_CONFIG, "dimension must be 2 or 3");
  if (D.num_levels < 2) throw PmgError(PMG_ERR_CONFIG, "need at least one refinement level");
  if (D.params.nu < 1 || D.params.mu < 1 || D.params.mu > 2) throw PmgError(PMG_ERR_CONFIG, "bad cycle parameters");
  c.lv.resize(c.nl);
  if (D.geometry) {
    c.geo.assign(D.geometry, D.geometry + D.num_patches);
    c.geo_ctrl.resize(D.num_patches);
    for (int k = 0; k < D.num_patches; ++k) {
      size_t n = D.dim;
      for (int a = 0; a < D.dim; ++a) n *= size_t(c.geo[k].elements[a] + c.geo[k].degree[a]);
      c.geo_ctrl[k].assign(D.geometry[k].ctrl, D.geometry[k].ctrl + n);
      c.geo[k].ctrl = c.geo_ctrl[k].data();
    }
  }
  fd_configure();
  size_t work_n = 1, tbuf_n = 1, face_n = 1;
  for (int l = 0; l < c.nl; ++l) {
    build_level(c, D, l);
    const pmg_level_desc& ld = D.levels[l];
    long long wi = 0, wf = 0;
    for (int i = 0; i < ld.num_pieces; ++i) {
      const pmg_piece_desc& pc = ld.pieces[i];
      if (pc.kind == PMG_PIECE_INTERIOR) wi += pc.ndofs;
      if (pc.kind == PMG_PIECE_FACE) wf += pc.ndofs;
    }
    work_n = std::max(work_n, size_t(std::max(wi, wf)));
    face_n = std::max(face_n, size_t(wf));
    if (l >= 1) {  // largest intermediate of the tensor transfer: ext_c * ext_f^(d-1) per patch
      long long t = c.lv[l - 1].ext;
      for (int a = 1; a < c.dim; ++a) t *= c.lv[l].ext;
      tbuf_n = std::max(tbuf_n, size_t(t * c.lv[l].K));
      tbuf_n = std::max(tbuf_n, size_t(c.lv[l].lat_n));
    }
  }
  c.work[0] = c.alloc<double>(work_n);
  c.work[1] = c.alloc<double>(work_n);
  c.face_buf[0] = c.alloc<double>(face_n);
  c.face_buf[1] = c.alloc<double>(face_n);
  c.tbuf[0] = c.alloc<double>(tbuf_n);
  c.tbuf[1] = c.alloc<double>(tbuf_n);
  // coarse solve (Hierarchy::coarse_solve): explicit inverse for a GEMV
  c.n0 = D.coarse_n;
  if (c.n0 != c.lv[0].N) throw PmgError(PMG_ERR_DOMAIN, "coarse matrix size does not match level 0");
  c.Ainv = c.upload(spd_inverse(c.n0, D.coarse_L));
  c.coarse_rhs = c.alloc<double>(size_t(c.n0));
  c.coarse_x = c.alloc<double>(size_t(c.n0));
  c.rank_buf = c.alloc<double>(size_t(c.size));
  c.coarse_parts = c.alloc<double>(size_t(c.size) * std::max(c.n0, 1));
  long long maxlat = 0;
  for (auto& L : c.lv) maxlat = std::max(maxlat, L.lat_n);
  c.partial_n = dot_blocks(maxlat);
  for (auto& L : c.lv) c.partial_n = std::max(c.partial_n, level_spmv_partials(c, L));
  c.partial = c.alloc<double>(size_t(c.partial_n));
  c.scal = c.alloc<double>(16);
  ck(cudaMemsetAsync(c.scal, 0, 16 * sizeof(double), c.stream), "memset");
  ck(cudaMallocHost(&c.h_scal, 16 * sizeof(double)), "cudaMallocHost");
  c.loop_state = c.alloc<PcgLoopState>(1);
  ck(cudaMallocHost(&c.h_loop, sizeof(PcgLoopState)), "cudaMallocHost");
  {
    const char* e = std::getenv("PMG_HOST_LOOP");
    c.device_loop = !(e && e[0] == '1') && !c.multi();
  }
  const DevLevel& F = c.lv.back();
  c.staging_n = std::max<long long>(F.N, 1);
  c.staging = c.alloc<double>(size_t(c.staging_n));
  for (double** v : {&c.pcg_r, &c.pcg_z, &c.pcg_p, &c.pcg_Ap, &c.pcg_acc, &c.pcg_u, &c.pcg_f}) {
    *v = c.alloc<double>(size_t(F.lat_n));
    ck(cudaMemsetAsync(*v, 0, sizeof(double) * F.lat_n, c.stream), "memset");
  }
  ck(cudaStreamSynchronize(c.stream), "build sync");
  ck(cudaGetLastError(), "build kernels");
}

// ================================================================ operations
// All launch on c.stream and count their kernels.

struct TimedScope {
  pmg_ctx& c;
  pmg_ctx::Timed t{};
  bool on;
  TimedScope(pmg_ctx& ctx, int cls, int level, double work) : c(ctx), on(ctx.profiling) {
    if (!on) return;
    t = pmg_ctx::Timed{cls, level, work, c.get_event(), c.get_event()};
    ck(cudaEventRecord(t.a, c.stream), "cudaEventRecord");
  }
  ~TimedScope() {
    if (!on) return;
    cudaEventRecord(t.b, c.stream);
    c.timed.push_back(t);
  }
};

// reference CSR entries per level (harness.cpp:274-282) for one patch
long long stored_per_patch(int degree, int elements, int dim) {
  const int extent = elements + degree;
  long long pairs = 0;
  for (int i = 0; i < extent; ++i) pairs += std::min(i + degree, extent - 1) - std::max(i - degree, 0) + 1;
  long long pp = 1;
  for (int a = 0; a < dim; ++a) pp *= pairs;
  return pp;
}

// dot partials one op_spmv launch of the level writes
int level_spmv_partials(const pmg_ctx& c, const DevLevel& L) {
  if (L.kron) return kron_partials(c.dim, c.degree, L.ext, L.S, L.K);
  return spmv_partials(c.dim, c.degree, L.S, L.K, L.Ob != L.O, c.sweep, c.sweep3);
}

void op_spmv(pmg_ctx& c, int l, const double* x, const double* f, double* y, double* dot_partial = nullptr) {
  const DevLevel& L = c.lv[l];
  if (L.kron) {
    // algorithmic bytes: x, y (and f) plus the 4-byte Dirichlet map per lattice row
    TimedScope ts(c, 0, l, (8.0 * (f ? 3 : 2) + 4.0) * L.lat_n);
    KronArgs a{c.dim, c.degree, L.ext, L.S, L.K, L.kron_M, L.kron_K, L.kron_g, L.l2g, x, f, y, dot_partial,
               L.kron_scratch};
    int n = 0;
    launch_kron_spmv(c.stream, a, &n);
    c.launches += n;
    c.spmv_launches++;
    return;
  }
  // algorithmic bytes: the stored entries of the reference's CSR (harness.cpp:274-282),
  // or with the symmetric half band (stored + diagonal) / 2
  const double entries = double(stored_per_patch(c.degree, L.n, c.dim));
  const double band_entries = L.Ob == L.O ? entries : 0.5 * (entries + double(L.S));
  const double bytes = 8.0 * band_entries * L.K + 8.0 * L.lat_n * (f ? 3 : 2);
  if (L.Ob != L.O && (reinterpret_cast<uintptr_t>(x) & 15))
    throw PmgError(PMG_ERR_CONFIG, "half-band SpMV needs a 16-byte aligned x (TMA window)");
  TimedScope ts(c, 0, l, bytes);
  SpmvArgs a{c.dim, c.degree, L.ext, L.S, L.K, L.band, x, f, y, dot_partial, L.Ob != L.O, L.Sp, c.sweep,
             L.sweep_scratch, L.sweep_flags, L.sweep_ticket, c.sweep3};
  launch_spmv(c.stream, a);
  c.launches++;
  c.spmv_launches++;
}

// flops of one pass over every interior piece of a level: 2 R K N per piece
double fd_pass_flops(const DevLevel& L, const std::vector<std::array<int, 3>>& dims, int naxes, int pass) {
  (void)L;
  double f = 0.0;
  for (const auto& d : dims) {
    double tot = 1.0;
    for (int a = 0; a < naxes; ++a) tot *= d[a];
    f += 2.0 * tot * d[pass % naxes];
  }
  return f;
}

// Sigma on the interface dofs of a distributed vector r: this rank's replica
// partials, the neighbour exchange, and the ascending-rank fold into L.if_t.
void op_iface_sum(pmg_ctx& c, int l, const double* r) {
  DevLevel& L = c.lv[l];
  launch_iface_partial(c.stream, L.n_iface, L.if_rep_off, L.if_rep_slot, r, L.if_tloc);
  if (L.n_iface) c.launches++;
  if (c.multi()) {
    launch_iface_pack(c.stream, L.n_send, L.if_send_idx, L.if_tloc, L.if_send);
    if (L.n_send) c.launches++;
    c.comm->exchange(c.stream, L.peers);
  }
  if (c.multi()) {  // on one rank the fold is the identity: totals = if_tloc
    launch_iface_combine(c.stream, L.n_iface, L.if_comb_off, L.if_comb_src, L.if_tloc, L.if_recv, L.if_t);
    if (L.n_iface) c.launches++;
  }
}

// smooth: interior FD, faces, edges + vertices.  out_mode SET: out = alpha z
// on every piece slot; ADD: out += alpha z.
void op_smooth_iface(pmg_ctx& c, int l, const double* r, double* out, bool add, double alpha);

void op_smooth(pmg_ctx& c, int l, const double* r, double* out, bool add, double alpha) {
  const DevLevel& L = c.lv[l];
  const int d = c.dim;
  const int np = 2 * d;
  // small levels on one rank: the whole smoother in one launch (interface
  // totals summed from the replicas inside the kernel)
  static const bool fused_ok = [] {
    const char* e = std::getenv("PMG_NO_FUSED_SMOOTH");
    return !(e && e[0] == '1');
  }();
  if (fused_ok && !c.multi() && L.int_small && (L.n_face == 0 || L.face_small)) {
    double flops = 0.0;
    for (int pass = 0; pass < np; ++pass) flops += fd_pass_flops(L, L.int_dims, d, pass);
    TimedScope ts(c, 1, l, flops);
    SmoothSmallArgs a{};
    a.d = d;
    a.ints = L.d_int;
    a.n_int = L.n_int;
    a.faces = L.d_face;
    a.n_face = L.n_face;
    a.face_iface = L.face_iface;
    a.edges = L.d_edges;
    a.edge_items = L.edge_items;
    a.n_edge_items = L.n_edge_items;
    a.edge_iface = L.edge_iface;
    a.vert_iface = L.vert_iface;
    a.vert_scalar = L.vert_scalar;
    a.nverts = L.n_verts;
    a.rep_off = L.if_rep_off;
    a.rep_slot = L.if_rep_slot;
    a.r = r;
    a.out = out;
    a.add = add ? 1 : 0;
    a.alpha = alpha;
    const size_t smem = std::max(fd_small_smem(L.int_max_total, L.int_max_dim, d),
                                 fd_small_smem(L.face_max_total, L.face_max_dim, 2));
    if (const char* dbg = std::getenv("PMG_DEBUG_SMOOTH")) {  // timing experiments only
      if (dbg[0] == '1') a.n_edge_items = a.nverts = 0;
      if (dbg[0] == '2') a.n_int = a.n_face = 0;
    }
    launch_smooth_small(c.stream, a, smem);
    c.launches++;
    return;
  }
  // interface pieces first, on the side stream when overlapping
  const cudaStream_t main = c.stream;
  const bool fork = c.overlap && !c.profiling && L.n_int > 0;
  if (fork) {
    ck(cudaEventRecord(c.ev_fork, main), "cudaEventRecord");
    ck(cudaStreamWaitEvent(c.side_stream, c.ev_fork, 0), "cudaStreamWaitEvent");
    c.stream = c.side_stream;
  }
  try {
    op_smooth_iface(c, l, r, out, add, alpha);
  } catch (...) {
    c.stream = main;
    throw;
  }
  if (fork) {
    ck(cudaEventRecord(c.ev_join, c.side_stream), "cudaEventRecord");
    c.stream = main;
  }
  if (L.int_small) {
    double flops = 0.0;
    for (int pass = 0; pass < np; ++pass) flops += fd_pass_flops(L, L.int_dims, d, pass);
    TimedScope ts(c, 1, l, flops);
    launch_fd_small(c.stream, L.d_int, L.n_int, d, L.int_max_total, L.int_max_dim, FD_IN_LATTICE,
                    add ? FD_OUT_LATTICE_ADD : FD_OUT_LATTICE_SET, r, out, alpha, nullptr, nullptr);
    if (L.n_int) c.launches++;
  }
  for (int pass = 0; pass < np && !L.int_small; ++pass) {
    const int in_mode = pass == 0 ? FD_IN_LATTICE : FD_IN_WORK;
    int out_mode = FD_OUT_WORK;
    if (pass == d - 1) out_mode = FD_OUT_WORK_DIAG;
    if (pass == np - 1) out_mode = add ? FD_OUT_LATTICE_ADD : FD_OUT_LATTICE_SET;
    TimedScope ts(c, 1, l, fd_pass_flops(L, L.int_dims, d, pass));
    launch_fd_pass(c.stream, L.d_int, L.int_items[pass], L.n_int_items[pass], L.int_ntc[pass], pass, d, in_mode,
                   out_mode, r, out,
                   alpha, c.work[(pass + 1) & 1], c.work[pass & 1], L.int_queue[pass]);
    if (L.n_int_items[pass]) c.launches++;
  }
  if (fork) ck(cudaStreamWaitEvent(main, c.ev_join, 0), "cudaStreamWaitEvent");
}

void op_smooth_iface(pmg_ctx& c, int l, const double* r, double* out, bool add, double alpha) {
  const DevLevel& L = c.lv[l];
  const int d = c.dim;
  // interface pieces act on the summed residual: Sigma over every replica
  // (all ranks), then each rank solves the pieces it touches and writes its
  // local replicas (ParallelBackend::smooth = accumulate(apply_pieces(r)),
  // parallel.cpp:353-355, with the sum taken before the linear piece solves)
  TimedScope ts_iface(c, 3, l, 0.0);
  op_iface_sum(c, l, r);
  if (d == 3 && L.n_face > 0) {
    launch_gather_t(c.stream, L.face_ndof, L.face_iface, L.if_total, c.face_buf[1]);
    c.launches++;
    const double* res = c.face_buf[1];
    if (L.face_small) {
      launch_fd_small(c.stream, L.d_face, L.n_face, 2, L.face_max_total, L.face_max_dim, FD_IN_WORK, FD_OUT_WORK,
                      nullptr, nullptr, 0.0, c.face_buf[1], c.face_buf[0]);
      c.launches++;
      res = c.face_buf[0];
    } else {
      for (int pass = 0; pass < 4; ++pass) {
        const int out_mode = pass == 1 ? FD_OUT_WORK_DIAG : FD_OUT_WORK;
        launch_fd_pass(c.stream, L.d_face, L.face_items[pass], L.n_face_items[pass], L.face_ntc[pass], pass, 2,
                       FD_IN_WORK, out_mode,
                       nullptr, nullptr, 0.0, c.face_buf[(pass + 1) & 1], c.face_buf[pass & 1], L.face_queue[pass]);
        c.launches++;
      }
    }
    launch_scatter_iface(c.stream, L.face_ndof, L.face_iface, L.if_rep_off, L.if_rep_slot, res, out, add ? 1 : 0,
                         alpha);
    c.launches++;
  }
  if (L.n_edges + L.n_verts > 0) {
    launch_edges_vertices(c.stream, L.d_edges, L.edge_items, L.n_edge_items, L.edge_iface, L.vert_iface,
                          L.vert_scalar, L.n_verts, L.if_rep_off, L.if_rep_slot, L.if_total, out, add ? 1 : 0, alpha);
    c.launches++;
  }
}

// one-pass tensor transfers for 2D and for small 3D lattices; large 3D
// lattices keep the axis-by-axis passes (fewer redundant loads)
bool fused_transfer(const pmg_ctx& c, const DevLevel& F) { return c.dim == 2 || F.S <= 40000; }
bool tiled_transfers() {
  static const bool on = [] {
    const char* e = std::getenv("PMG_NO_TILED_TRANSFER");
    return !(e && e[0] == '1');
  }();
  return on;
}

// restriction level l -> l-1 on distributed shares; out coarse (dist)
void op_restrict(pmg_ctx& c, int l, const double* r, double* out) {
  const DevLevel& F = c.lv[l];
  const DevLevel& C = c.lv[l - 1];
  TimedScope ts(c, 2, l, 0.0);
  if (c.dim == 2 && F.ts.rspan > 0 && tiled_transfers()) {
    launch_restrict_tile2d(c.stream, F.ts, F.K, F.ext, C.ext, r, out, C.l2g);
    c.launches++;
    return;
  }
  if (fused_transfer(c, F)) {
    launch_restrict_fused(c.stream, F.ts, F.K, c.dim, F.ext, C.ext, r, out, C.l2g);
    c.launches++;
    return;
  }
  int dims[3] = {F.ext, F.ext, F.ext};
  const double* src = r;
  for (int a = 0; a < c.dim; ++a) {
    const bool last = a == c.dim - 1;
    double* dst = last ? out : c.tbuf[a & 1];
    launch_ts_axis(c.stream, F.ts, true, F.K, c.dim, dims, a, src, dst, last ? 1 : 0, C.l2g);
    c.launches++;
    dims[a] = C.ext;
    src = dst;
  }
}

// u(level l) += coef * P coarse(level l-1)
void op_prolong_add(pmg_ctx& c, int l, const double* coarse, double coef, double* u) {
  const DevLevel& F = c.lv[l];
  const DevLevel& C = c.lv[l - 1];
  TimedScope ts(c, 2, l, 0.0);
  if (c.dim == 2 && F.ts.pspan > 0 && tiled_transfers()) {
    launch_prolong_tile2d(c.stream, F.ts, F.K, F.ext, C.ext, coarse, coef, u, F.l2g);
    c.launches++;
    return;
  }
  if (fused_transfer(c, F)) {
    launch_prolong_fused(c.stream, F.ts, F.K, c.dim, F.ext, C.ext, coarse, coef, u, F.l2g);
    c.launches++;
    return;
  }
  int dims[3] = {C.ext, C.ext, C.ext};
  const double* src = coarse;
  for (int a = 0; a < c.dim; ++a) {
    const bool last = a == c.dim - 1;
    double* dst = last ? u : c.tbuf[a & 1];
    launch_ts_axis(c.stream, F.ts, false, F.K, c.dim, dims, a, src, dst, last ? 2 : 0, F.l2g, coef);
    c.launches++;
    dims[a] = F.ext;
    src = dst;
  }
}

// coarse_solve (parallel.cpp:411-422): the global coarse residual is the sum
// of every replica share; on several ranks the per-rank partials go to rank 0,
// which sums them in ascending rank order, solves, and broadcasts the result
void op_coarse(pmg_ctx& c, const double* r, double* out) {
  const DevLevel& L = c.lv[0];
  TimedScope ts(c, 5, 0, 0.0);
  launch_coarse_gather(c.stream, L.rep_off, L.rep_slot, c.n0, r, c.coarse_rhs);
  c.launches++;
  if (c.multi()) {
    c.comm->gather(c.stream, c.coarse_rhs, c.coarse_parts, size_t(c.n0), 0);
    if (c.rank == 0) {
      launch_sum_ranks(c.stream, c.coarse_parts, c.size, c.n0, c.coarse_rhs);
      c.launches++;
    }
  }
  if (c.rank == 0) {
    launch_coarse_gemv(c.stream, c.Ainv, c.n0, c.coarse_rhs, c.coarse_x);
    c.launches++;
  }
  if (c.multi()) c.comm->broadcast(c.stream, c.coarse_x, size_t(c.n0), 0);
  launch_coarse_scatter(c.stream, L.l2g, L.lat_n, c.coarse_x, out);
  c.launches++;
}

// dot(dist a, acc b) into a device scalar, reduced over ranks in ascending
// rank order (Communicator::allreduce_sum, parallel.cpp:21-28)
void op_dot(pmg_ctx& c, int l, const double* a, const double* b, double* dst) {
  const DevLevel& L = c.lv[l];
  TimedScope ts(c, 4, l, 0.0);
  launch_dot_partial(c.stream, a, b, L.lat_n, c.partial);
  launch_sum_partials(c.stream, c.partial, dot_blocks(L.lat_n), dst);
  c.launches += 2;
  if (c.multi()) {
    c.comm->allgather(c.stream, dst, c.rank_buf, 1);
    launch_sum_ranks(c.stream, c.rank_buf, c.size, 1, dst);
    c.launches++;
  }
}

// accumulate (parallel.cpp:306-337): out = r with every interface replica
// replaced by the interface total
void op_accumulate(pmg_ctx& c, int l, const double* r, double* out) {
  DevLevel& L = c.lv[l];
  TimedScope ts(c, 4, l, 0.0);
  op_iface_sum(c, l, r);
  if (out != r) {
    launch_copy(c.stream, r, out, L.lat_n);
    c.launches++;
  }
  launch_iface_scatter(c.stream, L.n_iface, L.if_rep_off, L.if_rep_slot, L.if_total, out);
  if (L.n_iface) c.launches++;
}

// mg_cycle_generic (multigrid.hpp:120-141) on the ctx workspace.
// `zero` marks u == 0 on entry (every recursive call and mg_precondition).
void cycle(pmg_ctx& c, int l, double* u, const double* f, bool zero) {
  DevLevel& L = c.lv[l];
  const double tau = c.prm.tau;
  for (int i = 0; i < c.prm.nu; ++i) {
    if (zero && i == 0) {
      op_smooth(c, l, f, u, false, tau);  // u = 0 + tau L^-1 (f - A 0)
    } else {
      op_spmv(c, l, u, f, L.r);
      op_smooth(c, l, L.r, u, true, tau);
    }
  }
  op_spmv(c, l, u, f, L.r);
  DevLevel& C = c.lv[l - 1];
  op_restrict(c, l, L.r, C.f);
  if (l == 1) {
    op_coarse(c, C.f, C.u);
  } else {
    for (int i = 0; i < c.prm.mu; ++i) cycle(c, l - 1, C.u, C.f, i == 0);
  }
  op_prolong_add(c, l, C.u, c.prm.damp_coarse ? tau : 1.0, u);
  for (int i = 0; i < c.prm.nu; ++i) {
    op_spmv(c, l, u, f, L.r);
    op_smooth(c, l, L.r, u, true, tau);
  }
}

void precondition(pmg_ctx& c, const double* r, double* z) {
  // z starts as zero: every piece slot is written by the first smooth (SET),
  // Dirichlet slots of z are never written and stay 0
  cycle(c, c.nl - 1, z, r, true);
}

void sync_check(pmg_ctx& c) {
  ck(cudaStreamSynchronize(c.stream), "stream sync");
  ck(cudaGetLastError(), "kernel launch");
}

// The PCG iteration pieces shared by the host-driven and the device loop.
struct PcgParts {
  pmg_ctx& c;
  const double* f;
  double* u;
  int Lf;
  long long n;
  double *r, *z, *p, *Ap, *racc, *s;
  PcgParts(pmg_ctx& ctx, const double* f_, double* u_)
      : c(ctx), f(f_), u(u_), Lf(ctx.nl - 1), n(ctx.lv.back().lat_n), r(ctx.pcg_r), z(ctx.pcg_z), p(ctx.pcg_p),
        Ap(ctx.pcg_Ap), racc(ctx.pcg_acc), s(ctx.scal) {}
  void norm2() {  // sqrt(dot(r, accumulate(r)))
    op_accumulate(c, Lf, r, racc);
    op_dot(c, Lf, r, racc, s + 5);
    launch_pcg_scalars(c.stream, 2, s);
    c.launches++;
  }
  void start() {  // u = 0, r = f, |r0|
    launch_fill(c.stream, u, n, 0.0);
    launch_copy(c.stream, f, r, n);
    c.launches += 2;
    norm2();
  }
  // iteration front: Ap, alpha, u += alpha p, r -= alpha Ap, |r|
  void front() {
    const DevLevel& F = c.lv[Lf];
    op_spmv(c, Lf, p, nullptr, Ap, c.partial);  // Ap and the partials of Ap.p
    launch_sum_partials(c.stream, c.partial, level_spmv_partials(c, F), s + 1);
    if (c.multi()) {  // pAp over all ranks, ascending rank order
      c.comm->allgather(c.stream, s + 1, c.rank_buf, 1);
      launch_sum_ranks(c.stream, c.rank_buf, c.size, 1, s + 1);
      c.launches++;
    }
    launch_pcg_scalars(c.stream, 0, s);  // alpha = rz / pAp
    launch_axpy(c.stream, 0.0, s + 2, 1.0, p, u, n);
    launch_axpy(c.stream, 0.0, s + 2, -1.0, Ap, r, n);
    c.launches += 4;
    norm2();
  }
  // iteration back: z = M r, beta, p = z + beta p
  void back() {
    precondition(c, r, z);
    op_dot(c, Lf, r, z, s + 3);          // rz_next
    launch_pcg_scalars(c.stream, 1, s);  // beta, rz = rz_next
    launch_xpay(c.stream, z, 0.0, s + 4, p, n);
    c.launches += 2;
  }
};

// pcg_generic (multigrid.hpp:155-189) driven from the host: two graphs per
// iteration (front, back); the back half is enqueued before the host has
// seen |r|, so after the last iteration one V-cycle is computed and dropped.
// Multi-rank contexts and PMG_HOST_LOOP=1 take this path.
int pcg_host_loop(pmg_ctx& c, const double* f, double tol, int max_iter, double* u, double* history, int* iters) {
  PcgParts P(c, f, u);
  double* s = c.scal;
  auto read_scalars = [&]() {
    ck(cudaMemcpyAsync(c.h_scal, s, 8 * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "scalar D2H");
    sync_check(c);
  };
  P.start();
  read_scalars();
  const double r0 = c.h_scal[6];
  history[0] = r0;
  *iters = 0;
  if (r0 == 0.0) return PMG_OK;
  launch_fill(c.stream, P.z, P.n, 0.0);
  c.launches++;
  precondition(c, P.r, P.z);
  launch_copy(c.stream, P.z, P.p, P.n);
  c.launches++;
  op_dot(c, P.Lf, P.r, P.z, s + 0);  // rz
  auto front = [&]() {
    P.front();
    ck(cudaMemcpyAsync(c.h_scal, s, 8 * sizeof(double), cudaMemcpyDeviceToHost, c.stream), "scalar D2H");
  };
  auto back = [&]() { P.back(); };
  const bool graphs = c.use_graphs && !c.profiling;
  if (graphs && c.graph_u != u) {
    c.capture(c.graph_front, c.graph_front_launches, front);
    c.capture(c.graph_back, c.graph_back_launches, back);
    c.graph_u = u;
  }
  for (int k = 1; k <= max_iter; ++k) {
    if (graphs) {
      c.launch_graph(c.graph_front, c.graph_front_launches);
    } else {
      front();
    }
    ck(cudaEventRecord(c.ev_norm, c.stream), "cudaEventRecord");
    // with graphs the back half is enqueued speculatively (the GPU never
    // waits for the host); direct launches (profiling) stop exactly as
    // pcg_generic does, so an instrumented solve runs the device loop's kernels
    if (graphs && k < max_iter) c.launch_graph(c.graph_back, c.graph_back_launches);
    ck(cudaEventSynchronize(c.ev_norm), "cudaEventSynchronize");
    if (c.h_scal[7] != 0.0) {
      c.h_scal[7] = 0.0;
      sync_check(c);
      ck(cudaMemsetAsync(s + 7, 0, sizeof(double), c.stream), "memset");
      throw PmgError(PMG_ERR_DEFINITENESS, "pcg: search direction with nonpositive energy");
    }
    const double rn = c.h_scal[6];
    history[k] = rn;
    *iters = k;
    if (rn <= tol * r0) return PMG_OK;
    if (!graphs && k < max_iter) back();
  }
  return PMG_ERR_DIVERGENCE;
}

// Capture the whole solve as one graph: head (u = 0, r = f, |r0|, loop
// condition, z = p = 0, rz = +inf) and a WHILE node whose body is one PCG
// iteration in the order back, front, check.  With rz = +inf the first
// body's beta is 0 and p = z + 0 p = z exactly, and its rz = r.z is the same
// dot as the host loop's, so both loops produce the same bits.
void capture_loop(pmg_ctx& c, pmg_ctx::LoopGraph& g, const double* f, double* u) {
  if (g.exec) {
    cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
  }
  g.f = g.u = nullptr;
  PcgParts P(c, f, u);
  cudaGraph_t graph = nullptr;
  ck(cudaGraphCreate(&graph, 0), "cudaGraphCreate");
  cudaStream_t saved = c.stream;
  const long long before = c.launches;
  bool capturing = false;
  try {
    cudaGraphConditionalHandle handle;
    ck(cudaGraphConditionalHandleCreate(&handle, graph, 0, cudaGraphCondAssignDefault), "conditional handle");
    c.stream = c.own_stream;
    ck(cudaStreamBeginCaptureToGraph(c.own_stream, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
       "capture head");
    capturing = true;
    P.start();
    launch_pcg_check(c.stream, 1, c.loop_state, c.scal, c.loop_hist, handle);
    launch_fill(c.stream, P.z, P.n, 0.0);
    launch_fill(c.stream, P.p, P.n, 0.0);
    c.launches += 3;
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    ck(cudaStreamGetCaptureInfo(c.own_stream, &st, nullptr, nullptr, &deps, &ndeps), "capture info");
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    ck(cudaGraphAddNode(&cnode, graph, deps, ndeps, &cp), "while node");
    ck(cudaStreamUpdateCaptureDependencies(c.own_stream, &cnode, 1, cudaStreamSetCaptureDependencies),
       "capture dependencies");
    cudaGraph_t tmp = nullptr;
    capturing = false;
    ck(cudaStreamEndCapture(c.own_stream, &tmp), "end capture head");
    g.head = c.launches - before;
    const long long mid = c.launches;
    ck(cudaStreamBeginCaptureToGraph(c.own_stream, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal),
       "capture body");
    capturing = true;
    P.back();
    P.front();
    launch_pcg_check(c.stream, 0, c.loop_state, c.scal, c.loop_hist, handle);
    c.launches++;
    capturing = false;
    ck(cudaStreamEndCapture(c.own_stream, &tmp), "end capture body");
    g.body = c.launches - mid;
    ck(cudaGraphInstantiate(&g.exec, graph, 0), "instantiate loop graph");
  } catch (...) {
    if (capturing) {
      cudaGraph_t tmp = nullptr;
      cudaStreamEndCapture(c.own_stream, &tmp);
    }
    cudaGraphDestroy(graph);
    c.stream = saved;
    c.launches = before;
    throw;
  }
  cudaGraphDestroy(graph);
  c.stream = saved;
  c.launches = before;
  g.f = f;
  g.u = u;
}

int pcg_device_loop(pmg_ctx& c, const double* f, double tol, int max_iter, double* u, double* history, int* iters) {
  if (c.loop_hist_cap < max_iter + 1) {  // the history buffer is baked into the graphs
    const int cap = std::max(max_iter + 1, 501);
    if (c.loop_hist) c.release(c.loop_hist, size_t(c.loop_hist_cap));
    c.loop_hist = c.alloc<double>(size_t(cap));
    c.loop_hist_cap = cap;
    for (auto& g : c.loop) g.f = g.u = nullptr;
  }
  pmg_ctx::LoopGraph* g = nullptr;
  for (auto& cand : c.loop)
    if (cand.exec && cand.f == f && cand.u == u) g = &cand;
  if (!g) {
    g = &c.loop[c.loop_next];
    c.loop_next ^= 1;
    capture_loop(c, *g, f, u);
  }
  c.h_loop->k = 0;
  c.h_loop->status = 0;
  c.h_loop->max_iter = max_iter;
  c.h_loop->tol = tol;
  c.h_loop->r0 = 0.0;
  ck(cudaMemcpyAsync(c.loop_state, c.h_loop, sizeof(PcgLoopState), cudaMemcpyHostToDevice, c.stream), "state H2D");
  ck(cudaGraphLaunch(g->exec, c.stream), "cudaGraphLaunch");
  ck(cudaMemcpyAsync(c.h_loop, c.loop_state, sizeof(PcgLoopState), cudaMemcpyDeviceToHost, c.stream), "state D2H");
  sync_check(c);
  const int k = c.h_loop->k;
  ck(cudaMemcpy(history, c.loop_hist, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost), "history D2H");
  c.launches += g->head + (long long)k * g->body;
  *iters = k;
  switch (c.h_loop->status) {
    case 1: return PMG_OK;
    case 2: throw PmgError(PMG_ERR_DEFINITENESS, "pcg: search direction with nonpositive energy");
    case 3: return PMG_ERR_DIVERGENCE;
    default: throw PmgError(PMG_ERR_GENERIC, "pcg: device loop ended without a decision");
  }
}

int pcg_device(pmg_ctx& c, const double* f, double tol, int max_iter, double* u, double* history, int* iters) {
  if (c.device_loop && c.use_graphs && !c.profiling)
    return pcg_device_loop(c, f, tol, max_iter, u, history, iters);
  return pcg_host_loop(c, f, tol, max_iter, u, history, iters);
}

template <class F>
int guarded(pmg_ctx* c, F&& f) {
  try {
    if (c) ck(cudaSetDevice(c->device), "cudaSetDevice");
    f();
    return PMG_OK;
  } catch (const PmgError& e) {
    if (c) c->err = e.what();
    return e.code;
  } catch (const TransportFailure& e) {
    if (c) c->err = e.what();
    return PMG_ERR_TRANSPORT;
  } catch (const LaunchError& e) {
    if (c) c->err = e.what();
    return PMG_ERR_CUDA;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return PMG_ERR_GENERIC;
  }
}

void need(bool ok, int code, const char* msg) {
  if (!ok) throw PmgError(code, msg);
}

void check_vec(const pmg_ctx* c, const pmg_vec* v, int level) {
  need(v != nullptr && v->ctx == c, PMG_ERR_DOMAIN, "vector belongs to another context");
  need(v->level == level, PMG_ERR_DOMAIN, "vector level mismatch");
}

}  // namespace

// ================================================================ C ABI
extern "C" {

const char* pmg_last_error(pmg_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

int pmg_ctx_create(const pmg_hierarchy_desc* desc, int device, const pmg_comm_desc* comm, pmg_ctx** out) {
  if (!desc || !out) {
    g_create_error = "pmg_ctx_create: null argument";
    return PMG_ERR_CONFIG;
  }
  *out = nullptr;
  auto c = std::make_unique<pmg_ctx>();
  c->device = device;
  c->pb = 0;
  c->pe = desc->num_patches;
  try {
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    need(device >= 0 && device < ndev, PMG_ERR_CONFIG, "device index out of range");
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (comm) {
      need(comm->size >= 1 && comm->rank >= 0 && comm->rank < comm->size, PMG_ERR_CONFIG, "bad rank description");
      need(comm->size <= desc->num_patches && comm->size <= 64, PMG_ERR_CONFIG, "partition: bad rank count");
      // the exchange plans assume contiguous_partition (parallel.cpp:181-198)
      const pmgplan::Partition part = pmgplan::contiguous(desc->num_patches, comm->size);
      need(comm->patch_begin == part.patch_begin[comm->rank] && comm->patch_end == part.patch_begin[comm->rank + 1],
           PMG_ERR_CONFIG, "patch range is not the contiguous partition block of this rank");
      c->rank = comm->rank;
      c->size = comm->size;
      c->pb = comm->patch_begin;
      c->pe = comm->patch_end;
      if (comm->size > 1 || comm->transport == PMG_TRANSPORT_NCCL) {
        if (comm->transport == PMG_TRANSPORT_NCCL) {
          c->comm = make_nccl_transport(comm->nccl_id, comm->rank, comm->size);
        } else if (comm->transport == PMG_TRANSPORT_HUB) {
          need(comm->hub != nullptr && comm->hub->hub.ranks == comm->size, PMG_ERR_CONFIG, "hub / rank count mismatch");
          c->comm = make_hub_transport(&comm->hub->hub, comm->rank, device);
          c->use_graphs = false;  // host-mediated exchanges cannot be captured
        } else {
          throw PmgError(PMG_ERR_CONFIG, "multi-rank context without a transport");
        }
      }
    }
    ck(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    c->stream = c->own_stream;
    ck(cudaEventCreateWithFlags(&c->ev_norm, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "cudaEventCreate");
    {
      const char* e = std::getenv("PMG_NO_OVERLAP");
      c->overlap = !(e && e[0] == '1');
    }
    build_ctx(*c, *desc);
  } catch (const PmgError& e) {
    g_create_error = e.what();
    return e.code;
  } catch (const TransportFailure& e) {
    g_create_error = e.what();
    return PMG_ERR_TRANSPORT;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return PMG_ERR_GENERIC;
  }
  *out = c.release();
  return PMG_OK;
}

void pmg_ctx_destroy(pmg_ctx* ctx) { delete ctx; }

int pmg_nccl_unique_id(unsigned char* out) {
  const std::string e = nccl_unique_id(out);
  if (!e.empty()) {
    g_create_error = e;
    return PMG_ERR_TRANSPORT;
  }
  return PMG_OK;
}

int pmg_hub_create(int ranks, pmg_hub** out) {
  if (ranks < 1 || ranks > 64 || !out) {
    g_create_error = "hub: rank count outside [1, 64]";
    return PMG_ERR_CONFIG;
  }
  *out = new pmg_hub(ranks);
  return PMG_OK;
}

void pmg_hub_destroy(pmg_hub* hub) { delete hub; }

int pmg_hub_poison(pmg_hub* hub, const char* reason) {
  if (hub) hub->hub.poison(reason ? reason : "peer rank failed");
  return PMG_OK;
}

int pmg_comm_bytes(pmg_ctx* ctx, uint64_t* out) {
  return guarded(ctx, [&] { *out = ctx->comm ? ctx->comm->bytes_sent() : 0; });
}

int pmg_ctx_info(pmg_ctx* ctx, int what, int64_t* out) {
  return guarded(ctx, [&] {
    const int level = what >> 8;
    const int w = what & 0xff;
    need(level >= 0 && level < ctx->nl, PMG_ERR_DOMAIN, "level out of range");
    switch (w) {
      case 0: *out = ctx->nl - 1; break;
      case 1: *out = ctx->lv[level].lat_n; break;
      case 2: *out = int64_t(ctx->bytes); break;
      case 3: *out = ctx->lv[level].N; break;
      case 4: *out = ctx->pe - ctx->pb; break;
      case 5: *out = int64_t(ctx->assembly_seconds * 1e6); break;
      case 7: *out = int64_t(ctx->load_seconds * 1e6); break;
      case 6: *out = ctx->comm ? int64_t(ctx->comm->calls) : 0; break;
      default: throw PmgError(PMG_ERR_CONFIG, "unknown info query");
    }
  });
}

int pmg_assemble_load(pmg_ctx* ctx, int rhs_kind, uint64_t seed, pmg_vec* out) {
  return guarded(ctx, [&] {
    check_vec(ctx, out, ctx->nl - 1);
    need(!ctx->geo.empty(), PMG_ERR_CONFIG, "load vector assembly needs the patch geometry (desc.geometry)");
    const DevLevel& L = ctx->lv[ctx->nl - 1];
    try {
      ctx->load_seconds += assemble_load_device(ctx->stream, ctx->dim, ctx->degree, L.n, ctx->geo.data(), ctx->pb,
                                                L.K, rhs_kind, seed, L.l2g, out->d);
    } catch (const AssemblyError& e) {
      throw PmgError(PMG_ERR_GEOMETRY, e.what());
    }
  });
}

int pmg_band_download(pmg_ctx* ctx, int level, double* host, int64_t n) {
  return guarded(ctx, [&] {
    need(level >= 0 && level < ctx->nl, PMG_ERR_DOMAIN, "level out of range");
    const DevLevel& L = ctx->lv[level];
    const size_t per = size_t(L.O) * size_t(L.S);
    need(host != nullptr && n == int64_t(per) * L.K, PMG_ERR_DOMAIN,
         "band download: n must be local patches x (2p+1)^d x (n+p)^d");
    double* tmp = nullptr;
    ck(cudaMalloc(&tmp, per * sizeof(double)), "cudaMalloc band expand");
    try {
      for (int k = 0; k < L.K; ++k) {
        const double* src = L.sweep3_e2p > 0 ? L.band + size_t(k) * L.ext * L.Ob * L.sweep3_e2p
                            : L.sweep_tw > 0  ? L.band + size_t(k) * L.ext * L.Ob * L.sweep_tw
                                              : L.band + size_t(k) * L.Ob * L.Sp;
        launch_band_expand(ctx->stream, ctx->dim, ctx->degree, L.ext, L.S, L.Ob, L.Sp, L.sweep_tw, L.sweep3_front,
                           L.sweep3_e2p, src, tmp);
        ck(cudaGetLastError(), "band expand");
        ck(cudaMemcpyAsync(host + size_t(k) * per, tmp, per * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream),
           "band download");
        ck(cudaStreamSynchronize(ctx->stream), "band download");
      }
    } catch (...) {
      cudaFree(tmp);
      throw;
    }
    ck(cudaFree(tmp), "cudaFree");
  });
}

int pmg_set_stream(pmg_ctx* ctx, void* stream) {
  return guarded(ctx, [&] { ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream; });
}

int pmg_synchronize(pmg_ctx* ctx) {
  return guarded(ctx, [&] { sync_check(*ctx); });
}

int pmg_vec_create(pmg_ctx* ctx, int level, pmg_vec** out) {
  return guarded(ctx, [&] {
    need(level >= 0 && level < ctx->nl, PMG_ERR_DOMAIN, "level out of range");
    auto v = std::make_unique<pmg_vec>();
    v->ctx = ctx;
    v->level = level;
    v->n = ctx->lv[level].lat_n;
    ck(cudaMalloc(&v->d, sizeof(double) * std::max<long long>(v->n, 1) + 64), "cudaMalloc vec");
    ck(cudaMemsetAsync(v->d, 0, sizeof(double) * v->n, ctx->stream), "memset vec");
    *out = v.release();
  });
}

void pmg_vec_free(pmg_vec* v) {
  if (!v) return;
  cudaSetDevice(v->ctx->device);
  cudaFree(v->d);
  delete v;
}

int pmg_vec_upload(pmg_ctx* ctx, pmg_vec* v, int form, const double* host, int64_t n) {
  return guarded(ctx, [&] {
    check_vec(ctx, v, v ? v->level : 0);
    const DevLevel& L = ctx->lv[v->level];
    need(n == L.N, PMG_ERR_DOMAIN, "global vector size mismatch");
    need(L.N <= ctx->staging_n, PMG_ERR_DOMAIN, "staging too small");
    ck(cudaMemcpyAsync(ctx->staging, host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    launch_lattice_from_global(ctx->stream, L.l2g, L.owner, L.lat_n, form == PMG_DISTRIBUTED ? 1 : 0, ctx->staging,
                               v->d);
    ctx->launches++;
    sync_check(*ctx);
  });
}

int pmg_vec_download(pmg_ctx* ctx, pmg_vec* v, int form, double* host, int64_t n) {
  return guarded(ctx, [&] {
    check_vec(ctx, v, v ? v->level : 0);
    const DevLevel& L = ctx->lv[v->level];
    need(n == L.N, PMG_ERR_DOMAIN, "global vector size mismatch");
    launch_global_from_lattice(ctx->stream, L.rep_off, L.rep_slot, L.N, form == PMG_DISTRIBUTED ? 1 : 0, v->d,
                               ctx->staging);
    ctx->launches++;
    ck(cudaMemcpyAsync(host, ctx->staging, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync_check(*ctx);
  });
}

int pmg_vec_lattice_upload(pmg_ctx* ctx, pmg_vec* v, const double* host, int64_t n) {
  return guarded(ctx, [&] {
    check_vec(ctx, v, v ? v->level : 0);
    need(n == v->n, PMG_ERR_DOMAIN, "lattice size mismatch");
    ck(cudaMemcpyAsync(v->d, host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    sync_check(*ctx);
  });
}

int pmg_vec_lattice_download(pmg_ctx* ctx, pmg_vec* v, double* host, int64_t n) {
  return guarded(ctx, [&] {
    check_vec(ctx, v, v ? v->level : 0);
    need(n == v->n, PMG_ERR_DOMAIN, "lattice size mismatch");
    ck(cudaMemcpyAsync(host, v->d, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync_check(*ctx);
  });
}

int pmg_vec_zero(pmg_ctx* ctx, pmg_vec* v) {
  return guarded(ctx, [&] {
    check_vec(ctx, v, v ? v->level : 0);
    launch_fill(ctx->stream, v->d, v->n, 0.0);
    ctx->launches++;
  });
}

int pmg_vec_copy(pmg_ctx* ctx, const pmg_vec* src, pmg_vec* dst) {
  return guarded(ctx, [&] {
    check_vec(ctx, src, src ? src->level : 0);
    check_vec(ctx, dst, src->level);
    launch_copy(ctx->stream, src->d, dst->d, src->n);
    ctx->launches++;
  });
}

int pmg_apply_op(pmg_ctx* ctx, int level, const pmg_vec* u, pmg_vec* out) {
  return guarded(ctx, [&] {
    check_vec(ctx, u, level);
    check_vec(ctx, out, level);
    op_spmv(*ctx, level, u->d, nullptr, out->d);
  });
}

int pmg_residual(pmg_ctx* ctx, int level, const pmg_vec* f, const pmg_vec* u, pmg_vec* out) {
  return guarded(ctx, [&] {
    check_vec(ctx, f, level);
    check_vec(ctx, u, level);
    check_vec(ctx, out, level);
    op_spmv(*ctx, level, u->d, f->d, out->d);
  });
}

int pmg_accumulate(pmg_ctx* ctx, int level, const pmg_vec* r, pmg_vec* out) {
  return guarded(ctx, [&] {
    check_vec(ctx, r, level);
    check_vec(ctx, out, level);
    op_accumulate(*ctx, level, r->d, out->d);
  });
}

int pmg_smooth(pmg_ctx* ctx, int level, const pmg_vec* r, pmg_vec* out) {
  return guarded(ctx, [&] {
    check_vec(ctx, r, level);
    check_vec(ctx, out, level);
    need(r->d != out->d, PMG_ERR_DOMAIN, "smooth: input and output must differ");
    launch_fill(ctx->stream, out->d, out->n, 0.0);
    ctx->launches++;
    op_smooth(*ctx, level, r->d, out->d, false, 1.0);
  });
}

int pmg_restrict(pmg_ctx* ctx, int level, const pmg_vec* r, pmg_vec* out) {
  return guarded(ctx, [&] {
    need(level >= 1 && level < ctx->nl, PMG_ERR_DOMAIN, "restrict: level out of range");
    check_vec(ctx, r, level);
    check_vec(ctx, out, level - 1);
    op_restrict(*ctx, level, r->d, out->d);
  });
}

int pmg_add_prolonged(pmg_ctx* ctx, int level, const pmg_vec* coarse, double coef, pmg_vec* u) {
  return guarded(ctx, [&] {
    need(level >= 1 && level < ctx->nl, PMG_ERR_DOMAIN, "prolong: level out of range");
    check_vec(ctx, coarse, level - 1);
    check_vec(ctx, u, level);
    op_prolong_add(*ctx, level, coarse->d, coef, u->d);
  });
}

int pmg_coarse_solve(pmg_ctx* ctx, const pmg_vec* r, pmg_vec* out) {
  return guarded(ctx, [&] {
    check_vec(ctx, r, 0);
    check_vec(ctx, out, 0);
    op_coarse(*ctx, r->d, out->d);
  });
}

int pmg_dot(pmg_ctx* ctx, int level, const pmg_vec* a, const pmg_vec* b, double* out) {
  return guarded(ctx, [&] {
    check_vec(ctx, a, level);
    check_vec(ctx, b, level);
    op_dot(*ctx, level, a->d, b->d, ctx->scal + 8);
    ck(cudaMemcpyAsync(ctx->h_scal + 8, ctx->scal + 8, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync_check(*ctx);
    *out = ctx->h_scal[8];
  });
}

int pmg_axpy(pmg_ctx* ctx, double a, const pmg_vec* x, pmg_vec* y) {
  return guarded(ctx, [&] {
    check_vec(ctx, x, x ? x->level : 0);
    check_vec(ctx, y, x->level);
    launch_axpy(ctx->stream, a, nullptr, 1.0, x->d, y->d, x->n);
    ctx->launches++;
  });
}

int pmg_xpay(pmg_ctx* ctx, const pmg_vec* z, double beta, pmg_vec* p) {
  return guarded(ctx, [&] {
    check_vec(ctx, z, z ? z->level : 0);
    check_vec(ctx, p, z->level);
    launch_xpay(ctx->stream, z->d, beta, nullptr, p->d, z->n);
    ctx->launches++;
  });
}

int pmg_mg_cycle(pmg_ctx* ctx, int level, pmg_vec* u, const pmg_vec* f) {
  return guarded(ctx, [&] {
    need(level >= 1 && level < ctx->nl, PMG_ERR_DOMAIN, "cycle: level out of range");
    check_vec(ctx, u, level);
    check_vec(ctx, f, level);
    cycle(*ctx, level, u->d, f->d, false);
  });
}

int pmg_precondition(pmg_ctx* ctx, const pmg_vec* r, pmg_vec* z) {
  return guarded(ctx, [&] {
    check_vec(ctx, r, ctx->nl - 1);
    check_vec(ctx, z, ctx->nl - 1);
    need(r->d != z->d, PMG_ERR_DOMAIN, "precondition: input and output must differ");
    auto body = [&]() {
      launch_fill(ctx->stream, z->d, z->n, 0.0);
      ctx->launches++;
      precondition(*ctx, r->d, z->d);
    };
    if (ctx->use_graphs && !ctx->profiling) {  // one graph launch per V-cycle, cached by (r, z)
      if (!ctx->graph_pre || ctx->graph_pre_r != r->d || ctx->graph_pre_z != z->d) {
        ctx->capture(ctx->graph_pre, ctx->graph_pre_launches, body);
        ctx->graph_pre_r = r->d;
        ctx->graph_pre_z = z->d;
      }
      ctx->launch_graph(ctx->graph_pre, ctx->graph_pre_launches);
    } else {
      body();
    }
  });
}

int pmg_pcg_solve_device(pmg_ctx* ctx, const pmg_vec* f, double tol, int max_iter, pmg_vec* u, double* history,
                         int* iterations) {
  int rc = PMG_OK;
  int g = guarded(ctx, [&] {
    check_vec(ctx, f, ctx->nl - 1);
    check_vec(ctx, u, ctx->nl - 1);
    need(max_iter >= 1, PMG_ERR_CONFIG, "max-iter: must be positive");
    rc = pcg_device(*ctx, f->d, tol, max_iter, u->d, history, iterations);
    sync_check(*ctx);
  });
  if (g != PMG_OK) return g;
  if (rc == PMG_ERR_DIVERGENCE) ctx->err = "pcg: no convergence within the iteration limit";
  return rc;
}

int pmg_pcg_solve(pmg_ctx* ctx, const double* f_host, int64_t n, double tol, int max_iter, double* u_host,
                  double* history, int* iterations) {
  int rc = PMG_OK;
  int g = guarded(ctx, [&] {
    const DevLevel& F = ctx->lv.back();
    need(n == F.N, PMG_ERR_DOMAIN, "global vector size mismatch");
    need(max_iter >= 1, PMG_ERR_CONFIG, "max-iter: must be positive");
    ck(cudaMemcpyAsync(ctx->staging, f_host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream), "H2D");
    launch_lattice_from_global(ctx->stream, F.l2g, F.owner, F.lat_n, 1, ctx->staging, ctx->pcg_f);
    ctx->launches++;
    rc = pcg_device(*ctx, ctx->pcg_f, tol, max_iter, ctx->pcg_u, history, iterations);
    launch_global_from_lattice(ctx->stream, F.rep_off, F.rep_slot, F.N, 0, ctx->pcg_u, ctx->staging);
    ctx->launches++;
    ck(cudaMemcpyAsync(u_host, ctx->staging, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    sync_check(*ctx);
  });
  if (g != PMG_OK) return g;
  if (rc == PMG_ERR_DIVERGENCE) ctx->err = "pcg: no convergence within the iteration limit";
  return rc;
}

int pmg_profile(pmg_ctx* ctx, int enable) {
  return guarded(ctx, [&] { ctx->profiling = enable != 0; });
}

int pmg_profile_read(pmg_ctx* ctx, int kernel_class, int level, int64_t* launches, double* ms, double* work) {
  return guarded(ctx, [&] {
    sync_check(*ctx);
    int64_t n = 0;
    double t = 0.0, w = 0.0;
    std::vector<pmg_ctx::Timed> keep;
    for (auto& e : ctx->timed) {
      if (e.cls == kernel_class && e.level == level) {
        float dt = 0.f;
        ck(cudaEventElapsedTime(&dt, e.a, e.b), "cudaEventElapsedTime");
        n++;
        t += dt;
        w += e.work;
        ctx->event_pool.push_back(e.a);
        ctx->event_pool.push_back(e.b);
      } else {
        keep.push_back(e);
      }
    }
    ctx->timed.swap(keep);
    *launches = n;
    *ms = t;
    *work = w;
  });
}

int pmg_kernel_stats(pmg_ctx* ctx, int which, int64_t* count, double* reserved) {
  (void)reserved;
  return guarded(ctx, [&] {
    switch (which) {
      case 0: *count = ctx->launches; break;
      case 1: *count = ctx->spmv_launches; break;
      case 2:
        ctx->launches = ctx->spmv_launches = 0;
        if (count) *count = 0;
        break;
      default: throw PmgError(PMG_ERR_CONFIG, "unknown stats query");
    }
  });
}

}  // extern "C"
