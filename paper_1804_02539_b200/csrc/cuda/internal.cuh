// Internal device data layout and kernel launchers of libpmg_cuda.
//
// HBM layout (one context = the patches one GPU owns):
//   lattice vectors   double[K][S], S = (n+p)^d, patch-major, axis 0 fastest
//   band              double[K][Ob][Sp], O = (2p+1)^d offsets (Ob = (O+1)/2,
//                     the symmetric lower half, on TMA levels), offset-major:
//                     a warp's 32 consecutive rows read 256 contiguous bytes
//                     per offset; row stride Sp >= S (spmv_row_stride); every
//                     (row, column) pair outside the stencil, Dirichlet or
//                     padding holds an exact 0 (zero_dirichlet_band)
//   l2g               int32[K][S] (global dof or -1)
//   replica CSR       per global dof, its lattice slots in ascending (patch,
//                     local) order -- DofMapper::reps (topology.cpp:367-372)
//   FD work buffers   per interior/face piece, its tensor box contiguous
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "pmg_types.h"

namespace pmgcu {

constexpr int kThreads = 256;

// ---------------------------------------------------------------- launches
// Every kernel is launched with programmatic stream serialization (PDL): the
// next kernel in the stream is scheduled while this one runs, and waits in
// PMG_PDL_ENTRY (griddepcontrol.wait) until its predecessor has completed
// and flushed, so dependent kernels pay no launch gap.  A kernel reads no
// global data before PMG_PDL_ENTRY; completion is transitive, so waiting on
// the direct predecessor orders it after everything earlier in the stream.
// PMG_NO_PDL=1 launches without the attribute (the wait is then a no-op).
#define PMG_PDL_ENTRY()                                           \
  do {                                                            \
    asm volatile("griddepcontrol.wait;\n" ::: "memory");           \
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); \
  } while (0)

bool pdl_enabled();

// A failed launch (configuration, shared memory, ...) is an error of the call
// that issued it: launch_k throws, the C ABI maps it to PMG_ERR_CUDA.
struct LaunchError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  static_assert(sizeof...(KArgs) == sizeof...(Args), "kernel argument count");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) throw LaunchError(std::string("kernel launch: ") + cudaGetErrorString(e));
}

// Raise `kernel`'s dynamic shared-memory limit to `bytes` on the CURRENT
// device.  Function attributes belong to each device's context, so the record
// is keyed by (kernel, device); hub ranks on several devices of one process
// and concurrent rank threads are both safe.  Throws LaunchError on failure.
inline void ensure_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) throw LaunchError(std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  std::lock_guard<std::mutex> g(mu);
  size_t& have = done[{kernel, dev}];
  if (have >= bytes) return;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e != cudaSuccess)
    throw LaunchError(std::string("cudaFuncSetAttribute(MaxDynamicSharedMemorySize): ") + cudaGetErrorString(e));
  have = bytes;
}

// ---------------------------------------------------------------- assembly
// SingularGeometryError / bad geometry description of device assembly
struct AssemblyError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Assemble the band of the K patches [patch_begin, patch_begin + K) of one
// level into band ([K][Ob][Sp], rows < S; Ob offsets of the lower half or all
// O).  Returns wall seconds (stream-synchronous).  assembly.cu.
double assemble_level_device(cudaStream_t s, int dim, int degree, int elements, const pmg_patch_geometry* geo,
                             int patch_begin, int K, double* band, long long Sp, int Ob);

// Load vector (assemble_rhs, assembly.cpp:299-365) of the local patches as a
// distributed lattice vector [K][ext^d]; kind = a resolved PMGH_RHS_* source.
double assemble_load_device(cudaStream_t s, int dim, int degree, int elements, const pmg_patch_geometry* geo,
                            int patch_begin, int K, int kind, unsigned long long seed, const int* l2g, double* out);

// ---------------------------------------------------------------- FD
struct FdPiece {
  int dims[3];
  int naxes;
  long long total;
  long long lat_base;  // slot of the box corner (interior pieces)
  int ext;             // lattice extent (interior pieces)
  long long work_off;  // offset in the work buffers
  const double* B[3][2];  // [axis][0 fwd: B(k,n)=V(k,n) | 1 bwd: B(k,n)=V(n,k)], row-major k*N+n
  const double* diag;     // total, original (axis 0 fastest) layout
  const double* rdiag;    // 1 / diag (correctly rounded on the host): the resident-factor kernel multiplies
};

enum FdIn { FD_IN_WORK = 0, FD_IN_LATTICE = 1 };
enum FdOut { FD_OUT_WORK = 0, FD_OUT_WORK_DIAG = 1, FD_OUT_LATTICE_SET = 2, FD_OUT_LATTICE_ADD = 3 };

// One fast-diagonalization pass (contract one axis, rotate the layout).
// items: (first piece of a group of pieces sharing dims and factor, first row
// of the panel within the group, first column, rows of the group) per CTA;
// cfg = NTC | NW << 8: the column panel in 8-column tiles and the warps (8-row
// strips) of the CTA (fd_pick_cfg)
void launch_fd_pass(cudaStream_t s, const FdPiece* pieces, const int4* items, int nitems, int cfg, int pass,
                    int naxes, int in_mode, int out_mode, const double* lat_in, double* lat_out, double alpha,
                    const double* work_in, double* work_out, unsigned* queue = nullptr);
int fd_pick_cfg(const long long* cols, const long long* weight, int n);
bool fd_cfg_valid(int cfg);
// cfg | kFdResident: the resident-factor kernel for short contractions
// (K = N <= 88, many rows); its items come from fd_resident_items, and each
// items list needs its own zeroed strip counters: one unsigned per group + 1
constexpr int kFdResident = 1 << 16;
bool fd_cfg_resident(int cfg);
void fd_resident_items(const std::vector<std::pair<int, long long>>& groups, std::vector<int4>& items);
int fd_cfg_rows(int cfg);  // rows per CTA
int fd_cfg_cols(int cfg);  // columns per CTA
void fd_configure();  // per device, before the first pass
// whole solve of every piece in one launch, one CTA per piece, tensor, diagonal
// and every factor in shared memory: fd_small_smem(max_total, max_dim, naxes)
// = 3 max_total + 2 naxes max_dim^2 doubles <= kFdSmallDoubles
constexpr long long kFdSmallDoubles = 25000;
size_t fd_small_smem(long long max_total, int max_dim, int naxes);
void launch_fd_small(cudaStream_t s, const FdPiece* pieces, int npieces, int naxes, long long max_total,
                     int max_dim, int in_mode, int out_mode, const double* lat_in, double* lat_out, double alpha,
                     const double* work_in, double* work_out);

// ---------------------------------------------------------------- SpMV
struct SpmvArgs {
  int dim, degree, ext;
  long long S;         // rows per patch
  int K;               // patches
  const double* band;  // [K][Ob][Sp]
  const double* x;     // lattice vector (accumulated)
  const double* f;     // residual mode: f (distributed); nullptr for y = A x
  double* y;
  double* dot_partial; // optional: per-block partial of sum y*x (nullptr: none)
  int half = 0;        // band holds the lower half only ([K][(O+1)/2][Sp])
  long long Sp = 0;    // band row stride per (patch, offset): spmv_row_stride
  int sweep = 128;     // 2D half band: line-sweep kernel on lines of >= sweep rows (0: off)
  double* sweep_scratch = nullptr;  // sweep: per segment boundary, the carry rows (spmv_sweep_scratch)
  unsigned* sweep_flags = nullptr;  // sweep: per segment boundary, carry published (zeroed; reset by the reader)
  unsigned long long* sweep_ticket = nullptr;  // sweep: segment ticket counter (zeroed, 8-byte aligned)
  int sweep3 = 30;  // 3D half band: plane-sweep kernel on lattices of >= sweep3 rows per axis (0: off)
};
void launch_spmv(cudaStream_t s, const SpmvArgs& a);
int spmv_blocks(long long rows);
// band row stride per (patch, offset): S, or on levels streamed with TMA bulk
// copies S + halo rounded up to 256 (halo = p (1 + ext [+ ext^2]) + 2)
long long spmv_row_stride(int dim, int degree, int ext, long long S);
// levels whose SpMV streams the band with TMA (S >= 1024, specialised degree)
bool spmv_tma_level(int dim, int degree, long long S);
// band offsets stored per patch: (O+1)/2 (symmetric half) on TMA levels when
// allowed, else O
int spmv_stored_offsets(int dim, int degree, long long S, bool allow_half);
// number of dot partials one launch writes
int spmv_partials(int dim, int degree, long long S, int K, bool half, int sweep, int sweep3);
// scratch of a swept level: carry rows (doubles) and boundary flags (count)
// 2D line-sweep levels keep the band line-major ([K][ext][Ob][tw], zero
// padded): its size in doubles (0: the level is not swept), and the
// conversion from the offset-major band
long long spmv_sweep_band_doubles(int dim, int degree, int ext, long long S, int K, bool half, int sweep);
void spmv_sweep_scratch(int dim, int degree, int ext, long long S, int K, bool half, int sweep, long long* doubles,
                        long long* flags);
void launch_sweep_relayout(cudaStream_t s, int degree, int ext, long long S, int K, long long Sp, const double* src,
                           double* dst);
// One patch's device band (offset-major [Ob][Sp], line-major [ext][Ob][tw]
// when tw > 0, plane-major [ext][Ob][e2p] when e2p > 0) expanded to the reference's index-free full band [O][S]
// (offset o = sum_a (delta_a + p) (2p+1)^a, axis 0 fastest): stored offsets
// are copied, the upper half of a symmetric half band is the mirrored lower
// entry A(r, r+s) = A(r+s, r).  Pairs outside the lattice read 0.
void launch_band_expand(cudaStream_t s, int dim, int degree, int ext, long long S, int Ob, long long Sp, int tw,
                        int front, int e2p, const double* band_patch, double* full);
// 3D plane-sweep levels keep the band plane-major ([K][ext][Ob][e2p], each
// (plane, offset) row at [front, front + ext^2) between zero pads): its size
// in doubles (0: the level is not swept) with front / e2p, and the conversion
// from the offset-major band
long long spmv_sweep3_band_doubles(int dim, int degree, int ext, long long S, int K, bool half, int sweep3,
                                   int* front, int* e2p);
void launch_sweep3_relayout(cudaStream_t s, int degree, int ext, long long S, int K, long long Sp, const double* src,
                            double* dst);

// ---------------------------------------------------------------- Kronecker operator
// Matrix-free operator of a level whose patches are axis-aligned affine
// (PMG_BAND_KRONECKER, kernels_kron.cu): y = A x or y = f - A x with
// A = sum_a g[k][a] (x)_{b != a} M (x) K.
struct KronArgs {
  int dim, degree, ext;
  long long S;        // rows per patch
  int K;              // patches
  const double* M;    // univariate mass, full band [ext][2p+1] (zero outside the lattice)
  const double* Kst;  // univariate stiffness, same layout
  const double* g;    // [K][3] geometry factors
  const int* l2g;     // [K][S], < 0 on Dirichlet slots
  const double* x;
  const double* f;    // residual form; nullptr for y = A x
  double* y;
  double* dot_partial;  // optional: per-CTA partials of sum y x (kron_partials of them)
  double* scratch;      // 3D: 5 lattices
};
void launch_kron_spmv(cudaStream_t s, const KronArgs& a, int* launches);
int kron_partials(int dim, int degree, int ext, long long S, int K);
bool kron_supported(int dim, int degree, int ext);

// ---------------------------------------------------------------- device PCG loop
// State of a device-resident pcg_generic loop (multigrid.hpp:155-189): the
// iteration counter, the stopping decision and the residual norms stay on the
// device; a WHILE conditional graph node repeats the iteration body until
// pcg_check clears the condition.
struct PcgLoopState {
  int k;         // iterations done
  int status;    // 0 running, 1 converged, 2 non-positive energy, 3 iteration cap
  int max_iter;  // set by the host before each launch
  int pad;
  double tol;    // set by the host before each launch
  double r0;
};
// first != 0: history[0] = |r0| and the loop condition (|r0| != 0), and
// scal[0] = +inf so the first body's beta = rz / inf = 0 gives p = z exactly;
// else: history[++k] = |r_k| and the stop test (definiteness flag, tol, cap)
void launch_pcg_check(cudaStream_t s, int first, PcgLoopState* st, double* scal, double* history,
                      cudaGraphConditionalHandle handle);

// ---------------------------------------------------------------- misc kernels
void launch_fill(cudaStream_t s, double* x, long long n, double v);
void launch_copy(cudaStream_t s, const double* x, double* y, long long n);
void launch_axpy(cudaStream_t s, double a, const double* a_dev, double sign, const double* x, double* y, long long n);
void launch_xpay(cudaStream_t s, const double* z, double beta, const double* beta_dev, double* p, long long n);
void launch_scale_set(cudaStream_t s, double a, const double* x, double* y, long long n);  // y = a x
// deterministic dot: fixed grid -> partials -> one ordered final sum
int dot_blocks(long long n);
void launch_dot_partial(cudaStream_t s, const double* a, const double* b, long long n, double* partial);
void launch_sum_partials(cudaStream_t s, const double* partial, int nparts, double* out);
// Sigma: out = r, then every multi-replica dof gets the ordered sum written to all its replicas
void launch_group_sum(cudaStream_t s, const int* goff, const int* gslot, int ngroups, const double* r, double* out);
// gather-sum / scatter for interface piece dofs via the replica CSR of global dofs
void launch_gather_sum(cudaStream_t s, const int* dof_g, long long ndof, const int* rep_off, const int* rep_slot,
                       const double* r, double* buf);
void launch_scatter(cudaStream_t s, const int* dof_g, long long ndof, const int* rep_off, const int* rep_slot,
                    const double* buf, double* out, int add, double alpha);
// edges (dense inverse GEMV) and vertices (scalar) in one launch
struct EdgePiece {
  int m;
  long long dof_off;  // into the concatenated edge dof list
  const double* Linv; // column-major m x m
};
// one-launch smoother of a small level on one rank (kernels_fd.cu)
struct SmoothSmallArgs {
  int d;
  const FdPiece* ints;
  int n_int;
  const FdPiece* faces;  // 3D face pieces; dofs at face_iface[work_off..]
  int n_face;
  const int* face_iface;
  const EdgePiece* edges;
  const int2* edge_items;
  int n_edge_items;
  const int* edge_iface;
  const int* vert_iface;
  const double* vert_scalar;
  int nverts;
  const int* rep_off;  // interface replica CSR
  const int* rep_slot;
  const double* r;
  double* out;
  int add;
  double alpha;
};
void launch_smooth_small(cudaStream_t s, const SmoothSmallArgs& a, size_t smem);
// items: (edge, first row) per CTA, 32 rows each.  Piece dofs are interface
// indices: t holds their totals, rep_off/rep_slot their local replicas.
void launch_edges_vertices(cudaStream_t s, const EdgePiece* edges, const int2* items, int nitems,
                           const int* edge_iface, const int* vert_iface, const double* vert_scalar, int nverts,
                           const int* rep_off, const int* rep_slot, const double* t, double* out, int add,
                           double alpha);
// interface dofs: partial replica sums, exchange packing, ascending-rank fold,
// write-back to every local replica; piece gathers/scatters through t
void launch_iface_partial(cudaStream_t s, int n, const int* rep_off, const int* rep_slot, const double* r,
                          double* tloc);
void launch_iface_pack(cudaStream_t s, int n, const int* idx, const double* tloc, double* send);
void launch_iface_combine(cudaStream_t s, int n, const int* comb_off, const int* comb_src, const double* tloc,
                          const double* recv, double* t);
void launch_iface_scatter(cudaStream_t s, int n, const int* rep_off, const int* rep_slot, const double* t,
                          double* out);
void launch_gather_t(cudaStream_t s, long long n, const int* map, const double* t, double* buf);
void launch_scatter_iface(cudaStream_t s, long long n, const int* map, const int* rep_off, const int* rep_slot,
                          const double* buf, double* out, int add, double alpha);
void launch_sum_ranks(cudaStream_t s, const double* parts, int ranks, int n, double* out);
// global <-> lattice
void launch_lattice_from_global(cudaStream_t s, const int* l2g, const unsigned char* owner, long long n, int form,
                                const double* g, double* lat);
void launch_global_from_lattice(cudaStream_t s, const int* rep_off, const int* rep_slot, long long ndofs, int form,
                                const double* lat, double* g);
// coarse, in steps: rhs[g] = sum of local replicas; x = Ainv rhs; out[slot] = x[l2g]
void launch_coarse_gather(cudaStream_t s, const int* rep_off, const int* rep_slot, int n0, const double* r,
                          double* rhs);
void launch_coarse_gemv(cudaStream_t s, const double* Ainv, int n0, const double* rhs, double* x);
void launch_coarse_scatter(cudaStream_t s, const int* l2g, long long lat_n, const double* x, double* out);
// coarse: rhs[g] = sum reps; x = Ainv rhs; out[slot] = x[l2g]
void launch_coarse(cudaStream_t s, const int* rep_off, const int* rep_slot, const int* l2g, int n0, long long lat_n,
                   const double* Ainv, const double* r, double* rhs, double* x, double* out);
// two-scale passes
struct TsDev {
  int fine_dim, coarse_dim;
  const int* row_start;  // [fine]
  const int* row_len;
  const int* row_off;
  const double* vals;
  const int* col_off;    // transpose CSR: [coarse+1]
  const int* col_row;    // fine rows, ascending
  const double* col_val;
  // tiled 2D transfers: widest coarse range of kTileF consecutive fine rows,
  // widest fine range of kTileC consecutive coarse columns (0: not tileable)
  int pspan = 0, rspan = 0;
};
constexpr int kTileF = 32;  // prolongation: fine tile kTileF x kTileF
constexpr int kTileC = 16;  // restriction: coarse tile kTileC x kTileC
// 2D transfers through a shared-memory tile (axis 0 then axis 1, the
// reference's order per output); same results as the fused kernels
void launch_restrict_tile2d(cudaStream_t s, const TsDev& ts, int K, int ext_f, int ext_c, const double* r,
                            double* out, const int* l2g_c);
void launch_prolong_tile2d(cudaStream_t s, const TsDev& ts, int K, int ext_f, int ext_c, const double* c, double coef,
                           double* u, const int* l2g_f);
// one tensor axis pass over K patches: in dims -> out dims (axis changes
// extent).  mode 0 writes; 1 writes with Dirichlet slots zeroed (l2g of the
// output lattice); 2 adds coef * value on non-Dirichlet slots.
void launch_ts_axis(cudaStream_t s, const TsDev& ts, bool transpose, int K, int d, const int* in_dims, int axis,
                    const double* in, double* out, int mode = 0, const int* l2g = nullptr, double coef = 0.0);
// single-pass transfers (2D, and 3D levels with small lattices)
void launch_restrict_fused(cudaStream_t s, const TsDev& ts, int K, int d, int ext_f, int ext_c, const double* r,
                           double* out, const int* l2g_c);
void launch_prolong_fused(cudaStream_t s, const TsDev& ts, int K, int d, int ext_f, int ext_c, const double* c,
                          double coef, double* u, const int* l2g_f);
// final fine write of a prolongation: u[slot] += c * val where l2g >= 0
void launch_masked_axpy(cudaStream_t s, const int* l2g, long long n, double c, const double* val, double* u);
void launch_mask_dirichlet(cudaStream_t s, const int* l2g, long long n, double* v);
void launch_zero_dirichlet_band(cudaStream_t s, int dim, int degree, int ext, long long S, long long Sp, int K,
                                int stored_offsets, const int* l2g, double* band);
// scalar helpers on device: out = num/den ; check energy
void launch_pcg_scalars(cudaStream_t s, int op, double* scal);

}  // namespace pmgcu
