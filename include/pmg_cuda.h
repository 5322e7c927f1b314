/* libpmg_cuda.so -- the B200 (sm_100a) solve path of the PCG + V(1,1)-cycle
 * multigrid method for multi-patch IgA, behind a plain C ABI.
 *
 * Every entry point replaces one call of the reference's Backend concept
 * (the seam consumed by mg_cycle_generic / mg_precondition / pcg_generic,
 * /root/reference/proj/include/patchmg/multigrid.hpp:120-189), implemented by
 * SerialBackend (multigrid.hpp:80-114) and ParallelBackend
 * (parallel.hpp:267-341, parallel.cpp:247-468).
 *
 * Vector representation.  A pmg_vec holds one value per patch-lattice slot
 * (num_patches x (n+p)^dim, patch-major, axis 0 fastest), i.e. the paper's
 * accumulated (Type I) / distributed (Type II) vectors applied per patch:
 *   accumulated: every replica of a global dof holds its global value;
 *   distributed: the replicas' values sum to the global value.
 * Dirichlet slots hold 0.  Whether a vector is read as accumulated or
 * distributed is fixed by the operation, exactly as the reference's AccVec /
 * DistVec types fix it; pmg_vec_upload/download take the form explicitly.
 *
 * Errors: every function returns a PMG_* status (pmg_types.h) that maps 1:1
 * onto the reference exception classes; pmg_last_error() holds the message.
 * No function falls back to a CPU implementation.
 */
#ifndef PMG_CUDA_H
#define PMG_CUDA_H

#include "pmg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pmg_ctx pmg_ctx;
typedef struct pmg_vec pmg_vec;

enum { PMG_ACCUMULATED = 0, PMG_DISTRIBUTED = 1 };

/* In-process rank hub: R ranks as threads of one process exchanging through
 * host-mediated device copies (the reference's InProcHub, parallel.hpp:70-113). */
typedef struct pmg_hub pmg_hub;

enum { PMG_TRANSPORT_NONE = 0, PMG_TRANSPORT_NCCL = 1, PMG_TRANSPORT_HUB = 2 };

/* Multi-GPU placement: this context owns patches [patch_begin, patch_end), the
 * contiguous_partition block of `rank` (parallel.cpp:181-198).  With size > 1
 * the ranks exchange interface sums, scalar reductions and the coarse
 * residual over `transport`: NCCL (one process per GPU; every rank passes the
 * same nccl_id from pmg_nccl_unique_id) or an in-process hub. */
typedef struct {
  int rank;
  int size;
  int patch_begin;
  int patch_end;
  int transport;               /* PMG_TRANSPORT_* */
  unsigned char nccl_id[128];  /* ncclUniqueId */
  pmg_hub* hub;
} pmg_comm_desc;

int pmg_nccl_unique_id(unsigned char out[128]);
int pmg_hub_create(int ranks, pmg_hub** out);
void pmg_hub_destroy(pmg_hub* hub);
/* wake every rank blocked in the hub with a TransportError (run_ranks poison) */
int pmg_hub_poison(pmg_hub* hub, const char* reason);
/* payload bytes this rank pushed to peers (Communicator::bytes_sent) */
int pmg_comm_bytes(pmg_ctx* ctx, uint64_t* out);

/* Upload one hierarchy (Hierarchy, multigrid.hpp:42-75) to `device`.
 * comm == NULL: single GPU owning every patch. */
int pmg_ctx_create(const pmg_hierarchy_desc* desc, int device, const pmg_comm_desc* comm, pmg_ctx** out);
void pmg_ctx_destroy(pmg_ctx* ctx);
/* Message of the last failure on ctx (or of the last failed create when NULL). */
const char* pmg_last_error(pmg_ctx* ctx);
/* what: 0 finest level, 1 lattice slots of level `level`, 2 device bytes held,
 *       3 num_dofs of level `level`, 4 local patches, 5 microseconds spent in
 *       device stiffness assembly (PMG_BAND_ASSEMBLE levels), 6 collectives
 *       issued through the rank transport (a captured one counts once).
 *       level = what >> 8. */
int pmg_ctx_info(pmg_ctx* ctx, int what, int64_t* out);
/* The operator of `level` as held on the device, expanded to the reference's
 * index-free full band double[K_local][(2p+1)^d][(n+p)^d] (the host layout of
 * pmg_level_desc.band, PMG_BAND_TENSOR; the stored values behind
 * PatchOperator::apply_add, assembly.hpp:16-25).  The upper half of a
 * symmetric half band is the mirrored lower entry.  This is how a hierarchy
 * assembled on the device (PMG_BAND_ASSEMBLE) hands its stiffness to a host
 * consumer -- the CPU checker and baseline.  n = K_local (2p+1)^d (n+p)^d. */
int pmg_band_download(pmg_ctx* ctx, int level, double* host, int64_t n);
/* Assemble the finest-level load vector on the device (assemble_rhs,
 * assembly.cpp:299-365, by sum factorization over the patch quadrature grid)
 * into `out` as a DistributedVector: every local patch holds its own share,
 * Dirichlet slots 0.  rhs_kind = a resolved PMGH_RHS_* source of pmg_host.h
 * (1 one, 2 sine2d, 3 sine3d, 4 sine_pi, 5 random_nodes with `seed`, 6 zero).
 * Needs pmg_hierarchy_desc.geometry.  The sum order differs from the host
 * loop's element scatter, so entries agree to rounding, not bitwise. */
int pmg_assemble_load(pmg_ctx* ctx, int rhs_kind, uint64_t seed, pmg_vec* out);
/* Launch everything on this cudaStream_t from now on (NULL: the ctx stream). */
int pmg_set_stream(pmg_ctx* ctx, void* stream);
int pmg_synchronize(pmg_ctx* ctx);

/* Vectors (AccumulatedVector / DistributedVector, parallel.hpp:169-260). */
int pmg_vec_create(pmg_ctx* ctx, int level, pmg_vec** out);
void pmg_vec_free(pmg_vec* v);
/* global host vector (num_dofs) <-> lattice vector in the given form;
 * to_accumulated / to_distributed_owner / gather_global(_sum),
 * parallel.cpp:428-468 */
int pmg_vec_upload(pmg_ctx* ctx, pmg_vec* v, int form, const double* host, int64_t n);
int pmg_vec_download(pmg_ctx* ctx, pmg_vec* v, int form, double* host, int64_t n);
/* raw lattice copies (num local patches x (n+p)^dim) */
int pmg_vec_lattice_upload(pmg_ctx* ctx, pmg_vec* v, const double* host, int64_t n);
int pmg_vec_lattice_download(pmg_ctx* ctx, pmg_vec* v, double* host, int64_t n);
int pmg_vec_zero(pmg_ctx* ctx, pmg_vec* v);                  /* zero_acc */
int pmg_vec_copy(pmg_ctx* ctx, const pmg_vec* src, pmg_vec* dst);

/* Backend operations. */
/* apply_op: out(dist) = A u(acc)                 multigrid.hpp:93, parallel.cpp:281-300 */
int pmg_apply_op(pmg_ctx* ctx, int level, const pmg_vec* u, pmg_vec* out);
/* residual: out(dist) = f(dist) - A u(acc)       multigrid.hpp:94-96, parallel.cpp:302-304 */
int pmg_residual(pmg_ctx* ctx, int level, const pmg_vec* f, const pmg_vec* u, pmg_vec* out);
/* accumulate: interface sum Sigma               multigrid.hpp:97, parallel.cpp:306-337 */
int pmg_accumulate(pmg_ctx* ctx, int level, const pmg_vec* r, pmg_vec* out);
/* smooth: out(acc) = sum_T P_T L_T^-1 P_T^T r    multigrid.hpp:99, parallel.cpp:353-355 */
int pmg_smooth(pmg_ctx* ctx, int level, const pmg_vec* r, pmg_vec* out);
/* restrict_residual: level -> level-1 (dist)    multigrid.hpp:100-102, parallel.cpp:357-382 */
int pmg_restrict(pmg_ctx* ctx, int level, const pmg_vec* r, pmg_vec* out_coarse);
/* add_prolonged: u += c P coarse (acc)          multigrid.hpp:103-105, parallel.cpp:384-409 */
int pmg_add_prolonged(pmg_ctx* ctx, int level, const pmg_vec* coarse, double c, pmg_vec* u);
/* coarse_solve: out(acc) = A0^-1 r(dist)        multigrid.hpp:106, parallel.cpp:411-422 */
int pmg_coarse_solve(pmg_ctx* ctx, const pmg_vec* r, pmg_vec* out);
/* dot(dist, acc), globally reduced             multigrid.hpp:107, parallel.cpp:424-426 */
int pmg_dot(pmg_ctx* ctx, int level, const pmg_vec* a, const pmg_vec* b, double* out);
/* axpy_acc / axpy_dist: y += a x                 multigrid.hpp:108-109 */
int pmg_axpy(pmg_ctx* ctx, double a, const pmg_vec* x, pmg_vec* y);
/* xpay_acc: p = z + beta p                       multigrid.hpp:110 */
int pmg_xpay(pmg_ctx* ctx, const pmg_vec* z, double beta, pmg_vec* p);

/* Fused paths. */
/* mg_cycle_generic at `level`, in place on u(acc), f(dist)   multigrid.hpp:120-141 */
int pmg_mg_cycle(pmg_ctx* ctx, int level, pmg_vec* u, const pmg_vec* f);
/* mg_precondition: z(acc) = one cycle from zero on r(dist)   multigrid.hpp:144-149 */
int pmg_precondition(pmg_ctx* ctx, const pmg_vec* r, pmg_vec* z);
/* pcg_generic with the V-cycle preconditioner on device-resident vectors;
 * history has room for max_iter+1 norms; PMG_ERR_DIVERGENCE at the cap
 * (multigrid.hpp:155-189, multigrid.cpp:72-89). */
int pmg_pcg_solve_device(pmg_ctx* ctx, const pmg_vec* f, double tol, int max_iter, pmg_vec* u, double* history,
                         int* iterations);
/* The same from host memory: f_host is the global load vector (num_dofs of the
 * finest level), u_host receives the global solution -- the pcg_solve call of
 * the reference (multigrid.hpp:196-197) end to end, copies included. */
int pmg_pcg_solve(pmg_ctx* ctx, const double* f_host, int64_t n, double tol, int max_iter, double* u_host,
                  double* history, int* iterations);

/* Instrumentation: which = 0 kernel launches since ctx creation (count);
 * which = 1 launches of the band SpMV; which = 2 reset counters. */
int pmg_kernel_stats(pmg_ctx* ctx, int which, int64_t* count, double* reserved);

/* Live kernel timing with CUDA events on the launch stream.  While enabled,
 * every launch of the timed classes is bracketed by two events, kernels are
 * launched directly (no graphs) and a PCG solve stops exactly as
 * pcg_generic does, so an instrumented solve runs the same kernels as the
 * graph-replayed one.
 * kernel_class: 0 = band SpMV, 1 = fast-diagonalization pass, 2 = transfer
 * (restriction / prolongation), 3 = interface pieces of a smooth (Sigma,
 * face / edge / vertex solves; side stream), 4 = dot / accumulate,
 * 5 = coarse solve.
 * pmg_profile_read synchronizes and returns, for launches on `level` since the
 * last read: the launch count, the summed device milliseconds and the summed
 * algorithmic work: SpMV bytes = 8 B per stored band entry (the symmetric half
 * band: (S + D) / 2 entries, S = reference CSR entries, D = lattice rows;
 * SURVEY 8(d)) + 8 B per lattice row for x, y (and f when read); FD flops =
 * 2 per multiply-add; 0 for the other classes. */
int pmg_profile(pmg_ctx* ctx, int enable);
int pmg_profile_read(pmg_ctx* ctx, int kernel_class, int level, int64_t* launches, double* ms, double* work);

#ifdef __cplusplus
}
#endif

#endif /* PMG_CUDA_H */
