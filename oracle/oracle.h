/* CPU oracle of the PCG + V(1,1)-cycle solve path -- TEST INFRASTRUCTURE ONLY.
 *
 * This library is the parity checker for the CUDA path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  Nothing in paper_1804_02539_b200/ links or calls it.
 *
 * It restates, in plain C++ over the hierarchy descriptor of pmg_types.h, the
 * reference solve path of /root/reference/proj (which cannot be compiled here:
 * Eigen3 and its vendor/ headers are absent):
 *   SerialBackend, mg_cycle_generic, mg_precondition, pcg_generic
 *                                       include/patchmg/multigrid.hpp:80-189
 *   Hierarchy::coarse_solve             src/multigrid.cpp:52-55 (dense LLT)
 *   MultiPatchOperator::apply, PatchOperator::apply_add
 *                                       src/assembly.cpp:12-18,265-280
 *   HybridSmoother::apply, PieceSmoother::apply_add/solve
 *                                       src/smoother.cpp:20-44,110-115
 *   FastDiagonalSolver::solve, apply_along_axis(_transpose)
 *                                       src/tensor.cpp:18-102,132-140
 *   BandedCholesky::solve               src/banded.cpp:61-77
 *   TransferOperator::prolong(_patch), restrict_full/restrict_patch
 *                                       src/transfer.cpp:21-91
 *   ParallelBackend, RankLayout, contiguous_partition, Communicator,
 *   InProcHub, run_ranks                src/parallel.cpp:21-518
 * Pinning: tests/test_oracle_kats.py ports the reference's known-answer and
 * identity tests (tests/test_multigrid.cpp, test_parallel.cpp,
 * test_transfer.cpp, test_smoother.cpp) and runs them against this library.
 */
#ifndef PMG_ORACLE_H
#define PMG_ORACLE_H

#include "../include/pmg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_ctx oracle_ctx;

/* The descriptor's arrays are borrowed and must outlive the context. */
int oracle_create(const pmg_hierarchy_desc* desc, oracle_ctx** out);
void oracle_destroy(oracle_ctx* ctx);
const char* oracle_last_error(void);
int64_t oracle_num_dofs(oracle_ctx* ctx, int level);

/* SerialBackend operations on global dof vectors (multigrid.hpp:90-110). */
int oracle_apply_op(oracle_ctx* ctx, int level, const double* u, double* out);
int oracle_residual(oracle_ctx* ctx, int level, const double* f, const double* u, double* out);
int oracle_smooth(oracle_ctx* ctx, int level, const double* r, double* out);
int oracle_restrict(oracle_ctx* ctx, int level, const double* r, double* out_coarse);
int oracle_add_prolonged(oracle_ctx* ctx, int level, const double* coarse, double c, double* u);
int oracle_coarse_solve(oracle_ctx* ctx, const double* r, double* out);
int oracle_mg_cycle(oracle_ctx* ctx, int level, double* u, const double* f);
int oracle_precondition(oracle_ctx* ctx, const double* r, double* z);

/* Coarse solver of this context: 0 the dense LLT substitution (default,
 * Hierarchy::coarse_solve), 1 the explicit inverse L^-T L^-1 as a GEMV -- a
 * second exact solver with different rounding, used by the tests to measure
 * the conditioning limit kappa(A_0) eps that any two exact coarse solvers
 * differ by (the CUDA path applies the explicit inverse). */
int oracle_set_coarse_mode(oracle_ctx* ctx, int mode);

/* pcg_generic with the V-cycle preconditioner (multigrid.cpp:72-89).
 * history has room for max_iter+1 entries.  With allow_cap != 0 the
 * iteration cap returns PMG_OK instead of PMG_ERR_DIVERGENCE (bounded CPU
 * samples for the benchmark's baseline leg). */
int oracle_pcg_solve(oracle_ctx* ctx, const double* f, double tol, int max_iter, int allow_cap, double* u,
                     double* history, int* iterations, double* t_solve);

/* parallel_pcg_solve over R in-process ranks with the contiguous patch
 * partition (parallel.cpp:497-518): one std::thread per rank, one shared
 * read-only hierarchy. */
int oracle_parallel_pcg_solve(oracle_ctx* ctx, int ranks, const double* f, double tol, int max_iter,
                              int allow_cap, double* u, double* history, int* iterations, double* t_solve,
                              uint64_t* comm_bytes);

#ifdef __cplusplus
}
#endif

#endif /* PMG_ORACLE_H */
