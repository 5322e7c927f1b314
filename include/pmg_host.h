/* Host-side hierarchy builder (libpmg_host.so).
 *
 * Builds the multigrid hierarchy the solve path consumes -- the role of the
 * reference's Hierarchy constructor (multigrid.hpp:42-75, multigrid.cpp:16-50)
 * together with assemble_rhs (assembly.cpp:299-365) and the domain
 * generators (harness.cpp:118-178, tests/util.hpp:37-126).
 * A reference-side integration would fill pmg_hierarchy_desc from its own
 * Hierarchy instead; this library exists so the repository
 * can produce the same data without Eigen.
 */
#ifndef PMG_HOST_H
#define PMG_HOST_H

#include "pmg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pmgh_hierarchy pmgh_hierarchy;

/* Source term selection for the load vector. */
enum {
  PMGH_RHS_DEFAULT = 0, /* the config's own: c1 sine_pi, c2..c5 random_nodes, fixtures sine2d/3d */
  PMGH_RHS_ONE = 1,
  PMGH_RHS_SINE2D = 2,  /* harness.cpp:28-30 */
  PMGH_RHS_SINE3D = 3,  /* harness.cpp:32-35 */
  PMGH_RHS_SINE_PI = 4, /* 2 pi^2 sin(pi x) sin(pi y): BASELINE config 1 */
  PMGH_RHS_RANDOM_NODES = 5, /* uniform [-1,1] per quadrature node from the seed */
  PMGH_RHS_ZERO = 6
};

/* domain: c1..c5, unit_square_D|N, two_squares_D|N, two_squares_flipped_D|N,
 * lshape, fichera, unit_grid(kx,ky[,kz]), jitter(kx,ky,kz).
 * Level l has n0 * 2^l elements per patch direction, l = 0..levels. */
int pmgh_build(const char* domain, int split, int degree, int n0, int levels, const pmg_cycle_params* params,
               int rhs_kind, uint64_t seed, int threads, pmgh_hierarchy** out);
/* flags: PMGH_DEVICE_ASSEMBLY leaves the stiffness of levels >= 1 unassembled
 * (PMG_BAND_ASSEMBLE): the CUDA context assembles it from the patch geometry.
 * PMGH_KRONECKER describes levels >= 1 as PMG_BAND_KRONECKER: the CUDA context
 * applies the operator matrix-free (axis-aligned affine patch maps only); the
 * host band, when assembled, stays in the descriptor for host-side checkers. */
enum { PMGH_DEVICE_ASSEMBLY = 1, PMGH_KRONECKER = 2 };
int pmgh_build_ex(const char* domain, int split, int degree, int n0, int levels, const pmg_cycle_params* params,
                  int rhs_kind, uint64_t seed, int threads, int flags, pmgh_hierarchy** out);
void pmgh_free(pmgh_hierarchy* h);
const char* pmgh_last_error(void);

/* The source PMGH_RHS_DEFAULT stands for on this domain (a PMGH_RHS_* value);
 * other kinds are returned unchanged. */
int pmgh_resolve_rhs_kind(const char* domain, int dim, int rhs_kind);

/* Whole-hierarchy descriptor; pointers live as long as h. */
int pmgh_describe(pmgh_hierarchy* h, pmg_hierarchy_desc* out);
/* Finest-level load vector (num_dofs of the finest level). */
int pmgh_rhs(pmgh_hierarchy* h, const double** rhs, int64_t* n);
/* Reassemble the load vector with another source term. */
int pmgh_set_rhs(pmgh_hierarchy* h, int rhs_kind, uint64_t seed, int threads);
/* which: 0 setup seconds, 1 assembly seconds. */
double pmgh_seconds(pmgh_hierarchy* h, int which);
/* Stored CSR entry count of the reference layout (harness.cpp:274-282). */
int64_t pmgh_stored_entries(int degree, int elements, int dim, int patches);
/* Global dof replicas (DofMapper::reps, topology.cpp:367-372) of a level:
 * CSR offsets [num_dofs+1], patches, locals. */
int pmgh_reps(pmgh_hierarchy* h, int level, const int32_t** off, const int32_t** patch, const int32_t** local);
/* Interfaces found by build_topology: count, then 5 ints each
 * (patch_a, side_a, patch_b, side_b, orientation). */
int pmgh_interfaces(pmgh_hierarchy* h, int* count, const int32_t** data);

/* Interface-dof exchange plan of `rank` among `ranks` on `level` -- the plan
 * libpmg_cuda builds internally (csrc/common/rank_plan.hpp), exposed so the
 * CPU tests can run the exchange protocol over torch.distributed/gloo.
 * Arrays stay valid until the next call on h. */
typedef struct {
  int n_iface;
  const int32_t* iface_g;   /* [n_iface] global ids, ascending */
  const int32_t* rep_off;   /* [n_iface+1] local replicas (rank-local lattice slots) */
  const int32_t* rep_slot;
  const int32_t* comb_off;  /* [n_iface+1] fold sources, ascending rank */
  const int32_t* comb_src;  /* -1 = own partial, else index into the concatenated receive buffers */
  int n_neighbors;
  const int32_t* nb_rank;   /* [n_neighbors] ascending */
  const int32_t* nb_off;    /* [n_neighbors+1] into nb_iface */
  const int32_t* nb_iface;  /* interface positions exchanged with each neighbour, ascending */
} pmgh_rank_plan_view;
int pmgh_rank_plan(pmgh_hierarchy* h, int level, int ranks, int rank, pmgh_rank_plan_view* out);

/* ---- numerics hooks used by the known-answer tests ---- */
int pmgh_gauss_legendre(int points, double* nodes, double* weights);
/* first_index and values[degree+1] */
int pmgh_eval_basis(int degree, int elements, int left_elim, int right_elim, double x, int deriv, int* first_index,
                    double* values);
/* dense dim x dim, column-major; dim = returned via *dim when out == NULL */
int pmgh_gram(int degree, int elements, int left_elim, int right_elim, int deriv, int* dim, double* out);
int pmgh_two_scale(int degree, int elements, int left_elim, int right_elim, int* fine_dim, int* coarse_dim,
                   double* dense);
int pmgh_gen_eig(int n, const double* K, const double* M, double* eigenvalues, double* eigenvectors);
int pmgh_banded_cholesky_solve(int dim, int bw, const double* lower_band, const double* rhs, double* x);

#ifdef __cplusplus
}
#endif

#endif /* PMG_HOST_H */
