/* Plain-C description of one multigrid hierarchy: the data the PCG + V-cycle
 * path consumes.  Every pointer is borrowed; the consumer copies what it
 * keeps.  Each field names the reference object it carries:
 *
 *   pmg_level_desc.l2g        DofMapper::local_to_global     topology.hpp:89
 *   pmg_level_desc.band/csr_* PatchOperator {row_ptr,cols,vals}  assembly.hpp:16-25
 *   pmg_level_desc.ts_*       TwoScaleMatrix {row_start,row_vals} spline.hpp:76-85
 *   pmg_piece_desc            PieceSmoother + Piece          smoother.hpp:17-45, topology.hpp:104-110
 *     .V/.diag                FastDiagonalSolver vecs_/diag_ tensor.hpp:56-60
 *     .chol_*                 BandedCholesky l_              banded.hpp:46-58
 *     .scalar                 PieceSmoother::vertex_scalar   smoother.hpp:35
 *   pmg_hierarchy_desc.coarse_* Hierarchy coarse factorization multigrid.cpp:37-48
 *   pmg_cycle_params          CycleParams                    multigrid.hpp:21-27
 */
#ifndef PMG_TYPES_H
#define PMG_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  Nonzero codes correspond 1:1 to the reference's exception
 * classes (errors.hpp:9-56); the CLI mapping of harness.cpp:573-581 is
 * config -> 2, divergence -> 3, transport -> 4, everything else -> 1. */
enum {
  PMG_OK = 0,
  PMG_ERR_GENERIC = 1,
  PMG_ERR_CONFIG = 2,        /* ConfigError */
  PMG_ERR_DIVERGENCE = 3,    /* DivergenceError */
  PMG_ERR_TRANSPORT = 4,     /* TransportError */
  PMG_ERR_DOMAIN = 5,        /* DomainError: size / shape mismatch */
  PMG_ERR_DEFINITENESS = 6,  /* DefinitenessError */
  PMG_ERR_DECOMPOSITION = 7, /* DecompositionError */
  PMG_ERR_GEOMETRY = 8,      /* SingularGeometryError */
  PMG_ERR_NONMATCHING = 9,   /* NonMatchingError / NonManifoldError */
  PMG_ERR_CUDA = 10          /* device failure (no reference analogue) */
};

enum { PMG_PIECE_INTERIOR = 0, PMG_PIECE_FACE = 1, PMG_PIECE_EDGE = 2, PMG_PIECE_VERTEX = 3 };

/* Stiffness storage of one level.
 *   PMG_BAND_TENSOR:   index-free band[k][o][r], o = sum_a (delta_a+p)(2p+1)^a,
 *                      zero where the column leaves the patch lattice.
 *   PMG_BAND_CSR:      the reference PatchOperator triple per patch.
 *   PMG_BAND_ASSEMBLE: no values; the context assembles the band on the device
 *                      from pmg_hierarchy_desc.geometry (assemble_patch_stiffness,
 *                      assembly.cpp:127-248, with Gauss-Legendre p+1 points).
 *   PMG_BAND_KRONECKER: no values read; the context applies the patch operator
 *                      matrix-free as the Kronecker sum of the univariate mass
 *                      and stiffness matrices (the identity the reference tests in
 *                      test_assembly.cpp:112-146).  Every patch map in
 *                      pmg_hierarchy_desc.geometry must be axis-aligned affine,
 *                      x_a = c_a + h_a xi_a; pmg_ctx_create returns PMG_ERR_CONFIG
 *                      otherwise.  Results agree with the assembled band to
 *                      rounding (about 1e-15 relative), not bitwise. */
enum { PMG_BAND_TENSOR = 0, PMG_BAND_CSR = 1, PMG_BAND_ASSEMBLE = 2, PMG_BAND_KRONECKER = 3 };

/* Geometry of one patch (GeometryMap, geometry.hpp): a tensor B-spline map
 * whose axis a uses the uniform open-knot space of degree[a] with elements[a]
 * elements (free ends); ctrl holds prod(elements[a]+degree[a]) control points
 * of dim coordinates each, axis 0 fastest. */
typedef struct {
  int degree[3];
  int elements[3];
  const double* ctrl;
} pmg_patch_geometry;

typedef struct {
  int nu;
  int mu;
  double tau;
  double sigma_scale;
  int damp_coarse;
} pmg_cycle_params;

typedef struct {
  int kind; /* PMG_PIECE_* */
  int patch;
  int64_t ndofs;
  const int32_t* dofs; /* global dof ids, piece lattice order (first axis fastest) */
  /* interior / face: fast-diagonalization payload */
  int naxes;
  int dims[3];
  const double* V[3]; /* column-major dims[a] x dims[a], V^T M V = I */
  const double* diag; /* prod(dims): scale * (sigma + sum_a lambda_a) */
  /* edge: banded Cholesky factor, l[i*(bw+1) + (i-k)] */
  int chol_dim;
  int chol_bw;
  const double* chol_l;
  /* vertex: the diagonal value of L_T */
  double scalar;
} pmg_piece_desc;

typedef struct {
  int elements;
  int64_t num_dofs;
  const int32_t* l2g; /* [num_patches][ext^dim], -1 on Dirichlet */
  int band_format;
  const double* band;                    /* PMG_BAND_TENSOR */
  const int64_t* const* csr_row_ptr;     /* PMG_BAND_CSR, per patch */
  const int32_t* const* csr_cols;
  const double* const* csr_vals;
  /* two-scale factor from level-1 to this level (unused on level 0) */
  int ts_fine_dim;
  int ts_coarse_dim;
  const int32_t* ts_row_start; /* [fine_dim] first coarse column */
  const int32_t* ts_row_len;   /* [fine_dim] nonzeros in the row */
  const int32_t* ts_row_off;   /* [fine_dim] offset into ts_vals */
  const double* ts_vals;
  int num_pieces;
  const pmg_piece_desc* pieces;
} pmg_level_desc;

typedef struct {
  int dim;
  int degree;
  int num_patches;
  int num_levels; /* finest level = num_levels - 1 */
  pmg_cycle_params params;
  const pmg_level_desc* levels;
  int coarse_n;
  const double* coarse_A; /* dense, column-major */
  const double* coarse_L; /* lower Cholesky factor of coarse_A, column-major */
  /* per patch; required when a level uses PMG_BAND_ASSEMBLE or PMG_BAND_KRONECKER, else may be NULL */
  const pmg_patch_geometry* geometry;
} pmg_hierarchy_desc;

#ifdef __cplusplus
}
#endif

#endif /* PMG_TYPES_H */
