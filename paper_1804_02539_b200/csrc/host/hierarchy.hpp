// Grid hierarchy for the PCG + V-cycle path: per-level dof mappers, patch
// stiffness bands, two-scale factors, smoother pieces with their factorized
// payloads, the coarsest-level matrix and its Cholesky factor, and the load
// vector.  This is the setup the solve path consumes; it is built once on the
// host and handed, unchanged, to both the GPU context and the CPU oracle.
//
// Restates (Eigen-free):
//   Hierarchy ctor           /root/reference/proj/src/multigrid.cpp:16-50
//   assemble_patch_stiffness /root/reference/proj/src/assembly.cpp:127-248
//   assemble_rhs             /root/reference/proj/src/assembly.cpp:299-365
//   FastDiagonalSolver ctor  /root/reference/proj/src/tensor.cpp:104-130
//   smoother builders        /root/reference/proj/src/smoother.cpp:52-108
//   TransferOperator ctor    /root/reference/proj/src/transfer.cpp:10-19
//
// Deviation: the coarsest level has n0 elements per
// patch direction (level l has n0 * 2^l); the reference hard-codes n0 = 1.
//
// Stiffness storage: the reference's PatchOperator is CSR over the full patch
// lattice with the tensor-band pattern |i_a - j_a| <= p (assembly.cpp:63-111).
// Here the same values are kept index-free: band[k][o][r] with
// o = sum_a (delta_a + p) (2p+1)^a (axis 0 fastest, i.e. the CSR column order)
// and zeros where the column leaves the lattice.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

#include "topology.hpp"

namespace pmg {

struct CycleParams {  // multigrid.hpp:21-27
  int nu = 1;
  int mu = 1;
  double tau = 0.25;
  double sigma_scale = 0.2;
  bool damp_coarse = false;
};

/// Fast-diagonalization payload (tensor.hpp:42-63): per-axis generalized
/// eigenvector matrices (column-major m_a x m_a) and the diagonal
/// scale * (sigma + sum_a lambda_a) over the piece lattice, axis 0 fastest.
struct FDPayload {
  int naxes = 0;
  int dims[3] = {1, 1, 1};
  std::shared_ptr<const Dense> V[3];
  std::vector<double> diag;
};

struct PieceData {
  PieceKind kind;
  int patch;
  std::vector<std::int32_t> dofs;  // global ids, piece lattice order
  double scalar = 0.0;             // vertex: diagonal value of L_T
  BandedCholesky chol;             // edge
  FDPayload fd;                    // interior / face
};

struct Level {
  int elements = 0;
  std::unique_ptr<DofMapper> mapper;
  std::vector<std::int32_t> l2g;  // [K][ext^d] contiguous copy of local_to_global
  std::vector<double> band;       // [K][(2p+1)^d][ext^d]
  TwoScaleMatrix two_scale;       // from level-1 to this level (level >= 1)
  std::vector<PieceData> pieces;
};

/// Source term: a function of the physical point, or one value per
/// quadrature node drawn from a counter-based generator.
struct RhsSpec {
  enum Kind { function, random_nodes } kind = function;
  std::function<double(const double*)> f;
  std::uint64_t seed = 42;
  bool zero = false;  // f == 0: assemble_rhs returns zeros without the quadrature loop
};

class Hierarchy {
 public:
  // host_assembly = false leaves the bands of levels >= 1 empty: the device
  // context assembles them from the patch geometry (PMG_BAND_ASSEMBLE)
  Hierarchy(const MultiPatchDomain& domain, int degree, int n0, int levels, CycleParams params,
            const RhsSpec& rhs, int threads, bool host_assembly = true);
  int dim() const { return domain_->dim; }
  int degree() const { return degree_; }
  int n0() const { return n0_; }
  int num_levels() const { return int(levels_.size()); }
  int finest_level() const { return num_levels() - 1; }
  int num_patches() const { return domain_->num_patches(); }
  const MultiPatchDomain& domain() const { return *domain_; }
  const CycleParams& params() const { return params_; }
  const Level& level(int l) const { return levels_[l]; }
  const Dense& coarse_matrix() const { return coarse_A_; }
  const Dense& coarse_factor() const { return coarse_L_; }
  const std::vector<double>& rhs() const { return rhs_; }
  double setup_seconds() const { return t_setup_; }
  double assemble_seconds() const { return t_assemble_; }

 private:
  std::unique_ptr<MultiPatchDomain> domain_;
  int degree_, n0_;
  CycleParams params_;
  std::vector<Level> levels_;
  Dense coarse_A_, coarse_L_;
  std::vector<double> rhs_;
  double t_setup_ = 0.0, t_assemble_ = 0.0;
};

/// Band offsets per patch: (2p+1)^d.
inline int band_offsets(int dim, int degree) {
  int o = 1;
  for (int a = 0; a < dim; ++a) o *= 2 * degree + 1;
  return o;
}

/// Stiffness of one mapped patch into band[(2p+1)^d][ext^d]
/// (assembly.cpp:127-248); element layers are processed in fixed chunks so the
/// result does not depend on the thread count.
void assemble_patch_band(const GeometryMap& geo, int degree, int elements, double* band, int threads);

/// Load vector over the mapper's dofs (assembly.cpp:299-365).
std::vector<double> assemble_rhs(const DofMapper& mapper, const RhsSpec& rhs, int threads);

/// Counter-based uniform [-1,1) draw used for per-node source terms.
double node_uniform(std::uint64_t seed, std::uint64_t index);

/// Domain generators: reference fixtures (tests/util.hpp:37-126,
/// harness.cpp:118-178) and the BASELINE configs.
MultiPatchDomain make_domain(const std::string& spec, std::uint64_t seed);

/// Stored entry count of the reference CSR (harness.cpp:274-282).
std::int64_t stored_stiffness_entries(int degree, int elements, int dim, int patches);

}  // namespace pmg
