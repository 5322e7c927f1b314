// Geometry maps, multi-patch topology, dof identification and the additive
// piece decomposition used by the hybrid smoother.
//
// Restates, Eigen-free:
//   geometry.hpp/.cpp  (/root/reference/proj/src/geometry.cpp:10-202)
//   topology.hpp/.cpp  (/root/reference/proj/src/topology.cpp:25-600)
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "numerics.hpp"

namespace pmg {

// ---------------------------------------------------------------- geometry
/// Tensor B-spline map (0,1)^d -> R^d; control point f (axis 0 fastest) is
/// row f of `ctrl` stored as ctrl[f*d + c] (geometry.hpp:13-41).
class GeometryMap {
 public:
  GeometryMap() = default;
  GeometryMap(std::vector<UnivariateSpace> spaces, std::vector<double> ctrl);
  int dim() const { return int(spaces_.size()); }
  const std::vector<UnivariateSpace>& spaces() const { return spaces_; }
  const std::vector<double>& control_points() const { return ctrl_; }
  std::int64_t num_control_points() const { return std::int64_t(ctrl_.size()) / dim(); }
  void eval(const double* param, double* x) const;          // geometry.cpp:50-60
  void jacobian(const double* param, double* J) const;      // geometry.cpp:62-79, J[i*d+j] = dx_i/dxhat_j
  GeometryMap restrict_to_subcell(const std::vector<int>& cell, int m) const;  // geometry.cpp:140-191
  static GeometryMap axis_aligned_box(const std::vector<double>& corner,
                                      const std::vector<double>& extent);     // geometry.cpp:193-202

 private:
  std::vector<UnivariateSpace> spaces_;
  std::vector<double> ctrl_;
};

// ---------------------------------------------------------------- topology
enum class SideTag : std::uint8_t { dirichlet, neumann, matched };

inline int side_axis(int side) { return side / 2; }
inline int side_end(int side) { return side % 2; }
inline int side_of(int axis, int end) { return 2 * axis + end; }

struct Interface {
  int patch_a, side_a;
  int patch_b, side_b;
  std::uint8_t orientation;
};

std::vector<int> inside_axes(int dim, int side);
std::array<int, 2> map_side_index(int dim, std::uint8_t orientation, const std::array<int, 2>& idx,
                                  const std::array<int, 2>& sizes_b);
std::array<double, 2> map_side_param(int dim, std::uint8_t orientation, const std::array<double, 2>& uv);

struct MultiPatchDomain {
  int dim = 0;
  std::vector<GeometryMap> patches;
  std::vector<Interface> interfaces;
  std::vector<std::array<SideTag, 6>> side_tags;
  double geometric_tolerance = 0.0;
  int num_patches() const { return int(patches.size()); }
  SideTag tag(int patch, int side) const { return side_tags[patch][side]; }
  void side_point(int patch, int side, const std::array<double, 2>& uv, double* x) const;
};

/// Geometric interface discovery by side sampling (topology.cpp:132-210).
void build_topology(MultiPatchDomain& domain);
/// Split every patch into m^dim children (topology.cpp:212-252).
MultiPatchDomain split_patches(const MultiPatchDomain& domain, int m);

/// Per-patch tensor lattices -> global dof ids; -1 on Dirichlet
/// (topology.hpp:88-125, topology.cpp:280-372).
class DofMapper {
 public:
  DofMapper(const MultiPatchDomain& domain, int degree, int elements);
  const MultiPatchDomain& domain() const { return *domain_; }
  int degree() const { return degree_; }
  int elements() const { return elements_; }
  int extent() const { return elements_ + degree_; }
  std::int64_t lattice_size() const { return per_patch_; }
  std::int64_t num_dofs() const { return num_dofs_; }
  const std::vector<std::int32_t>& local_to_global(int patch) const { return l2g_[patch]; }
  std::int32_t global_of(int patch, std::int64_t local) const { return l2g_[patch][local]; }
  int rep_count(std::int32_t g) const { return rep_off_[g + 1] - rep_off_[g]; }
  std::int32_t owner_patch(std::int32_t g) const { return rep_patch_[rep_off_[g]]; }
  std::int64_t flat_of(const std::vector<int>& idx) const;
  const std::vector<std::int32_t>& rep_offsets() const { return rep_off_; }
  const std::vector<std::int32_t>& rep_patches() const { return rep_patch_; }
  const std::vector<std::int32_t>& rep_locals() const { return rep_local_; }

 private:
  const MultiPatchDomain* domain_;
  int degree_, elements_;
  std::int64_t per_patch_ = 0;
  std::int64_t num_dofs_ = 0;
  std::vector<std::vector<std::int32_t>> l2g_;
  std::vector<std::int32_t> rep_off_, rep_patch_, rep_local_;
};

enum class PieceKind { interior = 0, face = 1, edge = 2, vertex = 3 };

struct Piece {
  PieceKind kind;
  int patch;
  std::vector<std::int32_t> dofs;
  std::vector<UnivariateSpace> spaces;
};

/// Additive decomposition: interiors, faces (3D), edges, vertices
/// (topology.cpp:394-600).
std::vector<Piece> classify_dofs(const DofMapper& mapper);

}  // namespace pmg
