// Interface-dof exchange plan of one rank on one level -- header-only, shared
// by the CUDA context (libpmg_cuda) and the host library's test hook.
//
// Restates RankLayout (parallel.hpp:133-165, parallel.cpp:200-237) for the
// per-patch lattice layout: patches go to ranks in contiguous blocks
// (contiguous_partition, parallel.cpp:181-198); an "interface dof" of a rank
// is a global dof with at least two replicas overall (any rank) and at least
// one replica on this rank.  Its global value is the sum of the per-rank
// partial sums (each partial summed over the rank's replicas in ascending
// (patch, local) order), added in ascending rank order -- the fold of
// ParallelBackend::accumulate (parallel.cpp:306-337), so every sharing rank
// obtains the same bits.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace pmgplan {

struct Partition {
  int ranks = 1;
  std::vector<int> patch_begin;  // [ranks + 1]
  int rank_of(int patch) const {
    int r = int(std::upper_bound(patch_begin.begin(), patch_begin.end(), patch) - patch_begin.begin()) - 1;
    return r;
  }
};

// contiguous_partition (parallel.cpp:181-198)
inline Partition contiguous(int num_patches, int ranks) {
  if (ranks < 1 || ranks > num_patches || ranks > 64) throw std::invalid_argument("partition: bad rank count");
  Partition p;
  p.ranks = ranks;
  for (int r = 0; r <= ranks; ++r) p.patch_begin.push_back(int(int64_t(num_patches) * r / ranks));
  return p;
}

struct Neighbor {
  int rank;
  std::vector<int32_t> iface;  // positions in the rank's interface list, ascending global id
};

struct RankPlan {
  // interface dofs of this rank, ascending global id
  std::vector<int32_t> iface_g;
  std::vector<int32_t> rep_off;   // [n_iface + 1] local replicas (lattice slots of this rank)
  std::vector<int32_t> rep_slot;
  // fold order: for iface i, sources comb_src[comb_off[i] .. comb_off[i+1]) in
  // ascending rank order; -1 = this rank's partial, otherwise an index into
  // the concatenation of the receive buffers (neighbour order)
  std::vector<int32_t> comb_off;
  std::vector<int32_t> comb_src;
  std::vector<Neighbor> neighbors;  // ascending rank
  std::vector<int32_t> iface_of_g;  // [num_dofs] -> iface position or -1
};

// l2g_all: [num_patches][S] global ids (-1 Dirichlet) of one level
inline RankPlan build(const int32_t* l2g_all, int num_patches, int64_t S, int64_t num_dofs, const Partition& part,
                      int rank) {
  const int pb = part.patch_begin[rank], pe = part.patch_begin[rank + 1];
  // replica counts per rank for every global dof
  std::vector<int32_t> total(size_t(num_dofs), 0), mine(size_t(num_dofs), 0);
  std::vector<uint64_t> rank_mask(size_t(num_dofs), 0);
  for (int k = 0; k < num_patches; ++k) {
    const int r = part.rank_of(k);
    for (int64_t f = 0; f < S; ++f) {
      const int32_t g = l2g_all[size_t(k) * S + f];
      if (g < 0) continue;
      total[g]++;
      rank_mask[g] |= uint64_t(1) << r;
      if (k >= pb && k < pe) mine[g]++;
    }
  }
  RankPlan p;
  p.iface_of_g.assign(size_t(num_dofs), -1);
  for (int64_t g = 0; g < num_dofs; ++g)
    if (mine[g] > 0 && total[g] >= 2) {
      p.iface_of_g[g] = int32_t(p.iface_g.size());
      p.iface_g.push_back(int32_t(g));
    }
  const size_t n = p.iface_g.size();
  // local replicas in ascending (patch, local) order
  p.rep_off.assign(n + 1, 0);
  for (int k = pb; k < pe; ++k)
    for (int64_t f = 0; f < S; ++f) {
      const int32_t g = l2g_all[size_t(k) * S + f];
      if (g >= 0 && p.iface_of_g[g] >= 0) p.rep_off[p.iface_of_g[g] + 1]++;
    }
  for (size_t i = 0; i < n; ++i) p.rep_off[i + 1] += p.rep_off[i];
  p.rep_slot.resize(p.rep_off.back());
  std::vector<int32_t> cur(p.rep_off.begin(), p.rep_off.end() - 1);
  for (int k = pb; k < pe; ++k)
    for (int64_t f = 0; f < S; ++f) {
      const int32_t g = l2g_all[size_t(k) * S + f];
      if (g >= 0 && p.iface_of_g[g] >= 0) p.rep_slot[cur[p.iface_of_g[g]]++] = int32_t((k - pb) * S + f);
    }
  // neighbours and their shared lists (ascending global id == ascending iface position)
  std::vector<std::vector<int32_t>> shared(part.ranks);
  for (size_t i = 0; i < n; ++i) {
    const uint64_t m = rank_mask[p.iface_g[i]];
    for (int r = 0; r < part.ranks; ++r)
      if (r != rank && (m >> r & 1)) shared[r].push_back(int32_t(i));
  }
  std::vector<int> nb_index(part.ranks, -1);
  std::vector<int32_t> recv_base;
  int32_t base = 0;
  for (int r = 0; r < part.ranks; ++r)
    if (!shared[r].empty()) {
      nb_index[r] = int(p.neighbors.size());
      recv_base.push_back(base);
      base += int32_t(shared[r].size());
      p.neighbors.push_back({r, shared[r]});
    }
  // fold sources in ascending rank order
  std::vector<int32_t> cursor(p.neighbors.size(), 0);
  p.comb_off.assign(n + 1, 0);
  for (size_t i = 0; i < n; ++i) {
    const uint64_t m = rank_mask[p.iface_g[i]];
    for (int r = 0; r < part.ranks; ++r) {
      if (!(m >> r & 1)) continue;
      if (r == rank) {
        p.comb_src.push_back(-1);
      } else {
        const int j = nb_index[r];
        p.comb_src.push_back(recv_base[j] + cursor[j]++);
      }
    }
    p.comb_off[i + 1] = int32_t(p.comb_src.size());
  }
  return p;
}

}  // namespace pmgplan
