// swe/partition.hpp -- domain decomposition for multi-GPU runs (SURVEY.md
// §8(e); the reference has none: SPEC.md lists distributed memory as a
// non-goal).
//
// Recursive coordinate bisection of cell centroids into P parts.  Part p's
// local mesh holds its owned cells (first, in global order), a one-cell ghost
// layer (the non-owned neighbours across its edges), and every edge touching
// an owned cell, in global edge order with the global orientation.  Cut edges
// are therefore evaluated by both sides from identical inputs, and every
// owned cell sums the same three contributions in the same local order as on
// one device: a P-part run is bit-identical to the single-domain run.
// Exchange plan: part p sends to peer q the state of its owned cells that are
// ghosts of q, and receives its ghosts owned by q -- both lists ordered by
// global cell id, so sender and receiver agree without negotiation.
#pragma once

#include <algorithm>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "swe/mesh.hpp"

namespace swe {

/// part id per cell: recursive bisection of the longer bounding-box axis;
/// ties broken by cell id (deterministic).  Without weights the cut is the
/// median (equal cell counts); with per-cell weights (the step's cost per
/// cell, see cost_weights) it is the weighted median, so parts get equal
/// WORK -- on a partly dry domain equal counts leave the wet parts slower
/// (measured: a dry 1.28M-cell part steps in 0.027 ms, a wet one in 0.115).
namespace detail {
inline std::vector<int> rcb_partition_centroids(const std::vector<Vec2>& cent, int nparts,
                                                const std::vector<double>* weights) {
  if (nparts < 1) throw config_error("rcb_partition: nparts must be >= 1");
  const int C = static_cast<int>(cent.size());
  if (weights && static_cast<int>(weights->size()) != C)
    throw config_error("rcb_partition: one weight per cell required");
  std::vector<int> part(C, 0);
  std::vector<int> idx(C);
  std::iota(idx.begin(), idx.end(), 0);
  struct Job {
    int lo, hi, p0, np;
  };
  std::vector<Job> stack{{0, C, 0, nparts}};
  while (!stack.empty()) {
    const Job j = stack.back();
    stack.pop_back();
    if (j.np == 1 || j.hi - j.lo <= 1) {
      for (int i = j.lo; i < j.hi; ++i) part[idx[i]] = j.p0;
      continue;
    }
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int i = j.lo; i < j.hi; ++i) {
      const Vec2 c = cent[idx[i]];
      x0 = std::min(x0, c.x);
      x1 = std::max(x1, c.x);
      y0 = std::min(y0, c.y);
      y1 = std::max(y1, c.y);
    }
    const bool along_x = (x1 - x0) >= (y1 - y0);
    const int nleft = j.np / 2;
    auto key = [&](int c) { return along_x ? cent[c].x : cent[c].y; };
    auto less = [&](int a, int b) {
      const double ka = key(a), kb = key(b);
      return ka != kb ? ka < kb : a < b;
    };
    int cut = j.lo + static_cast<int>((static_cast<long long>(j.hi - j.lo) * nleft) / j.np);
    if (!weights) {
      std::nth_element(idx.begin() + j.lo, idx.begin() + cut, idx.begin() + j.hi, less);
    } else {  // weighted median: left gets nleft/np of the range's weight
      std::sort(idx.begin() + j.lo, idx.begin() + j.hi, less);
      double total = 0.0;
      for (int i = j.lo; i < j.hi; ++i) total += (*weights)[idx[i]];
      const double target = total * nleft / j.np;
      double acc = 0.0;
      cut = j.lo;
      while (cut < j.hi - 1 && acc + (*weights)[idx[cut]] <= target) acc += (*weights)[idx[cut++]];
      cut = std::max(cut, j.lo + 1);
    }
    stack.push_back({j.lo, cut, j.p0, nleft});
    stack.push_back({cut, j.hi, j.p0 + nleft, j.np - nleft});
  }
  return part;
}
}  // namespace detail

inline std::vector<int> rcb_partition(const Mesh& m, int nparts,
                                      const std::vector<double>* weights = nullptr) {
  return detail::rcb_partition_centroids(m.cell_centroid, nparts, weights);
}

/// Per-cell cost of the fused step for a weighted partition: 1 for a dry
/// cell, wet_cost for a wet one (h >= h_dry).  wet_cost = 5 fits the
/// measured part step times on B200 with dry-tile skipping (least squares
/// over 2/4/8-part splits of the 10M channel: 0.080 ms per million wet
/// cells, 0.015 per million dry ones, tools/scaling_proxy.py).
inline std::vector<double> cost_weights(const std::vector<double>& h, double h_dry,
                                        double wet_cost = 5.0) {
  std::vector<double> w(h.size());
  for (size_t c = 0; c < h.size(); ++c) w[c] = h[c] >= h_dry ? wet_cost : 1.0;
  return w;
}

/// One part's mesh in local numbering (owned cells first) plus its exchange plan.
struct LocalMesh {
  int part = 0;
  int n_owned = 0;
  std::vector<int> cells;  // local cell -> global cell
  std::vector<int> edges;  // local edge -> global edge
  // SoA arrays of swe_mesh_view (local numbering)
  std::vector<double> area, inradius, bed, manning, cx, cy;
  std::vector<int> cell_edge, cell_sign;  // [3 * n_cells]
  std::vector<int> edge_left, edge_right;
  std::vector<double> nx, ny, len;
  // exchange plan (local cell ids), one block per peer
  std::vector<int> peers;
  std::vector<std::vector<int>> send;  // owned cells peer needs
  std::vector<std::vector<int>> recv;  // ghosts owned by peer
};

inline LocalMesh build_local_mesh(const Mesh& m, const std::vector<int>& part, int p) {
  const int C = m.n_cells(), E = m.n_edges();
  if (static_cast<int>(part.size()) != C) throw config_error("build_local_mesh: part size");
  LocalMesh L;
  L.part = p;
  std::vector<int> local(C, -1);
  for (int c = 0; c < C; ++c)
    if (part[c] == p) {
      local[c] = static_cast<int>(L.cells.size());
      L.cells.push_back(c);
    }
  L.n_owned = static_cast<int>(L.cells.size());
  // edges touching an owned cell, global order; ghosts = their other cells
  std::vector<int> ghosts;
  for (int e = 0; e < E; ++e) {
    const int l = m.edge_left[e], r = m.edge_right[e];
    const bool ol = part[l] == p, orr = r >= 0 && part[r] == p;
    if (!ol && !orr) continue;
    L.edges.push_back(e);
    if (!ol) ghosts.push_back(l);
    if (r >= 0 && !orr) ghosts.push_back(r);
  }
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  for (int g : ghosts) {
    local[g] = static_cast<int>(L.cells.size());
    L.cells.push_back(g);
  }
  const int nl = static_cast<int>(L.cells.size()), ne = static_cast<int>(L.edges.size());
  std::vector<int> ledge(E, -1);
  for (int i = 0; i < ne; ++i) ledge[L.edges[i]] = i;

  L.area.resize(nl);
  L.inradius.resize(nl);
  L.bed.resize(nl);
  L.manning.resize(nl);
  L.cx.resize(nl);
  L.cy.resize(nl);
  L.cell_edge.resize(3 * static_cast<size_t>(nl));
  L.cell_sign.resize(3 * static_cast<size_t>(nl));
  for (int i = 0; i < nl; ++i) {
    const int c = L.cells[i];
    L.area[i] = m.cell_area[c];
    L.inradius[i] = m.cell_inradius[c];
    L.bed[i] = m.cell_bed[c];
    L.manning[i] = m.cell_manning[c];
    L.cx[i] = m.cell_centroid[c].x;
    L.cy[i] = m.cell_centroid[c].y;
    // owned cells keep all three incidences in reference order; a ghost's
    // missing incidences point at one of its present edges (ghosts are never
    // updated, so only the present edges' sides matter)
    int present = -1;
    for (int k = 0; k < 3; ++k)
      if (ledge[m.cell_edges[c][k].edge] >= 0) present = k;
    for (int k = 0; k < 3; ++k) {
      const int kk = ledge[m.cell_edges[c][k].edge] >= 0 ? k : present;
      L.cell_edge[3 * static_cast<size_t>(i) + k] = ledge[m.cell_edges[c][kk].edge];
      L.cell_sign[3 * static_cast<size_t>(i) + k] = m.cell_edges[c][kk].sign;
    }
  }
  L.edge_left.resize(ne);
  L.edge_right.resize(ne);
  L.nx.resize(ne);
  L.ny.resize(ne);
  L.len.resize(ne);
  for (int i = 0; i < ne; ++i) {
    const int e = L.edges[i];
    L.edge_left[i] = local[m.edge_left[e]];
    L.edge_right[i] = m.edge_right[e] < 0 ? -1 : local[m.edge_right[e]];
    L.nx[i] = m.edge_normal[e].x;
    L.ny[i] = m.edge_normal[e].y;
    L.len[i] = m.edge_length[e];
  }
  // exchange plan: recv = my ghosts grouped by owner; send = my owned cells
  // that are ghosts of each peer (a peer's ghost is a non-owned endpoint of
  // an edge touching one of its owned cells)
  const int P = 1 + *std::max_element(part.begin(), part.end());
  std::vector<std::vector<int>> send_g(P), recv_g(P);
  for (int g : ghosts) recv_g[part[g]].push_back(g);
  for (int e = 0; e < E; ++e) {
    const int l = m.edge_left[e], r = m.edge_right[e];
    if (r < 0) continue;
    if (part[l] == p && part[r] != p) send_g[part[r]].push_back(l);
    if (part[r] == p && part[l] != p) send_g[part[l]].push_back(r);
  }
  for (int q = 0; q < P; ++q) {
    auto& s = send_g[q];
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    if (s.empty() && recv_g[q].empty()) continue;
    L.peers.push_back(q);
    std::vector<int> sl, rl;
    for (int c : s) sl.push_back(local[c]);
    for (int c : recv_g[q]) rl.push_back(local[c]);
    L.send.push_back(std::move(sl));
    L.recv.push_back(std::move(rl));
  }
  return L;
}

}  // namespace swe
