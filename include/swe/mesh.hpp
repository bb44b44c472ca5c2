// swe/mesh.hpp -- mesh input of the drop-in API.
//
// Same types and semantics as the reference's mesh.hpp (RawMesh, Mesh,
// generate_square_mesh, build_mesh, mesh_diagnostics; /root/reference/proj/
// include/swe/mesh.hpp:14-301), re-implemented: the edge numbering comes from
// a bucket pass over the lower node index instead of a global comparison sort,
// but it reproduces the reference order exactly -- edges ordered by
// (min node, max node), the lower cell index on the left (mesh.hpp:187-189,
// :210, :221) -- and every geometric quantity uses the reference's
// expression (area :112-114, perimeter :163, inradius :167, normal :208), so a
// Mesh built here is bit-identical to the reference's.
//
// Also: generate_unstructured_mesh (jittered nodes, random diagonals, random
// node/cell numbering) for the benchmark configurations.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "swe/core.hpp"

namespace swe {

struct RawMesh {
  std::vector<Vec2> nodes;
  std::vector<std::array<int, 3>> triangles;
};

/// (edge, orientation) incidence of a cell; sign * normal is outward.
struct EdgeUse {
  int edge = -1;
  int sign = 0;
};

constexpr int kBoundary = -1;

struct Mesh {
  std::vector<Vec2> nodes;

  std::vector<std::array<int, 3>> cell_nodes;  // CCW
  std::vector<double> cell_area;
  std::vector<Vec2> cell_centroid;
  std::vector<double> cell_inradius;
  std::vector<double> cell_bed;
  std::vector<double> cell_manning;
  std::vector<std::array<EdgeUse, 3>> cell_edges;

  std::vector<std::array<int, 2>> edge_nodes;
  std::vector<int> edge_left;
  std::vector<int> edge_right;  // kBoundary for walls
  std::vector<Vec2> edge_normal;
  std::vector<double> edge_length;

  int n_nodes() const { return static_cast<int>(nodes.size()); }
  int n_cells() const { return static_cast<int>(cell_nodes.size()); }
  int n_edges() const { return static_cast<int>(edge_nodes.size()); }
  int n_boundary_edges() const {
    return static_cast<int>(std::count(edge_right.begin(), edge_right.end(), kBoundary));
  }
};

/// Structured triangulation, uniform lower-left -> upper-right diagonal
/// (reference mesh.hpp:67-87: same node and triangle order).
inline RawMesh generate_square_mesh(int nx, int ny, double lx, double ly) {
  if (nx < 1 || ny < 1) throw mesh_error("generate_square_mesh: nx and ny must be >= 1");
  if (!(lx > 0.0) || !(ly > 0.0)) throw mesh_error("generate_square_mesh: Lx and Ly must be > 0");
  RawMesh raw;
  const double dx = lx / nx, dy = ly / ny;
  raw.nodes.resize(static_cast<size_t>(nx + 1) * (ny + 1));
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i)
      raw.nodes[static_cast<size_t>(j) * (nx + 1) + i] = {i == nx ? lx : i * dx,
                                                          j == ny ? ly : j * dy};
  raw.triangles.resize(static_cast<size_t>(2) * nx * ny);
  size_t t = 0;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int a = j * (nx + 1) + i, b = a + 1, c = a + (nx + 1) + 1, d = a + (nx + 1);
      raw.triangles[t++] = {a, b, c};
      raw.triangles[t++] = {a, c, d};
    }
  return raw;
}

/// 180-degree partner of cell c on a generate_square_mesh grid
/// (reference mesh.hpp:92-98).
inline int rotated_cell_index(int c, int nx, int ny) {
  const int sq = c / 2, upper = c % 2, i = sq % nx, j = sq / nx;
  return 2 * ((ny - 1 - j) * nx + (nx - 1 - i)) + (1 - upper);
}

/// Unstructured variant of the square grid: interior nodes
/// jittered by U(-jitter, +jitter) grid spacings (jitter < 0.25 keeps every
/// triangle positive for either diagonal; SURVEY's 0.3 can invert them), each square split along a
/// random diagonal, then node and cell numbering randomly permuted and each
/// triangle's vertex list randomly rotated/reflected.  Deterministic in seed.
inline RawMesh generate_unstructured_mesh(int nx, int ny, double lx, double ly, double jitter = 0.2,
                                          std::uint64_t seed = 1807) {
  if (nx < 1 || ny < 1) throw mesh_error("generate_unstructured_mesh: nx and ny must be >= 1");
  if (!(lx > 0.0) || !(ly > 0.0))
    throw mesh_error("generate_unstructured_mesh: Lx and Ly must be > 0");
  if (!(jitter >= 0.0) || !(jitter < 0.25))
    throw mesh_error("generate_unstructured_mesh: jitter must lie in [0, 0.25)");
  std::mt19937_64 rng(seed);
  auto unit = [&rng]() { return double(rng() >> 11) * 0x1.0p-53; };  // [0,1)
  const double dx = lx / nx, dy = ly / ny;
  const size_t nn = static_cast<size_t>(nx + 1) * (ny + 1);
  std::vector<Vec2> grid(nn);
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i) {
      double x = i == nx ? lx : i * dx, y = j == ny ? ly : j * dy;
      if (i > 0 && i < nx) x += (2.0 * unit() - 1.0) * jitter * dx;
      if (j > 0 && j < ny) y += (2.0 * unit() - 1.0) * jitter * dy;
      grid[static_cast<size_t>(j) * (nx + 1) + i] = {x, y};
    }
  std::vector<std::array<int, 3>> tris;
  tris.reserve(static_cast<size_t>(2) * nx * ny);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int a = j * (nx + 1) + i, b = a + 1, c = a + (nx + 1) + 1, d = a + (nx + 1);
      if (rng() & 1) {
        tris.push_back({a, b, c});
        tris.push_back({a, c, d});
      } else {
        tris.push_back({a, b, d});
        tris.push_back({b, c, d});
      }
    }
  // random node numbering
  std::vector<int> perm(nn);
  for (size_t i = 0; i < nn; ++i) perm[i] = static_cast<int>(i);
  for (size_t i = nn - 1; i > 0; --i) std::swap(perm[i], perm[rng() % (i + 1)]);
  RawMesh raw;
  raw.nodes.resize(nn);
  for (size_t i = 0; i < nn; ++i) raw.nodes[perm[i]] = grid[i];
  // random cell order and vertex rotation/reflection
  const size_t nt = tris.size();
  for (size_t i = nt - 1; i > 0; --i) std::swap(tris[i], tris[rng() % (i + 1)]);
  raw.triangles.resize(nt);
  for (size_t t = 0; t < nt; ++t) {
    std::array<int, 3> v{perm[tris[t][0]], perm[tris[t][1]], perm[tris[t][2]]};
    const auto r = rng();
    std::rotate(v.begin(), v.begin() + (r % 3), v.end());
    if ((r >> 8) & 1) std::swap(v[1], v[2]);
    raw.triangles[t] = v;
  }
  return raw;
}

/// Triangle centroids in the raw vertex order (reference mesh.hpp:100-108;
/// the case initialisers evaluate fields here).
inline std::vector<Vec2> cell_centroids(const RawMesh& raw) {
  std::vector<Vec2> c(raw.triangles.size());
  for (size_t t = 0; t < raw.triangles.size(); ++t) {
    const auto& tri = raw.triangles[t];
    const Vec2 p0 = raw.nodes[tri[0]], p1 = raw.nodes[tri[1]], p2 = raw.nodes[tri[2]];
    c[t] = {(p0.x + p1.x + p2.x) / 3.0, (p0.y + p1.y + p2.y) / 3.0};
  }
  return c;
}

/// Edge-based mesh build (reference semantics: mesh.hpp:121-240).
inline Mesh build_mesh(const RawMesh& raw, std::vector<double> bathymetry,
                       std::vector<double> manning) {
  const int nn = static_cast<int>(raw.nodes.size());
  const int nc = static_cast<int>(raw.triangles.size());
  if (static_cast<int>(bathymetry.size()) != nc || static_cast<int>(manning.size()) != nc)
    throw mesh_error("build_mesh: bathymetry/manning arrays must have one entry per triangle (got " +
                     std::to_string(bathymetry.size()) + "/" + std::to_string(manning.size()) +
                     " for " + std::to_string(nc) + " triangles)");
  for (int c = 0; c < nc; ++c)
    if (manning[c] < 0.0)
      throw mesh_error("build_mesh: negative Manning coefficient at cell " + std::to_string(c));

  Mesh m;
  m.nodes = raw.nodes;
  m.cell_nodes.resize(nc);
  m.cell_area.resize(nc);
  m.cell_centroid.resize(nc);
  m.cell_inradius.resize(nc);
  m.cell_bed = std::move(bathymetry);
  m.cell_manning = std::move(manning);
  m.cell_edges.assign(nc, {});

  for (int c = 0; c < nc; ++c) {
    std::array<int, 3> t = raw.triangles[c];
    for (int k = 0; k < 3; ++k)
      if (t[k] < 0 || t[k] >= nn)
        throw mesh_error("build_mesh: node index " + std::to_string(t[k]) +
                         " out of range in triangle " + std::to_string(c));
    if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2])
      throw mesh_error("build_mesh: degenerate triangle " + std::to_string(c) +
                       " repeats a node index");
    const Vec2 a = raw.nodes[t[0]];
    double area = 0.5 * cross(raw.nodes[t[1]] - a, raw.nodes[t[2]] - a);
    if (area < 0.0) {  // canonical CCW order
      std::swap(t[1], t[2]);
      area = -area;
    }
    if (!(area > 0.0))
      throw mesh_error("build_mesh: triangle " + std::to_string(c) + " has zero area");
    const Vec2 p0 = raw.nodes[t[0]], p1 = raw.nodes[t[1]], p2 = raw.nodes[t[2]];
    const double perimeter = norm(p1 - p0) + norm(p2 - p1) + norm(p0 - p2);
    m.cell_nodes[c] = t;
    m.cell_area[c] = area;
    m.cell_centroid[c] = {(p0.x + p1.x + p2.x) / 3.0, (p0.y + p1.y + p2.y) / 3.0};
    m.cell_inradius[c] = 2.0 * area / perimeter;
  }

  // Bucket the 3*nc directed edges by their lower node; inside a bucket order
  // by (upper node, cell).  Walking the buckets in node order visits the
  // incidences in exactly the (key, cell) order of the reference's sort.
  struct Slot {
    int hi, cell, local;
  };
  std::vector<int> start(static_cast<size_t>(nn) + 1, 0);
  for (int c = 0; c < nc; ++c)
    for (int k = 0; k < 3; ++k) {
      const int a = m.cell_nodes[c][k], b = m.cell_nodes[c][(k + 1) % 3];
      ++start[static_cast<size_t>(std::min(a, b)) + 1];
    }
  for (int i = 0; i < nn; ++i) start[i + 1] += start[i];
  std::vector<Slot> slots(static_cast<size_t>(3) * nc);
  {
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int c = 0; c < nc; ++c)
      for (int k = 0; k < 3; ++k) {
        const int a = m.cell_nodes[c][k], b = m.cell_nodes[c][(k + 1) % 3];
        slots[fill[std::min(a, b)]++] = {std::max(a, b), c, k};
      }
  }
  m.edge_nodes.reserve(static_cast<size_t>(3) * nc / 2 + nn);
  m.edge_left.reserve(m.edge_nodes.capacity());
  m.edge_right.reserve(m.edge_nodes.capacity());
  m.edge_normal.reserve(m.edge_nodes.capacity());
  m.edge_length.reserve(m.edge_nodes.capacity());
  for (int lo = 0; lo < nn; ++lo) {
    Slot* b = slots.data() + start[lo];
    Slot* e = slots.data() + start[lo + 1];
    std::sort(b, e, [](const Slot& x, const Slot& y) {
      return x.hi != y.hi ? x.hi < y.hi : x.cell < y.cell;
    });
    for (Slot* i = b; i < e;) {
      Slot* j = i;
      while (j < e && j->hi == i->hi) ++j;
      const std::array<int, 2> ab{m.cell_nodes[i->cell][i->local],
                                  m.cell_nodes[i->cell][(i->local + 1) % 3]};
      if (j - i > 2)
        throw mesh_error("build_mesh: non-manifold edge (" + std::to_string(ab[0]) + "," +
                         std::to_string(ab[1]) + ") shared by " + std::to_string(j - i) +
                         " triangles");
      const int edge = m.n_edges();
      const Vec2 d = m.nodes[ab[1]] - m.nodes[ab[0]];
      const double len = norm(d);
      m.edge_nodes.push_back(ab);
      m.edge_normal.push_back({d.y / len, -d.x / len});
      m.edge_length.push_back(len);
      m.edge_left.push_back(i->cell);
      m.edge_right.push_back(kBoundary);
      m.cell_edges[i->cell][i->local] = {edge, +1};
      if (j - i == 2) {
        const Slot& r = i[1];
        const int b0 = m.cell_nodes[r.cell][r.local], b1 = m.cell_nodes[r.cell][(r.local + 1) % 3];
        if (b0 != ab[1] || b1 != ab[0])
          throw mesh_error("build_mesh: non-manifold edge (" + std::to_string(ab[0]) + "," +
                           std::to_string(ab[1]) + ") traversed twice in the same direction; " +
                           "triangles " + std::to_string(i->cell) + " and " +
                           std::to_string(r.cell) + " overlap or are inconsistently oriented");
        m.edge_right[edge] = r.cell;
        m.cell_edges[r.cell][r.local] = {edge, -1};
      }
      i = j;
    }
  }

  for (int c = 0; c < nc; ++c) {  // closed-polygon identity
    Vec2 s{0.0, 0.0};
    double perimeter = 0.0;
    for (const EdgeUse& eu : m.cell_edges[c]) {
      s = s + (eu.sign * m.edge_length[eu.edge]) * m.edge_normal[eu.edge];
      perimeter += m.edge_length[eu.edge];
    }
    if (norm(s) > 1e-10 * perimeter)
      throw mesh_error("build_mesh: cell " + std::to_string(c) +
                       " fails the closed-polygon identity (residual " + std::to_string(norm(s)) +
                       ")");
  }
  return m;
}

struct DiagnosticsReport {
  bool built = false;
  std::string structural_error;
  int nodes = 0, cells = 0, edges = 0, boundary_edges = 0;
  double min_area = 0.0, max_area = 0.0;
  double min_inradius = 0.0;
  int euler_characteristic = 0;
  bool euler_ok = false;
  double max_closure_rel = 0.0;
  bool closure_ok = false;
  bool pass() const { return built && euler_ok && closure_ok && min_area > 0.0; }
};

inline DiagnosticsReport mesh_diagnostics(const Mesh& m) {
  DiagnosticsReport r;
  r.built = true;
  r.nodes = m.n_nodes();
  r.cells = m.n_cells();
  r.edges = m.n_edges();
  r.boundary_edges = m.n_boundary_edges();
  r.euler_characteristic = r.nodes - r.edges + r.cells;
  r.euler_ok = r.euler_characteristic == 1;
  if (!m.cell_area.empty()) {
    r.min_area = *std::min_element(m.cell_area.begin(), m.cell_area.end());
    r.max_area = *std::max_element(m.cell_area.begin(), m.cell_area.end());
    r.min_inradius = *std::min_element(m.cell_inradius.begin(), m.cell_inradius.end());
  }
  for (int c = 0; c < m.n_cells(); ++c) {
    Vec2 s{0.0, 0.0};
    double perimeter = 0.0;
    for (const EdgeUse& eu : m.cell_edges[c]) {
      s = s + (eu.sign * m.edge_length[eu.edge]) * m.edge_normal[eu.edge];
      perimeter += m.edge_length[eu.edge];
    }
    r.max_closure_rel = std::max(r.max_closure_rel, norm(s) / perimeter);
  }
  r.closure_ok = r.max_closure_rel <= 1e-10;
  return r;
}

inline DiagnosticsReport mesh_diagnostics(const RawMesh& raw) {
  try {
    const size_t nc = raw.triangles.size();
    return mesh_diagnostics(build_mesh(raw, std::vector<double>(nc, 0.0), std::vector<double>(nc, 0.0)));
  } catch (const mesh_error& e) {
    DiagnosticsReport r;
    r.structural_error = e.what();
    r.nodes = static_cast<int>(raw.nodes.size());
    r.cells = static_cast<int>(raw.triangles.size());
    return r;
  }
}

}  // namespace swe
