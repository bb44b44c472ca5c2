// swe/vtk.hpp -- a parallel writer for the reference's VTK legacy snapshot
// (reference io.hpp:171-206 write_vtk_snapshot).
//
// The same file byte for byte -- the same sections, the same 17-significant-
// digit numbers (%.17g, io.hpp:24-28: std::to_chars with chars_format::general
// and precision 17 prints exactly what printf does), the same derived fields
// (eta = h + z, velocity() with the default dry threshold) -- but every
// section is formatted by all host threads into per-thread buffers and the
// buffers are written in order.  The reference streams ~60M lines through an
// ofstream one value at a time (a 10M-cell snapshot is ~1.4 GB of text).
#pragma once

#include <charconv>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "swe/engine.hpp"
#include "swe/kernels.hpp"
#include "swe/swemesh.hpp"

namespace swe {

namespace detail {

inline char* vtk_put_int(char* p, long long v) { return std::to_chars(p, p + 24, v).ptr; }

// one section of per-item lines, formatted by T threads into parts (appended)
template <class F>
void vtk_section(std::vector<std::string>& parts, size_t n, size_t bytes_per_item, int T, F&& line) {
  const size_t base = parts.size();
  parts.resize(base + (size_t)T);
  swemesh::detail::parallel(T, [&](int i) {
    const size_t a = n * i / T, b = n * (i + 1) / T;
    std::string& s = parts[base + i];
    s.resize(bytes_per_item * (b - a) + 16);
    char* p = s.data();
    for (size_t k = a; k < b; ++k) p = line(p, k);
    s.resize((size_t)(p - s.data()));
  });
}

}  // namespace detail

/// write_vtk_snapshot (io.hpp:171-206), byte-identical, formatted by
/// `threads` host threads (<= 0: all cores).
inline void write_vtk_snapshot_parallel(const Mesh& mesh, const FieldState& s, double t,
                                        const std::string& path, int threads = 0) {
  if (s.size() != mesh.n_cells())
    throw io_error("write_vtk_snapshot: state has " + std::to_string(s.size()) +
                   " cells, mesh has " + std::to_string(mesh.n_cells()));
  std::FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) throw io_error("cannot open '" + path + "' for writing");
  const size_t nn = mesh.nodes.size(), nc = (size_t)mesh.n_cells();
  const int T = swemesh::detail::thread_count(threads, 60 * (nn + 6 * nc));
  using swemesh::put_double;
  std::vector<std::string> parts;
  char buf[64];
  auto text = [&](const std::string& x) { parts.push_back(x); };
  text("# vtk DataFile Version 3.0\nswe snapshot t=" +
       std::string(buf, put_double(buf, t)) + "\nASCII\nDATASET UNSTRUCTURED_GRID\nPOINTS " +
       std::to_string(mesh.n_nodes()) + " double\n");
  detail::vtk_section(parts, nn, 56, T, [&](char* p, size_t k) {
    p = put_double(p, mesh.nodes[k].x);
    *p++ = ' ';
    p = put_double(p, mesh.nodes[k].y);
    *p++ = ' ';
    *p++ = '0';
    *p++ = '\n';
    return p;
  });
  text("CELLS " + std::to_string(mesh.n_cells()) + ' ' + std::to_string(4LL * mesh.n_cells()) + '\n');
  detail::vtk_section(parts, nc, 40, T, [&](char* p, size_t c) {
    *p++ = '3';
    for (int k = 0; k < 3; ++k) {
      *p++ = ' ';
      p = detail::vtk_put_int(p, mesh.cell_nodes[c][k]);
    }
    *p++ = '\n';
    return p;
  });
  text("CELL_TYPES " + std::to_string(mesh.n_cells()) + '\n');
  detail::vtk_section(parts, nc, 2, T, [](char* p, size_t) {
    *p++ = '5';
    *p++ = '\n';
    return p;
  });
  text("CELL_DATA " + std::to_string(mesh.n_cells()) + '\n');
  auto scalars = [&](const char* name, auto value) {
    text(std::string("SCALARS ") + name + " double 1\nLOOKUP_TABLE default\n");
    detail::vtk_section(parts, nc, 26, T, [&](char* p, size_t c) {
      p = put_double(p, value(c));
      *p++ = '\n';
      return p;
    });
  };
  scalars("h", [&](size_t c) { return s.h[c]; });
  scalars("eta", [&](size_t c) { return s.h[c] + mesh.cell_bed[c]; });
  scalars("z", [&](size_t c) { return mesh.cell_bed[c]; });
  text("VECTORS velocity double\n");
  const PhysParams pv;  // dry threshold only guards the division here (io.hpp:200)
  detail::vtk_section(parts, nc, 56, T, [&](char* p, size_t c) {
    const Vec2 v = velocity(s.cell((int)c), pv.h_dry);
    p = put_double(p, v.x);
    *p++ = ' ';
    p = put_double(p, v.y);
    *p++ = ' ';
    *p++ = '0';
    *p++ = '\n';
    return p;
  });
  bool ok = true;
  for (const std::string& x : parts) ok = ok && std::fwrite(x.data(), 1, x.size(), fp) == x.size();
  const int rc = std::fclose(fp);
  if (!ok || rc != 0) throw io_error("write failed for '" + path + "'");
}

}  // namespace swe
