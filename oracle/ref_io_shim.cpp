// ref_io_shim.cpp -- TEST INFRASTRUCTURE ONLY.  The reference's SWEMESH
// reader / writer (/root/reference/proj/include/swe/io.hpp:80-165), included
// in place and exported with a C ABI so the tests can check
// include/swe/swemesh.hpp against it (values, bytes written, error texts).
// Built by oracle/Makefile into oracle/_ref/libswe_ref_io.so; io.hpp needs
// nlohmann/json (found under site-packages).
#define swe ref_swe
#include "swe/io.hpp"
#undef swe

#include <cstring>
#include <sstream>
#include <string>

namespace {
void put(const std::exception& e, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
}
}  // namespace

#define EXPORT extern "C" __attribute__((visibility("default")))

// parse a text (read_mesh_native on an istringstream) or a file
EXPORT void* refio_parse(const char* text, long long n, char* err, int errlen) {
  try {
    std::istringstream in(std::string(text, (size_t)n));
    return new ref_swe::NativeMesh(ref_swe::read_mesh_native(in));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void* refio_read(const char* path, char* err, int errlen) {
  try {
    return new ref_swe::NativeMesh(ref_swe::read_mesh_native_file(path));
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return nullptr;
  }
}

EXPORT void refio_sizes(void* h, int* nn, int* nc) {
  const auto& m = *static_cast<ref_swe::NativeMesh*>(h);
  *nn = (int)m.raw.nodes.size();
  *nc = (int)m.raw.triangles.size();
}

EXPORT void refio_export(void* h, double* xy, int* tris, double* bed, double* man) {
  const auto& m = *static_cast<ref_swe::NativeMesh*>(h);
  for (size_t i = 0; i < m.raw.nodes.size(); ++i) {
    xy[2 * i] = m.raw.nodes[i].x;
    xy[2 * i + 1] = m.raw.nodes[i].y;
  }
  for (size_t c = 0; c < m.raw.triangles.size(); ++c)
    for (int k = 0; k < 3; ++k) tris[3 * c + k] = m.raw.triangles[c][k];
  std::memcpy(bed, m.bed.data(), m.bed.size() * sizeof(double));
  std::memcpy(man, m.manning.data(), m.manning.size() * sizeof(double));
}

EXPORT void refio_free(void* h) { delete static_cast<ref_swe::NativeMesh*>(h); }

EXPORT int refio_write(const char* path, int nn, const double* xy, int nc, const int* tris,
                       const double* bed, const double* man, char* err, int errlen) {
  try {
    ref_swe::RawMesh raw;
    raw.nodes.resize(nn);
    for (int i = 0; i < nn; ++i) raw.nodes[i] = {xy[2 * i], xy[2 * i + 1]};
    raw.triangles.resize(nc);
    for (int c = 0; c < nc; ++c) raw.triangles[c] = {tris[3 * c], tris[3 * c + 1], tris[3 * c + 2]};
    ref_swe::write_mesh_native_file(path, raw, std::vector<double>(bed, bed + nc),
                                    std::vector<double>(man, man + nc));
    return 0;
  } catch (const std::exception& e) {
    put(e, err, errlen);
    return 1;
  }
}
