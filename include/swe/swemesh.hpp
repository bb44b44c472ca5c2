// swe/swemesh.hpp -- parallel reader / writer of the reference's SWEMESH 1
// mesh format (reference io.hpp:30-165).
//
//   SWEMESH 1
//   <nnodes> <ncells>
//   x y                    (nnodes lines)
//   i j k z_b n_manning    (ncells lines, 0-based node indices)
//
// Same results and error texts as the reference's read_mesh_native /
// write_mesh_native (io.hpp:80-146): every number parses to the same double
// (correctly rounded std::from_chars == the reference's istream >> double),
// files are written with 17 significant digits exactly as its %.17g, and the
// FIRST offending line (in file order) is reported with its line / token.
// What changes is the machinery: the file is read into one buffer, threads
// count newlines in byte chunks, a prefix sum gives every chunk its global
// line number, and the chunks are parsed (or formatted) in parallel -- the
// reference parses one line at a time through std::istringstream.
#pragma once

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "swe/core.hpp"
#include "swe/mesh.hpp"

namespace swe::swemesh {

struct NativeFile {  // io.hpp NativeMesh
  RawMesh raw;
  std::vector<double> bed;
  std::vector<double> manning;
};

namespace detail {

inline bool is_space(char c) {  // std::isspace in the "C" locale
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// One token the way `std::istream >> T` reads it: skip whitespace, optional
// sign, the longest valid prefix; the next token starts right after it.
inline bool parse_int(const char*& p, const char* e, int& v) {
  while (p < e && is_space(*p)) ++p;
  const char* q = p;
  if (q < e && *q == '+') ++q;
  if (q >= e || !((*q >= '0' && *q <= '9') || (*q == '-' && q == p))) return false;
  const auto r = std::from_chars(q, e, v);
  if (r.ec != std::errc() || r.ptr == q) return false;
  p = r.ptr;
  return true;
}

inline bool parse_double(const char*& p, const char* e, double& v) {
  while (p < e && is_space(*p)) ++p;
  const char* q = p;
  if (q < e && *q == '+') ++q;
  const char* d = (q < e && *q == '-' && q == p) ? q + 1 : q;
  // digits or a decimal point must follow: istream has no inf / nan / hex
  if (d >= e || !((*d >= '0' && *d <= '9') || *d == '.')) return false;
  const auto r = std::from_chars(q, e, v, std::chars_format::general);
  if (r.ec != std::errc() || r.ptr == q) return false;
  p = r.ptr;
  return true;
}

struct Error {
  long long line = -1;  // -1: none
  std::string msg;
  void set(long long l, std::string m) {
    if (line < 0 || l < line) {
      line = l;
      msg = std::move(m);
    }
  }
};

inline std::string token_error(long long line, int col, const char* what) {
  return "line " + std::to_string(line) + ", token " + std::to_string(col) + ": expected " + what;
}

template <class T>
bool token(const char*& p, const char* e, T& v, long long line, int col, const char* what,
           Error& err) {
  bool ok;
  if constexpr (std::is_same_v<T, int>) ok = parse_int(p, e, v);
  else ok = parse_double(p, e, v);
  if (!ok) {
    err.set(line, token_error(line, col, what));
    return false;
  }
  if constexpr (std::is_floating_point_v<T>) {
    if (!std::isfinite(v)) {  // io.hpp:71-74
      err.set(line, "line " + std::to_string(line) + ", token " + std::to_string(col) +
                        ": non-finite number");
      return false;
    }
  }
  return true;
}

inline int thread_count(int threads, size_t work) {
  int t = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  const size_t per = 1 << 16;  // below ~64 KiB per thread, threads do not pay
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)t, (work + per - 1) / per));
}

template <class F>
void parallel(int n, F&& f) {
  if (n <= 1) {
    f(0);
    return;
  }
  std::vector<std::thread> ts;
  ts.reserve(n - 1);
  for (int i = 1; i < n; ++i) ts.emplace_back(f, i);
  f(0);
  for (auto& t : ts) t.join();
}

}  // namespace detail

// Parse a whole SWEMESH 1 text (io.hpp:80-132).  threads <= 0: all cores.
inline NativeFile parse(const char* data, size_t size, int threads = 0) {
  using detail::Error;
  const char* const end = data + size;
  auto line_end = [&](const char* p) {
    const void* nl = std::memchr(p, '\n', (size_t)(end - p));
    return nl ? static_cast<const char*>(nl) : end;
  };
  // line 1: magic + version
  if (size == 0) throw io_error("line 1: empty stream, expected 'SWEMESH 1'");
  const char* l1e = line_end(data);
  {
    const char* p = data;
    while (p < l1e && detail::is_space(*p)) ++p;
    const char* m0 = p;
    while (p < l1e && !detail::is_space(*p)) ++p;
    const std::string magic(m0, p);
    int version = 0;
    if (magic != "SWEMESH" || !detail::parse_int(p, l1e, version) || version != 1)
      throw io_error("line 1: bad magic, expected 'SWEMESH 1', got '" + std::string(data, l1e) +
                     "'");
  }
  // line 2: counts
  const char* l2 = l1e < end ? l1e + 1 : end;
  if (l2 >= end) throw io_error("line 2: expected '<nnodes> <ncells>'");
  const char* l2e = line_end(l2);
  int nn = 0, nc = 0;
  {
    Error err;
    const char* p = l2;
    if (!detail::token(p, l2e, nn, 2, 1, "node count", err) ||
        !detail::token(p, l2e, nc, 2, 2, "cell count", err))
      throw io_error(err.msg);
  }
  if (nn < 0 || nc < 0) throw io_error("line 2: negative counts");

  NativeFile f;
  f.raw.nodes.resize((size_t)nn);
  f.raw.triangles.resize((size_t)nc);
  f.bed.resize((size_t)nc);
  f.manning.resize((size_t)nc);
  const char* body = l2e < end ? l2e + 1 : end;
  const size_t bsize = (size_t)(end - body);
  const long long want = (long long)nn + nc;  // body lines the format declares

  // chunks of the body, each starting at a line start
  const int T = detail::thread_count(threads, bsize);
  std::vector<const char*> cs(T + 1);
  cs[0] = body;
  cs[T] = end;
  for (int i = 1; i < T; ++i) {
    const char* p = body + bsize * (size_t)i / (size_t)T;
    p = std::max(p, cs[i - 1]);
    if (p > body && p < end && p[-1] != '\n') p = line_end(p) < end ? line_end(p) + 1 : end;
    cs[i] = p;
  }
  // lines per chunk (a final line without '\n' still counts, like getline)
  std::vector<long long> nl(T + 1, 0);
  detail::parallel(T, [&](int i) {
    long long n = 0;
    for (const char* p = cs[i]; p < cs[i + 1];) {
      const char* q = static_cast<const char*>(std::memchr(p, '\n', (size_t)(cs[i + 1] - p)));
      ++n;
      if (!q) break;
      p = q + 1;
    }
    nl[i + 1] = n;
  });
  for (int i = 0; i < T; ++i) nl[i + 1] += nl[i];
  const long long have = nl[T];

  std::vector<Error> errs(T);
  detail::parallel(T, [&](int i) {
    Error& err = errs[i];
    long long j = nl[i];  // body line index of the chunk's first line
    for (const char* p = cs[i]; p < cs[i + 1] && j < want; ++j) {
      const char* e = static_cast<const char*>(std::memchr(p, '\n', (size_t)(cs[i + 1] - p)));
      if (!e) e = cs[i + 1];
      const long long line = j + 3;
      const char* q = p;
      if (j < nn) {  // io.hpp:100-109
        double x, y;
        if (detail::token(q, e, x, line, 1, "x coordinate", err) &&
            detail::token(q, e, y, line, 2, "y coordinate", err))
          f.raw.nodes[(size_t)j] = Vec2{x, y};
      } else {  // io.hpp:113-129
        const size_t c = (size_t)(j - nn);
        std::array<int, 3> tri{};
        bool ok = true;
        for (int k = 0; k < 3 && ok; ++k) {
          ok = detail::token(q, e, tri[k], line, k + 1, "node index", err);
          if (ok && (tri[k] < 0 || tri[k] >= nn)) {
            err.set(line, "line " + std::to_string(line) + ", token " + std::to_string(k + 1) +
                              ": node index " + std::to_string(tri[k]) + " out of range [0," +
                              std::to_string(nn) + ")");
            ok = false;
          }
        }
        double z = 0.0, n = 0.0;
        if (ok && detail::token(q, e, z, line, 4, "bathymetry", err) &&
            detail::token(q, e, n, line, 5, "manning coefficient", err)) {
          f.raw.triangles[c] = tri;
          f.bed[c] = z;
          f.manning[c] = n;
        }
      }
      if (err.line >= 0) break;  // later lines of this chunk cannot win
      p = e < cs[i + 1] ? e + 1 : cs[i + 1];
    }
  });
  Error first;
  for (const Error& e : errs)
    if (e.line >= 0) first.set(e.line, e.msg);
  if (have < want) {  // io.hpp:101-103, :114-116
    const long long line = have + 3;
    if (have < nn)
      first.set(line, "line " + std::to_string(line) + ": file ends after " +
                          std::to_string(have) + " of " + std::to_string(nn) + " node lines");
    else
      first.set(line, "line " + std::to_string(line) + ": file ends after " +
                          std::to_string(have - nn) + " of " + std::to_string(nc) +
                          " cell lines");
  }
  if (first.line >= 0) throw io_error(first.msg);
  return f;
}

inline NativeFile read_file(const std::string& path, int threads = 0) {  // io.hpp:148-156
  std::FILE* fp = std::fopen(path.c_str(), "rb");
  if (!fp) throw io_error("cannot open mesh file '" + path + "'");
  std::string buf;
  std::fseek(fp, 0, SEEK_END);
  const long sz = std::ftell(fp);
  std::fseek(fp, 0, SEEK_SET);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = buf.empty() ? 0 : std::fread(buf.data(), 1, buf.size(), fp);
  std::fclose(fp);
  if (got != buf.size()) throw io_error("cannot read mesh file '" + path + "'");
  try {
    return parse(buf.data(), buf.size(), threads);
  } catch (const io_error& e) {
    throw io_error(path + ": " + e.what());
  }
}

// io.hpp format_double: %.17g (std::to_chars with precision is printf-exact)
inline char* put_double(char* p, double v) {
  return std::to_chars(p, p + 32, v, std::chars_format::general, 17).ptr;
}

// The SWEMESH 1 text of a mesh (io.hpp:134-146), formatted in parallel:
// parts[0] header, then per thread its node lines, then per thread its cell
// lines (the file is their concatenation in this order).
inline std::vector<std::string> format_parts(const RawMesh& raw, const std::vector<double>& bed,
                                             const std::vector<double>& manning, int threads = 0) {
  const size_t nn = raw.nodes.size(), nc = raw.triangles.size();
  if (bed.size() != nc || manning.size() != nc)
    throw io_error("write_mesh_native: bed / manning size != cell count");
  const int T = detail::thread_count(threads, 50 * (nn + nc));
  std::vector<std::string> parts(1 + 2 * (size_t)T);
  parts[0] = "SWEMESH 1\n" + std::to_string(nn) + ' ' + std::to_string(nc) + '\n';
  detail::parallel(T, [&](int i) {
    const size_t n0 = nn * i / T, n1 = nn * (i + 1) / T;
    const size_t c0 = nc * i / T, c1 = nc * (i + 1) / T;
    std::string& s = parts[1 + i];
    s.resize(52 * (n1 - n0) + 16);
    char* p = s.data();
    for (size_t k = n0; k < n1; ++k) {
      p = put_double(p, raw.nodes[k].x);
      *p++ = ' ';
      p = put_double(p, raw.nodes[k].y);
      *p++ = '\n';
    }
    s.resize((size_t)(p - s.data()));
    std::string& t = parts[1 + T + i];
    t.resize(110 * (c1 - c0) + 16);
    p = t.data();
    for (size_t c = c0; c < c1; ++c) {
      for (int k = 0; k < 3; ++k) {
        p = std::to_chars(p, p + 12, raw.triangles[c][k]).ptr;
        *p++ = ' ';
      }
      p = put_double(p, bed[c]);
      *p++ = ' ';
      p = put_double(p, manning[c]);
      *p++ = '\n';
    }
    t.resize((size_t)(p - t.data()));
  });
  return parts;
}

inline std::string format(const RawMesh& raw, const std::vector<double>& bed,
                          const std::vector<double>& manning, int threads = 0) {
  std::string out;
  for (const std::string& s : format_parts(raw, bed, manning, threads)) out += s;
  return out;
}

inline void write_file(const std::string& path, const RawMesh& raw, const std::vector<double>& bed,
                       const std::vector<double>& manning, int threads = 0) {  // io.hpp:158-165
  const std::vector<std::string> parts = format_parts(raw, bed, manning, threads);
  std::FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) throw io_error("cannot open '" + path + "' for writing");
  bool ok = true;
  for (const std::string& s : parts) ok = ok && std::fwrite(s.data(), 1, s.size(), fp) == s.size();
  const int rc = std::fclose(fp);
  if (!ok || rc != 0) throw io_error("write failed for '" + path + "'");
}

}  // namespace swe::swemesh
