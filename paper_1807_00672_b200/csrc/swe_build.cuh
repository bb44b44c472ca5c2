// swe_build.cuh -- build_mesh (reference mesh.hpp:121-240) on the device
// (SURVEY.md §8(f) row 3).  Same numbering and geometry bit for bit as the
// host build_mesh (include/swe/mesh.hpp): every operation is an IEEE-exact
// + - * / sqrt in the reference's expression order (--fmad=false), and the
// edge numbering is the (lower node, upper node, cell) order of the
// reference's incidence sort, obtained here from a stable 64-bit radix sort
// of the 3C directed incidences that start in (cell, local edge) order.
// Errors: each kernel records the FIRST offending item (atomicMin of its
// index in the serial loop's order); the host formats the reference's text.
#pragma once

#include <climits>

namespace swe_b200 {

struct BuildErr {
  int cell;     // first triangle failing range / degeneracy / area (loop 1)
  int run;      // sorted position of the first bad edge run (non-manifold)
  int closure;  // first cell failing the closed-polygon identity
  int pad;
};

__device__ __forceinline__ double bnorm(double x, double y) { return sqrt(x * x + y * y); }

// mesh.hpp:189-212: CCW order, area, centroid, inradius
__global__ void kb_cells(int nn, int nc, const double* __restrict__ xy, const int* __restrict__ tri,
                         int* cn, double* area, double* cx, double* cy, double* inr,
                         BuildErr* err) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  int t0 = tri[3 * (size_t)c], t1 = tri[3 * (size_t)c + 1], t2 = tri[3 * (size_t)c + 2];
  if (t0 < 0 || t0 >= nn || t1 < 0 || t1 >= nn || t2 < 0 || t2 >= nn || t0 == t1 || t1 == t2 ||
      t0 == t2) {
    atomicMin(&err->cell, c);
    return;
  }
  const double ax = xy[2 * (size_t)t0], ay = xy[2 * (size_t)t0 + 1];
  // 0.5 * cross(n1 - a, n2 - a)
  const double ux = xy[2 * (size_t)t1] - ax, uy = xy[2 * (size_t)t1 + 1] - ay;
  const double vx = xy[2 * (size_t)t2] - ax, vy = xy[2 * (size_t)t2 + 1] - ay;
  double ar = 0.5 * (ux * vy - uy * vx);
  if (ar < 0.0) {
    const int s = t1;
    t1 = t2;
    t2 = s;
    ar = -ar;
  }
  if (!(ar > 0.0)) {
    atomicMin(&err->cell, c);
    return;
  }
  const double p0x = xy[2 * (size_t)t0], p0y = xy[2 * (size_t)t0 + 1];
  const double p1x = xy[2 * (size_t)t1], p1y = xy[2 * (size_t)t1 + 1];
  const double p2x = xy[2 * (size_t)t2], p2y = xy[2 * (size_t)t2 + 1];
  const double per = bnorm(p1x - p0x, p1y - p0y) + bnorm(p2x - p1x, p2y - p1y) +
                     bnorm(p0x - p2x, p0y - p2y);
  cn[3 * (size_t)c] = t0;
  cn[3 * (size_t)c + 1] = t1;
  cn[3 * (size_t)c + 2] = t2;
  area[c] = ar;
  cx[c] = (p0x + p1x + p2x) / 3.0;
  cy[c] = (p0y + p1y + p2y) / 3.0;
  inr[c] = 2.0 * ar / per;
}

// directed incidence (c, k) -> key (lower node, upper node), value 3c + k
__global__ void kb_keys(int nc, const int* __restrict__ cn, unsigned long long* key, int* val) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= 3LL * nc) return;
  const int c = (int)(i / 3), k = (int)(i % 3);
  const int a = cn[3 * (size_t)c + k], b = cn[3 * (size_t)c + (k + 1) % 3];
  key[i] = ((unsigned long long)min(a, b) << 32) | (unsigned)max(a, b);
  val[i] = (int)i;
}

__global__ void kb_heads(long long n, const unsigned long long* __restrict__ key, int* head) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// mesh.hpp:247-276: one thread per run head of the sorted incidences;
// eid[i] = inclusive scan of heads (edge = eid - 1)
__global__ void kb_edges(long long n, const unsigned long long* __restrict__ key,
                         const int* __restrict__ val, const int* __restrict__ head,
                         const int* __restrict__ eid, const int* __restrict__ cn,
                         const double* __restrict__ xy, int* en, int* el, int* er, double* nx,
                         double* ny, double* len, int* ce, int* cs, BuildErr* err) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n || !head[i]) return;
  const bool two = i + 1 < n && key[i + 1] == key[i];
  if (two && i + 2 < n && key[i + 2] == key[i]) {  // shared by > 2 triangles
    atomicMin(&err->run, (int)i);
    return;
  }
  const int e = eid[i] - 1;
  const int v = val[i], c = v / 3, k = v % 3;
  const int a = cn[3 * (size_t)c + k], b = cn[3 * (size_t)c + (k + 1) % 3];
  const double dx = xy[2 * (size_t)b] - xy[2 * (size_t)a];
  const double dy = xy[2 * (size_t)b + 1] - xy[2 * (size_t)a + 1];
  const double l = bnorm(dx, dy);
  en[2 * (size_t)e] = a;
  en[2 * (size_t)e + 1] = b;
  nx[e] = dy / l;
  ny[e] = -dx / l;
  len[e] = l;
  el[e] = c;
  er[e] = -1;
  ce[3 * (size_t)c + k] = e;
  cs[3 * (size_t)c + k] = 1;
  if (two) {
    const int w = val[i + 1], rc = w / 3, rk = w % 3;
    if (cn[3 * (size_t)rc + rk] != b || cn[3 * (size_t)rc + (rk + 1) % 3] != a) {
      atomicMin(&err->run, (int)i);
      return;
    }
    er[e] = rc;
    ce[3 * (size_t)rc + rk] = e;
    cs[3 * (size_t)rc + rk] = -1;
  }
}

// mesh.hpp:280-291: closed-polygon identity
__global__ void kb_closure(int nc, const int* __restrict__ ce, const int* __restrict__ cs,
                           const double* __restrict__ nx, const double* __restrict__ ny,
                           const double* __restrict__ len, BuildErr* err) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double sx = 0.0, sy = 0.0, per = 0.0;
  for (int k = 0; k < 3; ++k) {
    const int e = ce[3 * (size_t)c + k];
    const double s = cs[3 * (size_t)c + k] * len[e];
    sx = sx + s * nx[e];
    sy = sy + s * ny[e];
    per += len[e];
  }
  if (bnorm(sx, sy) > 1e-10 * per) atomicMin(&err->closure, c);
}

}  // namespace swe_b200
