// swe_step.cuh -- the explicit step kernels.
//
//   k_tile   fused one-pass step (default): per tile of T Morton-consecutive
//            cells, stage the cells' state in shared memory, evaluate the
//            fluxes of the tile's owned edges and of its halo edges (edges
//            owned by a neighbouring tile; evaluated by both tiles from the
//            same inputs, so bit-identical), keep the edge records in shared
//            memory, then update the tile's cells.
//   k_face + k_cell   two-phase path (edge records through HBM), also used by
//            compute_fluxes.
// Both reproduce engine.hpp:138-170 + :248-290 bit for bit; the cell update
// also produces the next step's CFL bound and the post-step mass.
#pragma once

#include "swe_ctl.cuh"

#ifndef SWE_FACE_MINB
#define SWE_FACE_MINB 6
#endif
#ifndef SWE_CELL_MINB
#define SWE_CELL_MINB 4
#endif
#ifndef SWE_TILE_MINB
#define SWE_TILE_MINB 3
#endif

namespace swe_b200 {

// per-thread accumulators of the cell update
struct CellAcc {
  double lo, hi, mass, clip;
  long long ev;
};

// engine.hpp:254-289 for one cell given its three applied edge fluxes in the
// reference's local order: (fm, fx, fy) per unit length, edge length l and
// outward normal (ox, oy) = sign * n.  Writes the new state and accumulates
// clip ledger, mass and the next step's CFL bound.
__device__ __forceinline__ void cell_update(const Dev& d, int c, double h, double qx, double qy,
                                            const double* fm, const double* fx, const double* fy,
                                            const double* l, const double* ox, const double* oy,
                                            double dt, double* NH, double* NQX, double* NQY,
                                            CellAcc& a) {
  const Phys& P = d.P;
  const double own = ((0.5 * P.g) * h) * h;  // engine.hpp:254
  double am = 0.0, ax = 0.0, ay = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {  // engine.hpp:256-264
    am += fm[k] * l[k];
    ax += (fx[k] - own * ox[k]) * l[k];
    ay += (fy[k] - own * oy[k]) * l[k];
  }
  const double area = __ldg(d.area + c);
  const double scale = dt / area;  // engine.hpp:265-268
  Cons u{h - scale * am, qx - scale * ax, qy - scale * ay};
  u = friction(u, __ldg(d.man + c), dt, P);  // engine.hpp:269
  if (u.h < -1e-14 * P.h_ref || !isfinite(u.h) || !isfinite(u.qx) || !isfinite(u.qy)) {
    atomicMin(&d.ctl->bad_cell, __ldg(d.c_orig + c));  // engine.hpp:273-279
    NH[c] = u.h;
    NQX[c] = u.qx;
    NQY[c] = u.qy;
    return;
  }
  if (u.h < 0.0) {  // clamp_dry, kernels.hpp:205-216
    a.clip += (-u.h) * area;
    a.ev += 1;
    u = Cons{0.0, 0.0, 0.0};
  } else if (u.h < P.h_dry) {
    u = Cons{u.h, 0.0, 0.0};
  }
  NH[c] = u.h;
  NQX[c] = u.qx;
  NQY[c] = u.qy;
  a.mass += u.h * area;
  if (!(u.h < P.h_dry)) {  // next step's CFL bound, engine.hpp:192-200
    const double s = signal_speed(u, P);
    if (!isfinite(s)) {
      atomicMin(&d.ctl->bad_speed, __ldg(d.c_orig + c));
    } else {
      a.lo = sel_min(a.lo, __ldg(d.inr + c) / s);
      a.hi = sel_max(a.hi, s);
    }
  }
}

// ---------------------------------------------------------------------------
// two-phase path: k_face (engine.hpp:138-170) then k_cell (:248-290)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock, SWE_FACE_MINB) k_face(Dev d) {
  const Ctl* ctl = d.ctl;
  if (!ctl->active) return;
  const int cur = ctl->cur;
  const double* __restrict__ H = d.h[cur];
  const double* __restrict__ QX = d.qx[cur];
  const double* __restrict__ QY = d.qy[cur];
  const int stride = gridDim.x * blockDim.x;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d.E; e += stride) {
    const int cl = __ldg(d.el + e), cr = __ldg(d.er + e);
    const double nx = __ldg(d.nx + e), ny = __ldg(d.ny + e);
    const Cons uL{__ldg(H + cl), __ldg(QX + cl), __ldg(QY + cl)};
    if (cr >= 0) {
      const Cons uR{__ldg(H + cr), __ldg(QX + cr), __ldg(QY + cr)};
      if (uL.h < 0.0 || uR.h < 0.0) {  // engine.hpp:147-153
        atomicMin(&d.ctl->bad_edge, __ldg(d.e_orig + e));
        d.M[e] = d.LX[e] = d.LY[e] = d.RX[e] = d.RY[e] = 0.0;
        continue;
      }
      double f0, lx, ly, rx, ry;
      interior_edge(uL, __ldg(d.z + cl), uR, __ldg(d.z + cr), nx, ny, d.P, f0, lx, ly, rx, ry);
      d.M[e] = f0;
      d.LX[e] = lx;
      d.LY[e] = ly;
      d.RX[e] = rx;
      d.RY[e] = ry;
    } else {
      if (uL.h < 0.0) {
        atomicMin(&d.ctl->bad_edge, __ldg(d.e_orig + e));
        d.M[e] = d.LX[e] = d.LY[e] = 0.0;
        continue;
      }
      const Flux f = wall(uL, nx, ny, d.P);  // engine.hpp:155-159
      d.M[e] = f.m;
      d.LX[e] = f.fx;
      d.LY[e] = f.fy;
    }
  }
}

__global__ void __launch_bounds__(kBlock, SWE_CELL_MINB) k_cell(Dev d) {
  Ctl* ctl = d.ctl;
  if (!ctl->active) return;
  const int cur = ctl->cur;
  const double dt = step_dt(ctl, d.sp->t_end, nullptr);
  const double* __restrict__ H = d.h[cur];
  const double* __restrict__ QX = d.qx[cur];
  const double* __restrict__ QY = d.qy[cur];
  double* NH = d.h[cur ^ 1];
  double* NQX = d.qx[cur ^ 1];
  double* NQY = d.qy[cur ^ 1];
  CellAcc a{INFINITY, 0.0, 0.0, 0.0, 0};
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d.C; c += stride) {
    const int inc[3] = {__ldg(d.inc0 + c), __ldg(d.inc1 + c), __ldg(d.inc2 + c)};
    double fm[3], fx[3], fy[3], l[3], ox[3], oy[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int e = inc[k] >> 1;
      const bool neg = inc[k] & 1;
      const double m = d.M[e];
      fm[k] = neg ? -m : m;
      fx[k] = neg ? d.RX[e] : d.LX[e];
      fy[k] = neg ? d.RY[e] : d.LY[e];
      l[k] = __ldg(d.len + e);
      const double enx = __ldg(d.nx + e), eny = __ldg(d.ny + e);
      ox[k] = neg ? -enx : enx;  // double(sign) * n, engine.hpp:259-260
      oy[k] = neg ? -eny : eny;
    }
    cell_update(d, c, H[c], QX[c], QY[c], fm, fx, fy, l, ox, oy, dt, NH, NQX, NQY, a);
  }
  block_reduce_part(a.lo, a.hi, a.mass, a.clip, a.ev, d.part + blockIdx.x);
}

// ---------------------------------------------------------------------------
// fused tile kernel
// shared memory: staged tile state [4*T] (h, qx, qy, z) + per slot
// [8*S] (f0, left mom x/y, right mom x/y, nx, ny, len)
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT, SWE_TILE_MINB * 256 / NT) k_tile(Dev d) {
  extern __shared__ double smem[];
  Ctl* ctl = d.ctl;
  if (!ctl->active) return;
  const int cur = ctl->cur;
  const double dt = step_dt(ctl, d.sp->t_end, nullptr);
  const double* __restrict__ H = d.h[cur];
  const double* __restrict__ QX = d.qx[cur];
  const double* __restrict__ QY = d.qy[cur];
  double* NH = d.h[cur ^ 1];
  double* NQX = d.qx[cur ^ 1];
  double* NQY = d.qy[cur ^ 1];
  const int T = d.T, S = d.max_slots;
  double* sh = smem;
  double* sq = sh + T;
  double* sr = sq + T;
  double* sz = sr + T;
  double* rM = sz + T;
  double* rLX = rM + S;
  double* rLY = rLX + S;
  double* rRX = rLY + S;
  double* rRY = rRX + S;
  double* rNX = rRY + S;
  double* rNY = rNX + S;
  double* rL = rNY + S;
  const Phys P = d.P;
  CellAcc a{INFINITY, 0.0, 0.0, 0.0, 0};

  for (int t = blockIdx.x; t < d.ntiles; t += gridDim.x) {
    const int c0 = t * T;
    const int nc = min(T, d.C - c0);
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {  // stage the tile
      sh[i] = H[c0 + i];
      sq[i] = QX[c0 + i];
      sr[i] = QY[c0 + i];
      sz[i] = __ldg(d.z + c0 + i);
    }
    const int e0 = __ldg(d.eoff + t), no = __ldg(d.eoff + t + 1) - e0;
    const int h0 = __ldg(d.hoff + t), ns = no + __ldg(d.hoff + t + 1) - h0;
    __syncthreads();

    // phase 1: fluxes of owned + halo edges into the slot records
    for (int j = threadIdx.x; j < ns; j += blockDim.x) {
      const int e = j < no ? e0 + j : __ldg(d.halo + h0 + (j - no));
      const int cl = __ldg(d.el + e), cr = __ldg(d.er + e);
      const double nx = __ldg(d.nx + e), ny = __ldg(d.ny + e);
      rNX[j] = nx;
      rNY[j] = ny;
      rL[j] = __ldg(d.len + e);
      const int il = cl - c0;
      Cons uL;
      double zl;
      if ((unsigned)il < (unsigned)nc) {
        uL = Cons{sh[il], sq[il], sr[il]};
        zl = sz[il];
      } else {
        uL = Cons{__ldg(H + cl), __ldg(QX + cl), __ldg(QY + cl)};
        zl = __ldg(d.z + cl);
      }
      if (cr >= 0) {
        const int ir = cr - c0;
        Cons uR;
        double zr;
        if ((unsigned)ir < (unsigned)nc) {
          uR = Cons{sh[ir], sq[ir], sr[ir]};
          zr = sz[ir];
        } else {
          uR = Cons{__ldg(H + cr), __ldg(QX + cr), __ldg(QY + cr)};
          zr = __ldg(d.z + cr);
        }
        if (uL.h < 0.0 || uR.h < 0.0) {  // engine.hpp:147-153
          atomicMin(&ctl->bad_edge, __ldg(d.e_orig + e));
          rM[j] = rLX[j] = rLY[j] = rRX[j] = rRY[j] = 0.0;
          continue;
        }
        double f0, lx, ly, rx, ry;
        interior_edge(uL, zl, uR, zr, nx, ny, P, f0, lx, ly, rx, ry);
        rM[j] = f0;
        rLX[j] = lx;
        rLY[j] = ly;
        rRX[j] = rx;
        rRY[j] = ry;
      } else {
        if (uL.h < 0.0) {
          atomicMin(&ctl->bad_edge, __ldg(d.e_orig + e));
          rM[j] = rLX[j] = rLY[j] = 0.0;
          continue;
        }
        const Flux f = wall(uL, nx, ny, P);  // engine.hpp:155-159
        rM[j] = f.m;
        rLX[j] = f.fx;
        rLY[j] = f.fy;
      }
    }
    __syncthreads();

    // phase 2: cell update from the slot records
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      const int c = c0 + i;
      const ushort4 s = d.slots[c];
      const int sl[3] = {s.x, s.y, s.z};
      double fm[3], fx[3], fy[3], l[3], ox[3], oy[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int j = sl[k] >> 1;
        const bool neg = sl[k] & 1;
        const double m = rM[j];
        fm[k] = neg ? -m : m;
        fx[k] = neg ? rRX[j] : rLX[j];
        fy[k] = neg ? rRY[j] : rLY[j];
        l[k] = rL[j];
        ox[k] = neg ? -rNX[j] : rNX[j];
        oy[k] = neg ? -rNY[j] : rNY[j];
      }
      cell_update(d, c, sh[i], sq[i], sr[i], fm, fx, fy, l, ox, oy, dt, NH, NQX, NQY, a);
    }
    __syncthreads();
  }
  block_reduce_part(a.lo, a.hi, a.mass, a.clip, a.ev, d.part + blockIdx.x);
}

}  // namespace swe_b200
