// swe_dev.cu -- B200 (sm_100a) explicit HLLC shallow-water step behind the
// C-ABI of include/swe_dev.h.
//
// Hot path (reference: /root/reference/proj/include/swe/engine.hpp:226-319):
//   face kernel   one thread per edge: hydrostatic reconstruction + HLLC (or
//                 the mirror wall flux) -> 5-double edge record
//                 {f0, left momentum, right momentum} (engine.hpp:138-170)
//   cell kernel   atomic-free gather of the cell's 3 records in the
//                 reference's local edge order, explicit Euler update,
//                 Manning friction, blow-up check, dry clamp, clip ledger
//                 (engine.hpp:248-290) + the NEXT step's CFL bound and the
//                 post-step mass fused in (engine.hpp:179-216, :128-132)
//   finalize      one block: fixed-order reduction of the cell-block
//                 partials, error promotion, clock commit, Δt for the next
//                 step with t_end truncation (engine.hpp:235-237, :300-307),
//                 per-step record, loop condition for the CUDA graph.
// The run() loop (engine.hpp:355-380) is one CUDA graph launch: a gate kernel
// and a conditional WHILE node whose body is {face, cell, finalize}.
//
// Layout in HBM (all SoA, FP64 unless noted), in a Morton renumbering of the
// cells and an edge order sorted by (wall?, lower new cell) built on the device
// at create time; orientation (left = reference left cell) and each cell's
// local edge order are preserved, so results are bit-identical to the
// reference numbering.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "swe_dev.h"
#include "swe_phys.cuh"

using namespace swe_b200;

namespace {

thread_local std::string g_last_error;
long long g_launches = 0;

// resident blocks per SM the kernels are register-budgeted for (ncu r01:
// 48/74 registers left them latency-bound at 62%/37% occupancy; 6/4 blocks
// measured 0.333/0.375 ms vs 0.416/0.474 ms at 10M cells)
#ifndef SWE_FACE_MINB
#define SWE_FACE_MINB 6
#endif
#ifndef SWE_CELL_MINB
#define SWE_CELL_MINB 4
#endif

constexpr int kNone = INT_MAX;
constexpr int kBlock = 256;  // threads per block of the face/cell kernels

struct StepParams {  // written by the host before a launch sequence
  double t_end;
  long long max_steps;
  double next_snap;
  long long rec_cap;
  int ring;  // records wrap instead of stopping the loop
  int mode;  // 0 run loop, 1 single advance_step (no t/max_steps gate), 2 flux only
};

struct Ctl {
  // committed clock and ledger
  double t;
  long long step;
  double clipped;
  long long events;
  // CFL cache of the current state
  double dts;        // cfl * min(r / speed), or dt_max when all dry
  double max_speed;  // of the current state
  double mass;       // of the current state (fixed-order tree sum)
  int cfl_valid;
  int cfl_bad;  // lowest reference cell with a non-finite speed, or kNone
  // loop state
  int cur;     // which buffer holds the current state
  int active;  // kernels run only when set
  long long n_rec;
  // outcome
  int status;
  int err_index;
  long long err_step;
  double err_dt;
  double err_h;
  // per-step error scratch (lowest reference index, kNone = none)
  int bad_edge;
  int bad_cell;
  int bad_speed;
  int pad;
};

struct Part {  // one cell-kernel block's partial results
  double lo, hi, mass, clip;
  long long events;
  long long pad;
};

struct Dev {
  int C, E, E_int;  // cells, edges, interior edges (walls are [E_int, E))
  // cells (device order)
  const double *area, *inr, *z, *man;
  const int *inc0, *inc1, *inc2;  // (new edge << 1) | (sign < 0)
  const int *c_orig;               // device cell -> reference cell
  const int *c_new;                // reference cell -> device cell
  // edges (device order)
  const int *el, *er;
  const double *nx, *ny, *len;
  const int* e_orig;
  // state, double-buffered
  double *h[2], *qx[2], *qy[2];
  // edge records
  double *M, *LX, *LY, *RX, *RY;
  // control
  Ctl* ctl;
  const StepParams* sp;
  Part* part;
  int n_part;
  swe_step_record* rec;
  Phys P;
};

__device__ __forceinline__ double step_dt(const Ctl* c, double t_end, bool* last_out) {
  // engine.hpp:236-237
  const bool last = c->t + c->dts >= t_end;
  if (last_out) *last_out = last;
  return last ? t_end - c->t : c->dts;
}

// ---------------------------------------------------------------------------
// face kernel: engine.hpp:138-170 over the device edge order
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
    const int cl = __ldg(d.el + e);
    const double nx = __ldg(d.nx + e), ny = __ldg(d.ny + e);
    const Cons uL{__ldg(H + cl), __ldg(QX + cl), __ldg(QY + cl)};
    if (e < d.E_int) {
      const int cr = __ldg(d.er + e);
      const Cons uR{__ldg(H + cr), __ldg(QX + cr), __ldg(QY + cr)};
      if (uL.h < 0.0 || uR.h < 0.0) {  // engine.hpp:147-153
        atomicMin(&d.ctl->bad_edge, __ldg(d.e_orig + e));
        d.M[e] = 0.0;
        d.LX[e] = 0.0;
        d.LY[e] = 0.0;
        d.RX[e] = 0.0;
        d.RY[e] = 0.0;
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
        d.M[e] = 0.0;
        d.LX[e] = 0.0;
        d.LY[e] = 0.0;
        continue;
      }
      const Flux f = wall(uL, nx, ny, d.P);  // engine.hpp:155-159
      d.M[e] = f.m;
      d.LX[e] = f.fx;
      d.LY[e] = f.fy;
    }
  }
}

// ---------------------------------------------------------------------------
// block reduction of the per-thread partials in a fixed tree order
// ---------------------------------------------------------------------------
__device__ __forceinline__ void block_reduce_part(double lo, double hi, double mass, double clip,
                                                  long long ev, Part* out) {
  __shared__ double s_lo[kBlock / 32], s_hi[kBlock / 32], s_m[kBlock / 32], s_c[kBlock / 32];
  __shared__ long long s_e[kBlock / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = sel_min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = sel_max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    mass += __shfl_xor_sync(0xffffffffu, mass, o);
    clip += __shfl_xor_sync(0xffffffffu, clip, o);
    ev += __shfl_xor_sync(0xffffffffu, ev, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_lo[w] = lo;
    s_hi[w] = hi;
    s_m[w] = mass;
    s_c[w] = clip;
    s_e[w] = ev;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Part p{s_lo[0], s_hi[0], s_m[0], s_c[0], s_e[0], 0};
    for (int i = 1; i < kBlock / 32; ++i) {
      p.lo = sel_min(p.lo, s_lo[i]);
      p.hi = sel_max(p.hi, s_hi[i]);
      p.mass += s_m[i];
      p.clip += s_c[i];
      p.events += s_e[i];
    }
    *out = p;
  }
}

// ---------------------------------------------------------------------------
// cell kernel: engine.hpp:248-290, + CFL (engine.hpp:186-204) and mass of the
// new state for the next step
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock, SWE_CELL_MINB) k_cell(Dev d) {
  Ctl* ctl = d.ctl;
  if (!ctl->active) return;
  const int cur = ctl->cur;
  if (ctl->bad_edge != kNone) return;  // compute_fluxes threw before the update
  const double dt = step_dt(ctl, d.sp->t_end, nullptr);
  const double* __restrict__ H = d.h[cur];
  const double* __restrict__ QX = d.qx[cur];
  const double* __restrict__ QY = d.qy[cur];
  double* __restrict__ NH = d.h[cur ^ 1];
  double* __restrict__ NQX = d.qx[cur ^ 1];
  double* __restrict__ NQY = d.qy[cur ^ 1];
  const Phys P = d.P;
  const double g_half = 0.5 * P.g;
  const double tol = -1e-14 * P.h_ref;

  double lo = INFINITY, hi = 0.0, mass = 0.0, clip = 0.0;
  long long ev = 0;
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d.C; c += stride) {
    const double h = H[c], qx = QX[c], qy = QY[c];
    const double own = (g_half * h) * h;  // engine.hpp:254
    const int inc[3] = {__ldg(d.inc0 + c), __ldg(d.inc1 + c), __ldg(d.inc2 + c)};
    double am = 0.0, ax = 0.0, ay = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // engine.hpp:256-264, local order k
      const int e = inc[k] >> 1;
      const bool neg = inc[k] & 1;
      const double m = d.M[e];
      const double fm = neg ? -m : m;
      const double fx = neg ? d.RX[e] : d.LX[e];
      const double fy = neg ? d.RY[e] : d.LY[e];
      const double l = __ldg(d.len + e);
      const double enx = __ldg(d.nx + e), eny = __ldg(d.ny + e);
      const double ox = neg ? -enx : enx, oy = neg ? -eny : eny;
      am += fm * l;
      ax += (fx - own * ox) * l;
      ay += (fy - own * oy) * l;
    }
    const double area = __ldg(d.area + c);
    const double scale = dt / area;  // engine.hpp:265-268
    Cons u{h - scale * am, qx - scale * ax, qy - scale * ay};
    u = friction(u, __ldg(d.man + c), dt, P);  // engine.hpp:269
    if (u.h < tol || !isfinite(u.h) || !isfinite(u.qx) || !isfinite(u.qy)) {
      atomicMin(&ctl->bad_cell, __ldg(d.c_orig + c));  // engine.hpp:273-279
      NH[c] = u.h;
      NQX[c] = u.qx;
      NQY[c] = u.qy;
      continue;
    }
    if (u.h < 0.0) {  // clamp_dry, kernels.hpp:205-216
      clip += (-u.h) * area;
      ev += 1;
      u = Cons{0.0, 0.0, 0.0};
    } else if (u.h < P.h_dry) {
      u = Cons{u.h, 0.0, 0.0};
    }
    NH[c] = u.h;
    NQX[c] = u.qx;
    NQY[c] = u.qy;
    mass += u.h * area;
    if (!(u.h < P.h_dry)) {  // next step's CFL bound, engine.hpp:192-200
      const double s = signal_speed(u, P);
      if (!isfinite(s)) {
        atomicMin(&ctl->bad_speed, __ldg(d.c_orig + c));
      } else {
        lo = sel_min(lo, __ldg(d.inr + c) / s);
        hi = sel_max(hi, s);
      }
    }
  }
  block_reduce_part(lo, hi, mass, clip, ev, d.part + blockIdx.x);
}

// standalone CFL + mass of the current state (first step after set_state),
// engine.hpp:179-216 and :128-132
__global__ void __launch_bounds__(kBlock) k_cfl(Dev d) {
  Ctl* ctl = d.ctl;
  const int cur = ctl->cur;
  const double* __restrict__ H = d.h[cur];
  const double* __restrict__ QX = d.qx[cur];
  const double* __restrict__ QY = d.qy[cur];
  double lo = INFINITY, hi = 0.0, mass = 0.0;
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d.C; c += stride) {
    const Cons u{H[c], QX[c], QY[c]};
    mass += u.h * __ldg(d.area + c);
    if (u.h < d.P.h_dry) continue;
    const double s = signal_speed(u, d.P);
    if (!isfinite(s)) {
      atomicMin(&ctl->bad_speed, __ldg(d.c_orig + c));
      continue;
    }
    lo = sel_min(lo, __ldg(d.inr + c) / s);
    hi = sel_max(hi, s);
  }
  block_reduce_part(lo, hi, mass, 0.0, 0, d.part + blockIdx.x);
}

// fixed-order reduction of the block partials by one block
__device__ Part reduce_parts(const Dev& d) {
  __shared__ Part s[kBlock];
  Part p{INFINITY, 0.0, 0.0, 0.0, 0, 0};
  for (int i = threadIdx.x; i < d.n_part; i += blockDim.x) {
    const Part q = d.part[i];
    p.lo = sel_min(p.lo, q.lo);
    p.hi = sel_max(p.hi, q.hi);
    p.mass += q.mass;
    p.clip += q.clip;
    p.events += q.events;
  }
  s[threadIdx.x] = p;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      Part a = s[threadIdx.x];
      const Part b = s[threadIdx.x + o];
      a.lo = sel_min(a.lo, b.lo);
      a.hi = sel_max(a.hi, b.hi);
      a.mass += b.mass;
      a.clip += b.clip;
      a.events += b.events;
      s[threadIdx.x] = a;
    }
    __syncthreads();
  }
  return s[0];
}

__device__ __forceinline__ void set_cfl_cache(Ctl* ctl, const Part& p, const Phys& P) {
  ctl->dts = isfinite(p.lo) ? P.cfl * p.lo : P.dt_max;  // engine.hpp:214
  ctl->max_speed = p.hi;
  ctl->mass = p.mass;
  ctl->cfl_bad = ctl->bad_speed;
  ctl->bad_speed = kNone;
  ctl->cfl_valid = 1;
}

// prepare: reduce k_cfl's partials into the CFL cache
__global__ void __launch_bounds__(kBlock) k_prepare(Dev d) {
  const Part p = reduce_parts(d);
  if (threadIdx.x == 0) set_cfl_cache(d.ctl, p, d.P);
}

// gate: opens a launch sequence (run() loop entry, engine.hpp:355-358)
__global__ void k_gate(Dev d, cudaGraphConditionalHandle cond, int use_cond) {
  Ctl* c = d.ctl;
  const StepParams* sp = d.sp;
  c->status = SWE_OK;
  c->n_rec = 0;
  c->bad_edge = kNone;
  c->bad_cell = kNone;
  c->bad_speed = kNone;
  int go = sp->mode != 0 ||
           (c->t < sp->t_end && c->step < sp->max_steps && (sp->ring || sp->rec_cap > 0));
  if (go && sp->mode != 2 && c->cfl_bad != kNone) {  // stable_dt would throw (engine.hpp:205-206)
    c->status = SWE_NONFINITE_SPEED;
    c->err_index = c->cfl_bad;
    go = 0;
  }
  c->active = go;
  if (use_cond) cudaGraphSetConditional(cond, go);
}

// finalize: engine.hpp:292-307 + the fused CFL cache for the next step
__global__ void __launch_bounds__(kBlock) k_finalize(Dev d, cudaGraphConditionalHandle cond,
                                                     int use_cond) {
  Ctl* c = d.ctl;
  if (!c->active) {
    if (threadIdx.x == 0 && use_cond) cudaGraphSetConditional(cond, 0);
    return;
  }
  const Part p = reduce_parts(d);
  if (threadIdx.x != 0) return;
  const StepParams* sp = d.sp;
  bool last;
  const double dt = step_dt(c, sp->t_end, &last);
  int go = 1;
  if (c->bad_edge != kNone) {  // engine.hpp:168-169
    c->status = SWE_NEGATIVE_DEPTH;
    c->err_index = c->bad_edge;
    go = 0;
  } else if (c->bad_cell != kNone) {  // engine.hpp:292-297; state is not committed
    c->status = SWE_BLOWUP;
    c->err_index = c->bad_cell;
    c->err_step = c->step;
    c->err_dt = dt;
    c->err_h = d.h[c->cur ^ 1][d.c_new[c->bad_cell]];
    go = 0;
  }
  if (!go) {
    c->bad_edge = kNone;
    c->bad_cell = kNone;
    c->bad_speed = kNone;
    c->active = 0;
    if (use_cond) cudaGraphSetConditional(cond, 0);
    return;
  }
  // commit (engine.hpp:300-307)
  const double max_speed_pre = c->max_speed;
  c->clipped += p.clip;
  c->events += p.events;
  c->cur ^= 1;
  c->t = last ? sp->t_end : c->t + dt;
  c->step += 1;
  const long long slot = sp->ring ? (c->n_rec % sp->rec_cap) : c->n_rec;
  if (slot < sp->rec_cap) {
    swe_step_record r;
    r.step = c->step;
    r.t = c->t;
    r.dt = dt;
    r.max_speed = max_speed_pre;
    r.mass = p.mass;
    d.rec[slot] = r;
  }
  c->n_rec += 1;
  set_cfl_cache(c, p, d.P);
  // continue? (engine.hpp:355-358, :374-375)
  go = c->t < sp->t_end && c->step < sp->max_steps && !(c->t >= sp->next_snap - 1e-12) &&
       (sp->ring || c->n_rec < sp->rec_cap);
  if (go && c->cfl_bad != kNone) {
    c->status = SWE_NONFINITE_SPEED;
    c->err_index = c->cfl_bad;
    go = 0;
  }
  c->active = go;
  if (use_cond) cudaGraphSetConditional(cond, go);
}

// ---------------------------------------------------------------------------
// device preprocessor (mesh.hpp layout -> renumbered SoA)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned spread16(unsigned v) {
  v &= 0xffffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

__global__ void k_morton(int C, const double* cx, const double* cy, double x0, double y0,
                         double sx, double sy, unsigned* key, int* idx) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double fx = (cx[c] - x0) * sx, fy = (cy[c] - y0) * sy;
  fx = fmin(fmax(fx, 0.0), 65535.0);
  fy = fmin(fmax(fy, 0.0), 65535.0);
  key[c] = spread16((unsigned)fx) | (spread16((unsigned)fy) << 1);
  idx[c] = c;
}

__global__ void k_iota(int n, int* v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void k_invert(int n, const int* p, int* inv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) inv[p[i]] = i;
}

__global__ void k_edge_keys(int E, const int* el, const int* er, const int* c_new, unsigned* key,
                            int* idx) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int l = c_new[el[e]];
  const int r = er[e];
  unsigned k;
  if (r < 0) {
    k = 0x80000000u | (unsigned)l;
  } else {
    const int rn = c_new[r];
    k = (unsigned)(l < rn ? l : rn);
  }
  key[e] = k;
  idx[e] = e;
}

template <class T>
__global__ void k_gather(int n, const int* perm, const T* src, T* dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

__global__ void k_edges_new(int E, const int* e_orig, const int* el, const int* er,
                            const int* c_new, int* nel, int* ner) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int o = e_orig[e];
  nel[e] = c_new[el[o]];
  ner[e] = er[o] < 0 ? -1 : c_new[er[o]];
}

__global__ void k_inc_new(int C, const int* c_orig, const int* cell_edge, const int* cell_sign,
                          const int* e_new, int* i0, int* i1, int* i2, int* bad) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int o = c_orig[c];
  int v[3];
  for (int k = 0; k < 3; ++k) {
    const int e = cell_edge[3 * (size_t)o + k];
    const int s = cell_sign[3 * (size_t)o + k];
    if (s != 1 && s != -1) atomicExch(bad, 1);
    v[k] = (e_new[e] << 1) | (s < 0 ? 1 : 0);
  }
  i0[c] = v[0];
  i1[c] = v[1];
  i2[c] = v[2];
}

// state permutation: reference order <-> device order
__global__ void k_state_in(int C, const int* c_orig, const double* h, const double* qx,
                           const double* qy, double* dh, double* dqx, double* dqy) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int o = c_orig[c];
  dh[c] = h[o];
  dqx[c] = qx[o];
  dqy[c] = qy[o];
}

__global__ void k_state_out(int C, const int* c_new, const double* dh, const double* dqx,
                            const double* dqy, double* h, double* qx, double* qy) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= C) return;
  const int c = c_new[o];
  h[o] = dh[c];
  qx[o] = dqx[c];
  qy[o] = dqy[c];
}

// edge records -> reference left/right Flux3 arrays (compute_fluxes layout)
__global__ void k_flux_out(Dev d, double* left, double* right) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E) return;
  const int o = d.e_orig[e];
  const bool wall_e = e >= d.E_int;
  left[3 * (size_t)o] = d.M[e];
  left[3 * (size_t)o + 1] = d.LX[e];
  left[3 * (size_t)o + 2] = d.LY[e];
  right[3 * (size_t)o] = wall_e ? 0.0 : -d.M[e];
  right[3 * (size_t)o + 1] = wall_e ? 0.0 : d.RX[e];
  right[3 * (size_t)o + 2] = wall_e ? 0.0 : d.RY[e];
}

// point physics over arrays (kernel-level parity tests)
__global__ void k_point(int kind, long long n, Phys P, const double* l, const double* r,
                        const double* z, const double* nrm, double* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Cons a{l[3 * i], l[3 * i + 1], l[3 * i + 2]};
  if (kind == 0) {
    const Cons b{r[3 * i], r[3 * i + 1], r[3 * i + 2]};
    const Flux f = hllc(a, b, nrm[2 * i], nrm[2 * i + 1], P);
    out[3 * i] = f.m;
    out[3 * i + 1] = f.fx;
    out[3 * i + 2] = f.fy;
  } else if (kind == 1) {
    const Flux f = wall(a, nrm[2 * i], nrm[2 * i + 1], P);
    out[3 * i] = f.m;
    out[3 * i + 1] = f.fx;
    out[3 * i + 2] = f.fy;
  } else if (kind == 2) {
    const Cons b{r[3 * i], r[3 * i + 1], r[3 * i + 2]};
    double f0, lx, ly, rx, ry;
    interior_edge(a, z[2 * i], b, z[2 * i + 1], nrm[2 * i], nrm[2 * i + 1], P, f0, lx, ly, rx, ry);
    out[6 * i] = f0;
    out[6 * i + 1] = lx;
    out[6 * i + 2] = ly;
    out[6 * i + 3] = -f0;
    out[6 * i + 4] = rx;
    out[6 * i + 5] = ry;
  } else if (kind == 3) {
    const Cons u = friction(a, z[2 * i], z[2 * i + 1], P);
    out[3 * i] = u.h;
    out[3 * i + 1] = u.qx;
    out[3 * i + 2] = u.qy;
  } else if (kind == 4) {
    out[i] = swe_pow43(a.h);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}

#define CK(call)                               \
  do {                                         \
    if (!cuda_ok((call), #call)) return SWE_CUDA; \
  } while (0)

int blocks_for(long long n, int b = kBlock) { return (int)((n + b - 1) / b); }

}  // namespace

struct swe_dev_ctx {
  int device = 0;
  unsigned flags = 0;
  cudaStream_t stream = nullptr;
  Dev d{};
  std::vector<void*> allocs;
  long long bytes = 0;
  Ctl* ctl = nullptr;          // device
  StepParams* sp = nullptr;    // device
  Ctl* h_ctl = nullptr;        // pinned host mirror
  StepParams* h_sp = nullptr;  // pinned host
  swe_step_record* rec = nullptr;
  long long rec_cap = 0;
  double *stage_h = nullptr, *stage_qx = nullptr, *stage_qy = nullptr;
  int grid_face = 0, grid_cell = 0;
  // graph
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond{};
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> events;
  double kms[4] = {0, 0, 0, 0};
  long long klaunch[4] = {0, 0, 0, 0};

  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, n * sizeof(T) + 16) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    bytes += (long long)(n * sizeof(T));
    return static_cast<T*>(p);
  }
};

namespace {

int launch_face(swe_dev_ctx* x) {
  k_face<<<x->grid_face, kBlock, 0, x->stream>>>(x->d);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_face") ? SWE_OK : SWE_CUDA;
}

int launch_cell(swe_dev_ctx* x) {
  k_cell<<<x->grid_cell, kBlock, 0, x->stream>>>(x->d);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_cell") ? SWE_OK : SWE_CUDA;
}

int launch_finalize(swe_dev_ctx* x, cudaGraphConditionalHandle h, int use_cond) {
  k_finalize<<<1, kBlock, 0, x->stream>>>(x->d, h, use_cond);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_finalize") ? SWE_OK : SWE_CUDA;
}

int launch_gate(swe_dev_ctx* x) {
  k_gate<<<1, 1, 0, x->stream>>>(x->d, cudaGraphConditionalHandle{}, 0);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_gate") ? SWE_OK : SWE_CUDA;
}

// CFL cache of the current state if stale (after set_state)
int ensure_cfl(swe_dev_ctx* x, bool force = false) {
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  if (x->h_ctl->cfl_valid && !force) return SWE_OK;
  k_cfl<<<x->grid_cell, kBlock, 0, x->stream>>>(x->d);
  ++g_launches;
  CK(cudaGetLastError());
  k_prepare<<<1, kBlock, 0, x->stream>>>(x->d);
  ++g_launches;
  CK(cudaGetLastError());
  return SWE_OK;
}

int write_params(swe_dev_ctx* x, double t_end, long long max_steps, double next_snap,
                 long long rec_cap, int ring, int mode = 0) {
  x->h_sp->t_end = t_end;
  x->h_sp->max_steps = max_steps;
  x->h_sp->next_snap = next_snap;
  x->h_sp->rec_cap = rec_cap;
  x->h_sp->ring = ring;
  x->h_sp->mode = mode;
  CK(cudaMemcpyAsync(x->sp, x->h_sp, sizeof(StepParams), cudaMemcpyHostToDevice, x->stream));
  return SWE_OK;
}

int read_status(swe_dev_ctx* x, swe_status* st) {
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  const Ctl& c = *x->h_ctl;
  if (st) {
    st->code = c.status;
    st->index = c.err_index;
    st->step = c.err_step;
    st->dt = c.err_dt;
    st->h = c.err_h;
  }
  return c.status;
}

int build_graph(swe_dev_ctx* x) {
  CK(cudaGraphCreate(&x->graph, 0));
  CK(cudaGraphConditionalHandleCreate(&x->cond, x->graph, 0, cudaGraphCondAssignDefault));
  // gate kernel node
  cudaKernelNodeParams kp{};
  Dev dcopy = x->d;
  cudaGraphConditionalHandle hc = x->cond;
  int use = 1;
  void* args[] = {&dcopy, &hc, &use};
  kp.func = (void*)k_gate;
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(1);
  kp.kernelParams = args;
  cudaGraphNode_t gate;
  CK(cudaGraphAddKernelNode(&gate, x->graph, nullptr, 0, &kp));
  // WHILE node
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = x->cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wnode;
  CK(cudaGraphAddNode(&wnode, x->graph, &gate, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  // body: face -> cell -> finalize, captured into the body graph
  CK(cudaStreamBeginCaptureToGraph(x->stream, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  k_face<<<x->grid_face, kBlock, 0, x->stream>>>(x->d);
  k_cell<<<x->grid_cell, kBlock, 0, x->stream>>>(x->d);
  k_finalize<<<1, kBlock, 0, x->stream>>>(x->d, x->cond, 1);
  cudaGraph_t captured = nullptr;
  CK(cudaStreamEndCapture(x->stream, &captured));
  CK(cudaGraphInstantiate(&x->exec, x->graph, 0));
  return SWE_OK;
}

int fail_invalid(const char* msg) {
  g_last_error = msg;
  return SWE_INVALID;
}

}  // namespace

extern "C" {

const char* swe_dev_strerror(int code) {
  switch (code) {
    case SWE_OK: return "ok";
    case SWE_NONFINITE_SPEED: return "non-finite velocity";
    case SWE_NEGATIVE_DEPTH: return "negative depth";
    case SWE_BLOWUP: return "numeric blowup";
    case SWE_CUDA: return "CUDA error";
    case SWE_NCCL: return "NCCL error";
    case SWE_INVALID: return "invalid argument";
  }
  return "unknown";
}

const char* swe_dev_last_error(void) { return g_last_error.c_str(); }

long long swe_dev_launch_count(void) { return g_launches; }

int swe_dev_create(const swe_mesh_view* m, const swe_params* params, int device, unsigned flags,
                   swe_dev_ctx** out) {
  if (!m || !params || !out) return fail_invalid("swe_dev_create: null argument");
  if (m->n_cells <= 0 || m->n_edges <= 0) return fail_invalid("swe_dev_create: empty mesh");
  if (!m->area || !m->inradius || !m->bed || !m->manning || !m->cell_edge || !m->cell_sign ||
      !m->edge_left || !m->edge_right || !m->nx || !m->ny || !m->len)
    return fail_invalid("swe_dev_create: missing mesh array");
  const int C = m->n_cells, E = m->n_edges;
  int n_wall = 0;
  for (int e = 0; e < E; ++e) {
    const int l = m->edge_left[e], r = m->edge_right[e];
    if (l < 0 || l >= C || r < -1 || r >= C) return fail_invalid("swe_dev_create: edge cell out of range");
    n_wall += (r < 0);
  }
  for (long long i = 0; i < 3LL * C; ++i)
    if (m->cell_edge[i] < 0 || m->cell_edge[i] >= E)
      return fail_invalid("swe_dev_create: cell edge out of range");

  auto* x = new swe_dev_ctx();
  x->device = device;
  x->flags = flags;
  auto bail = [&](int rc) {
    swe_dev_destroy(x);
    return rc;
  };
  if (!cuda_ok(cudaSetDevice(device), "cudaSetDevice")) return bail(SWE_CUDA);
  if (!cuda_ok(cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking), "stream"))
    return bail(SWE_CUDA);
  cudaStream_t s = x->stream;

  Dev& d = x->d;
  d.C = C;
  d.E = E;
  d.E_int = E - n_wall;
  d.P = Phys{params->g, params->h_dry, params->cfl, params->dt_max, params->h_ref};

  // -- permanent arrays
  double* area = x->alloc<double>(C);
  double* inr = x->alloc<double>(C);
  double* z = x->alloc<double>(C);
  double* man = x->alloc<double>(C);
  int* inc0 = x->alloc<int>(C);
  int* inc1 = x->alloc<int>(C);
  int* inc2 = x->alloc<int>(C);
  int* c_orig = x->alloc<int>(C);
  int* c_new = x->alloc<int>(C);
  int* el = x->alloc<int>(E);
  int* er = x->alloc<int>(E);
  double* nx = x->alloc<double>(E);
  double* ny = x->alloc<double>(E);
  double* len = x->alloc<double>(E);
  int* e_orig = x->alloc<int>(E);
  for (int b = 0; b < 2; ++b) {
    d.h[b] = x->alloc<double>(C);
    d.qx[b] = x->alloc<double>(C);
    d.qy[b] = x->alloc<double>(C);
  }
  d.M = x->alloc<double>(E);
  d.LX = x->alloc<double>(E);
  d.LY = x->alloc<double>(E);
  d.RX = x->alloc<double>(E);
  d.RY = x->alloc<double>(E);
  x->stage_h = x->alloc<double>(C);
  x->stage_qx = x->alloc<double>(C);
  x->stage_qy = x->alloc<double>(C);
  x->ctl = x->alloc<Ctl>(1);
  x->sp = x->alloc<StepParams>(1);
  x->rec_cap = 1 << 16;
  x->rec = x->alloc<swe_step_record>(x->rec_cap);
  if (!x->rec || !x->stage_qy || !d.RY || !e_orig) {
    g_last_error = "swe_dev_create: cudaMalloc failed";
    return bail(SWE_CUDA);
  }
  if (!cuda_ok(cudaMallocHost(&x->h_ctl, sizeof(Ctl)), "cudaMallocHost")) return bail(SWE_CUDA);
  if (!cuda_ok(cudaMallocHost(&x->h_sp, sizeof(StepParams)), "cudaMallocHost")) return bail(SWE_CUDA);

  // grid sizes: a fixed number of resident blocks (multiple of the SM count)
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int occ_face = 0, occ_cell = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_face, k_face, kBlock, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_cell, k_cell, kBlock, 0);
  x->grid_face = std::max(1, std::min(blocks_for(E), sms * std::max(1, occ_face)));
  x->grid_cell = std::max(1, std::min(blocks_for(C), sms * std::max(1, occ_cell)));
  d.n_part = x->grid_cell;
  d.part = x->alloc<Part>(d.n_part);

  // -- temporary reference-order arrays
  std::vector<void*> tmp;
  auto talloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes + 16) != cudaSuccess) return nullptr;
    tmp.push_back(p);
    return p;
  };
  auto free_tmp = [&]() {
    for (void* p : tmp) cudaFree(p);
    tmp.clear();
  };
  int* r_cell_edge = (int*)talloc(sizeof(int) * 3 * (size_t)C);
  int* r_cell_sign = (int*)talloc(sizeof(int) * 3 * (size_t)C);
  int* r_el = (int*)talloc(sizeof(int) * E);
  int* r_er = (int*)talloc(sizeof(int) * E);
  double* r_buf = (double*)talloc(sizeof(double) * (size_t)std::max(C, E));
  unsigned* key_in = (unsigned*)talloc(sizeof(unsigned) * (size_t)std::max(C, E));
  unsigned* key_out = (unsigned*)talloc(sizeof(unsigned) * (size_t)std::max(C, E));
  int* idx_in = (int*)talloc(sizeof(int) * (size_t)std::max(C, E));
  int* e_new = (int*)talloc(sizeof(int) * E);
  int* bad = (int*)talloc(sizeof(int));
  double* r_cx = (double*)talloc(sizeof(double) * C);
  double* r_cy = (double*)talloc(sizeof(double) * C);
  if (!r_cy) {
    free_tmp();
    g_last_error = "swe_dev_create: cudaMalloc (temporaries) failed";
    return bail(SWE_CUDA);
  }
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "upload");
  };
  bool ok = up(r_cell_edge, m->cell_edge, sizeof(int) * 3 * (size_t)C) &&
            up(r_cell_sign, m->cell_sign, sizeof(int) * 3 * (size_t)C) &&
            up(r_el, m->edge_left, sizeof(int) * E) && up(r_er, m->edge_right, sizeof(int) * E);
  ok = ok && cuda_ok(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");

  // 1. cell order: Morton code of the centroid (stable radix sort; ties keep
  //    reference order), or identity
  const bool morton = !(flags & SWE_FLAG_IDENTITY_ORDER) && m->cx && m->cy;
  if (ok && morton) {
    double x0 = m->cx[0], x1 = x0, y0 = m->cy[0], y1 = y0;
    for (int c = 1; c < C; ++c) {
      x0 = std::min(x0, m->cx[c]);
      x1 = std::max(x1, m->cx[c]);
      y0 = std::min(y0, m->cy[c]);
      y1 = std::max(y1, m->cy[c]);
    }
    const double span = std::max(x1 - x0, y1 - y0);
    const double sc = span > 0 ? 65535.0 / span : 0.0;
    ok = up(r_cx, m->cx, sizeof(double) * C) && up(r_cy, m->cy, sizeof(double) * C);
    k_morton<<<blocks_for(C), kBlock, 0, s>>>(C, r_cx, r_cy, x0, y0, sc, sc, key_in, idx_in);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key_in, key_out, idx_in, c_orig, C, 0, 32, s);
    void* tstore = talloc(tb);
    ok = ok && tstore &&
         cuda_ok(cub::DeviceRadixSort::SortPairs(tstore, tb, key_in, key_out, idx_in, c_orig, C, 0,
                                                 32, s),
                 "cub sort cells");
  } else if (ok) {
    k_iota<<<blocks_for(C), kBlock, 0, s>>>(C, c_orig);
  }
  if (ok) k_invert<<<blocks_for(C), kBlock, 0, s>>>(C, c_orig, c_new);

  // 2. edge order: interior edges by their lower device cell, walls last
  if (ok) {
    k_edge_keys<<<blocks_for(E), kBlock, 0, s>>>(E, r_el, r_er, c_new, key_in, idx_in);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key_in, key_out, idx_in, e_orig, E, 0, 32, s);
    void* tstore = talloc(tb);
    ok = tstore && cuda_ok(cub::DeviceRadixSort::SortPairs(tstore, tb, key_in, key_out, idx_in,
                                                           e_orig, E, 0, 32, s),
                           "cub sort edges");
  }
  if (ok) {
    k_invert<<<blocks_for(E), kBlock, 0, s>>>(E, e_orig, e_new);
    k_edges_new<<<blocks_for(E), kBlock, 0, s>>>(E, e_orig, r_el, r_er, c_new, el, er);
    k_inc_new<<<blocks_for(C), kBlock, 0, s>>>(C, c_orig, r_cell_edge, r_cell_sign, e_new, inc0,
                                               inc1, inc2, bad);
  }
  // 3. permuted geometry
  auto permute_d = [&](const double* host, int n, const int* perm, double* dst) {
    if (!ok) return;
    ok = up(r_buf, host, sizeof(double) * n);
    k_gather<double><<<blocks_for(n), kBlock, 0, s>>>(n, perm, r_buf, dst);
  };
  permute_d(m->area, C, c_orig, area);
  permute_d(m->inradius, C, c_orig, inr);
  permute_d(m->bed, C, c_orig, z);
  permute_d(m->manning, C, c_orig, man);
  permute_d(m->nx, E, e_orig, nx);
  permute_d(m->ny, E, e_orig, ny);
  permute_d(m->len, E, e_orig, len);
  int h_bad = 0;
  ok = ok && cuda_ok(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h") &&
       cuda_ok(cudaStreamSynchronize(s), "preprocess");
  free_tmp();
  if (!ok) return bail(SWE_CUDA);
  if (h_bad) {
    g_last_error = "swe_dev_create: cell_sign must be +1/-1";
    return bail(SWE_INVALID);
  }

  d.area = area;
  d.inr = inr;
  d.z = z;
  d.man = man;
  d.inc0 = inc0;
  d.inc1 = inc1;
  d.inc2 = inc2;
  d.c_orig = c_orig;
  d.c_new = c_new;
  d.el = el;
  d.er = er;
  d.nx = nx;
  d.ny = ny;
  d.len = len;
  d.e_orig = e_orig;
  d.ctl = x->ctl;
  d.sp = x->sp;
  d.rec = x->rec;

  // initial control block: zero state at t = 0
  Ctl c0{};
  c0.cfl_bad = kNone;
  c0.bad_edge = kNone;
  c0.bad_cell = kNone;
  c0.bad_speed = kNone;
  *x->h_ctl = c0;
  if (!cuda_ok(cudaMemcpyAsync(x->ctl, x->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s), "ctl"))
    return bail(SWE_CUDA);
  for (int b = 0; b < 2; ++b) {
    cudaMemsetAsync(d.h[b], 0, sizeof(double) * C, s);
    cudaMemsetAsync(d.qx[b], 0, sizeof(double) * C, s);
    cudaMemsetAsync(d.qy[b], 0, sizeof(double) * C, s);
  }
  if (!(flags & SWE_FLAG_NO_GRAPH)) {
    const int rc = build_graph(x);
    if (rc != SWE_OK) return bail(rc);
  }
  if (!cuda_ok(cudaStreamSynchronize(s), "create")) return bail(SWE_CUDA);
  *out = x;
  return SWE_OK;
}

int swe_dev_destroy(swe_dev_ctx* x) {
  if (!x) return SWE_OK;
  if (x->stream) cudaStreamSynchronize(x->stream);
  if (x->exec) cudaGraphExecDestroy(x->exec);
  if (x->graph) cudaGraphDestroy(x->graph);
  for (cudaEvent_t e : x->events) cudaEventDestroy(e);
  for (void* p : x->allocs) cudaFree(p);
  if (x->h_ctl) cudaFreeHost(x->h_ctl);
  if (x->h_sp) cudaFreeHost(x->h_sp);
  if (x->stream) cudaStreamDestroy(x->stream);
  delete x;
  return SWE_OK;
}

static int set_state_impl(swe_dev_ctx* x, const double* h, const double* qx, const double* qy,
                          double t, long long step, cudaMemcpyKind kind) {
  if (!x || !h || !qx || !qy) return fail_invalid("swe_dev_set_state: null argument");
  const int C = x->d.C;
  cudaStream_t s = x->stream;
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  Ctl c = *x->h_ctl;
  CK(cudaMemcpyAsync(x->stage_h, h, sizeof(double) * C, kind, s));
  CK(cudaMemcpyAsync(x->stage_qx, qx, sizeof(double) * C, kind, s));
  CK(cudaMemcpyAsync(x->stage_qy, qy, sizeof(double) * C, kind, s));
  k_state_in<<<blocks_for(C), kBlock, 0, s>>>(C, x->d.c_orig, x->stage_h, x->stage_qx,
                                               x->stage_qy, x->d.h[c.cur], x->d.qx[c.cur],
                                               x->d.qy[c.cur]);
  ++g_launches;
  CK(cudaGetLastError());
  c.t = t;
  c.step = step;
  c.cfl_valid = 0;
  c.cfl_bad = kNone;
  c.status = SWE_OK;
  c.active = 0;
  c.bad_edge = c.bad_cell = c.bad_speed = kNone;
  *x->h_ctl = c;
  CK(cudaMemcpyAsync(x->ctl, x->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  return SWE_OK;
}

int swe_dev_set_state(swe_dev_ctx* x, const double* h, const double* qx, const double* qy,
                      double t, long long step) {
  return set_state_impl(x, h, qx, qy, t, step, cudaMemcpyHostToDevice);
}

int swe_dev_set_state_device(swe_dev_ctx* x, const double* h, const double* qx, const double* qy,
                             double t, long long step) {
  return set_state_impl(x, h, qx, qy, t, step, cudaMemcpyDeviceToDevice);
}

static int get_state_impl(swe_dev_ctx* x, double* h, double* qx, double* qy, double* t,
                          long long* step, cudaMemcpyKind kind) {
  if (!x) return fail_invalid("swe_dev_get_state: null context");
  const int C = x->d.C;
  cudaStream_t s = x->stream;
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int cur = x->h_ctl->cur;
  if (t) *t = x->h_ctl->t;
  if (step) *step = x->h_ctl->step;
  if (!h && !qx && !qy) return SWE_OK;
  k_state_out<<<blocks_for(C), kBlock, 0, s>>>(C, x->d.c_new, x->d.h[cur], x->d.qx[cur],
                                                x->d.qy[cur], x->stage_h, x->stage_qx,
                                                x->stage_qy);
  ++g_launches;
  CK(cudaGetLastError());
  if (h) CK(cudaMemcpyAsync(h, x->stage_h, sizeof(double) * C, kind, s));
  if (qx) CK(cudaMemcpyAsync(qx, x->stage_qx, sizeof(double) * C, kind, s));
  if (qy) CK(cudaMemcpyAsync(qy, x->stage_qy, sizeof(double) * C, kind, s));
  CK(cudaStreamSynchronize(s));
  return SWE_OK;
}

int swe_dev_get_state(swe_dev_ctx* x, double* h, double* qx, double* qy, double* t,
                      long long* step) {
  return get_state_impl(x, h, qx, qy, t, step, cudaMemcpyDeviceToHost);
}

int swe_dev_get_state_device(swe_dev_ctx* x, double* h, double* qx, double* qy) {
  return get_state_impl(x, h, qx, qy, nullptr, nullptr, cudaMemcpyDeviceToDevice);
}

int swe_dev_get_ledger(swe_dev_ctx* x, double* clipped, long long* events) {
  if (!x) return fail_invalid("null context");
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  if (clipped) *clipped = x->h_ctl->clipped;
  if (events) *events = x->h_ctl->events;
  return SWE_OK;
}

int swe_dev_set_ledger(swe_dev_ctx* x, double clipped, long long events) {
  if (!x) return fail_invalid("null context");
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  x->h_ctl->clipped = clipped;
  x->h_ctl->events = events;
  CK(cudaMemcpyAsync(x->ctl, x->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  return SWE_OK;
}

// launches of one step with plain kernels (optionally bracketed by events)
static int plain_step(swe_dev_ctx* x, size_t ev_base) {
  const bool prof = x->profiling;
  if (prof) CK(cudaEventRecord(x->events[ev_base + 0], x->stream));
  if (int rc = launch_face(x)) return rc;
  if (prof) CK(cudaEventRecord(x->events[ev_base + 1], x->stream));
  if (int rc = launch_cell(x)) return rc;
  if (prof) CK(cudaEventRecord(x->events[ev_base + 2], x->stream));
  if (int rc = launch_finalize(x, cudaGraphConditionalHandle{}, 0)) return rc;
  if (prof) CK(cudaEventRecord(x->events[ev_base + 3], x->stream));
  return SWE_OK;
}

int swe_dev_step(swe_dev_ctx* x, double t_end, swe_step_record* rec, swe_status* st) {
  if (!x) return fail_invalid("null context");
  if (int rc = ensure_cfl(x)) return rc;
  if (int rc = write_params(x, t_end, LLONG_MAX, INFINITY, 1, 0, 1)) return rc;
  if (int rc = launch_gate(x)) return rc;
  const bool prof = x->profiling;
  x->profiling = false;
  int rc = plain_step(x, 0);
  x->profiling = prof;
  if (rc) return rc;
  const int code = read_status(x, st);
  if (code == SWE_OK && rec) CK(cudaMemcpy(rec, x->rec, sizeof(swe_step_record), cudaMemcpyDeviceToHost));
  return code;
}

int swe_dev_advance(swe_dev_ctx* x, double t_end, long long max_steps, double next_snap,
                    swe_step_record* series, long long max_records, long long* n_done,
                    swe_status* st) {
  if (!x) return fail_invalid("null context");
  if (n_done) *n_done = 0;
  const long long cap = std::min<long long>(max_records > 0 ? max_records : x->rec_cap, x->rec_cap);
  if (int rc = ensure_cfl(x)) return rc;
  if (int rc = write_params(x, t_end, max_steps, next_snap, cap, 0)) return rc;
  if (x->exec) {
    CK(cudaGraphLaunch(x->exec, x->stream));
    ++g_launches;
  } else {
    // no graph: step until the device says stop (checked every 64 steps)
    if (int rc = launch_gate(x)) return rc;
    for (long long k = 0; k < cap; ++k) {
      if (int rc = plain_step(x, 0)) return rc;
      if ((k & 63) == 63) {
        read_status(x, nullptr);
        if (!x->h_ctl->active) break;
      }
    }
  }
  const int code = read_status(x, st);
  const long long n = x->h_ctl->n_rec;
  if (n_done) *n_done = n;
  if (series && n > 0)
    CK(cudaMemcpy(series, x->rec, sizeof(swe_step_record) * (size_t)std::min(n, cap),
                  cudaMemcpyDeviceToHost));
  return code;
}

int swe_dev_advance_n_async(swe_dev_ctx* x, long long n, double t_end) {
  if (!x) return fail_invalid("null context");
  if (int rc = ensure_cfl(x)) return rc;
  if (int rc = write_params(x, t_end, LLONG_MAX, INFINITY, x->rec_cap, 1)) return rc;
  if (int rc = launch_gate(x)) return rc;
  if (x->profiling) {
    const size_t need = 4 * (size_t)n;
    while (x->events.size() < need) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      x->events.push_back(e);
    }
  }
  for (long long k = 0; k < n; ++k)
    if (int rc = plain_step(x, 4 * (size_t)k)) return rc;
  if (x->profiling) {
    CK(cudaStreamSynchronize(x->stream));
    for (long long k = 0; k < n; ++k) {
      for (int j = 0; j < 3; ++j) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, x->events[4 * k + j], x->events[4 * k + j + 1]));
        x->kms[j] += ms;
        x->klaunch[j] += 1;
      }
    }
  }
  return SWE_OK;
}

int swe_dev_synchronize(swe_dev_ctx* x, swe_status* st) {
  if (!x) return fail_invalid("null context");
  return read_status(x, st);
}

int swe_dev_compute_fluxes(swe_dev_ctx* x, double* left, double* right, swe_status* st) {
  if (!x || !left || !right) return fail_invalid("swe_dev_compute_fluxes: null argument");
  const int E = x->d.E;
  // one face pass on the current state (no commit): active gate only
  if (int rc = write_params(x, INFINITY, LLONG_MAX, INFINITY, 1, 0, 2)) return rc;
  if (int rc = launch_gate(x)) return rc;
  if (int rc = launch_face(x)) return rc;
  double *dl = nullptr, *dr = nullptr;
  CK(cudaMalloc(&dl, sizeof(double) * 3 * (size_t)E));
  CK(cudaMalloc(&dr, sizeof(double) * 3 * (size_t)E));
  k_flux_out<<<blocks_for(E), kBlock, 0, x->stream>>>(x->d, dl, dr);
  ++g_launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(left, dl, sizeof(double) * 3 * (size_t)E, cudaMemcpyDeviceToHost, x->stream));
  CK(cudaMemcpyAsync(right, dr, sizeof(double) * 3 * (size_t)E, cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  cudaFree(dl);
  cudaFree(dr);
  // promote a negative depth into the status, then clear the gate
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  Ctl c = *x->h_ctl;
  int code = SWE_OK;
  if (c.bad_edge != kNone) {
    code = SWE_NEGATIVE_DEPTH;
    if (st) {
      st->code = code;
      st->index = c.bad_edge;
    }
  } else if (st) {
    st->code = SWE_OK;
  }
  c.bad_edge = kNone;
  c.active = 0;
  *x->h_ctl = c;
  CK(cudaMemcpyAsync(x->ctl, x->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  return code;
}

int swe_dev_total_mass(swe_dev_ctx* x, double* mass) {
  if (!x || !mass) return fail_invalid("null argument");
  // recompute the CFL cache (which carries the mass) for the current state;
  // a pending non-finite speed is preserved by k_cfl/k_prepare
  if (int rc = ensure_cfl(x, true)) return rc;
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  *mass = x->h_ctl->mass;
  return SWE_OK;
}

int swe_dev_set_profiling(swe_dev_ctx* x, int on) {
  if (!x) return fail_invalid("null context");
  x->profiling = on != 0;
  for (int i = 0; i < 4; ++i) {
    x->kms[i] = 0;
    x->klaunch[i] = 0;
  }
  return SWE_OK;
}

int swe_dev_kernel_times(swe_dev_ctx* x, double* ms, long long* launches, int n) {
  if (!x) return fail_invalid("null context");
  for (int i = 0; i < n && i < 4; ++i) {
    if (ms) ms[i] = x->kms[i];
    if (launches) launches[i] = x->klaunch[i];
  }
  return SWE_OK;
}

void* swe_dev_stream(swe_dev_ctx* x) { return x ? (void*)x->stream : nullptr; }

long long swe_dev_memory_bytes(swe_dev_ctx* x) { return x ? x->bytes : 0; }

int swe_dev_point_eval(int kind, long long n, const swe_params* p, const double* l,
                       const double* r, const double* z, const double* nrm, double* out) {
  if (n <= 0) return SWE_OK;
  if (!p || !l || !out) return fail_invalid("swe_dev_point_eval: null argument");
  const size_t outw = kind == 2 ? 6 : (kind == 4 ? 1 : 3);
  double *dl = nullptr, *dr = nullptr, *dz = nullptr, *dn = nullptr, *dout = nullptr;
  CK(cudaMalloc(&dl, sizeof(double) * 3 * n));
  CK(cudaMalloc(&dr, sizeof(double) * 3 * n));
  CK(cudaMalloc(&dz, sizeof(double) * 2 * n));
  CK(cudaMalloc(&dn, sizeof(double) * 2 * n));
  CK(cudaMalloc(&dout, sizeof(double) * outw * n));
  CK(cudaMemcpy(dl, l, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
  if (r) CK(cudaMemcpy(dr, r, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
  if (z) CK(cudaMemcpy(dz, z, sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
  if (nrm) CK(cudaMemcpy(dn, nrm, sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
  const Phys P{p->g, p->h_dry, p->cfl, p->dt_max, p->h_ref};
  k_point<<<blocks_for(n), kBlock>>>(kind, n, P, dl, dr, dz, dn, dout);
  ++g_launches;
  CK(cudaGetLastError());
  CK(cudaMemcpy(out, dout, sizeof(double) * outw * n, cudaMemcpyDeviceToHost));
  cudaFree(dl);
  cudaFree(dr);
  cudaFree(dz);
  cudaFree(dn);
  cudaFree(dout);
  return SWE_OK;
}

}  // extern "C"
