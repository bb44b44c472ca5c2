// swe_step.cuh -- the explicit step kernels.
//
// The reference's cell update (engine.hpp:254-268) sums, for each cell c and
// local edge k = 0,1,2, the three terms
//     F.mass * l,   (F.momx - own_c * ox) * l,   (F.momy - own_c * oy) * l
// with own_c = 0.5 g h_c^2 and (ox, oy) = sign * n.  Every input of a term is
// known where the edge flux is evaluated (both cells' depths are loaded
// there), so the edge evaluation emits these per-incidence CONTRIBUTIONS --
// the very same FP64 values -- into the slot 3c+k of the cell they belong to,
// and the update reduces three contiguous slots in the reference's order.
//
//   k_tile    fused step (default): per tile of T Morton-consecutive cells,
//             stage the tile's state in shared memory, evaluate the tile's
//             owned edges and its halo edges (owned by a neighbouring tile,
//             evaluated by both from identical inputs -> identical bits),
//             write contributions of in-tile sides to shared memory, update.
//   k_face_c + k_cell_c   two-phase step: contributions through HBM; the
//             update is a pure streaming kernel.
//   k_face    edge records for the compute_fluxes API (engine.hpp:138-170).
// All reproduce engine.hpp:138-170 + :248-290 bit for bit; the update also
// produces the next step's CFL bound and the post-step mass.
#pragma once

#include "swe_ctl.cuh"

// resident-block budgets (registers) measured on B200 at 10M cells:
// face 5 (48 regs), cell 4 (64), tile 4 x 256-thread equivalents (64 regs)
#ifndef SWE_FACE_MINB
#define SWE_FACE_MINB 5
#endif
#ifndef SWE_CELL_MINB
#define SWE_CELL_MINB 4
#endif
#ifndef SWE_TILE_MINB
#define SWE_TILE_MINB 4
#endif

namespace swe_b200 {

// SWE_CHECKED=1 (test builds, tools/checked_build.sh): device-side bounds
// checks of every index the step kernels compute -- tiles, cells, edges,
// shared-memory slots, halo pushes -- trapping on a violation (this pool's
// compute-sanitizer is closed; profiles/r02_sanitizer_closed.txt)
#ifndef SWE_CHECKED
#define SWE_CHECKED 0
#endif
#if SWE_CHECKED
#define SWE_CHECK(cond)                                                              \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("SWE_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,   \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                           \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define SWE_CHECK(cond) ((void)0)
#endif

// per-thread accumulators of the cell update
struct CellAcc {
  double lo, hi, mass, clip;
  long long ev;
};

// contributions of one edge to its left / right cell (terms of
// engine.hpp:261-263); walls contribute to the left cell only
struct EdgeTerms {
  double lm, lx, ly, rm, rx, ry;
};

// evaluate one edge from its two states (engine.hpp:147-166); returns false
// on a negative depth (engine.hpp:147-153)
__device__ __forceinline__ bool edge_terms(const Cons& uL, double zl, const Cons& uR, double zr,
                                           bool is_wall, double nx, double ny, double len,
                                           const Phys& P, EdgeTerms& t) {
  const double hg = 0.5 * P.g;
  const double ownL = (hg * uL.h) * uL.h;
  if (!is_wall) {
    if (uL.h < 0.0 || uR.h < 0.0) return false;
    double f0, lx, ly, rx, ry;
    interior_edge(uL, zl, uR, zr, nx, ny, P, f0, lx, ly, rx, ry);
    const double ownR = (hg * uR.h) * uR.h;
    t.lm = f0 * len;
    t.lx = (lx - ownL * nx) * len;
    t.ly = (ly - ownL * ny) * len;
    t.rm = (-f0) * len;  // right.mass = -f.mass
    t.rx = (rx - ownR * (-nx)) * len;
    t.ry = (ry - ownR * (-ny)) * len;
  } else {
    if (uL.h < 0.0) return false;
    const Flux f = wall(uL, nx, ny, P);  // engine.hpp:155-159
    t.lm = f.m * len;
    t.lx = (f.fx - ownL * nx) * len;
    t.ly = (f.fy - ownL * ny) * len;
  }
  return true;
}

// engine.hpp:265-289 given the cell's summed fluxes and its area / Manning n /
// inradius; writes the new state and accumulates the clip ledger, the mass
// and the next step's CFL bound
__device__ __forceinline__ Cons cell_finish_v(const Dev& d, int c, double h, double qx, double qy,
                                              double am, double ax, double ay, double dt,
                                              double area, double man, double inr, double* NH,
                                              double* NQX, double* NQY, CellAcc& a) {
  const Phys& P = d.P;
  const double scale = dt / area;  // engine.hpp:265-268
  Cons u{h - scale * am, qx - scale * ax, qy - scale * ay};
  u = friction(u, man, dt, P);  // engine.hpp:269
  if (u.h < -1e-14 * P.h_ref || !isfinite(u.h) || !isfinite(u.qx) || !isfinite(u.qy)) {
    atomicMin(&d.ctl->bad_cell, __ldg(d.c_orig + c));  // engine.hpp:273-279
    NH[c] = u.h;
    NQX[c] = u.qx;
    NQY[c] = u.qy;
    return u;
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
      a.lo = sel_min(a.lo, inr / s);
      a.hi = sel_max(a.hi, s);
    }
  }
  return u;
}

__device__ __forceinline__ Cons cell_finish(const Dev& d, int c, double h, double qx, double qy,
                                            double am, double ax, double ay, double dt,
                                            double* NH, double* NQX, double* NQY, CellAcc& a) {
  return cell_finish_v(d, c, h, qx, qy, am, ax, ay, dt, __ldg(d.area + c), __ldg(d.man + c),
                __ldg(d.inr + c), NH, NQX, NQY, a);
}

// ---------------------------------------------------------------------------
// k_face: edge records {f0, left momentum, right momentum} for compute_fluxes
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

// ---------------------------------------------------------------------------
// two-phase step: k_face_c (contributions to HBM) then k_cell_c (streaming)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock, SWE_FACE_MINB) k_face_c(Dev d) {
  Ctl* ctl = d.ctl;
  if (!ctl->active) return;
  const int cur = ctl->cur;
  const double* __restrict__ H = d.h[cur];
  const double* __restrict__ QX = d.qx[cur];
  const double* __restrict__ QY = d.qy[cur];
  const int stride = gridDim.x * blockDim.x;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < d.E; e += stride) {
    const int cl = __ldg(d.el + e), cr = __ldg(d.er + e);
    const double nx = __ldg(d.nx + e), ny = __ldg(d.ny + e), len = __ldg(d.len + e);
    const Cons uL{__ldg(H + cl), __ldg(QX + cl), __ldg(QY + cl)};
    const bool w = cr < 0;
    const int crs = w ? cl : cr;
    const Cons uR{__ldg(H + crs), __ldg(QX + crs), __ldg(QY + crs)};
    EdgeTerms t;
    if (!edge_terms(uL, __ldg(d.z + cl), uR, __ldg(d.z + crs), w, nx, ny, len, d.P, t)) {
      atomicMin(&ctl->bad_edge, __ldg(d.e_orig + e));
      continue;
    }
    const int sl = 3 * cl + __ldg(d.kl + e);
    d.TM[sl] = t.lm;
    d.TX[sl] = t.lx;
    d.TY[sl] = t.ly;
    if (!w) {
      const int sr = 3 * cr + __ldg(d.kr + e);
      d.TM[sr] = t.rm;
      d.TX[sr] = t.rx;
      d.TY[sr] = t.ry;
    }
  }
}

__global__ void __launch_bounds__(kBlock, SWE_CELL_MINB) k_cell_c(Dev d) {
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
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d.C_own; c += stride) {
    double am = 0.0, ax = 0.0, ay = 0.0;  // engine.hpp:255-264, local order k
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      am += d.TM[3 * c + k];
      ax += d.TX[3 * c + k];
      ay += d.TY[3 * c + k];
    }
    cell_finish(d, c, H[c], QX[c], QY[c], am, ax, ay, dt, NH, NQX, NQY, a);
  }
  block_reduce_part(a.lo, a.hi, a.mass, a.clip, a.ev, d.part + blockIdx.x);
}

// linked two-phase step: push the new state of the cells peers hold as ghosts
__global__ void __launch_bounds__(kBlock) k_push(Dev d) {
  const Ctl* ctl = d.ctl;
  if (!ctl->active) return;
  const int nxt = ctl->cur ^ 1;
  const int n = d.L.tile_push[d.ntiles];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int c = d.L.push_cell[j], g = d.L.push_ghost[j];
  double* const* dst = d.L.state + 6 * d.L.push_rank[j] + 3 * nxt;
  dst[0][g] = d.h[nxt][c];
  dst[1][g] = d.qx[nxt][c];
  dst[2][g] = d.qy[nxt][c];
  __threadfence_system();
}

// ---------------------------------------------------------------------------
// fused tile kernel.  Per tile of T Morton-consecutive cells: stage the
// tile's state and bed in shared memory, evaluate the owned + halo edges
// into per-incidence contributions in shared memory, update the cells.
// Tiles whose cells and ring are dry and at rest skip the edge evaluation
// (exact).  Shared memory: state+bed [4T], contributions [9T]
// -- kept small on purpose: the FP64 dependency chains of the flux need
// resident warps more than staged data (a variant staging every array needed
// 65 KB per 256-cell tile and ran 1.3x slower; a TMA bulk L2 prefetch of the
// next tile's ranges (cp.async.bulk.prefetch.L2) cost 6%).
// ---------------------------------------------------------------------------
// streamed loads that no other warp of the CTA re-reads kept out of L1
// (SWE_L1_HINTS=1: ld.global.L1::no_allocate for the edge records and the
// staged state) -- measured no faster than the default allocation
#ifndef SWE_L1_HINTS
#define SWE_L1_HINTS 0
#endif
#if SWE_L1_HINTS
__device__ __forceinline__ double ld_na(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_na(const double2* p) {
  double2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ int2 ld_na(const int2* p) {
  int2 v;
  asm("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
// state of the current step: written by the previous launch, read-only here
__device__ __forceinline__ double ld_na_state(const double* p) {
  double v;
  asm("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
#define SWE_LD_STREAM(p) ld_na(p)
#define SWE_LD_STATE(p) ld_na_state(p)
#else
#define SWE_LD_STREAM(p) __ldg(p)
#define SWE_LD_STATE(p) (*(p))
#endif
// one 256-bit read-only load of a cell record (sm_100: LDG.E.ENL2.256)
__device__ __forceinline__ CellGeo ldg_geo(const CellGeo* p) {
  CellGeo g;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(g.z), "=d"(g.area), "=d"(g.man), "=d"(g.inr)
      : "l"(p));
  return g;
}
// SWE_TILE_TMA=1 (experiment build, tools/variant_build.sh): the tile's state
// arrives by TMA bulk copies (cp.async.bulk + mbarrier complete_tx) into one of
// two shared buffers, the next computed tile's copy issued when a tile starts,
// so it lands while the current tile is evaluated.  16T doubles of shared
// memory: 7 CTAs per SM at T = 224.
#ifndef SWE_TILE_TMA
#define SWE_TILE_TMA 0
#endif
__host__ __device__ constexpr size_t tile_smem_bytes(int T, int S) {
  // state+bed [4T], contributions [9T] (TMA: two state buffers [6T] + bed [T])
  // (SWE_TILE_TMA=2: one buffer, the tile's own copy only: 13T, 8 CTAs per SM)
  return sizeof(double) * (SWE_TILE_TMA == 1 ? 16 : 13) * (size_t)T + 0 * (size_t)S;
}

#if SWE_TILE_TMA
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// one tile's h / qx / qy (3 x bytes) into dst[0..3T): issued by one thread
__device__ __forceinline__ void tma_state(double* dst, int T, const double* H, const double* QX,
                                          const double* QY, int c0, unsigned bytes,
                                          unsigned long long* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after generic reads of dst
  const unsigned b = smem_u32(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(3 * bytes)
               : "memory");
  const double* src[3] = {H + c0, QX + c0, QY + c0};
#pragma unroll
  for (int k = 0; k < 3; ++k)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst + k * T)),
        "l"(src[k]), "r"(bytes), "r"(b)
        : "memory");
}
#endif

// Skip decision of tile tk for the step with tag `tag` (thread 0, kAhead
// tiles ahead): 0 compute, 1 skip, 2 skip without writing the tile's next
// state.  A tile that k_tile skipped at the two previous steps already holds
// the state it would write in the next buffer: the step two back wrote
// (h, 0, 0) there, and the step between copied the same h (skipped tiles keep
// h bit for bit and zero q).  streak[tk] = {tag of its last skip by k_tile,
// consecutive skips}; any other writer of the state (set_state, link, other
// step kernels) breaks or clears the chain.
__device__ __forceinline__ int skip_code(const Dev& d, int tk, int tag) {
  if (tk >= d.ntiles) return 0;
  const int m = __ldg(d.skipmask + tk);
  const int2 st = d.streak ? d.streak[tk] : make_int2(0, 0);
  if (m != tag) return 0;
  if (!d.streak) return 1;
  const bool chain = st.x == tag - 1;
  d.streak[tk] = make_int2(tag, chain ? st.y + 1 : 1);
  return chain && st.y >= 2 ? 2 : 1;
}

// LINK: linked context -- after the update, push the tile's cells that peers
// hold as ghosts into the peers' next state buffers (see Link, swe_ctl.cuh).
// (Finalizing in the kernel's last block instead of a separate launch was
// measured slower: its register copies spill into the main loop.)
template <int NT, bool LINK>
#ifndef SWE_TILE_BLOCKS
#if SWE_TILE_TMA == 1
#define SWE_TILE_BLOCKS(NT) (896 / (NT))
#else
#define SWE_TILE_BLOCKS(NT) (SWE_TILE_MINB * 256 / (NT))
#endif
#endif
__global__ void __launch_bounds__(NT, SWE_TILE_BLOCKS(NT)) k_tile(Dev d) {
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
  const int T = d.T;
#if SWE_TILE_TMA
  double* const tbuf = smem;  // [2][3T]: the tile's state / the next computed tile's
  double *sh = tbuf, *sq = sh + T, *sr = sq + T;
  double* sz = smem + (SWE_TILE_TMA == 1 ? 6 : 3) * T;
  __shared__ __align__(8) unsigned long long s_bar[2];
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned ph = 0;  // bit b: parity of buffer b's next completion
  int pf_tile = -1, pf_buf = 0;
#else
  double* sh = smem;
  double* sq = sh + T;
  double* sr = sq + T;
  double* sz = sr + T;
#endif
  double* tm = sz + T;
  double* tx = tm + 3 * T;
  double* ty = tx + 3 * T;
  const Phys P = d.P;
  CellAcc a{INFINITY, 0.0, 0.0, 0.0, 0};

#ifndef SWE_SKIP_AHEAD
#define SWE_SKIP_AHEAD 4
#endif
  constexpr int kAhead = SWE_SKIP_AHEAD;  // skip decisions known ahead per CTA (ring s_dec)
  constexpr int kRing = 2 * kAhead, kMask = kRing - 1;
  static_assert((kAhead & (kAhead - 1)) == 0 && kAhead <= 16, "SWE_SKIP_AHEAD: a power of two");
  __shared__ int s_next, s_skip, s_dec[kRing];
  // dry-tile skipping: skipmask[t] == tag(state) <=> tile t and its ring were
  // dry and at rest (computed by the finalize launch from the flags this
  // kernel writes, tagged with the step of the state they describe).  With
  // the static schedule the decisions of this CTA's next kAhead tiles sit in
  // s_dec[it .. it + kAhead) (mod 8), refilled by thread 0.
  const int tag = (int)(ctl->step + 1);
  const bool ahead = d.skip && !d.dyn;
  if (ahead && threadIdx.x == 0)
    for (int k = 0; k < kAhead; ++k) {
      const int tk = blockIdx.x + k * gridDim.x;
      s_dec[k] = skip_code(d, tk, tag);
    }
  __syncthreads();
  int it = 0;
  for (int t = blockIdx.x; t < d.ntiles;) {
    const int c0 = t * T;
    SWE_CHECK(t >= 0 && t < d.ntiles && c0 < d.C_own);
    const int nc = min(T, d.C_own - c0);
    const bool pre_skip = ahead && s_dec[it & kMask] != 0;
    if (pre_skip) {
      // skipped tiles, fast path: a run of up to kAhead consecutive skipped
      // tiles of this CTA in one round trip, no shared memory (a tile with
      // halo pushes is never in the skip mask)
      int run = 1;
      while (run < kAhead && s_dec[(it + run) & kMask]) ++run;
      if (threadIdx.x == 0) {
        int held = 0;
        for (int k = 0; k < run; ++k) {
          held += s_dec[(it + k) & kMask] == 2;
          const int tk = t + (kAhead + k) * gridDim.x;
          s_dec[(it + kAhead + k) & kMask] = skip_code(d, tk, tag);
          d.dryflag[t + k * gridDim.x] = tag + 1;
        }
        atomicAdd(&ctl->skipped, (unsigned long long)run);
        if (held) atomicAdd(&ctl->held, (unsigned long long)held);
      }
#ifndef SWE_SKIP_HOIST
#define SWE_SKIP_HOIST 1
#endif
      if (SWE_SKIP_HOIST && T <= 2 * NT) {
        // every load of the run first (up to kAhead tiles x 2 cells per
        // thread), then the stores and the mass in tile, cell order: one
        // round trip for the run instead of one per cell
        double hv[kAhead][2], av[kAhead][2];
#pragma unroll
        for (int k = 0; k < kAhead; ++k) {
          const int ck = (t + k * gridDim.x) * T;
          const int nk = k < run ? min(T, d.C_own - ck) : 0;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int i = threadIdx.x + j * NT;
            hv[k][j] = i < nk ? H[ck + i] : 0.0;
            av[k][j] = i < nk ? __ldg(d.area + ck + i) : 0.0;
          }
        }
#pragma unroll
        for (int k = 0; k < kAhead; ++k) {
          if (k >= run) break;
          const int ck = (t + k * gridDim.x) * T;
          const int nk = min(T, d.C_own - ck);
          const bool held = s_dec[(it + k) & kMask] == 2;  // the next buffer holds it already
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int i = threadIdx.x + j * NT;
            if (i < nk) {
              if (!held) {
                NH[ck + i] = hv[k][j];
                NQX[ck + i] = 0.0;
                NQY[ck + i] = 0.0;
              }
              a.mass += hv[k][j] * av[k][j];
            }
          }
        }
      } else {
        for (int k = 0; k < run; ++k) {  // tile order, then cell order: the mass sums' order
          const int ck = (t + k * gridDim.x) * T;
          const int nk = min(T, d.C_own - ck);
          const bool held = s_dec[(it + k) & kMask] == 2;  // the next buffer holds it already
          for (int i = threadIdx.x; i < nk; i += NT) {
            const double h = H[ck + i];
            if (!held) {
              NH[ck + i] = h;
              NQX[ck + i] = 0.0;
              NQY[ck + i] = 0.0;
            }
            a.mass += h * __ldg(d.area + ck + i);
          }
        }
      }
      __syncthreads();  // s_dec refill
      t += run * gridDim.x;
      it += run;
      continue;
    }
#if SWE_TILE_TMA
    const bool full = nc == T;  // T * 8 bytes: a multiple of 16
    int cb = 0;
    if (pf_tile == t) {
      cb = pf_buf;
    } else if (full && threadIdx.x == 0) {
      tma_state(tbuf, T, H, QX, QY, c0, (unsigned)(T * sizeof(double)), &s_bar[0]);
    }
    sh = tbuf + cb * 3 * T;
    sq = sh + T;
    sr = sq + T;
    {  // the next tile's state (if it is computed), in flight during this one
      const int tn = t + gridDim.x;
      pf_tile = -1;
      if (SWE_TILE_TMA == 1 && tn < d.ntiles && (tn + 1) * T <= d.C_own &&
          !(ahead && s_dec[(it + 1) & kMask])) {
        if (threadIdx.x == 0)
          tma_state(tbuf + (cb ^ 1) * 3 * T, T, H, QX, QY, tn * T, (unsigned)(T * sizeof(double)),
                    &s_bar[cb ^ 1]);
        pf_tile = tn;
        pf_buf = cb ^ 1;
      }
    }
    for (int i = threadIdx.x; i < nc; i += NT) {
      if (!full) {  // the last, partial tile: plain loads
        sh[i] = SWE_LD_STATE(H + c0 + i);
        sq[i] = SWE_LD_STATE(QX + c0 + i);
        sr[i] = SWE_LD_STATE(QY + c0 + i);
      }
      sz[i] = ldg_geo(d.cg + c0 + i).z;
    }
    if (full) {
      mbar_wait(&s_bar[cb], (ph >> cb) & 1u);
      ph ^= 1u << cb;
    }
#else
    for (int i = threadIdx.x; i < nc; i += NT) {  // stage the tile (a skipped one needs h only)
      sh[i] = SWE_LD_STATE(H + c0 + i);
      if (!pre_skip) {
        sq[i] = SWE_LD_STATE(QX + c0 + i);
        sr[i] = SWE_LD_STATE(QY + c0 + i);
        sz[i] = ldg_geo(d.cg + c0 + i).z;  // area, n, r come along (read at the update)
      }
    }
#endif
    const int e0 = __ldg(d.eoff + t), no = __ldg(d.eoff + t + 1) - e0;
    const int h0 = __ldg(d.hoff + t), ns = no + __ldg(d.hoff + t + 1) - h0;
    int p0 = 0, p1 = 0;  // push-list range of the tile (linked)
    if (LINK) {
      p0 = __ldg(d.L.tile_push + t);
      p1 = __ldg(d.L.tile_push + t + 1);
    }
    // dry-tile skip: the tile and its ring were dry and at rest after the
    // previous step -> every mass flux is exactly +-0, h stays bit-identical,
    // the dry clamp zeroes q, no CFL contribution
    if (threadIdx.x == 0) {
      int sk;
      if (ahead) {
        sk = pre_skip;  // decided ahead; refill the ring
        const int tk = t + kAhead * gridDim.x;
        s_dec[(it + kAhead) & kMask] = skip_code(d, tk, tag);
      } else {
        sk = d.skip && __ldg(d.skipmask + t) == tag;
      }
      if (sk) atomicAdd(&ctl->skipped, 1ULL);
      s_skip = sk;
    }
    __syncthreads();
    const bool skip = s_skip != 0;

    // owned + halo edges -> contributions of the in-tile sides
    for (int j = threadIdx.x; j < (skip ? 0 : ns); j += NT) {
      const int e = j < no ? e0 + j : __ldg(d.halo + h0 + (j - no));
      SWE_CHECK(e >= 0 && e < d.E);
      const int2 ek = SWE_LD_STREAM(d.ek + e);
      const double2 nn = SWE_LD_STREAM(d.enxy + e);
      const double nx = nn.x, ny = nn.y, len = SWE_LD_STREAM(d.len + e);
      const int cl = ek.x & 0x3fffffff, cr = ek.y & 0x3fffffff;
      SWE_CHECK(cl < d.C && (ek.y == -1 || cr < d.C));
      const bool w = ek.y == -1;
      const int il = cl - c0, ir = (w ? cl : cr) - c0;
      const bool inL = (unsigned)il < (unsigned)nc, inR = !w && (unsigned)ir < (unsigned)nc;
      Cons uL, uR;
      double zl, zr;
      if (inL) {
        uL = Cons{sh[il], sq[il], sr[il]};
        zl = sz[il];
      } else {
        uL = Cons{__ldg(H + cl), __ldg(QX + cl), __ldg(QY + cl)};
        zl = __ldg(d.z + cl);
      }
      if ((unsigned)ir < (unsigned)nc) {
        uR = Cons{sh[ir], sq[ir], sr[ir]};
        zr = sz[ir];
      } else {
        const int c = ir + c0;
        uR = Cons{__ldg(H + c), __ldg(QX + c), __ldg(QY + c)};
        zr = __ldg(d.z + c);
      }
      // edge_terms() inlined with every contribution stored as soon as it is
      // formed (shorter live ranges than a six-value record)
      if (uL.h < 0.0 || (!w && uR.h < 0.0)) {  // engine.hpp:147-153
        atomicMin(&ctl->bad_edge, __ldg(d.e_orig + e));
        continue;
      }
      const double hg = 0.5 * P.g;
      const int sl = 3 * il + (int)((unsigned)ek.x >> 30);
      if (!w) {
        double f0, lx, ly, rx, ry;
        interior_edge(uL, zl, uR, zr, nx, ny, P, f0, lx, ly, rx, ry);
        // the edge's index record and length are re-read (L1) rather than
        // held in registers across the Riemann solver
        (void)inR;
        const int2 ek2 = __ldg(d.ek + e);
        const double len2 = __ldg(d.len + e);
        const int il2 = (ek2.x & 0x3fffffff) - c0, ir2 = (ek2.y & 0x3fffffff) - c0;
        if ((unsigned)il2 < (unsigned)nc) {
          const int s2 = 3 * il2 + (int)((unsigned)ek2.x >> 30);
          SWE_CHECK(s2 >= 0 && s2 < 3 * nc);
          const double ownL = (hg * uL.h) * uL.h;
          tm[s2] = f0 * len2;
          tx[s2] = (lx - ownL * nx) * len2;
          ty[s2] = (ly - ownL * ny) * len2;
        }
        if ((unsigned)ir2 < (unsigned)nc) {
          const int sr = 3 * ir2 + (int)((unsigned)ek2.y >> 30);
          SWE_CHECK(sr >= 0 && sr < 3 * nc);
          const double ownR = (hg * uR.h) * uR.h;
          tm[sr] = (-f0) * len2;  // right.mass = -f.mass
          tx[sr] = (rx - ownR * (-nx)) * len2;
          ty[sr] = (ry - ownR * (-ny)) * len2;
        }
      } else if (inL) {
        const Flux f = wall(uL, nx, ny, P);  // engine.hpp:155-159
        const double ownL = (hg * uL.h) * uL.h;
        tm[sl] = f.m * len;
        tx[sl] = (f.fx - ownL * nx) * len;
        ty[sl] = (f.fy - ownL * ny) * len;
      }
    }
    __syncthreads();

    // cell update from the three contribution slots
    int dry = 1;  // every cell of the tile dry and at rest afterwards
    for (int i = threadIdx.x; i < nc; i += NT) {
      if (skip) {  // cell_finish of a dry cell with zero mass flux, exactly
        const double h = sh[i];
        NH[c0 + i] = h;
        NQX[c0 + i] = 0.0;
        NQY[c0 + i] = 0.0;
        a.mass += h * __ldg(d.area + c0 + i);
        if (LINK && p1 > p0) {
          sq[i] = 0.0;
          sr[i] = 0.0;
        }
        continue;
      }
      double am = 0.0, ax = 0.0, ay = 0.0;  // engine.hpp:255-264, local order k
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        am += tm[3 * i + k];
        ax += tx[3 * i + k];
        ay += ty[3 * i + k];
      }
      const CellGeo g = ldg_geo(d.cg + c0 + i);
      const Cons u = cell_finish_v(d, c0 + i, sh[i], sq[i], sr[i], am, ax, ay, dt, g.area, g.man,
                                   g.inr, NH, NQX, NQY, a);
      dry &= (0.0 <= u.h && u.h < P.h_dry) ? 1 : 0;
      if (LINK && p1 > p0) {  // the tile's new state, for the push below
        sh[i] = u.h;
        sq[i] = u.qx;
        sr[i] = u.qy;
      }
    }
    if (d.skip) {
      dry = __syncthreads_and(dry);
      if (threadIdx.x == 0) d.dryflag[t] = dry ? tag + 1 : 0;  // describes the next state
    } else {
      __syncthreads();
    }
    if (LINK && p1 > p0) {
      for (int j = p0 + threadIdx.x; j < p1; j += NT) {
        const int i = __ldg(d.L.push_cell + j) - c0, g = __ldg(d.L.push_ghost + j);
        SWE_CHECK(i >= 0 && i < nc && g >= 0);
        double* const* dst = d.L.state + 6 * __ldg(d.L.push_rank + j) + 3 * (cur ^ 1);
        dst[0][g] = sh[i];
        dst[1][g] = sq[i];
        dst[2][g] = sr[i];
      }
      __threadfence_system();
      __syncthreads();
    }
    if (d.dyn) {  // next tile from a shared counter (experiment, SWE_DYN_TILES=1)
      if (threadIdx.x == 0) s_next = gridDim.x + atomicAdd(&ctl->tile_next, 1);
      __syncthreads();
      t = s_next;
    } else {
      t += gridDim.x;
    }
    ++it;
  }
  block_reduce_part(a.lo, a.hi, a.mass, a.clip, a.ev, d.part + blockIdx.x);
}

// ---------------------------------------------------------------------------
// persistent step kernel (default run loop).  One cooperative launch steps
// until the loop stops (t_end, max_steps, snapshot due, record buffer full,
// error): every CTA owns the same round-robin tiles as k_tile, and the steps
// are separated by a grid barrier instead of kernel boundaries --
//   * arrival: each CTA adds one to sync->arrive after its partials; the
//     LAST to arrive reduces the partials and commits the step exactly as
//     k_finalize / k_exchange do (same code, same fixed order -> the same
//     bits), then publishes it as sync->epoch;
//   * overlap: a CTA does not wait for the commit to start the next step: as
//     soon as every CTA has arrived (the new state is complete) it decides
//     its tiles' dry-tile skips and evaluates its first tile's edges -- the
//     flux needs no dt (engine.hpp:138 takes none) -- and waits for the
//     epoch (dt, stop) only before the first update.  So the commit, and on a
//     linked context the whole exchange with the peers, runs behind flux
//     work.  Linked tiles that read ghost cells wait for the epoch first.
// Memory model: the state arrays are rewritten during the launch, so they
// are read with plain (L1-cached, not .nc) loads after an acquire, which
// invalidates L1 (ld.acquire.gpu -> LDG.STRONG.GPU + CCTL.IVALL on sm_100);
// dry-tile flags are double-buffered by step parity (pflag) so a flag is
// never rewritten while another CTA may still read it.
// Results (state, dt, records, mass, ledger) equal k_tile + k_finalize's bit
// for bit: the same per-thread tile order, partials and reduction.
// ---------------------------------------------------------------------------
constexpr int kRunDec = 128;  // skip decisions held per CTA (recomputed in chunks)

// SWE_RUN_TIMING=1 (experiment builds): per-CTA globaltimer sums of the
// persistent loop's phases in Sync::pad, read by swe_dev_run_timing
#ifndef SWE_RUN_TIMING
#define SWE_RUN_TIMING 0
#endif
#if SWE_RUN_TIMING
#define RUN_T(k, v) atomicAdd(&sy->timing[k], (unsigned long long)(v))
#else
#define RUN_T(k, v) ((void)0)
#endif

__device__ __forceinline__ bool run_skip(const Dev& d, const int* fl, int t, int tag) {
  // three round trips, not one per neighbour: the own flag and the list
  // bounds together, then up to 8 neighbour ids, then their flags
  const int own = __ldcg(fl + t);
  const int v0 = __ldg(d.nbr_off + t), v1 = __ldg(d.nbr_off + t + 1);
  if (own != tag) return false;
  bool ok = true;
  for (int v = v0; v < v1; v += 8) {
    int nbv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) nbv[k] = v + k < v1 ? __ldg(d.nbr + v + k) : -1;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int q = nbv[k];
      const int f = q < 0 ? tag : (q < d.ntiles ? __ldcg(fl + q) : 0);
      ok &= f == tag;
    }
  }
  // a tile whose cells peers hold as ghosts is computed (its pushes run there)
  if (d.L.nranks > 0 && __ldg(d.L.tile_push + t + 1) > __ldg(d.L.tile_push + t)) ok = false;
  return ok;
}

// The control CTA of the persistent kernel (the grid's last block; it owns no
// tiles): per step it waits for every worker's arrival, reduces their
// partials in the fixed order and commits the step -- k_finalize /
// k_exchange's code, so the same bits -- then publishes it as the next epoch.
// The workers meanwhile start the next step's fluxes.  Its Dev lives in its
// shared memory (the tile buffers are free), off the L1 the per-step acquire
// invalidates; kept out of line so it costs the workers no registers.
constexpr size_t kRunCtlOff = (sizeof(Part) * kBlock + 63) / 64 * 64;  // Dev, Ctl, StepParams
constexpr size_t kRunCtlSmem =
    kRunCtlOff + (sizeof(Dev) + 63) / 64 * 64 + (sizeof(Ctl) + 63) / 64 * 64 + sizeof(StepParams);

template <bool LINK>
__device__ __noinline__ void run_control(const Dev* dg, Sync* sy, int nb) {
  extern __shared__ double smem[];
  // the tile buffers of this block hold: partial scratch, its Dev, the
  // authoritative control block during the launch, the step parameters
  char* base = reinterpret_cast<char*>(smem);
  Part* scratch = reinterpret_cast<Part*>(base);
  Dev* ds = reinterpret_cast<Dev*>(base + kRunCtlOff);
  Ctl& s_c = *reinterpret_cast<Ctl*>(base + kRunCtlOff + (sizeof(Dev) + 63) / 64 * 64);
  StepParams& s_sp = *reinterpret_cast<StepParams*>(base + kRunCtlOff + (sizeof(Dev) + 63) / 64 * 64 +
                                                    (sizeof(Ctl) + 63) / 64 * 64);
  __shared__ int s_go, s_tmo;
  __shared__ double s_lo, s_hi;
  __shared__ CommitInfo s_ci;
  {
    const unsigned* src = reinterpret_cast<const unsigned*>(dg);
    unsigned* dst = reinterpret_cast<unsigned*>(ds);
    for (int i = threadIdx.x; i < (int)(sizeof(Dev) / 4); i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const Dev& d = *ds;
  if (threadIdx.x == 0) {
    s_c = load_ctl(d.ctl);  // as the gate left it
    s_sp = *d.sp;
    s_go = s_c.active;
  }
  __syncthreads();
  if (!s_go) return;  // the gate closed the loop: no worker runs a step
  for (unsigned it = 0;; ++it) {
    const unsigned long long w0 = SWE_RUN_TIMING ? global_ns() : 0;
    const int par = (int)(s_c.step & 1);
    const Part* parts = d.part + (size_t)par * nb;
    if (LINK) {
      // split exchange (swe_ctl.cuh): post the CFL bound / max speed (the
      // workers' atomics) and the error slots at once, commit the head from
      // the combined posts and publish it; then reduce and exchange the sums
      unsigned long long c0 = 0, c1 = 0;
      if (threadIdx.x == 0) {
        poll_until(&sy->arrive, (unsigned)nb * (it + 1));
        fence_acq_rel_gpu();
        if (SWE_RUN_TIMING) c0 = global_ns();
        s_lo = __longlong_as_double((long long)__ldcg(&sy->lo[par]));
        s_hi = __longlong_as_double((long long)__ldcg(&sy->hi[par]));
        sy->lo[par] = 0x7ff0000000000000ULL;  // this parity's next use: two steps on
        sy->hi[par] = 0ULL;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        post_outcome(d, Part{s_lo, s_hi, 0.0, 0.0, 0, 0}, 0);
        CommitInfo ci;
        ci.ok = false;
        bool tmo = false;
        const int go = wait_commit_head(d, s_sp, ci, tmo);
        if (threadIdx.x == 0) {
          s_ci = ci;
          s_go = go;
          s_tmo = tmo;
          s_c.step = __ldcg(&d.ctl->step);  // (the parity of the next step's slots)
          const double t = __ldcg(&d.ctl->t), dts = __ldcg(&d.ctl->dts);
          view_publish(&sy->view, it + 1, go, (t + dts >= s_sp.t_end) ? s_sp.t_end - t : dts);
          if (SWE_RUN_TIMING) c1 = global_ns();
        }
      }
      __syncthreads();
      if (!s_tmo) {  // off the critical path: the sums in the fixed order, then across ranks
        const Part p = reduce_parts_into(parts, nb, scratch);
        if (threadIdx.x < 32) {
          const CommitInfo ci = s_ci;
          const int ok = post_wait_sums(d, s_sp, p, ci);
          if (threadIdx.x == 0 && !ok && s_go) {  // stop the workers at their next view
            s_go = 0;
            view_publish(&sy->view, it + 2, 0, 0.0);
          }
        }
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        RUN_T(2, c0 - w0);
        RUN_T(3, c1 - c0);
        RUN_T(7, global_ns() - c1);
        RUN_T(5, 1);
      }
      __syncthreads();
      if (!s_go) return;
      continue;
    }
    if (threadIdx.x == 0) {
      poll_until(&sy->arrive, (unsigned)nb * (it + 1));
      fence_acq_rel_gpu();  // every worker's partials, error slots and state
      const unsigned long long c0 = SWE_RUN_TIMING ? global_ns() : 0;
      const double lo = __longlong_as_double((long long)__ldcg(&sy->lo[par]));
      const double hi = __longlong_as_double((long long)__ldcg(&sy->hi[par]));
      const int bad_edge = __ldcg(&d.ctl->bad_edge), bad_cell = __ldcg(&d.ctl->bad_cell);
      const int bad_speed = __ldcg(&d.ctl->bad_speed);
      sy->lo[par] = 0x7ff0000000000000ULL;  // this parity's next use: two steps on
      sy->hi[par] = 0ULL;
      int status = SWE_OK, index = kNone;  // finalize_local (engine.hpp:168-169, :292-297)
      double err_h = 0.0;
      if (bad_edge != kNone) {
        status = SWE_NEGATIVE_DEPTH;
        index = bad_edge;
      } else if (bad_cell != kNone) {
        status = SWE_BLOWUP;
        index = bad_cell;
        err_h = d.h[s_c.cur ^ 1][d.c_new[bad_cell]];
      }
      Ctl c = s_c;
      c.bad_speed = bad_speed;
      CommitInfo ci;
      s_go = commit_head(c, s_sp, lo, hi, status, index, err_h, d.P, ci);
      store_commit(d.ctl, c);
      s_c = c;
      s_ci = ci;
      // the next step's dt as the workers' step_dt forms it (engine.hpp:236-237)
      view_publish(&sy->view, it + 1, s_go,
                   (c.t + c.dts >= s_sp.t_end) ? s_sp.t_end - c.t : c.dts);
      RUN_T(3, global_ns() - c0);
      RUN_T(5, 1);
      RUN_T(2, c0 - w0);
    }
    __syncthreads();
    // off the critical path: the step's sums in the fixed order (the same
    // bits as k_finalize), the clip ledger and the record
    const unsigned long long r0 = SWE_RUN_TIMING ? global_ns() : 0;
    const Part p = reduce_parts_into(parts, nb, scratch);
    if (threadIdx.x == 0) {
      Ctl c = s_c;
      commit_tail(c, s_sp, p, s_ci, d.rec);
      d.ctl->clipped = c.clipped;
      d.ctl->events = c.events;
      d.ctl->mass = c.mass;
      s_c = c;
      RUN_T(7, global_ns() - r0);
    }
    __syncthreads();
    if (!s_go) return;
  }
}

// staging + edge evaluation of one computed tile of the persistent kernel
// (k_tile's code).  CG: the state is read through L2 (ld.global.cg) -- the
// first tile of a step runs before the CTA's acquire of the new epoch, and L1
// may still hold lines of this buffer from two steps ago.
#ifndef SWE_RUN_NC
#define SWE_RUN_NC 0  // experiment only: .nc loads of the state (not valid across steps)
#endif
template <bool CG>
__device__ __forceinline__ double ld_state(const double* p) {
  if (CG) return __ldcg(p);
#if SWE_RUN_NC
  return __ldg(p);
#else
  return *p;
#endif
}

template <int NT, bool CG>
__device__ __forceinline__ void run_tile_edges(const Dev& d, const double* H, const double* QX,
                                               const double* QY, int t, int c0, int nc,
                                               double* sh, double* sq, double* sr, double* sz,
                                               double* tm, double* tx, double* ty) {
  Ctl* ctl = d.ctl;
  const Phys P = d.P;
  for (int i = threadIdx.x; i < nc; i += NT) {
    sh[i] = ld_state<CG>(H + c0 + i);
    sq[i] = ld_state<CG>(QX + c0 + i);
    sr[i] = ld_state<CG>(QY + c0 + i);
    sz[i] = ldg_geo(d.cg + c0 + i).z;
  }
  const int e0 = __ldg(d.eoff + t), no = __ldg(d.eoff + t + 1) - e0;
  const int h0 = __ldg(d.hoff + t), ns = no + __ldg(d.hoff + t + 1) - h0;
  __syncthreads();
  for (int jj = threadIdx.x; jj < ns; jj += NT) {
    const int e = jj < no ? e0 + jj : __ldg(d.halo + h0 + (jj - no));
    SWE_CHECK(e >= 0 && e < d.E);
    const int2 ek = __ldg(d.ek + e);
    const double2 nn = __ldg(d.enxy + e);
    const double nx = nn.x, ny = nn.y, len = __ldg(d.len + e);
    const int cl = ek.x & 0x3fffffff, cr = ek.y & 0x3fffffff;
    SWE_CHECK(cl < d.C && (ek.y == -1 || cr < d.C));
    const bool w = ek.y == -1;
    const int il = cl - c0, ir = (w ? cl : cr) - c0;
    const bool inL = (unsigned)il < (unsigned)nc;
    Cons uL, uR;
    double zl, zr;
    if (inL) {
      uL = Cons{sh[il], sq[il], sr[il]};
      zl = sz[il];
    } else {
      uL = Cons{ld_state<CG>(H + cl), ld_state<CG>(QX + cl), ld_state<CG>(QY + cl)};
      zl = __ldg(d.z + cl);
    }
    if ((unsigned)ir < (unsigned)nc) {
      uR = Cons{sh[ir], sq[ir], sr[ir]};
      zr = sz[ir];
    } else {
      const int c = ir + c0;
      uR = Cons{ld_state<CG>(H + c), ld_state<CG>(QX + c), ld_state<CG>(QY + c)};
      zr = __ldg(d.z + c);
    }
    if (uL.h < 0.0 || (!w && uR.h < 0.0)) {  // engine.hpp:147-153
      atomicMin(&ctl->bad_edge, __ldg(d.e_orig + e));
      continue;
    }
    const double hg = 0.5 * P.g;
    const int sl = 3 * il + (int)((unsigned)ek.x >> 30);
    if (!w) {
      double f0, lx, ly, rx, ry;
      interior_edge(uL, zl, uR, zr, nx, ny, P, f0, lx, ly, rx, ry);
      const int2 ek2 = __ldg(d.ek + e);
      const double len2 = __ldg(d.len + e);
      const int il2 = (ek2.x & 0x3fffffff) - c0, ir2 = (ek2.y & 0x3fffffff) - c0;
      if ((unsigned)il2 < (unsigned)nc) {
        const int s2 = 3 * il2 + (int)((unsigned)ek2.x >> 30);
        SWE_CHECK(s2 >= 0 && s2 < 3 * nc);
        const double ownL = (hg * uL.h) * uL.h;
        tm[s2] = f0 * len2;
        tx[s2] = (lx - ownL * nx) * len2;
        ty[s2] = (ly - ownL * ny) * len2;
      }
      if ((unsigned)ir2 < (unsigned)nc) {
        const int s3 = 3 * ir2 + (int)((unsigned)ek2.y >> 30);
        SWE_CHECK(s3 >= 0 && s3 < 3 * nc);
        const double ownR = (hg * uR.h) * uR.h;
        tm[s3] = (-f0) * len2;
        tx[s3] = (rx - ownR * (-nx)) * len2;
        ty[s3] = (ry - ownR * (-ny)) * len2;
      }
    } else if (inL) {
      const Flux f = wall(uL, nx, ny, P);  // engine.hpp:155-159
      const double ownL = (hg * uL.h) * uL.h;
      tm[sl] = f.m * len;
      tx[sl] = (f.fx - ownL * nx) * len;
      ty[sl] = (f.fy - ownL * ny) * len;
    }
  }
}

template <int NT, bool LINK>
__device__ __forceinline__ void run_body(const Dev& d, const Dev* dg, Sync* sy, const int bid,
                                         const int nb) {
  extern __shared__ double smem[];
  Ctl* ctl = d.ctl;
  const int T = d.T;
  double* sh = smem;
  double* sq = sh + T;
  double* sr = sq + T;
  double* sz = sr + T;
  double* tm = sz + T;
  double* tx = tm + 3 * T;
  double* ty = tx + 3 * T;
  const Phys P = d.P;
  __shared__ unsigned char s_dec[kRunDec];
  __shared__ int s_cur, s_active;
  __shared__ long long s_step;
  __shared__ double s_dt;

  // the committed view of the step a CTA is about to update: published by the
  // finalizing CTA (epoch >= it), read by thread 0 after the acquire
  auto read_view = [&](unsigned it) {
    if (threadIdx.x == 0) {
      if (it > 0) {  // relaxed polls (an acquire per poll would flush L1 each time)
        const unsigned long long w0 = SWE_RUN_TIMING ? global_ns() : 0;
        unsigned int e, ns = 32;
        int act;
        double dtv;
        for (;;) {
          view_load(&sy->view, e, act, dtv);
          if (e >= it) break;
          __nanosleep(ns);
          ns = ns < 1024 ? 2 * ns : 1024;
        }
        // acquire the commit (and the peers' halo pushes); run_noacq: the
        // state is read through L2 only (ld.cg after the observed epoch, as
        // before it), so L1 keeps the geometry across steps
        if (!d.run_noacq) fence_acq_rel_gpu();
        s_active = act;
        s_dt = dtv;
        RUN_T(1, global_ns() - w0);
      } else {  // the launch's first step: the control block as the gate left it
        s_cur = __ldcg(&ctl->cur);
        s_step = __ldcg(&ctl->step);
        s_active = __ldcg(&ctl->active);
        const double t = __ldcg(&ctl->t), dts = __ldcg(&ctl->dts), t_end = __ldcg(&d.sp->t_end);
        s_dt = (t + dts >= t_end) ? t_end - t : dts;  // engine.hpp:236-237 (step_dt)
      }
    }
    __syncthreads();
    return s_active != 0;
  };
  if (!read_view(0)) return;
  int cur = s_cur;
  long long step = s_step;
  double dt = s_dt;
  const int ntl = bid < d.ntiles ? (d.ntiles - bid + nb - 1) / nb : 0;  // this CTA's tiles

  unsigned long long t_step = SWE_RUN_TIMING ? global_ns() : 0;
  for (unsigned it = 0;; ++it) {
    const int tag = (int)(step + 1);
    const int* fl = d.pflag + (size_t)(step & 1) * d.ntiles;       // flags of this state
    int* fl_next = d.pflag + (size_t)((step + 1) & 1) * d.ntiles;  // of the next state
    const double* H = d.h[cur];
    const double* QX = d.qx[cur];
    const double* QY = d.qy[cur];
    double* NH = d.h[cur ^ 1];
    double* NQX = d.qx[cur ^ 1];
    double* NQY = d.qy[cur ^ 1];
    CellAcc a{INFINITY, 0.0, 0.0, 0.0, 0};
    bool viewed = it == 0;  // dt / stop of this step known
#ifndef SWE_RUN_OVERLAP
#define SWE_RUN_OVERLAP 1  // 0 (experiment): wait for the commit before the first tile
#endif
    if (!SWE_RUN_OVERLAP && !viewed) {
      if (!read_view(it)) return;
      viewed = true;
      dt = s_dt;
    }
    for (int j = 0; j < ntl;) {
      if (j % kRunDec == 0) {  // skip decisions of the next chunk of tiles
        const unsigned long long q0 = SWE_RUN_TIMING && j == 0 ? global_ns() : 0;
        __syncthreads();
        for (int k = threadIdx.x; k < kRunDec && j + k < ntl; k += NT)
          s_dec[k] = d.skip && run_skip(d, fl, bid + (j + k) * nb, tag);
        __syncthreads();
        if (SWE_RUN_TIMING && j == 0 && threadIdx.x == 0) RUN_T(8, global_ns() - q0);
      }
      const int t = bid + j * nb;
      const int c0 = t * T;
      SWE_CHECK(t >= 0 && t < d.ntiles && c0 < d.C_own);
      const int nc = min(T, d.C_own - c0);
      if (s_dec[j % kRunDec]) {
        // a run of consecutive skipped tiles (as k_tile's fast path): h kept,
        // q zeroed, mass in tile then cell order; no shared memory
        int run = 1;
        while (j + run < ntl && (j + run) % kRunDec != 0 && s_dec[(j + run) % kRunDec]) ++run;
        if (!viewed) {
          if (!read_view(it)) return;
          viewed = true;
          dt = s_dt;
        }
        if (threadIdx.x == 0) {
          for (int k = 0; k < run; ++k) __stcg(fl_next + t + k * nb, tag + 1);
          atomicAdd(&ctl->skipped, (unsigned long long)run);
        }
        for (int k = 0; k < run; ++k) {
          const int ck = (t + k * nb) * T;
          const int nk = min(T, d.C_own - ck);
          for (int i = threadIdx.x; i < nk; i += NT) {
            const double h = __ldcg(H + ck + i);
            NH[ck + i] = h;
            NQX[ck + i] = 0.0;
            NQY[ck + i] = 0.0;
            a.mass += h * __ldg(d.area + ck + i);
          }
        }
        j += run;
        continue;
      }
      // a linked tile that reads ghost cells needs the peers' pushes: the epoch
      if (LINK && !viewed && __ldg(d.tile_ghost + t)) {
        if (!read_view(it)) return;
        viewed = true;
        dt = s_dt;
      }
      const unsigned long long q1 = SWE_RUN_TIMING && j == 0 ? global_ns() : 0;
      if (viewed && (it == 0 || !d.run_noacq))
        run_tile_edges<NT, false>(d, H, QX, QY, t, c0, nc, sh, sq, sr, sz, tm, tx, ty);
      else  // before the epoch: L1 may hold this buffer from two steps ago
        run_tile_edges<NT, true>(d, H, QX, QY, t, c0, nc, sh, sq, sr, sz, tm, tx, ty);
      __syncthreads();
      const unsigned long long q2 = SWE_RUN_TIMING && j == 0 ? global_ns() : 0;
      if (SWE_RUN_TIMING && j == 0 && threadIdx.x == 0) RUN_T(9, q2 - q1);
      if (!viewed) {  // the first computed tile's edges are done: now dt / stop
        if (!read_view(it)) return;
        viewed = true;
        dt = s_dt;
      }
      const unsigned long long q3 = SWE_RUN_TIMING && j == 0 ? global_ns() : 0;
      if (SWE_RUN_TIMING && j == 0 && threadIdx.x == 0) RUN_T(10, q3 - q2);
      int p0 = 0, p1 = 0;
      if (LINK) {
        p0 = __ldg(d.L.tile_push + t);
        p1 = __ldg(d.L.tile_push + t + 1);
      }
      int dry = 1;
      for (int i = threadIdx.x; i < nc; i += NT) {
        double am = 0.0, ax = 0.0, ay = 0.0;  // engine.hpp:255-264, local order k
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          am += tm[3 * i + k];
          ax += tx[3 * i + k];
          ay += ty[3 * i + k];
        }
        const CellGeo g = ldg_geo(d.cg + c0 + i);
        const Cons u = cell_finish_v(d, c0 + i, sh[i], sq[i], sr[i], am, ax, ay, dt, g.area, g.man,
                                     g.inr, NH, NQX, NQY, a);
        dry &= (0.0 <= u.h && u.h < P.h_dry) ? 1 : 0;
        if (LINK && p1 > p0) {
          sh[i] = u.h;
          sq[i] = u.qx;
          sr[i] = u.qy;
        }
      }
      dry = __syncthreads_and(dry);
      if (SWE_RUN_TIMING && j == 0 && threadIdx.x == 0) RUN_T(11, global_ns() - q3);
      if (threadIdx.x == 0 && d.skip) __stcg(fl_next + t, dry ? tag + 1 : 0);
      if (LINK && p1 > p0) {
        for (int q = p0 + threadIdx.x; q < p1; q += NT) {
          const int i = __ldg(d.L.push_cell + q) - c0, g = __ldg(d.L.push_ghost + q);
          SWE_CHECK(i >= 0 && i < nc && g >= 0);
          double* const* dst = d.L.state + 6 * __ldg(d.L.push_rank + q) + 3 * (cur ^ 1);
          dst[0][g] = sh[i];
          dst[1][g] = sq[i];
          dst[2][g] = sr[i];
        }
        __threadfence_system();
        __syncthreads();
      }
      ++j;
    }
    if (!viewed) {  // a CTA without tiles still follows the loop
      if (!read_view(it)) return;
      viewed = true;
    }
    const int par = (int)(step & 1);
    const Part bp = block_reduce_part_ret(a.lo, a.hi, a.mass, a.clip, a.ev,
                                          d.part + (size_t)par * nb + bid);
    // fold the CFL bound / max speed in (exact, order-independent), then
    // arrive (a release: this CTA's state, flags and partials are in L2)
    if (threadIdx.x == 0) {
      if (SWE_RUN_TIMING) {
        RUN_T(0, global_ns() - t_step);
        RUN_T(4, 1);
      }
      atomicMin(&sy->lo[par], (unsigned long long)__double_as_longlong(bp.lo));
      atomicMax(&sy->hi[par], (unsigned long long)__double_as_longlong(bp.hi));
      atom_add_release_gpu(&sy->arrive, 1u);
    }
    // every worker has arrived: the next state and its dry-tile flags are
    // complete.  Relaxed polls: the CTA reads them through L2 (ld.cg) until
    // its acquire of the epoch, which flushes L1 once per step
    if (threadIdx.x == 0) {
      const unsigned long long w0 = SWE_RUN_TIMING ? global_ns() : 0;
      poll_until(&sy->arrive, (unsigned)nb * (it + 1));
      if (SWE_RUN_TIMING) {
        t_step = global_ns();
        RUN_T(6, t_step - w0);
      }
    }
    __syncthreads();
    cur ^= 1;  // the next step, provisionally (confirmed by its epoch)
    step += 1;
  }
}

// swe_dev_cell_skip of a persistent context: the decisions k_run makes next
__global__ void k_cell_skip_run(Dev d, long long step, unsigned char* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d.C) return;
  const int* fl = d.pflag + (size_t)(step & 1) * d.ntiles;
  out[d.c_orig[c]] = (c < d.C_own && run_skip(d, fl, c / d.T, (int)(step + 1))) ? 1 : 0;
}

template <int NT, bool LINK>
__global__ void __launch_bounds__(NT, SWE_TILE_BLOCKS(NT)) k_run(Dev d, const Dev* dg) {
  const int nb = gridDim.x - 1;  // workers; the last block controls
  if ((int)blockIdx.x == nb) run_control<LINK>(dg, d.sync, nb);
  else run_body<NT, LINK>(d, dg, d.sync, blockIdx.x, nb);
}

// P linked ranks' persistent kernels as ONE cooperative launch on one device
// (blocks [r G, (r+1) G) run rank r): the ranks' CTAs spin on each other's
// mailboxes truly concurrently, which separate launches sharing a device
// cannot guarantee.  Test path for the linked exchange (B200_PROFILING.md).
template <int NT>
__global__ void __launch_bounds__(NT, SWE_TILE_BLOCKS(NT)) k_run_ranks(const Dev* devs, int G) {
  const Dev& d = devs[blockIdx.x / G];
  const int b = blockIdx.x % G, nb = G - 1;  // G - 1 workers and a control block per rank
  if (b == nb) run_control<true>(&d, d.sync, nb);
  else run_body<NT, true>(d, &d, d.sync, b, nb);
}

// ---------------------------------------------------------------------------
// staged tile kernel (option, SWE_TILE_STAGE=1): every contiguous input of a
// tile -- state, bed, area, n, r of its cells and the per-tile slot arrays
// (owned + halo edges copied in tile order at create) -- is brought into
// shared memory by one batch of cp.async copies, so a tile costs one memory
// round trip instead of several dependent ones.  128-cell tiles keep it at
// ~25 KB per CTA (8 CTAs/SM, as the default kernel).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__host__ __device__ constexpr size_t tile_stage_smem_bytes(int T, int S) {
  return sizeof(double) * (16 * (size_t)T + 3 * (size_t)S) + sizeof(int) * 3 * (size_t)S;
}

template <int NT, bool LINK>
__global__ void __launch_bounds__(NT, SWE_TILE_MINB * 256 / NT) k_tile_s(Dev d) {
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
  double* sa = sz + T;
  double* sm = sa + T;
  double* si = sm + T;
  double* tm = si + T;
  double* tx = tm + 3 * T;
  double* ty = tx + 3 * T;
  double* gnx = ty + 3 * T;
  double* gny = gnx + S;
  double* gln = gny + S;
  int* gel = reinterpret_cast<int*>(gln + S);
  int* ger = gel + S;
  int* gkk = ger + S;
  const Phys P = d.P;
  CellAcc a{INFINITY, 0.0, 0.0, 0.0, 0};

  for (int t = blockIdx.x; t < d.ntiles; t += gridDim.x) {
    const int c0 = t * T;
    SWE_CHECK(t >= 0 && t < d.ntiles && c0 < d.C_own);
    const int nc = min(T, d.C_own - c0);
    const int s0 = __ldg(d.soff + t), ns = __ldg(d.soff + t + 1) - s0;
    for (int i = threadIdx.x; i < nc; i += NT) {
      cp_async8(sh + i, H + c0 + i);
      cp_async8(sq + i, QX + c0 + i);
      cp_async8(sr + i, QY + c0 + i);
      cp_async8(sz + i, d.z + c0 + i);
      cp_async8(sa + i, d.area + c0 + i);
      cp_async8(sm + i, d.man + c0 + i);
      cp_async8(si + i, d.inr + c0 + i);
    }
    for (int j = threadIdx.x; j < ns; j += NT) {
      cp_async4(gel + j, d.sel + s0 + j);
      cp_async4(ger + j, d.ser + s0 + j);
      cp_async4(gkk + j, d.skk + s0 + j);
      cp_async8(gnx + j, d.snx + s0 + j);
      cp_async8(gny + j, d.sny + s0 + j);
      cp_async8(gln + j, d.slen + s0 + j);
    }
    int p0 = 0, p1 = 0;
    if (LINK) {
      p0 = __ldg(d.L.tile_push + t);
      p1 = __ldg(d.L.tile_push + t + 1);
    }
    cp_async_wait_all();
    __syncthreads();

    for (int j = threadIdx.x; j < ns; j += NT) {
      const int cl = gel[j], cr = ger[j];
      const double nx = gnx[j], ny = gny[j], len = gln[j];
      const bool w = cr < 0;
      const int il = cl - c0, ir = (w ? cl : cr) - c0;
      const bool inL = (unsigned)il < (unsigned)nc, inR = !w && (unsigned)ir < (unsigned)nc;
      Cons uL, uR;
      double zl, zr;
      if (inL) {
        uL = Cons{sh[il], sq[il], sr[il]};
        zl = sz[il];
      } else {
        uL = Cons{__ldg(H + cl), __ldg(QX + cl), __ldg(QY + cl)};
        zl = __ldg(d.z + cl);
      }
      if ((unsigned)ir < (unsigned)nc) {
        uR = Cons{sh[ir], sq[ir], sr[ir]};
        zr = sz[ir];
      } else {
        const int c = ir + c0;
        uR = Cons{__ldg(H + c), __ldg(QX + c), __ldg(QY + c)};
        zr = __ldg(d.z + c);
      }
      EdgeTerms et;
      if (!edge_terms(uL, zl, uR, zr, w, nx, ny, len, P, et)) {
        atomicMin(&ctl->bad_edge, __ldg(d.e_orig + __ldg(d.sedge + s0 + j)));
        continue;
      }
      const int kk = gkk[j];
      if (inL) {
        const int s = 3 * il + (kk & 0xff);
        tm[s] = et.lm;
        tx[s] = et.lx;
        ty[s] = et.ly;
      }
      if (inR) {
        const int s = 3 * ir + (kk >> 8);
        tm[s] = et.rm;
        tx[s] = et.rx;
        ty[s] = et.ry;
      }
    }
    __syncthreads();

    for (int i = threadIdx.x; i < nc; i += NT) {
      double am = 0.0, ax = 0.0, ay = 0.0;  // engine.hpp:255-264, local order k
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        am += tm[3 * i + k];
        ax += tx[3 * i + k];
        ay += ty[3 * i + k];
      }
      const Cons u = cell_finish_v(d, c0 + i, sh[i], sq[i], sr[i], am, ax, ay, dt, sa[i], sm[i],
                                   si[i], NH, NQX, NQY, a);
      if (LINK && p1 > p0) {
        sh[i] = u.h;
        sq[i] = u.qx;
        sr[i] = u.qy;
      }
    }
    __syncthreads();
    if (LINK && p1 > p0) {
      for (int j = p0 + threadIdx.x; j < p1; j += NT) {
        const int i = __ldg(d.L.push_cell + j) - c0, g = __ldg(d.L.push_ghost + j);
        SWE_CHECK(i >= 0 && i < nc && g >= 0);
        double* const* dst = d.L.state + 6 * __ldg(d.L.push_rank + j) + 3 * (cur ^ 1);
        dst[0][g] = sh[i];
        dst[1][g] = sq[i];
        dst[2][g] = sr[i];
      }
      __threadfence_system();
      __syncthreads();
    }
  }
  block_reduce_part(a.lo, a.hi, a.mass, a.clip, a.ev, d.part + blockIdx.x);
}

}  // namespace swe_b200
