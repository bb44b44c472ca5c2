// swe_ctl.cuh -- device control block, launch-sequence kernels and the
// fixed-order reductions of the explicit step (engine.hpp:179-216, :226-319,
// :355-380).  Included by swe_dev.cu only.
#pragma once

#include <climits>

#include "swe_dev.h"
#include "swe_phys.cuh"

namespace swe_b200 {

constexpr int kNone = INT_MAX;  // "no error index"
constexpr int kBlock = 256;     // threads per block of the step kernels

struct StepParams {  // written by the host before a launch sequence
  double t_end;
  long long max_steps;
  double next_snap;
  long long rec_cap;
  int ring;  // records wrap instead of stopping the loop
  int mode;  // 0 run loop, 1 single advance_step (no t/max_steps gate), 2 flux only
  long long add_steps;  // > 0: the gate sets max_steps = step + add_steps (exactly n steps)
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
  int link_err;  // a peer exchange timed out (sticky until set_state)
  unsigned long long xseq;  // exchanges posted so far (linked contexts)
  unsigned int done;        // blocks of the running step kernel that finished
  int tile_next;            // dynamic tile counter of k_tile (reset by finalize)
  unsigned long long skipped;  // dry tiles skipped by k_tile (cumulative)
  unsigned long long held;     // ... of which held: next state already in place, no writes
};

struct Part {  // one block's partial results
  double lo, hi, mass, clip;
  long long events;
  long long pad;
};

// ---------------------------------------------------------------------------
// Linked contexts (multi-device).  Every rank's state arrays and
// mailbox live in one device allocation (the arena) that its peers map (CUDA
// IPC across processes, plain pointers within one).  Per step:
//   k_tile   pushes the new state of the owned cells a peer holds as ghosts
//            straight into that peer's next state buffer (P2P stores);
//   k_post   posts the rank's step outcome (reduced CFL bound, speed, mass,
//            clip ledger, error) into every rank's mailbox slot, then
//            releases a flag;
//   k_wait   acquires all ranks' flags and combines the posts in rank order,
//            so every rank commits the same global dt, record and ledger.
// No host round trip: the whole loop stays in the CUDA graph.
// ---------------------------------------------------------------------------
constexpr int kMaxRanks = 64;

struct XPost {  // one rank's contribution to one exchange
  double lo, hi, mass, clip;
  long long events;
  unsigned long long tag;
  int status;     // local outcome of the step
  int index;      // global id of the offending edge / cell
  int bad_speed;  // global id of the lowest cell with a non-finite speed, or kNone
  int pad;
  double err_h;   // depth of the blown-up cell (BLOWUP)
};

struct XSums {  // one rank's deferred sums (persistent kernel: posted after the commit)
  double mass, clip;
  long long events;
  unsigned long long tag;
};

struct Mailbox {
  unsigned long long flag[kMaxRanks];  // flag[q]: last tag rank q posted here
  XPost slot[2][kMaxRanks];            // [tag & 1][q]
  unsigned long long dflag[kMaxRanks];  // dflag[q]: last tag of rank q's deferred sums
  XSums sums[2][kMaxRanks];
};

struct Link {
  int rank, nranks;  // nranks == 0: not linked
  Mailbox* mine;
  Mailbox* const* box;        // [nranks] every rank's mailbox, mapped here
  double* const* state;       // [6 * nranks] h0 qx0 qy0 h1 qx1 qy1 of every rank
  const int* tile_push;       // [ntiles + 1] push-list range of each tile
  const int* push_cell;       // device cell of each push entry (sorted)
  const int* push_rank;       // destination rank
  const int* push_ghost;      // ghost cell id on the destination rank
  const int* gcell;           // reference-local cell -> global id
  const int* gedge;           // reference-local edge -> global id
  unsigned long long timeout_ns;
};

// Step barrier of the persistent step kernel (k_run): CTAs count their
// arrivals at the end of every step (monotonic within a launch); the last to
// arrive commits the step and publishes it as the next epoch.  k_gate resets
// both before a launch.  One 128-byte line.
// the committed view the workers need to update a step: published by the
// control CTA as ONE 16-byte store after its commit, polled by the workers
// with one 16-byte load (epoch, stop flag and the step's dt together: one
// round trip instead of a poll and then the control block's fields)
struct __align__(16) View {
  unsigned int epoch;
  int active;
  double dt;
};

struct __align__(128) Sync {
  unsigned int arrive;
  View view;
  // the step's CFL bound and max speed (bits of non-negative doubles, so
  // integer atomicMin / atomicMax order them exactly), double-buffered by
  // step parity: min and max are order-independent, so the workers fold them
  // in at arrival and the commit needs no reduction on its critical path
  unsigned long long lo[2], hi[2];
  unsigned long long timing[12];  // SWE_RUN_TIMING builds
};

struct __align__(32) CellGeo {
  double z, area, man, inr;
};

struct Dev {
  int C, E;
  int C_own;  // cells [0, C_own) are owned (updated); [C_own, C) are ghosts of a multi-device run
  // halo exchange plan (device ids): owned cells to pack, ghost cells to unpack
  int n_send, n_recv;
  const int *send_cells, *recv_cells;
  // cells (device order)
  const double *area, *inr, *z, *man;
  const int *inc0, *inc1, *inc2;  // (device edge << 1) | (sign < 0), reference local order
  const int* c_orig;              // device cell -> reference cell
  const int* c_new;               // reference cell -> device cell
  // edges (device order: owner tile, walls last within a tile, lower cell)
  const int *el, *er;  // er < 0: reflective wall
  const double *nx, *ny, *len;
  const int* e_orig;
  const unsigned char *kl, *kr;  // local index k of the edge in its left / right cell
  // k_tile's edge records: ek = {el | kl << 30, er | kr << 30 (-1: wall)},
  // enxy = {nx, ny}; one 8 B and one 16 B load instead of six (fused path)
  const int2* ek;
  const double2* enxy;
  // k_tile's cell record {z, area, manning, inradius}: one 32 B load (fused path)
  const struct CellGeo* cg;
  // tiles of T consecutive cells (fused path)
  int T, ntiles, max_slots;  // max_slots: most edges (owned + halo) of one tile
  const int* eoff;  // [ntiles+1] owned edge range of each tile
  const int* hoff;  // [ntiles+1] halo list range of each tile
  const int* halo;  // halo edges (owned by another tile, touching this one)
  // staged tiles (k_tile_s): every slot (owned + halo edge) of every tile in
  // tile order, so a tile's slot data is one contiguous range [soff[t], soff[t+1])
  int stage;
  int dyn;  // k_tile fetches tiles from a counter instead of round robin
  // dry-tile skipping: dryflag[t] = tag of the state (step + 1) in which every
  // owned cell of tile t is dry and at rest (0 <= h < h_dry, q = 0), else 0;
  // skipmask[t] = that tag when tile t AND every tile holding its ring cells
  // carry it (nbr[nbr_off[t] .. nbr_off[t+1]); ntiles = a ghost cell of a
  // multi-device part: never skip)
  int skip;
  int* dryflag;
  int* skipmask;
  int2* streak;  // [ntiles] k_tile's consecutive skips (skip_code, swe_step.cuh)
  const int *nbr_off, *nbr;
  const int* soff;
  // persistent step kernel (k_run): barrier, double-buffered dry-tile flags
  // pflag[(step & 1) * ntiles + t] = tag of the state `step` if tile t is dry
  // and at rest in it (written during the previous step, read in this one),
  // tiles with an edge on a ghost cell (linked: they wait for the exchange)
  Sync* sync;
  int* pflag;
  const unsigned char* tile_ghost;
  int run_noacq;  // no L1-invalidating acquire per step (state via ld.cg only)
  const int *sel, *ser, *skk, *sedge;  // cells, kl | kr << 8, device edge (error path)
  const double *snx, *sny, *slen;
  // state, double-buffered
  double *h[2], *qx[2], *qy[2];
  // per-incidence contributions [3C] of the two-phase step
  double *TM, *TX, *TY;
  // edge records [E] of compute_fluxes
  double *M, *LX, *LY, *RX, *RY;
  // control
  Ctl* ctl;
  const StepParams* sp;
  Part* part;
  swe_step_record* rec;
  Phys P;
  Link L;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// relaxed (no L1 invalidation) poll; acquire fence (MEMBAR + CCTL.IVALL on
// sm_100) once the value is seen; release atomic add (MEMBAR, no IVALL)
__device__ __forceinline__ unsigned int ld_relaxed_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// wait until *p >= v: relaxed polls with exponential back-off (every CTA's
// thread 0 polls the same line; 20 ns polls made ~6M L2 requests per step
// at 10M cells and slowed every CTA's L2 traffic)
__device__ __forceinline__ void poll_until(const unsigned int* p, unsigned int v) {
  unsigned int ns = 32;
  while (ld_relaxed_gpu(p) < v) {
    __nanosleep(ns);
    ns = ns < 1024 ? 2 * ns : 1024;
  }
}

__device__ __forceinline__ void view_load(const View* v, unsigned int& epoch, int& active,
                                          double& dt) {
  unsigned long long a, b;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(v) : "memory");
  epoch = (unsigned int)a;
  active = (int)(a >> 32);
  dt = __longlong_as_double((long long)b);
}

// after a fence: the commit's stores are ordered before the view
__device__ __forceinline__ void view_publish(View* v, unsigned int epoch, int active, double dt) {
  const unsigned long long a =
      (unsigned long long)epoch | ((unsigned long long)(unsigned int)active << 32);
  const unsigned long long b = (unsigned long long)__double_as_longlong(dt);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(v), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned int atom_add_release_gpu(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// engine.hpp:236-237
__device__ __forceinline__ double step_dt(const Ctl* c, double t_end, bool* last_out) {
  const bool last = c->t + c->dts >= t_end;
  if (last_out) *last_out = last;
  return last ? t_end - c->t : c->dts;
}

// block reduction of per-thread partials in a fixed tree order
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
    for (int i = 1; i < (int)(blockDim.x / 32); ++i) {
      p.lo = sel_min(p.lo, s_lo[i]);
      p.hi = sel_max(p.hi, s_hi[i]);
      p.mass += s_m[i];
      p.clip += s_c[i];
      p.events += s_e[i];
    }
    *out = p;
  }
}

// block_reduce_part that also hands the block's partial to thread 0
__device__ __forceinline__ Part block_reduce_part_ret(double lo, double hi, double mass, double clip,
                                                      long long ev, Part* out) {
  __shared__ Part s_p;
  block_reduce_part(lo, hi, mass, clip, ev, &s_p);
  Part p{};
  if (threadIdx.x == 0) {
    p = s_p;
    *out = p;
  }
  return p;
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
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < d.C_own; c += stride) {
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

// fixed-order reduction of n block partials by one block: a tree of kBlock
// virtual lanes whatever blockDim.x is (k_finalize runs 256 threads, the
// persistent kernel's committing CTA 128), so every path forms the same sums
// in the same order; s: kBlock Parts of shared scratch.  Loads bypass L1 (the
// partials were written by other SMs of the same launch when called from a
// step kernel's last block).
__device__ Part reduce_parts_into(const Part* part, int n, Part* s) {
  for (int v = threadIdx.x; v < kBlock; v += blockDim.x) {
    Part p{INFINITY, 0.0, 0.0, 0.0, 0, 0};
    for (int base = v; base < n; base += 8 * kBlock) {
      Part q[8];  // 8 independent loads in flight, folded in index order
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = base + k * kBlock;
        if (i < n) {
          q[k].lo = __ldcg(&part[i].lo);
          q[k].hi = __ldcg(&part[i].hi);
          q[k].mass = __ldcg(&part[i].mass);
          q[k].clip = __ldcg(&part[i].clip);
          q[k].events = __ldcg(&part[i].events);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (base + k * kBlock < n) {
          p.lo = sel_min(p.lo, q[k].lo);
          p.hi = sel_max(p.hi, q[k].hi);
          p.mass += q[k].mass;
          p.clip += q[k].clip;
          p.events += q[k].events;
        }
      }
    }
    s[v] = p;
  }
  __syncthreads();
  for (int o = kBlock / 2; o > 0; o >>= 1) {
    for (int v = threadIdx.x; v < o; v += blockDim.x) {
      Part a = s[v];
      const Part b = s[v + o];
      a.lo = sel_min(a.lo, b.lo);
      a.hi = sel_max(a.hi, b.hi);
      a.mass += b.mass;
      a.clip += b.clip;
      a.events += b.events;
      s[v] = a;
    }
    __syncthreads();
  }
  return s[0];
}

__device__ Part reduce_parts(const Dev& d, int n) {
  __shared__ Part s[kBlock];
  return reduce_parts_into(d.part, n, s);
}

__device__ __forceinline__ void set_cfl_cache(Ctl* ctl, const Part& p, const Phys& P) {
  ctl->dts = isfinite(p.lo) ? P.cfl * p.lo : P.dt_max;  // engine.hpp:214
  ctl->max_speed = p.hi;
  ctl->mass = p.mass;
  ctl->cfl_bad = ctl->bad_speed;
  ctl->bad_speed = kNone;
  ctl->cfl_valid = 1;
}

// prepare: reduce k_cfl's n partials into the CFL cache
__global__ void __launch_bounds__(kBlock) k_prepare(Dev d, int n) {
  const Part p = reduce_parts(d, n);
  if (threadIdx.x == 0) set_cfl_cache(d.ctl, p, d.P);
}

__global__ void k_set_params(StepParams* sp, StepParams v) { *sp = v; }

// gate: opens a launch sequence (run() loop entry, engine.hpp:355-358)
__device__ __forceinline__ void gate(const Dev& d, cudaGraphConditionalHandle cond, int use_cond) {
  Ctl* c = d.ctl;
  StepParams* sp = const_cast<StepParams*>(d.sp);
  if (sp->add_steps > 0) {
    sp->max_steps = c->step + sp->add_steps;
    sp->add_steps = 0;
  }
  c->status = SWE_OK;
  c->n_rec = 0;
  if (d.sync) {  // the persistent kernel's barrier starts over with every launch
    d.sync->arrive = 0;
    d.sync->view.epoch = 0;
    for (int k = 0; k < 2; ++k) {
      d.sync->lo[k] = 0x7ff0000000000000ULL;  // +inf
      d.sync->hi[k] = 0ULL;                   // +0
    }
  }
  c->tile_next = 0;
  c->bad_edge = kNone;
  c->bad_cell = kNone;
  c->bad_speed = kNone;
  int go = sp->mode != 0 ||
           (c->t < sp->t_end && c->step < sp->max_steps && (sp->ring || sp->rec_cap > 0));
  if (go && sp->mode != 2 && c->cfl_bad != kNone) {  // stable_dt throws (engine.hpp:205-206)
    c->status = SWE_NONFINITE_SPEED;
    c->err_index = c->cfl_bad;
    go = 0;
  }
  if (go && sp->mode != 2 && c->link_err) {
    c->status = SWE_NCCL;
    c->err_index = -1;
    go = 0;
  }
  c->active = go;
  if (use_cond) cudaGraphSetConditional(cond, go);
}

__global__ void k_gate(Dev d, cudaGraphConditionalHandle cond, int use_cond) {
  gate(d, cond, use_cond);
}

// the step parameters and the gate in one launch (the persistent loop's prologue)
__global__ void k_gate_params(Dev d, StepParams v) {
  *const_cast<StepParams*>(d.sp) = v;
  gate(d, cudaGraphConditionalHandle{}, 0);
}

// Ctl through L2 (ld.cg): a step kernel's last block reads fields other
// blocks of the same launch updated with atomics, and its own SM may hold
// stale L1 lines of the block from the launch's start
static_assert(sizeof(Ctl) % 8 == 0, "Ctl is copied as 8-byte words");
__device__ __forceinline__ Ctl load_ctl(const Ctl* c) {
  Ctl v;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(c);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(&v);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Ctl) / 8); ++i) dst[i] = __ldcg(src + i);
  return v;
}

// write back the fields the committing thread owns.  The error slots
// bad_edge / bad_cell and the counters (skipped) are left alone: in the
// persistent kernel other CTAs may already be evaluating the next step's
// fluxes and atomicMin-ing bad_edge while the step is committed (a slot is
// only ever set by a failing step, which stops the loop; k_gate clears them)
__device__ __forceinline__ void store_commit(Ctl* g, const Ctl& c) {
  g->t = c.t;
  g->step = c.step;
  g->clipped = c.clipped;
  g->events = c.events;
  g->dts = c.dts;
  g->max_speed = c.max_speed;
  g->mass = c.mass;
  g->cfl_valid = c.cfl_valid;
  g->cfl_bad = c.cfl_bad;
  g->cur = c.cur;
  g->n_rec = c.n_rec;
  g->status = c.status;
  g->err_index = c.err_index;
  g->err_step = c.err_step;
  g->err_dt = c.err_dt;
  g->err_h = c.err_h;
  g->bad_speed = c.bad_speed;
  g->tile_next = c.tile_next;
  g->active = c.active;
}

// engine.hpp:292-307 + the fused CFL cache for the next step, given the
// step's reduced partials p and outcome (status, index, err_h).  One thread;
// works on a register copy of the control block (one batch of loads).
// the commit arithmetic on a control-block copy c (no global loads), in two
// parts: commit_head -- everything the NEXT step depends on (clock, buffer,
// CFL bound from the min / max lo, hi, stop decision) -- and commit_tail --
// the fixed-order sums (mass, clip ledger) and the step's record, which
// nothing in the next step reads.  k_finalize runs both back to back; the
// persistent kernel's control block publishes the step after the head.
struct CommitInfo {
  long long slot, step;
  double t, dt, max_speed_pre;
  int ok;
};

__device__ __forceinline__ int commit_head(Ctl& c, const StepParams& sp, double lo, double hi,
                                           int status, int index, double err_h, const Phys& P,
                                           CommitInfo& ci) {
  c.tile_next = 0;
  const bool last = c.t + c.dts >= sp.t_end;  // engine.hpp:236-237
  const double dt = last ? sp.t_end - c.t : c.dts;
  ci.ok = status == SWE_OK;
  if (status != SWE_OK) {  // engine.hpp:168-169, :292-297; state is not committed
    c.status = status;
    c.err_index = index;
    if (status == SWE_BLOWUP) {
      c.err_step = c.step;
      c.err_dt = dt;
      c.err_h = err_h;
    }
    c.bad_speed = kNone;
    c.active = 0;
    return 0;
  }
  // commit (engine.hpp:300-307)
  ci.max_speed_pre = c.max_speed;
  c.cur ^= 1;
  c.t = last ? sp.t_end : c.t + dt;
  c.step += 1;
  ci.slot = sp.ring ? (c.n_rec % sp.rec_cap) : c.n_rec;
  ci.step = c.step;
  ci.t = c.t;
  ci.dt = dt;
  c.n_rec += 1;
  // set_cfl_cache without the mass (engine.hpp:214)
  c.dts = isfinite(lo) ? P.cfl * lo : P.dt_max;
  c.max_speed = hi;
  c.cfl_bad = c.bad_speed;
  c.bad_speed = kNone;
  c.cfl_valid = 1;
  // continue? (engine.hpp:355-358, :374-375)
  int go = c.t < sp.t_end && c.step < sp.max_steps && !(c.t >= sp.next_snap - 1e-12) &&
           (sp.ring || c.n_rec < sp.rec_cap);
  if (go && c.cfl_bad != kNone) {
    c.status = SWE_NONFINITE_SPEED;
    c.err_index = c.cfl_bad;
    go = 0;
  }
  c.active = go;
  return go;
}

__device__ __forceinline__ void commit_tail(Ctl& c, const StepParams& sp, const Part& p,
                                            const CommitInfo& ci, swe_step_record* rec) {
  if (!ci.ok) return;
  c.clipped += p.clip;
  c.events += p.events;
  c.mass = p.mass;
  if (ci.slot < sp.rec_cap) {
    swe_step_record r;
    r.step = ci.step;
    r.t = ci.t;
    r.dt = ci.dt;
    r.max_speed = ci.max_speed_pre;
    r.mass = p.mass;
    rec[ci.slot] = r;
  }
}

__device__ __forceinline__ int commit_core(Ctl& c, const StepParams& sp, const Part& p, int status,
                                           int index, double err_h, const Phys& P,
                                           swe_step_record* rec) {
  CommitInfo ci;
  const int go = commit_head(c, sp, p.lo, p.hi, status, index, err_h, P, ci);
  commit_tail(c, sp, p, ci, rec);
  return go;
}

__device__ void finalize_step(const Dev& d, const Part& p, int status, int index, double err_h,
                              cudaGraphConditionalHandle cond, int use_cond) {
  Ctl c = load_ctl(d.ctl);
  const StepParams sp = *d.sp;
  const int go = commit_core(c, sp, p, status, index, err_h, d.P, d.rec);
  store_commit(d.ctl, c);
  if (use_cond) cudaGraphSetConditional(cond, go);
}

// single-domain step outcome from the reduced partials p (thread 0)
__device__ void finalize_local(const Dev& d, const Part& p, cudaGraphConditionalHandle cond,
                               int use_cond) {
  const Ctl c = load_ctl(d.ctl);
  int status = SWE_OK, index = kNone;
  double err_h = 0.0;
  if (c.bad_edge != kNone) {  // engine.hpp:168-169
    status = SWE_NEGATIVE_DEPTH;
    index = c.bad_edge;
  } else if (c.bad_cell != kNone) {  // engine.hpp:292-297
    status = SWE_BLOWUP;
    index = c.bad_cell;
    err_h = d.h[c.cur ^ 1][d.c_new[c.bad_cell]];
  }
  finalize_step(d, p, status, index, err_h, cond, use_cond);
}

// ---- linked contexts: post / wait (see Link) ------------------------------
// Executed by one full warp: lane q serves ranks q, q+32, ...
// kind 0: a step's outcome (partials of the step kernel, error slots);
// kind 1: the CFL bound of the current state (partials of k_cfl).
__device__ void post_outcome(const Dev& d, const Part& p, int kind) {
  const int lane = threadIdx.x & 31;
  const Ctl c = load_ctl(d.ctl);
  const Link& L = d.L;
  XPost x;
  x.lo = p.lo;
  x.hi = p.hi;
  x.mass = p.mass;
  x.clip = p.clip;
  x.events = p.events;
  x.status = SWE_OK;
  x.index = kNone;
  x.err_h = 0.0;
  x.pad = 0;
  if (kind == 0 && c.bad_edge != kNone) {
    x.status = SWE_NEGATIVE_DEPTH;
    x.index = L.gedge[c.bad_edge];
  } else if (kind == 0 && c.bad_cell != kNone) {
    x.status = SWE_BLOWUP;
    x.index = L.gcell[c.bad_cell];
    x.err_h = d.h[c.cur ^ 1][d.c_new[c.bad_cell]];
  }
  x.bad_speed = c.bad_speed == kNone ? kNone : L.gcell[c.bad_speed];
  const unsigned long long tag = c.xseq + 1;
  x.tag = tag;
  __syncwarp();
  if (lane == 0) {  // (bad_edge / bad_cell only fail a step: see store_commit)
    d.ctl->bad_speed = kNone;
    d.ctl->xseq = tag;
  }
  // the step kernel's halo pushes were fenced at system scope by their
  // writers; this lane's slot write is ordered before its flag by the release
  for (int q = lane; q < L.nranks; q += 32) {
    L.box[q]->slot[tag & 1][L.rank] = x;
    st_release_sys(&L.box[q]->flag[L.rank], tag);
  }
  __syncwarp();
}

// wait for every rank's post of exchange `tag` and combine them in rank order
// (one warp; every lane ends with the same result)
struct XCombined {
  Part g;
  int neg, blow, bad;
  double err_h;
  bool timeout;
};

__device__ XCombined wait_combine(const Dev& d, unsigned long long tag) {
  const int lane = threadIdx.x & 31;
  const Link& L = d.L;
  Mailbox* m = L.mine;
  const unsigned long long t0 = global_ns();
  bool timeout = false;
  for (int q = lane; q < L.nranks && !timeout; q += 32)
    while (ld_acquire_sys(&m->flag[q]) < tag) {
      if (global_ns() - t0 > L.timeout_ns) {
        timeout = true;
        break;
      }
      __nanosleep(64);
    }
  // combine in rank order: every rank forms the same sums
  XCombined r;
  r.g = Part{INFINITY, 0.0, 0.0, 0.0, 0, 0};
  r.neg = kNone;
  r.blow = kNone;
  r.bad = kNone;
  r.err_h = 0.0;
  for (int base = 0; base < L.nranks; base += 32) {
    const int q = base + lane;
    XPost s{};
    if (q < L.nranks && !timeout) {
      const volatile XPost* v = &m->slot[tag & 1][q];
      s.lo = v->lo;
      s.hi = v->hi;
      s.mass = v->mass;
      s.clip = v->clip;
      s.events = v->events;
      s.tag = v->tag;
      s.status = v->status;
      s.index = v->index;
      s.bad_speed = v->bad_speed;
      s.err_h = v->err_h;
      if (s.tag != tag) timeout = true;  // a post from a different exchange
    }
    const int cnt = min(32, L.nranks - base);
    for (int j = 0; j < cnt; ++j) {  // fold lane j's post (rank base + j)
      const double lo = __shfl_sync(0xffffffffu, s.lo, j);
      const double hi = __shfl_sync(0xffffffffu, s.hi, j);
      const double ms = __shfl_sync(0xffffffffu, s.mass, j);
      const double cl = __shfl_sync(0xffffffffu, s.clip, j);
      const long long ev = __shfl_sync(0xffffffffu, s.events, j);
      const int st = __shfl_sync(0xffffffffu, s.status, j);
      const int ix = __shfl_sync(0xffffffffu, s.index, j);
      const int bs = __shfl_sync(0xffffffffu, s.bad_speed, j);
      const double eh = __shfl_sync(0xffffffffu, s.err_h, j);
      r.g.lo = sel_min(r.g.lo, lo);
      r.g.hi = sel_max(r.g.hi, hi);
      r.g.mass += ms;
      r.g.clip += cl;
      r.g.events += ev;
      if (st == SWE_NEGATIVE_DEPTH) r.neg = min(r.neg, ix);
      if (st == SWE_BLOWUP && ix < r.blow) {
        r.blow = ix;
        r.err_h = eh;
      }
      r.bad = min(r.bad, bs);
    }
  }
  r.timeout = __any_sync(0xffffffffu, timeout);
  return r;
}

__device__ __forceinline__ void link_timeout(Ctl* c) {
  c->link_err = 1;
  c->status = SWE_NCCL;
  c->err_index = -1;
  c->active = 0;
  c->cfl_valid = 0;
}

// wait for every rank's post, combine in rank order, commit (one warp)
__device__ void wait_and_commit(const Dev& d, int kind, cudaGraphConditionalHandle cond,
                                int use_cond) {
  const int lane = threadIdx.x & 31;
  const XCombined r = wait_combine(d, __ldcg(&d.ctl->xseq));
  if (lane != 0) return;
  Ctl* c = d.ctl;
  if (r.timeout) {
    link_timeout(c);
    if (use_cond) cudaGraphSetConditional(cond, 0);
    return;
  }
  c->bad_speed = r.bad;
  if (kind == 1) {
    Ctl v = load_ctl(c);
    set_cfl_cache(&v, r.g, d.P);
    *c = v;
    return;
  }
  const int status =
      r.neg != kNone ? SWE_NEGATIVE_DEPTH : (r.blow != kNone ? SWE_BLOWUP : SWE_OK);
  finalize_step(d, r.g, status, status == SWE_NEGATIVE_DEPTH ? r.neg : r.blow, r.err_h, cond,
                use_cond);
}

// ---- the persistent kernel's split exchange (linked ranks) -----------------
// The step's commit needs only the CFL bound, the max speed and the error
// slots: the control CTA posts those as soon as its workers have arrived
// (bound and speed folded in by the workers' atomics), commits the head
// (clock, buffer, stop) from the combined posts and publishes it; the mass /
// clip sums follow in a second post (sums[], dflag[]) once reduced, and the
// record / ledger are completed from their rank-order combination.

// the head: wait + combine the critical posts, commit_head (warp 0; lane 0
// holds go and ci).  Returns go (0 on timeout: the loop stops)
__device__ int wait_commit_head(const Dev& d, const StepParams& sp, CommitInfo& ci, bool& tmo) {
  const int lane = threadIdx.x & 31;
  const XCombined r = wait_combine(d, __ldcg(&d.ctl->xseq));
  tmo = r.timeout;
  int go = 0;
  if (lane == 0) {
    if (r.timeout) {
      link_timeout(d.ctl);
      ci.ok = false;
    } else {
      Ctl c = load_ctl(d.ctl);
      c.bad_speed = r.bad;
      const int status =
          r.neg != kNone ? SWE_NEGATIVE_DEPTH : (r.blow != kNone ? SWE_BLOWUP : SWE_OK);
      go = commit_head(c, sp, r.g.lo, r.g.hi, status,
                       status == SWE_NEGATIVE_DEPTH ? r.neg : r.blow, r.err_h, d.P, ci);
      store_commit(d.ctl, c);
    }
  }
  return __shfl_sync(0xffffffffu, go, 0);
}

// the tail: post this rank's sums, wait for every rank's, combine in rank
// order, complete the record and the ledger (warp 0).  Returns 0 on timeout.
__device__ int post_wait_sums(const Dev& d, const StepParams& sp, const Part& p,
                              const CommitInfo& ci) {
  const int lane = threadIdx.x & 31;
  const Link& L = d.L;
  const unsigned long long tag = __ldcg(&d.ctl->xseq);
  XSums x;
  x.mass = p.mass;
  x.clip = p.clip;
  x.events = p.events;
  x.tag = tag;
  __syncwarp();
  for (int q = lane; q < L.nranks; q += 32) {
    L.box[q]->sums[tag & 1][L.rank] = x;
    st_release_sys(&L.box[q]->dflag[L.rank], tag);
  }
  Mailbox* m = L.mine;
  const unsigned long long t0 = global_ns();
  bool timeout = false;
  for (int q = lane; q < L.nranks && !timeout; q += 32)
    while (ld_acquire_sys(&m->dflag[q]) < tag) {
      if (global_ns() - t0 > L.timeout_ns) {
        timeout = true;
        break;
      }
      __nanosleep(64);
    }
  Part g{INFINITY, 0.0, 0.0, 0.0, 0, 0};
  for (int base = 0; base < L.nranks; base += 32) {
    const int q = base + lane;
    double ms = 0.0, cl = 0.0;
    long long ev = 0;
    if (q < L.nranks && !timeout) {
      const volatile XSums* v = &m->sums[tag & 1][q];
      ms = v->mass;
      cl = v->clip;
      ev = v->events;
      if (v->tag != tag) timeout = true;
    }
    const int cnt = min(32, L.nranks - base);
    for (int j = 0; j < cnt; ++j) {
      g.mass += __shfl_sync(0xffffffffu, ms, j);
      g.clip += __shfl_sync(0xffffffffu, cl, j);
      g.events += __shfl_sync(0xffffffffu, ev, j);
    }
  }
  timeout = __any_sync(0xffffffffu, timeout);
  if (lane == 0) {
    if (timeout) {
      link_timeout(d.ctl);
    } else if (ci.ok) {
      Ctl c = load_ctl(d.ctl);
      commit_tail(c, sp, g, ci, d.rec);
      d.ctl->clipped = c.clipped;
      d.ctl->events = c.events;
      d.ctl->mass = c.mass;
    }
  }
  return timeout ? 0 : 1;
}

// skip mask of tile u for the next step (blocks >= 1 of the finalize /
// exchange / post launch, one thread per tile; reads the flags k_tile wrote)
__device__ __forceinline__ bool skip_mask_blocks(const Dev& d) {
  if (blockIdx.x == 0) return false;
  const int u = (blockIdx.x - 1) * blockDim.x + threadIdx.x;
  if (d.skip && u < d.ntiles) {
    const int f = d.dryflag[u];
    const int v0 = d.nbr_off[u], v1 = d.nbr_off[u + 1];
    int ok = f != 0;
    // no early exit: the neighbour loads are independent and issue together
#pragma unroll 4
    for (int v = v0; v < v1; ++v) {
      const int nb = d.nbr[v];
      const int fl = nb < d.ntiles ? d.dryflag[nb] : 0;
      ok &= fl == f ? 1 : 0;
    }
    // a tile whose cells peers hold as ghosts is computed, never skipped: its
    // halo pushes run on the computed path (computing it is exact anyway)
    if (d.L.nranks > 0 && d.L.tile_push[u + 1] > d.L.tile_push[u]) ok = 0;
    d.skipmask[u] = ok ? f : 0;
  }
  return true;
}

// kernel forms
__global__ void __launch_bounds__(kBlock) k_finalize(Dev d, int n, cudaGraphConditionalHandle cond,
                                                     int use_cond) {
  if (skip_mask_blocks(d)) return;
  if (!d.ctl->active) {
    if (threadIdx.x == 0 && use_cond) cudaGraphSetConditional(cond, 0);
    return;
  }
  const Part p = reduce_parts(d, n);
  if (threadIdx.x == 0) finalize_local(d, p, cond, use_cond);
}

__global__ void __launch_bounds__(kBlock) k_post(Dev d, int n, int kind) {
  if (skip_mask_blocks(d)) return;
  if (kind == 0 && !d.ctl->active) return;
  const Part p = reduce_parts(d, n);
  if (threadIdx.x < 32) post_outcome(d, p, kind);
}

// post + wait in one launch (the graph / plain path of a linked context)
__global__ void __launch_bounds__(kBlock) k_exchange(Dev d, int n, int kind,
                                                     cudaGraphConditionalHandle cond, int use_cond) {
  if (skip_mask_blocks(d)) return;
  if (kind == 0 && !d.ctl->active) {
    if (threadIdx.x == 0 && use_cond) cudaGraphSetConditional(cond, 0);
    return;
  }
  const Part p = reduce_parts(d, n);
  if (threadIdx.x >= 32) return;
  post_outcome(d, p, kind);
  wait_and_commit(d, kind, cond, use_cond);
}

__global__ void k_wait(Dev d, int kind, cudaGraphConditionalHandle cond, int use_cond) {
  if (kind == 0 && !d.ctl->active) {
    if (use_cond) cudaGraphSetConditional(cond, 0);
    return;
  }
  wait_and_commit(d, kind, cond, use_cond);
}

}  // namespace swe_b200
