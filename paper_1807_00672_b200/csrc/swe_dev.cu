// swe_dev.cu -- B200 (sm_100a) explicit HLLC shallow-water step behind the
// C-ABI of include/swe_dev.h (host side: context, device preprocessor driver,
// CUDA graph of the time loop).  Kernels: swe_step.cuh (step), swe_ctl.cuh
// (gate / reductions / finalize), swe_prep.cuh (renumbering, tile tables).
//
// Step (reference: /root/reference/proj/include/swe/engine.hpp:226-319):
//   default   k_tile (fused flux + update per Morton tile) -> k_finalize
//   two-phase k_face (edge records to HBM) -> k_cell -> k_finalize
// k_finalize commits the step, reduces the CFL bound and mass the update
// kernel produced for the NEXT step, and sets the loop condition.  run()'s loop
// (engine.hpp:355-380) is one CUDA graph launch: k_gate + a conditional WHILE
// node over the step.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "swe_build.cuh"
#include "swe_ctl.cuh"
#include "swe_dev.h"
#include "swe_prep.cuh"
#include "swe_step.cuh"

using namespace swe_b200;

namespace {

thread_local std::string g_last_error;
long long g_launches = 0;

bool cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}

#define CK(call)                                  \
  do {                                            \
    if (!cuda_ok((call), #call)) return SWE_CUDA; \
  } while (0)

int blocks_for(long long n, int b = kBlock) { return (int)((n + b - 1) / b); }

// arena layout: [Mailbox][h0][qx0][qy0][h1][qx1][qy1], 256-byte aligned;
// arena_offset(C, k) = byte offset of state array k (k = 6: total size)
size_t arena_offset(long long C, int k) {
  const size_t box = (sizeof(Mailbox) + 255) & ~(size_t)255;
  const size_t arr = ((size_t)C * sizeof(double) + 255) & ~(size_t)255;
  return box + (size_t)k * arr;
}

// run loop choice by owned cells: the persistent kernel up to
// here, the CUDA graph above.  (Linked parts too: the persistent kernel's
// split exchange costs +1 us per step against the graph's +4.6 us at 1.28M
// cells, but the 10M channel's measured-cost parts step slower on it:
// 0.0845 vs 0.0768 ms at N = 8, profiles/r02_scaling_proxy_*.)
constexpr int kPersistentMaxCells = 600000;

int fail_invalid(const char* msg) {
  g_last_error = msg;
  return SWE_INVALID;
}

}  // namespace

struct swe_dev_ctx {
  int device = 0;
  unsigned flags = 0;
  bool fused = true;
  cudaStream_t stream = nullptr;
  Dev d{};
  std::vector<void*> allocs;
  long long bytes = 0;
  Ctl* ctl = nullptr;          // device
  StepParams* sp = nullptr;    // device
  Ctl* h_ctl = nullptr;        // pinned host mirror
  swe_step_record* rec = nullptr;
  long long rec_cap = 0;
  double *stage_h = nullptr, *stage_qx = nullptr, *stage_qy = nullptr;
  int grid_face = 0, grid_cell = 0, grid_tile = 0;
  int tile_threads = 128;  // measured best with 256-cell tiles
  int* halo_send = nullptr;  // device ids of the halo plan
  int* halo_recv = nullptr;
  size_t tile_smem = 0;
  int max_slots = 0;  // most edges (owned + halo) one tile evaluates
  long long n_halo = 0;
  // linked contexts (multi-device)
  char* arena = nullptr;  // mailbox + state arrays, mapped by the peers
  size_t arena_bytes = 0;
  bool linked = false;
  bool cfl_posted = false;  // link_phase: a CFL exchange awaits its wait
  bool cfl_host_valid = false;  // the device CFL cache is known valid (no sync needed)
  int graph_unroll = 8;         // steps per WHILE iteration of the graph (SWE_GRAPH_UNROLL)
  bool persistent = false;      // run loop = one cooperative k_run launch (SWE_PERSISTENT=0: graph)
  Dev* d_dev = nullptr;         // device copy of d for k_run's commit path
  Dev d_dev_host{};             // what d_dev holds
  bool d_dev_valid = false;
  int grid_run = 0;             // CTAs of k_run (= grid_tile when the occupancies agree)
  std::vector<void*> link_allocs;  // device tables of the link
  std::vector<void*> ipc_mapped;   // peers' arenas opened through CUDA IPC
  // asynchronous snapshots: device staging slots, copy stream, events
  double* snap[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t snap_ready[2] = {nullptr, nullptr}, snap_done[2] = {nullptr, nullptr};
  // state transfers: one event per array + one for the main stream's position
  cudaStream_t xfer_stream = nullptr;
  cudaEvent_t xfer_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // graph
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond{};
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> events;
  double kms[4] = {0, 0, 0, 0};
  long long klaunch[4] = {0, 0, 0, 0};

  template <class V>
  V* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, n * sizeof(V) + 16) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    bytes += (long long)(n * sizeof(V));
    return static_cast<V*>(p);
  }
  int n_step_parts() const { return fused ? grid_tile : grid_cell; }
  int n_push = 0;
};

namespace {

const void* tile_kernel(int threads, bool link, bool stage = false) {
  if (stage) {
    if (threads == 128)
      return link ? (const void*)k_tile_s<128, true> : (const void*)k_tile_s<128, false>;
    return link ? (const void*)k_tile_s<256, true> : (const void*)k_tile_s<256, false>;
  }
  if (threads == 128) return link ? (const void*)k_tile<128, true> : (const void*)k_tile<128, false>;
  return link ? (const void*)k_tile<256, true> : (const void*)k_tile<256, false>;
}

// the step kernel(s) before finalize
int launch_update(swe_dev_ctx* x) {
  if (x->fused) {
    const bool L = x->linked;
    const int g = x->grid_tile;
    const size_t sm = x->tile_smem;
    if (x->d.stage) {
      if (x->tile_threads == 128) {
        if (L) k_tile_s<128, true><<<g, 128, sm, x->stream>>>(x->d);
        else k_tile_s<128, false><<<g, 128, sm, x->stream>>>(x->d);
      } else {
        if (L) k_tile_s<256, true><<<g, 256, sm, x->stream>>>(x->d);
        else k_tile_s<256, false><<<g, 256, sm, x->stream>>>(x->d);
      }
      ++g_launches;
      return cuda_ok(cudaGetLastError(), "k_tile_s") ? SWE_OK : SWE_CUDA;
    }
    if (x->tile_threads == 128) {
      if (L) k_tile<128, true><<<g, 128, sm, x->stream>>>(x->d);
      else k_tile<128, false><<<g, 128, sm, x->stream>>>(x->d);
    } else {
      if (L) k_tile<256, true><<<g, 256, sm, x->stream>>>(x->d);
      else k_tile<256, false><<<g, 256, sm, x->stream>>>(x->d);
    }
    ++g_launches;
    return cuda_ok(cudaGetLastError(), "k_tile") ? SWE_OK : SWE_CUDA;
  }
  k_face_c<<<x->grid_face, kBlock, 0, x->stream>>>(x->d);
  k_cell_c<<<x->grid_cell, kBlock, 0, x->stream>>>(x->d);
  g_launches += 2;
  if (x->linked) {
    k_push<<<blocks_for(std::max(1, x->n_push)), kBlock, 0, x->stream>>>(x->d);
    ++g_launches;
  }
  return cuda_ok(cudaGetLastError(), "k_face_c/k_cell_c") ? SWE_OK : SWE_CUDA;
}

// linked: post this rank's outcome / CFL bound, then wait for every rank's
// extra blocks of the launch after the step kernel: the next step's skip mask
int mask_blocks(const swe_dev_ctx* x) { return x->d.skip ? blocks_for(x->d.ntiles) : 0; }

int launch_post(swe_dev_ctx* x, int n, int kind) {
  k_post<<<1 + (kind == 0 ? mask_blocks(x) : 0), kBlock, 0, x->stream>>>(x->d, n, kind);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_post") ? SWE_OK : SWE_CUDA;
}

int launch_wait(swe_dev_ctx* x, int kind, cudaGraphConditionalHandle h, int use_cond) {
  k_wait<<<1, 32, 0, x->stream>>>(x->d, kind, h, use_cond);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_wait") ? SWE_OK : SWE_CUDA;
}

int launch_exchange(swe_dev_ctx* x, int n, int kind, cudaGraphConditionalHandle h, int use_cond) {
  k_exchange<<<1 + (kind == 0 ? mask_blocks(x) : 0), kBlock, 0, x->stream>>>(x->d, n, kind, h,
                                                                            use_cond);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_exchange") ? SWE_OK : SWE_CUDA;
}

int launch_finalize(swe_dev_ctx* x, cudaGraphConditionalHandle h, int use_cond) {
  if (x->linked) return launch_exchange(x, x->n_step_parts(), 0, h, use_cond);
  k_finalize<<<1 + mask_blocks(x), kBlock, 0, x->stream>>>(x->d, x->n_step_parts(), h, use_cond);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_finalize") ? SWE_OK : SWE_CUDA;
}

int launch_gate(swe_dev_ctx* x) {
  k_gate<<<1, 1, 0, x->stream>>>(x->d, cudaGraphConditionalHandle{}, 0);
  ++g_launches;
  return cuda_ok(cudaGetLastError(), "k_gate") ? SWE_OK : SWE_CUDA;
}

const void* run_kernel(int threads, bool link) {
  if (threads == 128) return link ? (const void*)k_run<128, true> : (const void*)k_run<128, false>;
  return link ? (const void*)k_run<256, true> : (const void*)k_run<256, false>;
}

// the run loop as one cooperative launch of the persistent step kernel,
// after its prologue (step parameters + gate in one launch)
int launch_run(swe_dev_ctx* x, const StepParams& v) {
  k_gate_params<<<1, 1, 0, x->stream>>>(x->d, v);
  ++g_launches;
  CK(cudaGetLastError());
  Dev dcopy = x->d;
  // the commit path reads the context's Dev from global memory (stream-ordered
  // copy, only when it changed: a pageable copy costs ~10 us per launch)
  if (!x->d_dev_valid || std::memcmp(&x->d_dev_host, &x->d, sizeof(Dev)) != 0) {
    CK(cudaMemcpyAsync(x->d_dev, &x->d, sizeof(Dev), cudaMemcpyHostToDevice, x->stream));
    x->d_dev_host = x->d;
    x->d_dev_valid = true;
  }
  const Dev* dg = x->d_dev;
  void* args[] = {&dcopy, &dg};
  CK(cudaLaunchCooperativeKernel(run_kernel(x->tile_threads, x->linked), dim3(x->grid_run),
                                 dim3(x->tile_threads), args, x->tile_smem, x->stream));
  ++g_launches;
  return SWE_OK;
}

int sync_ctl(swe_dev_ctx* x) {
  CK(cudaMemcpyAsync(x->h_ctl, x->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  return SWE_OK;
}

// CFL cache of the current state if stale (after set_state)
// (no host sync when the host already knows the cache is valid: the step
// kernels keep it valid; set_state / link invalidate it)
int ensure_cfl(swe_dev_ctx* x, bool force = false) {
  if (x->cfl_host_valid && !force) return SWE_OK;
  if (int rc = sync_ctl(x)) return rc;
  if (x->h_ctl->cfl_valid && !force) {
    x->cfl_host_valid = true;
    return SWE_OK;
  }
  k_cfl<<<x->grid_cell, kBlock, 0, x->stream>>>(x->d);
  ++g_launches;
  x->cfl_host_valid = true;
  if (x->linked)  // the global bound: every rank posts, then waits
    return launch_exchange(x, x->grid_cell, 1, cudaGraphConditionalHandle{}, 0);
  k_prepare<<<1, kBlock, 0, x->stream>>>(x->d, x->grid_cell);
  ++g_launches;
  CK(cudaGetLastError());
  return SWE_OK;
}

// step parameters travel as a kernel argument (captured at launch: no
// host buffer to race with when launches are only enqueued)
StepParams make_params(double t_end, long long max_steps, double next_snap, long long rec_cap,
                       int ring, int mode = 0, long long add_steps = 0) {
  StepParams v;
  v.add_steps = add_steps;
  v.t_end = t_end;
  v.max_steps = max_steps;
  v.next_snap = next_snap;
  v.rec_cap = rec_cap;
  v.ring = ring;
  v.mode = mode;
  return v;
}

int write_params(swe_dev_ctx* x, double t_end, long long max_steps, double next_snap,
                 long long rec_cap, int ring, int mode = 0, long long add_steps = 0) {
  StepParams v;
  v.add_steps = add_steps;
  v.t_end = t_end;
  v.max_steps = max_steps;
  v.next_snap = next_snap;
  v.rec_cap = rec_cap;
  v.ring = ring;
  v.mode = mode;
  k_set_params<<<1, 1, 0, x->stream>>>(x->sp, v);
  ++g_launches;
  CK(cudaGetLastError());
  return SWE_OK;
}

int read_status(swe_dev_ctx* x, swe_status* st) {
  if (int rc = sync_ctl(x)) return rc;
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
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = x->cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wnode;
  CK(cudaGraphAddNode(&wnode, x->graph, &gate, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(x->stream, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  const long long before = g_launches;
  // the WHILE body holds `graph_unroll` steps: a step that finds the loop
  // stopped exits at once, and the conditional node's per-iteration cost
  // (~2-3 us) is shared (measured 1 -> 4 steps: -0.8% at 10M cells, -7% at 1M,
  // -19% at 10k; 4 -> 8: -0.5%, -1.5%, -4%; an advance() that stops mid-body
  // pays <= 7 no-op step pairs, ~2.5 us each)
  for (int u = 0; u < x->graph_unroll; ++u) {
    launch_update(x);
    launch_finalize(x, x->cond, 1);
  }
  g_launches = before;  // captured, not launched
  cudaGraph_t captured = nullptr;
  CK(cudaStreamEndCapture(x->stream, &captured));
  CK(cudaGraphInstantiate(&x->exec, x->graph, 0));
  return SWE_OK;
}

// ---------------------------------------------------------------------------
// device preprocessor driver
// ---------------------------------------------------------------------------
struct Temps {
  std::vector<void*> p;
  void* get(size_t bytes) {
    void* q = nullptr;
    if (cudaMalloc(&q, bytes + 16) != cudaSuccess) return nullptr;
    p.push_back(q);
    return q;
  }
  ~Temps() {
    for (void* q : p) cudaFree(q);
  }
};

template <class K, class V>
bool radix_sort(Temps& tmp, const K* kin, K* kout, const V* vin, V* vout, int n, int end_bit,
                cudaStream_t s) {
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, end_bit, s);
  void* store = tmp.get(tb);
  return store && cuda_ok(cub::DeviceRadixSort::SortPairs(store, tb, kin, kout, vin, vout, n, 0,
                                                          end_bit, s),
                          "cub radix sort");
}

template <class K>
bool radix_sort_keys(Temps& tmp, const K* kin, K* kout, int n, int end_bit, cudaStream_t s) {
  size_t tb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, kin, kout, n, 0, end_bit, s);
  void* store = tmp.get(tb);
  return store && cuda_ok(cub::DeviceRadixSort::SortKeys(store, tb, kin, kout, n, 0, end_bit, s),
                          "cub radix sort (keys)");
}

int bits_for(long long v) {
  int b = 1;
  while ((1LL << b) <= v) ++b;
  return b;
}

// dry-tile skipping: per tile the distinct tiles holding its ring cells
int build_tile_neighbours(swe_dev_ctx* x) {
  Dev& d = x->d;
  cudaStream_t s = x->stream;
  Temps tmp;
  const long long np = 2 * ((long long)d.E + x->n_halo);
  auto* k0 = (unsigned long long*)tmp.get(8 * (size_t)std::max(1LL, np));
  auto* k1 = (unsigned long long*)tmp.get(8 * (size_t)std::max(1LL, np));
  auto* k2 = (unsigned long long*)tmp.get(8 * (size_t)std::max(1LL, np));
  int* nsel = (int*)tmp.get(sizeof(int));
  if (!k0 || !k1 || !k2 || !nsel) return fail_invalid("dry-skip tables: cudaMalloc failed"), SWE_CUDA;
  k_tile_pairs<<<blocks_for(32LL * d.ntiles), kBlock, 0, s>>>(d, k0);
  if (!radix_sort_keys(tmp, k0, k1, (int)np, 32 + bits_for(d.ntiles + 1), s)) return SWE_CUDA;
  size_t tb = 0;
  cub::DeviceSelect::Unique(nullptr, tb, k1, k2, nsel, (int)np, s);
  void* store = tmp.get(tb);
  if (!store || !cuda_ok(cub::DeviceSelect::Unique(store, tb, k1, k2, nsel, (int)np, s), "unique"))
    return SWE_CUDA;
  int nu = 0;
  CK(cudaMemcpyAsync(&nu, nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  int* off = x->alloc<int>(d.ntiles + 1);
  int* nbr = x->alloc<int>(std::max(1, nu));
  d.dryflag = x->alloc<int>(d.ntiles);
  d.skipmask = x->alloc<int>(d.ntiles);
  d.streak = std::getenv("SWE_NO_HELD") ? nullptr : x->alloc<int2>(d.ntiles);
  if (!off || !nbr || !d.skipmask) return fail_invalid("dry-skip tables: cudaMalloc failed"), SWE_CUDA;
  if (d.streak) CK(cudaMemsetAsync(d.streak, 0, sizeof(int2) * d.ntiles, s));
  k_pair_bounds<<<blocks_for(nu), kBlock, 0, s>>>(nu, k2, d.ntiles, off, nbr);
  CK(cudaMemsetAsync(d.dryflag, 0, sizeof(int) * d.ntiles, s));
  CK(cudaMemsetAsync(d.skipmask, 0, sizeof(int) * d.ntiles, s));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  d.nbr_off = off;
  d.nbr = nbr;
  return SWE_OK;
}

int preprocess(swe_dev_ctx* x, const swe_mesh_view* m) {
  Dev& d = x->d;
  const int C = d.C, E = d.E, T = d.T;
  cudaStream_t s = x->stream;
  Temps tmp;
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "upload");
  };
  int* r_cell_edge = (int*)tmp.get(sizeof(int) * 3 * (size_t)C);
  int* r_cell_sign = (int*)tmp.get(sizeof(int) * 3 * (size_t)C);
  int* r_el = (int*)tmp.get(sizeof(int) * E);
  int* r_er = (int*)tmp.get(sizeof(int) * E);
  double* r_buf = (double*)tmp.get(sizeof(double) * (size_t)std::max(C, E));
  unsigned long long* k64a = (unsigned long long*)tmp.get(8 * (size_t)std::max(C, E));
  unsigned long long* k64b = (unsigned long long*)tmp.get(8 * (size_t)std::max(C, E));
  int* idx = (int*)tmp.get(sizeof(int) * (size_t)std::max(C, E));
  int* e_new = (int*)tmp.get(sizeof(int) * E);
  int* flags = (int*)tmp.get(2 * sizeof(int));
  if (!flags) return fail_invalid("swe_dev_create: cudaMalloc (temporaries) failed"), SWE_CUDA;
  bool ok = up(r_cell_edge, m->cell_edge, sizeof(int) * 3 * (size_t)C) &&
            up(r_cell_sign, m->cell_sign, sizeof(int) * 3 * (size_t)C) &&
            up(r_el, m->edge_left, sizeof(int) * E) && up(r_er, m->edge_right, sizeof(int) * E) &&
            cuda_ok(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s), "memset");
  int* c_orig = const_cast<int*>(d.c_orig);
  int* c_new = const_cast<int*>(d.c_new);
  int* e_orig = const_cast<int*>(d.e_orig);

  // 1. cells: blocked-Hilbert order of the owned cells' centroids (stable:
  //    ties keep reference order); ghost cells keep their place after the
  //    owned ones
  const int Co = d.C_own;
  const bool curve = !(x->flags & SWE_FLAG_IDENTITY_ORDER) && m->cx && m->cy;
  if (ok) k_iota<<<blocks_for(C), kBlock, 0, s>>>(C, c_orig);
  if (ok && curve) {
    double x0 = m->cx[0], x1 = x0, y0 = m->cy[0], y1 = y0;
    for (int c = 1; c < Co; ++c) {
      x0 = std::min(x0, m->cx[c]);
      x1 = std::max(x1, m->cx[c]);
      y0 = std::min(y0, m->cy[c]);
      y1 = std::max(y1, m->cy[c]);
    }
    const double span = std::max(x1 - x0, y1 - y0);
    double* dcx = (double*)tmp.get(sizeof(double) * Co);
    double* dcy = (double*)tmp.get(sizeof(double) * Co);
    ok = dcx && dcy && up(dcx, m->cx, sizeof(double) * Co) && up(dcy, m->cy, sizeof(double) * Co);
    if (ok) {
      const double side = std::max(std::min(x1 - x0, y1 - y0), span / 255.0) * (1.0 + 1e-9);
      k_hilbert_blocks<<<blocks_for(Co), kBlock, 0, s>>>(Co, dcx, dcy, x0, y0,
                                                          side > 0 ? side : 1.0,
                                                          (y1 - y0) > (x1 - x0), k64a, idx);
      ok = radix_sort(tmp, k64a, k64b, idx, c_orig, Co, 40, s);
    }
  }
  if (ok) k_invert<<<blocks_for(C), kBlock, 0, s>>>(C, c_orig, c_new);

  // 2. edges: (owner tile, wall?, lower device cell)
  if (ok) {
    k_edge_keys<<<blocks_for(E), kBlock, 0, s>>>(E, r_el, r_er, c_new, T, k64a, idx);
    ok = radix_sort(tmp, k64a, k64b, idx, e_orig, E, 33 + bits_for(d.ntiles), s);
  }
  int *el = const_cast<int*>(d.el), *er = const_cast<int*>(d.er);
  int *i0 = const_cast<int*>(d.inc0), *i1 = const_cast<int*>(d.inc1), *i2 = const_cast<int*>(d.inc2);
  if (ok) {
    k_invert<<<blocks_for(E), kBlock, 0, s>>>(E, e_orig, e_new);
    k_edges_new<<<blocks_for(E), kBlock, 0, s>>>(E, e_orig, r_el, r_er, c_new, el, er);
    k_inc_new<<<blocks_for(C), kBlock, 0, s>>>(C, c_orig, r_cell_edge, r_cell_sign, e_new, i0, i1,
                                               i2, flags);
  }
  // 3. geometry in device order
  auto permute = [&](const double* host, int n, const int* perm, const double* dst) {
    if (!ok) return;
    ok = up(r_buf, host, sizeof(double) * n);
    k_gather<double><<<blocks_for(n), kBlock, 0, s>>>(n, perm, r_buf, const_cast<double*>(dst));
  };
  permute(m->area, C, c_orig, d.area);
  permute(m->inradius, C, c_orig, d.inr);
  permute(m->bed, C, c_orig, d.z);
  permute(m->manning, C, c_orig, d.man);
  permute(m->nx, E, e_orig, d.nx);
  permute(m->ny, E, e_orig, d.ny);
  permute(m->len, E, e_orig, d.len);

  // 4. tile tables: owned edge ranges, halo lists, per-cell slots
  int *eoff = const_cast<int*>(d.eoff), *hoff = const_cast<int*>(d.hoff);
  int* halo = const_cast<int*>(d.halo);
  int* hcount = flags + 1;
  if (ok) {
    k_tile_bounds<<<blocks_for(E), kBlock, 0, s>>>(E, el, er, T, d.ntiles, eoff);
    k_halo_keys<<<blocks_for(E), kBlock, 0, s>>>(E, el, er, T, Co, k64a, hcount);
    ok = cuda_ok(cudaGetLastError(), "tile tables");
  }
  int h_flags[2] = {0, 0};
  ok = ok && cuda_ok(cudaMemcpyAsync(h_flags, flags, sizeof(h_flags), cudaMemcpyDeviceToHost, s),
                     "d2h") &&
       cuda_ok(cudaStreamSynchronize(s), "preprocess");
  if (!ok) return SWE_CUDA;
  if (h_flags[0]) return fail_invalid("swe_dev_create: cell_sign must be +1/-1");
  const int nh = h_flags[1];
  x->n_halo = nh;
  if (nh > 0) {
    ok = radix_sort_keys(tmp, k64a, k64b, nh, 32 + bits_for(d.ntiles), s);
    k_halo_bounds<<<blocks_for(nh), kBlock, 0, s>>>(nh, k64b, d.ntiles, hoff, halo);
  } else {
    k_fill_int<<<blocks_for(d.ntiles + 1), kBlock, 0, s>>>(d.ntiles + 1, hoff, 0);
  }
  unsigned char* kl = const_cast<unsigned char*>(d.kl);
  unsigned char* kr = const_cast<unsigned char*>(d.kr);
  ok = ok && cuda_ok(cudaMemsetAsync(kl, 0xff, E, s), "memset") &&
       cuda_ok(cudaMemsetAsync(kr, 0xff, E, s), "memset");
  k_local_index<<<blocks_for(C), kBlock, 0, s>>>(C, i0, i1, i2, kl, kr);
  k_local_check<<<blocks_for(E), kBlock, 0, s>>>(E, er, kl, kr, flags);
  if (d.ek)
    k_pack_edges<<<blocks_for(E), kBlock, 0, s>>>(E, el, er, kl, kr, d.nx, d.ny,
                                                  const_cast<int2*>(d.ek),
                                                  const_cast<double2*>(d.enxy));
  std::vector<int> h_eoff(d.ntiles + 1), h_hoff(d.ntiles + 1);
  ok = ok && cuda_ok(cudaGetLastError(), "local index") &&
       cuda_ok(cudaMemcpyAsync(h_eoff.data(), eoff, sizeof(int) * (d.ntiles + 1),
                               cudaMemcpyDeviceToHost, s), "d2h") &&
       cuda_ok(cudaMemcpyAsync(h_hoff.data(), hoff, sizeof(int) * (d.ntiles + 1),
                               cudaMemcpyDeviceToHost, s), "d2h") &&
       cuda_ok(cudaMemcpyAsync(h_flags, flags, sizeof(h_flags), cudaMemcpyDeviceToHost, s), "d2h") &&
       cuda_ok(cudaStreamSynchronize(s), "preprocess");
  if (!ok) return SWE_CUDA;
  int max_slots = 1;
  for (int t = 0; t < d.ntiles; ++t)
    max_slots = std::max(max_slots, (h_eoff[t + 1] - h_eoff[t]) + (h_hoff[t + 1] - h_hoff[t]));
  if (h_flags[0] == 2)
    return fail_invalid("swe_dev_create: an edge is not referenced by its cells (cell_edges)");
  x->max_slots = max_slots;
  d.max_slots = max_slots;
  return SWE_OK;
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
  // PhysParams invariants (SPEC.md kernels module: g > 0, 0 < h_dry, 0 < cfl < 1
  // is the reference's contract; cfl is not range-checked by it, so neither here)
  if (!(params->g > 0.0) || !(params->h_dry > 0.0))
    return fail_invalid("swe_dev_create: PhysParams needs g > 0 and h_dry > 0");
  if (!m->area || !m->inradius || !m->bed || !m->manning || !m->cell_edge || !m->cell_sign ||
      !m->edge_left || !m->edge_right || !m->nx || !m->ny || !m->len)
    return fail_invalid("swe_dev_create: missing mesh array");
  const int C = m->n_cells, E = m->n_edges;
  if (C >= (1 << 30))  // packed edge records keep k in the top two bits
    return fail_invalid("swe_dev_create: more than 2^30 - 1 cells");
  for (int e = 0; e < E; ++e) {
    const int l = m->edge_left[e], r = m->edge_right[e];
    if (l < 0 || l >= C || r < -1 || r >= C)
      return fail_invalid("swe_dev_create: edge cell out of range");
  }
  for (long long i = 0; i < 3LL * C; ++i)
    if (m->cell_edge[i] < 0 || m->cell_edge[i] >= E)
      return fail_invalid("swe_dev_create: cell edge out of range");
  for (int c = 0; c < C; ++c)  // the select-form reconstruction assumes ordered beds
    if (!std::isfinite(m->bed[c])) return fail_invalid("swe_dev_create: non-finite bathymetry");
  if (m->n_owned < 0 || m->n_owned > C) return fail_invalid("swe_dev_create: n_owned out of range");
  if (m->n_owned > 0) {  // every edge of a partial mesh must touch an owned cell
    for (int e = 0; e < E; ++e)
      if (m->edge_left[e] >= m->n_owned && (m->edge_right[e] < 0 || m->edge_right[e] >= m->n_owned))
        return fail_invalid("swe_dev_create: an edge touches no owned cell");
  }

  auto* x = new swe_dev_ctx();
  x->device = device;
  x->flags = flags;
  x->fused = !(flags & SWE_FLAG_TWO_PHASE);
  auto bail = [&](int rc) {
    swe_dev_destroy(x);
    return rc;
  };
  if (!cuda_ok(cudaSetDevice(device), "cudaSetDevice")) return bail(SWE_CUDA);
  if (!cuda_ok(cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking), "stream"))
    return bail(SWE_CUDA);

  Dev& d = x->d;
  d.C = C;
  d.E = E;
  d.C_own = (m->n_owned > 0 && m->n_owned <= C) ? m->n_owned : C;
  d.P = Phys{params->g, params->h_dry, params->cfl, params->dt_max, params->h_ref};
  if (const char* env = std::getenv("SWE_TILE_THREADS")) x->tile_threads = std::atoi(env) == 128 ? 128 : 256;
  // tile size: at most 256 cells (measured best), shrunk so the tiles
  // fill whole waves of the persistent grid (a 1.28M-cell part has 4.2 waves
  // of 256-cell tiles: the last one 23% busy)
  if (const char* env = std::getenv("SWE_TILE_STAGE")) d.stage = std::atoi(env) != 0;
  if (const char* env = std::getenv("SWE_DYN_TILES")) d.dyn = std::atoi(env) != 0;
  if (const char* env = std::getenv("SWE_GRAPH_UNROLL")) x->graph_unroll = std::max(1, std::atoi(env));
  // run loop: the persistent kernel where a step's fixed cost matters (10k
  // cells 7.1 vs 11.4 us per step), the CUDA graph of k_tile + k_finalize
  // above (1M 31.2 vs 31.5 us, 2.56M 129.3 vs 128.2, 10M 475 vs 460;
  // DESIGN.md §4).  SWE_PERSISTENT=0/1 forces either.
  x->persistent = d.C_own <= kPersistentMaxCells;
  if (const char* env = std::getenv("SWE_PERSISTENT")) x->persistent = std::atoi(env) != 0;
  d.skip = 1;  // dry-tile skipping (fused kernel); SWE_NO_DRY_SKIP=1 turns it off
  if (const char* env = std::getenv("SWE_NO_DRY_SKIP")) d.skip = std::atoi(env) == 0;
  // tile size: 224 cells, a sharp measured optimum on B200 (3-7%
  // ahead of 216, 232 or 256 on every configuration, with and without dry-tile
  // skipping; 8 CTAs x 23.3 KB keep the 196 KB shared-memory carveout and
  // ~60 KB of L1 for the gathers).  Meshes smaller than one wave of such
  // tiles get smaller tiles so that every SM has work.
  const int t_max = d.stage ? 128 : 224;  // staged tiles: ~25 KB of shared memory at 128 cells
  int T = t_max;
  if (const char* env = std::getenv("SWE_TILE_CELLS")) {
    T = std::max(32, std::atoi(env));
  } else {
    int sms = 148, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaFuncSetAttribute(tile_kernel(x->tile_threads, false),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_smem_bytes(t_max, 0));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tile_kernel(x->tile_threads, false),
                                                  x->tile_threads, tile_smem_bytes(t_max, 0));
    const long long grid = (long long)sms * std::max(1, occ);
    if (d.C_own < (long long)t_max * grid) {
      const long long t = (d.C_own + grid - 1) / grid;
      T = (int)std::min((long long)t_max, std::max(32LL, (t + 7) / 8 * 8));
    }
    cudaGetLastError();
  }
  d.T = T;
  d.ntiles = (d.C_own + T - 1) / T;

  d.area = x->alloc<double>(C);
  d.inr = x->alloc<double>(C);
  d.z = x->alloc<double>(C);
  d.man = x->alloc<double>(C);
  d.inc0 = x->alloc<int>(C);
  d.inc1 = x->alloc<int>(C);
  d.inc2 = x->alloc<int>(C);
  d.c_orig = x->alloc<int>(C);
  d.c_new = x->alloc<int>(C);
  d.el = x->alloc<int>(E);
  d.er = x->alloc<int>(E);
  d.nx = x->alloc<double>(E);
  d.ny = x->alloc<double>(E);
  d.len = x->alloc<double>(E);
  d.e_orig = x->alloc<int>(E);
  d.eoff = x->alloc<int>(d.ntiles + 1);
  d.hoff = x->alloc<int>(d.ntiles + 1);
  d.halo = x->alloc<int>(E);
  d.kl = x->alloc<unsigned char>(E);
  d.kr = x->alloc<unsigned char>(E);
  if (x->fused) {
    d.ek = x->alloc<int2>(E);
    d.enxy = x->alloc<double2>(E);
    d.cg = x->alloc<CellGeo>(C);
    if (!d.enxy || !d.cg) {
      g_last_error = "swe_dev_create: cudaMalloc failed";
      return bail(SWE_CUDA);
    }
  }
  // state arrays + mailbox in one allocation (the arena peers map)
  x->arena_bytes = arena_offset(C, 6);
  x->arena = x->alloc<char>(x->arena_bytes);
  if (!x->arena) {
    g_last_error = "swe_dev_create: cudaMalloc failed";
    return bail(SWE_CUDA);
  }
  for (int b = 0; b < 2; ++b) {
    d.h[b] = (double*)(x->arena + arena_offset(C, 3 * b));
    d.qx[b] = (double*)(x->arena + arena_offset(C, 3 * b + 1));
    d.qy[b] = (double*)(x->arena + arena_offset(C, 3 * b + 2));
  }
  d.L.mine = (Mailbox*)x->arena;
  // edge records: compute_fluxes (engine.hpp:138-170)
  d.M = x->alloc<double>(E);
  d.LX = x->alloc<double>(E);
  d.LY = x->alloc<double>(E);
  d.RX = x->alloc<double>(E);
  d.RY = x->alloc<double>(E);
  bool two_ok = true;
  if (!x->fused) {  // per-incidence contributions of the two-phase step
    d.TM = x->alloc<double>(3 * (size_t)C);
    d.TX = x->alloc<double>(3 * (size_t)C);
    d.TY = x->alloc<double>(3 * (size_t)C);
    two_ok = d.TY != nullptr;
  }
  x->stage_h = x->alloc<double>(C);
  x->stage_qx = x->alloc<double>(C);
  x->stage_qy = x->alloc<double>(C);
  x->ctl = x->alloc<Ctl>(1);
  x->sp = x->alloc<StepParams>(1);
  x->rec_cap = 1 << 16;
  x->rec = x->alloc<swe_step_record>(x->rec_cap);
  if (!x->rec || !x->stage_qy || !d.RY || !d.kr || !d.e_orig || !two_ok) {
    g_last_error = "swe_dev_create: cudaMalloc failed";
    return bail(SWE_CUDA);
  }
  if (!cuda_ok(cudaMallocHost(&x->h_ctl, sizeof(Ctl)), "cudaMallocHost")) return bail(SWE_CUDA);
  d.ctl = x->ctl;
  d.sp = x->sp;
  d.rec = x->rec;

  if (int rc = preprocess(x, m)) return bail(rc);
  if (d.cg) {
    k_pack_cells<<<blocks_for(C), kBlock, 0, x->stream>>>(C, d.z, d.area, d.man, d.inr,
                                                        const_cast<CellGeo*>(d.cg));
    if (!cuda_ok(cudaGetLastError(), "k_pack_cells")) return bail(SWE_CUDA);
  }
  if (!x->fused || d.stage) d.skip = 0;
  // plain launches (SWE_FLAG_NO_GRAPH) keep the one-kernel-per-phase path
  if (!x->fused || d.stage || d.dyn || (flags & SWE_FLAG_NO_GRAPH)) x->persistent = false;
  if (d.skip)
    if (int rc = build_tile_neighbours(x)) return bail(rc);
  if (x->persistent) {
    d.sync = x->alloc<Sync>(1);
    d.pflag = x->alloc<int>(2 * (size_t)d.ntiles);
    x->d_dev = x->alloc<Dev>(1);
    if (!d.sync || !d.pflag || !x->d_dev) {
      g_last_error = "swe_dev_create: cudaMalloc failed";
      return bail(SWE_CUDA);
    }
    cudaMemsetAsync(d.sync, 0, sizeof(Sync), x->stream);
    cudaMemsetAsync(d.pflag, 0, sizeof(int) * 2 * (size_t)d.ntiles, x->stream);
    // state through L2 only, no per-step L1 invalidation (10k cells 7.33 vs
    // 8.06 us per step, 1M 31.3 vs 32.1); SWE_RUN_NOACQ=0: acquire
    d.run_noacq = 1;
    if (const char* env = std::getenv("SWE_RUN_NOACQ")) d.run_noacq = std::atoi(env) != 0;
  }
  if (d.stage) {  // slot arrays of the staged tile kernel
    const size_t ns = (size_t)E + (size_t)x->n_halo;
    int* soff = x->alloc<int>(d.ntiles + 1);
    int* sel = x->alloc<int>(ns);
    int* ser = x->alloc<int>(ns);
    int* skk = x->alloc<int>(ns);
    int* sedge = x->alloc<int>(ns);
    double* snx = x->alloc<double>(ns);
    double* sny = x->alloc<double>(ns);
    double* slen = x->alloc<double>(ns);
    if (!slen) {
      g_last_error = "swe_dev_create: cudaMalloc (slot arrays) failed";
      return bail(SWE_CUDA);
    }
    k_slots<<<blocks_for(32LL * d.ntiles), kBlock, 0, x->stream>>>(d, soff, sel, ser, skk, sedge,
                                                                  snx, sny, slen);
    if (!cuda_ok(cudaGetLastError(), "k_slots")) return bail(SWE_CUDA);
    d.soff = soff;
    d.sel = sel;
    d.ser = ser;
    d.skk = skk;
    d.sedge = sedge;
    d.snx = snx;
    d.sny = sny;
    d.slen = slen;
  }

  // grid sizes: resident blocks per SM x SM count (persistent grid-stride)
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int occ_face = 0, occ_cell = 0, occ_tile = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_face, k_face_c, kBlock, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_cell, k_cell_c, kBlock, 0);
  x->tile_smem = d.stage ? tile_stage_smem_bytes(d.T, d.max_slots) : tile_smem_bytes(d.T, d.max_slots);
  if (x->persistent)  // k_run's control block keeps its scratch + Dev in the tile buffers
    x->tile_smem = std::max(x->tile_smem, kRunCtlSmem);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if ((long long)x->tile_smem + 1024 > smem_optin) {
    g_last_error = "swe_dev_create: tile of " + std::to_string(d.T) + " cells needs " +
                   std::to_string(x->tile_smem) + " B of shared memory (limit " +
                   std::to_string(smem_optin) + "); use a smaller SWE_TILE_CELLS";
    return bail(SWE_INVALID);
  }
  const void* ktile = tile_kernel(x->tile_threads, false, d.stage);
  for (int L = 0; L < 2; ++L) {
    if (!cuda_ok(cudaFuncSetAttribute(tile_kernel(x->tile_threads, L, d.stage),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)x->tile_smem),
                 "tile smem attribute"))
      return bail(SWE_CUDA);
    if (const char* env = std::getenv("SWE_CARVEOUT"))  // experiment: shared-memory share of L1
      cudaFuncSetAttribute(tile_kernel(x->tile_threads, L, d.stage),
                           cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(env));
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_tile, ktile, x->tile_threads, x->tile_smem);
  if (x->persistent) {
    int occ_run = 0;
    for (int L = 0; L < 2; ++L) {
      int o = 0;
      if (!cuda_ok(cudaFuncSetAttribute(run_kernel(x->tile_threads, L),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)x->tile_smem),
                   "run smem attribute"))
        return bail(SWE_CUDA);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, run_kernel(x->tile_threads, L),
                                                    x->tile_threads, x->tile_smem);
      occ_run = L == 0 ? o : std::min(occ_run, o);
    }
    if (occ_run < 1 || sms * occ_run < 2) x->persistent = false;
    // cooperative launch: every CTA resident at once -- W workers (as many
    // as k_tile's grid, so both loops form the same partial sums) + 1 control
    int W = std::max(1, std::min(d.ntiles, sms * std::max(1, occ_run) - 1));
    if (const char* env = std::getenv("SWE_RUN_GRID"))  // test hook: fewer CTAs, more tiles each
      W = std::max(1, std::min(W, std::atoi(env)));
    x->grid_run = W + 1;
  }
  x->grid_face = std::max(1, std::min(blocks_for(E), sms * std::max(1, occ_face)));
  x->grid_cell = std::max(1, std::min(blocks_for(C), sms * std::max(1, occ_cell)));
  // one resident CTA short of a full wave: the persistent kernel's control
  // block takes that slot, so both run loops form the same partial sums
  x->grid_tile = std::max(1, std::min(d.ntiles, sms * std::max(1, occ_tile) - 1));
  if (x->persistent) x->grid_tile = std::min(x->grid_tile, x->grid_run - 1);
  // (two parities of the persistent kernel's worker partials)
  d.part = x->alloc<Part>(2 * (size_t)std::max(std::max(x->grid_cell, x->grid_tile), x->grid_run));
  if (!d.part) return bail(SWE_CUDA);

  Ctl c0{};
  c0.cfl_bad = kNone;
  c0.bad_edge = kNone;
  c0.bad_cell = kNone;
  c0.bad_speed = kNone;
  *x->h_ctl = c0;
  cudaStream_t s = x->stream;
  if (!cuda_ok(cudaMemcpyAsync(x->ctl, x->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s), "ctl"))
    return bail(SWE_CUDA);
  cudaMemsetAsync(x->arena, 0, x->arena_bytes, s);  // mailbox flags 0, state 0
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
  for (void* p : x->link_allocs) cudaFree(p);
  for (void* p : x->ipc_mapped) cudaIpcCloseMemHandle(p);
  if (x->copy_stream) cudaStreamSynchronize(x->copy_stream);
  for (int i = 0; i < 2; ++i) {
    for (int k = 0; k < 3; ++k) cudaFree(x->snap[i][k]);
    if (x->snap_ready[i]) cudaEventDestroy(x->snap_ready[i]);
    if (x->snap_done[i]) cudaEventDestroy(x->snap_done[i]);
  }
  if (x->copy_stream) cudaStreamDestroy(x->copy_stream);
  if (x->xfer_stream) cudaStreamSynchronize(x->xfer_stream), cudaStreamDestroy(x->xfer_stream);
  for (cudaEvent_t e : x->xfer_ev)
    if (e) cudaEventDestroy(e);
  cudaFree(x->halo_send);
  cudaFree(x->halo_recv);
  if (x->h_ctl) cudaFreeHost(x->h_ctl);
  if (x->stream) cudaStreamDestroy(x->stream);
  delete x;
  return SWE_OK;
}

// the state transfers' own stream and events (created on first use)
static int ensure_xfer(swe_dev_ctx* x) {
  if (x->xfer_stream) return SWE_OK;
  CK(cudaStreamCreateWithFlags(&x->xfer_stream, cudaStreamNonBlocking));
  for (cudaEvent_t& e : x->xfer_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SWE_OK;
}

// Host state in: each array's copy runs on the transfer stream while the
// previous array is permuted into device order on the main stream (one array
// per gather: its 82 MB source at 10M cells stays in L2 for the random reads)
static int set_state_impl(swe_dev_ctx* x, const double* h, const double* qx, const double* qy,
                          double t, long long step, cudaMemcpyKind kind) {
  if (!x || !h || !qx || !qy) return fail_invalid("swe_dev_set_state: null argument");
  const int C = x->d.C;
  cudaStream_t s = x->stream;
  CK(cudaSetDevice(x->device));
  if (int rc = sync_ctl(x)) return rc;
  if (int rc = ensure_xfer(x)) return rc;
  Ctl c = *x->h_ctl;
  const double* src[3] = {h, qx, qy};
  double* stg[3] = {x->stage_h, x->stage_qx, x->stage_qy};
  double* dst[3] = {x->d.h[c.cur], x->d.qx[c.cur], x->d.qy[c.cur]};
  CK(cudaEventRecord(x->xfer_ev[3], s));  // the staging buffers are free from here
  CK(cudaStreamWaitEvent(x->xfer_stream, x->xfer_ev[3], 0));
  for (int k = 0; k < 3; ++k) {
    CK(cudaMemcpyAsync(stg[k], src[k], sizeof(double) * C, kind, x->xfer_stream));
    CK(cudaEventRecord(x->xfer_ev[k], x->xfer_stream));
    CK(cudaStreamWaitEvent(s, x->xfer_ev[k], 0));
    k_gather<double><<<blocks_for(C), kBlock, 0, s>>>(C, x->d.c_orig, stg[k], dst[k]);
    ++g_launches;
    CK(cudaGetLastError());
  }
  c.t = t;
  c.step = step;
  c.cfl_valid = 0;
  c.cfl_bad = kNone;
  c.status = SWE_OK;
  c.active = 0;
  c.bad_edge = c.bad_cell = c.bad_speed = kNone;
  c.link_err = 0;
  x->cfl_host_valid = false;
  if (x->d.skip) {  // a new state: no tile is known dry
    CK(cudaMemsetAsync(x->d.dryflag, 0, sizeof(int) * x->d.ntiles, s));
    CK(cudaMemsetAsync(x->d.skipmask, 0, sizeof(int) * x->d.ntiles, s));
  }
  if (x->d.streak) CK(cudaMemsetAsync(x->d.streak, 0, sizeof(int2) * x->d.ntiles, s));
  if (x->d.pflag) CK(cudaMemsetAsync(x->d.pflag, 0, sizeof(int) * 2 * (size_t)x->d.ntiles, s));
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
  if (int rc = sync_ctl(x)) return rc;
  const int cur = x->h_ctl->cur;
  if (t) *t = x->h_ctl->t;
  if (step) *step = x->h_ctl->step;
  if (!h && !qx && !qy) return SWE_OK;
  CK(cudaSetDevice(x->device));
  if (int rc = ensure_xfer(x)) return rc;
  // each array permuted to reference order on the main stream, then copied
  // out on the transfer stream while the next one is permuted
  double* out[3] = {h, qx, qy};
  const double* dev[3] = {x->d.h[cur], x->d.qx[cur], x->d.qy[cur]};
  double* stg[3] = {x->stage_h, x->stage_qx, x->stage_qy};
  for (int k = 0; k < 3; ++k) {
    if (!out[k]) continue;
    k_gather<double><<<blocks_for(C), kBlock, 0, s>>>(C, x->d.c_new, dev[k], stg[k]);
    ++g_launches;
    CK(cudaGetLastError());
    CK(cudaEventRecord(x->xfer_ev[k], s));
    CK(cudaStreamWaitEvent(x->xfer_stream, x->xfer_ev[k], 0));
    CK(cudaMemcpyAsync(out[k], stg[k], sizeof(double) * C, kind, x->xfer_stream));
  }
  CK(cudaStreamSynchronize(x->xfer_stream));
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
  if (int rc = sync_ctl(x)) return rc;
  if (clipped) *clipped = x->h_ctl->clipped;
  if (events) *events = x->h_ctl->events;
  return SWE_OK;
}

int swe_dev_set_ledger(swe_dev_ctx* x, double clipped, long long events) {
  if (!x) return fail_invalid("null context");
  if (int rc = sync_ctl(x)) return rc;
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
  if (x->fused) {
    if (int rc = launch_update(x)) return rc;
    if (prof) CK(cudaEventRecord(x->events[ev_base + 1], x->stream));
    if (prof) CK(cudaEventRecord(x->events[ev_base + 2], x->stream));
  } else {
    k_face_c<<<x->grid_face, kBlock, 0, x->stream>>>(x->d);
    if (prof) CK(cudaEventRecord(x->events[ev_base + 1], x->stream));
    k_cell_c<<<x->grid_cell, kBlock, 0, x->stream>>>(x->d);
    g_launches += 2;
    CK(cudaGetLastError());
    if (prof) CK(cudaEventRecord(x->events[ev_base + 2], x->stream));
  }
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
  if (code == SWE_OK && rec)
    CK(cudaMemcpy(rec, x->rec, sizeof(swe_step_record), cudaMemcpyDeviceToHost));
  return code;
}

int swe_dev_advance(swe_dev_ctx* x, double t_end, long long max_steps, double next_snap,
                    swe_step_record* series, long long max_records, long long* n_done,
                    swe_status* st) {
  if (!x) return fail_invalid("null context");
  if (n_done) *n_done = 0;
  const long long cap = std::min<long long>(max_records > 0 ? max_records : x->rec_cap, x->rec_cap);
  if (int rc = ensure_cfl(x)) return rc;
  if (x->persistent) {
    if (int rc = launch_run(x, make_params(t_end, max_steps, next_snap, cap, 0))) return rc;
  } else if (x->exec) {
    if (int rc = write_params(x, t_end, max_steps, next_snap, cap, 0)) return rc;
    CK(cudaGraphLaunch(x->exec, x->stream));
    ++g_launches;
  } else {
    // no graph: step until the device says stop (checked every 64 steps)
    if (int rc = write_params(x, t_end, max_steps, next_snap, cap, 0)) return rc;
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

int swe_dev_advance_async(swe_dev_ctx* x, double t_end, long long max_steps, double next_snap,
                          long long max_records) {
  if (!x) return fail_invalid("null context");
  if (!x->exec && !x->persistent)
    return fail_invalid("swe_dev_advance_async: context was created without a graph");
  const long long cap = std::min<long long>(max_records > 0 ? max_records : x->rec_cap, x->rec_cap);
  if (int rc = ensure_cfl(x)) return rc;
  if (x->persistent) return launch_run(x, make_params(t_end, max_steps, next_snap, cap, 0));
  if (int rc = write_params(x, t_end, max_steps, next_snap, cap, 0)) return rc;
  CK(cudaGraphLaunch(x->exec, x->stream));
  ++g_launches;
  return SWE_OK;
}

int swe_dev_records(swe_dev_ctx* x, swe_step_record* series, long long max_records,
                    long long* n_done, swe_status* st) {
  if (!x) return fail_invalid("null context");
  const int code = read_status(x, st);
  const long long n = x->h_ctl->n_rec;
  if (n_done) *n_done = n;
  const long long m = std::min(n, std::min<long long>(max_records, x->rec_cap));
  if (series && m > 0)
    CK(cudaMemcpy(series, x->rec, sizeof(swe_step_record) * (size_t)m, cudaMemcpyDeviceToHost));
  return code;
}

int swe_dev_advance_n_async(swe_dev_ctx* x, long long n, double t_end) {
  if (!x) return fail_invalid("null context");
  if (int rc = ensure_cfl(x)) return rc;
  if (!x->profiling && x->persistent)  // exactly n steps: the gate sets max_steps = step + n
    return launch_run(x, make_params(t_end, LLONG_MAX, INFINITY, x->rec_cap, 1, 0, n));
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
        x->klaunch[j] += (x->fused && j == 1) ? 0 : 1;
      }
    }
  }
  return SWE_OK;
}

int swe_dev_set_halo_plan(swe_dev_ctx* x, int n_send, const int* send_cells, int n_recv,
                          const int* recv_cells) {
  if (!x || n_send < 0 || n_recv < 0 || (n_send && !send_cells) || (n_recv && !recv_cells))
    return fail_invalid("swe_dev_set_halo_plan: bad argument");
  for (int i = 0; i < n_send; ++i)
    if (send_cells[i] < 0 || send_cells[i] >= x->d.C_own)
      return fail_invalid("swe_dev_set_halo_plan: send cell is not owned");
  for (int i = 0; i < n_recv; ++i)
    if (recv_cells[i] < x->d.C_own || recv_cells[i] >= x->d.C)
      return fail_invalid("swe_dev_set_halo_plan: recv cell is not a ghost");
  cudaFree(x->halo_send);
  cudaFree(x->halo_recv);
  x->halo_send = x->halo_recv = nullptr;
  CK(cudaMalloc(&x->halo_send, sizeof(int) * (size_t)std::max(1, n_send)));
  CK(cudaMalloc(&x->halo_recv, sizeof(int) * (size_t)std::max(1, n_recv)));
  if (n_send)
    CK(cudaMemcpyAsync(x->halo_send, send_cells, sizeof(int) * n_send, cudaMemcpyHostToDevice,
                       x->stream));
  if (n_recv)
    CK(cudaMemcpyAsync(x->halo_recv, recv_cells, sizeof(int) * n_recv, cudaMemcpyHostToDevice,
                       x->stream));
  // reference-local ids -> device ids
  if (n_send) k_map_cells<<<blocks_for(n_send), kBlock, 0, x->stream>>>(n_send, x->d.c_new, x->halo_send);
  if (n_recv) k_map_cells<<<blocks_for(n_recv), kBlock, 0, x->stream>>>(n_recv, x->d.c_new, x->halo_recv);
  CK(cudaGetLastError());
  x->d.n_send = n_send;
  x->d.n_recv = n_recv;
  x->d.send_cells = x->halo_send;
  x->d.recv_cells = x->halo_recv;
  CK(cudaStreamSynchronize(x->stream));
  return SWE_OK;
}

int swe_dev_pack_halo(swe_dev_ctx* x, double* buf) {
  if (!x || (x->d.n_send && !buf)) return fail_invalid("swe_dev_pack_halo: bad argument");
  if (x->d.n_send) {
    k_halo_pack<<<blocks_for(x->d.n_send), kBlock, 0, x->stream>>>(x->d, buf);
    ++g_launches;
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(x->stream));
  return SWE_OK;
}

int swe_dev_unpack_halo(swe_dev_ctx* x, const double* buf) {
  if (!x || (x->d.n_recv && !buf)) return fail_invalid("swe_dev_unpack_halo: bad argument");
  if (x->d.n_recv) {
    k_halo_unpack<<<blocks_for(x->d.n_recv), kBlock, 0, x->stream>>>(x->d, buf);
    ++g_launches;
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(x->stream));
  return SWE_OK;
}

int swe_dev_local_cfl(swe_dev_ctx* x, double* dts, double* max_speed, double* mass,
                      swe_status* st) {
  if (!x) return fail_invalid("null context");
  if (int rc = ensure_cfl(x)) return rc;
  if (int rc = sync_ctl(x)) return rc;
  const Ctl& c = *x->h_ctl;
  if (dts) *dts = c.dts;
  if (max_speed) *max_speed = c.max_speed;
  if (mass) *mass = c.mass;
  if (c.cfl_bad != kNone) {
    if (st) {
      st->code = SWE_NONFINITE_SPEED;
      st->index = c.cfl_bad;
    }
    return SWE_NONFINITE_SPEED;
  }
  if (st) st->code = SWE_OK;
  return SWE_OK;
}

int swe_dev_step_global(swe_dev_ctx* x, double t_end, double dts, double max_speed,
                        swe_step_record* rec, swe_status* st) {
  if (!x) return fail_invalid("null context");
  if (int rc = ensure_cfl(x)) return rc;
  if (int rc = sync_ctl(x)) return rc;
  x->h_ctl->dts = dts;
  x->h_ctl->max_speed = max_speed;
  x->h_ctl->cfl_valid = 1;
  x->h_ctl->cfl_bad = kNone;  // the driver checked every part's bound
  CK(cudaMemcpyAsync(x->ctl, x->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, x->stream));
  if (int rc = write_params(x, t_end, LLONG_MAX, INFINITY, 1, 0, 1)) return rc;
  if (int rc = launch_gate(x)) return rc;
  const bool prof = x->profiling;
  x->profiling = false;
  const int rc = plain_step(x, 0);
  x->profiling = prof;
  if (rc) return rc;
  const int code = read_status(x, st);
  if (code == SWE_OK && rec)
    CK(cudaMemcpy(rec, x->rec, sizeof(swe_step_record), cudaMemcpyDeviceToHost));
  return code;
}

int swe_dev_synchronize(swe_dev_ctx* x, swe_status* st) {
  if (!x) return fail_invalid("null context");
  return read_status(x, st);
}

int swe_dev_compute_fluxes(swe_dev_ctx* x, double* left, double* right, swe_status* st) {
  if (!x || !left || !right) return fail_invalid("swe_dev_compute_fluxes: null argument");
  const int E = x->d.E;
  // one face pass on the current state (no commit)
  if (int rc = write_params(x, INFINITY, LLONG_MAX, INFINITY, 1, 0, 2)) return rc;
  if (int rc = launch_gate(x)) return rc;
  k_face<<<x->grid_face, kBlock, 0, x->stream>>>(x->d);
  ++g_launches;
  CK(cudaGetLastError());
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
  if (int rc = sync_ctl(x)) return rc;
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
  if (int rc = ensure_cfl(x, true)) return rc;
  if (int rc = sync_ctl(x)) return rc;
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

int swe_dev_info(swe_dev_ctx* x, long long* out, int n) {
  if (!x || !out) return fail_invalid("null argument");
  if (n > 11)
    if (int rc = sync_ctl(x)) return rc;
  const long long v[16] = {x->fused ? 1 : 0, x->d.T, x->d.ntiles, x->max_slots, x->n_halo,
                           x->grid_tile, x->grid_face, x->grid_cell, (long long)x->tile_smem,
                           x->d.E, x->d.skip, n > 11 ? (long long)x->h_ctl->skipped : 0,
                           x->graph_unroll, x->persistent ? 1 : 0, x->grid_run,
                           n > 15 ? (long long)x->h_ctl->held : 0};
  for (int i = 0; i < n && i < 16; ++i) out[i] = v[i];
  return SWE_OK;
}

// ---------------------------------------------------------------------------
// linked contexts (multi-device); see Link in swe_ctl.cuh
// ---------------------------------------------------------------------------
int swe_dev_link_export(swe_dev_ctx* x, void** arena, unsigned char* ipc_handle) {
  if (!x) return fail_invalid("null context");
  if (arena) *arena = x->arena;
  if (ipc_handle) {
    CK(cudaSetDevice(x->device));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, x->arena));
    std::memcpy(ipc_handle, &h, sizeof(h));
  }
  return SWE_OK;
}

int swe_dev_link(swe_dev_ctx* x, int rank, int nranks, void* const* arenas,
                 const unsigned char* ipc_handles, const long long* peer_cells, int n_push,
                 const int* push_cell, const int* push_rank, const int* push_ghost,
                 const int* gcell, const int* gedge, double timeout_s) {
  if (!x) return fail_invalid("null context");
  if (x->linked) return fail_invalid("swe_dev_link: context is already linked");
  if (const char* env = std::getenv("SWE_LINK_FAIL"))  // test hook: an IPC-less platform
    if (std::atoi(env) == 1 + rank || std::atoi(env) == -1) {
      g_last_error = "swe_dev_link: peer memory unavailable (SWE_LINK_FAIL)";
      return SWE_CUDA;
    }
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || !peer_cells ||
      (!arenas && !ipc_handles) || n_push < 0 ||
      (n_push && (!push_cell || !push_rank || !push_ghost)))
    return fail_invalid("swe_dev_link: bad argument");
  Dev& d = x->d;
  if (peer_cells[rank] != d.C) return fail_invalid("swe_dev_link: peer_cells[rank] != n_cells");
  for (int j = 0; j < n_push; ++j) {
    const int q = push_rank[j];
    if (push_cell[j] < 0 || push_cell[j] >= d.C_own || q < 0 || q >= nranks || q == rank ||
        push_ghost[j] < 0 || push_ghost[j] >= peer_cells[q])
      return fail_invalid("swe_dev_link: bad push entry");
  }
  CK(cudaSetDevice(x->device));
  // peers' arenas in this process
  std::vector<char*> base(nranks, nullptr);
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) {
      base[q] = x->arena;
    } else if (arenas && arenas[q]) {  // a context of this process
      base[q] = (char*)arenas[q];
      cudaPointerAttributes a{};
      CK(cudaPointerGetAttributes(&a, base[q]));
      if (a.device != x->device) {  // another device of this process
        const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else CK(e);
      }
    } else {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, ipc_handles + sizeof(h) * q, sizeof(h));
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      x->ipc_mapped.push_back(p);
      base[q] = (char*)p;
    }
  }
  std::vector<Mailbox*> boxes(nranks);
  std::vector<double*> states(6 * (size_t)nranks);
  for (int q = 0; q < nranks; ++q) {
    boxes[q] = (Mailbox*)base[q];
    for (int k = 0; k < 6; ++k) states[6 * q + k] = (double*)(base[q] + arena_offset(peer_cells[q], k));
  }
  // push list in device cell order, grouped by tile
  std::vector<int> c_new(d.C);
  CK(cudaMemcpy(c_new.data(), d.c_new, sizeof(int) * d.C, cudaMemcpyDeviceToHost));
  std::vector<int> order(n_push);
  for (int j = 0; j < n_push; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return c_new[push_cell[a]] < c_new[push_cell[b]];
  });
  std::vector<int> pc(std::max(1, n_push)), pr(std::max(1, n_push)), pg(std::max(1, n_push));
  std::vector<int> tp(d.ntiles + 1, 0);
  for (int j = 0; j < n_push; ++j) {
    const int o = order[j];
    pc[j] = c_new[push_cell[o]];
    pr[j] = push_rank[o];
    pg[j] = push_ghost[o];  // ghosts keep their local ids on the device
    ++tp[pc[j] / d.T + 1];
  }
  for (int t = 0; t < d.ntiles; ++t) tp[t + 1] += tp[t];
  std::vector<int> gc(d.C), ge(d.E);
  for (int c = 0; c < d.C; ++c) gc[c] = gcell ? gcell[c] : c;
  for (int e = 0; e < d.E; ++e) ge[e] = gedge ? gedge[e] : e;
  auto upload = [&](const void* src, size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    x->link_allocs.push_back(p);
    if (cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return p;
  };
  Link L{};
  L.rank = rank;
  L.nranks = nranks;
  L.mine = (Mailbox*)x->arena;
  L.box = (Mailbox* const*)upload(boxes.data(), sizeof(Mailbox*) * nranks);
  L.state = (double* const*)upload(states.data(), sizeof(double*) * states.size());
  L.tile_push = (const int*)upload(tp.data(), sizeof(int) * tp.size());
  L.push_cell = (const int*)upload(pc.data(), sizeof(int) * pc.size());
  L.push_rank = (const int*)upload(pr.data(), sizeof(int) * pr.size());
  L.push_ghost = (const int*)upload(pg.data(), sizeof(int) * pg.size());
  L.gcell = (const int*)upload(gc.data(), sizeof(int) * gc.size());
  L.gedge = (const int*)upload(ge.data(), sizeof(int) * ge.size());
  L.timeout_ns = (unsigned long long)((timeout_s > 0 ? timeout_s : 60.0) * 1e9);
  if (!L.box || !L.state || !L.tile_push || !L.push_cell || !L.push_rank || !L.push_ghost ||
      !L.gcell || !L.gedge) {
    g_last_error = "swe_dev_link: device tables: " + std::string(cudaGetErrorString(cudaGetLastError()));
    return SWE_CUDA;
  }
  d.L = L;
  x->n_push = n_push;
  x->linked = true;
  if (x->persistent) {  // tiles whose edges read ghost cells wait for the exchange
    unsigned char* tg = nullptr;
    CK(cudaMalloc(&tg, std::max(1, d.ntiles)));
    x->link_allocs.push_back(tg);
    k_tile_ghost<<<blocks_for(d.ntiles), kBlock, 0, x->stream>>>(d, tg);
    CK(cudaGetLastError());
    d.tile_ghost = tg;
  }
  // the CFL cache must be re-formed globally; the graph gains the exchange
  if (int rc = sync_ctl(x)) return rc;
  // every rank starts linked with its current state in buffer 0 and no
  // exchange posted: a step kernel pushes ghosts into the PEER's buffer
  // (sender's cur ^ 1) and mailbox slots are tagged by the exchange count, so
  // contexts stepped different numbers of times before linking (e.g. an
  // unlinked warm-up) would otherwise write into a peer's live buffer
  if (x->h_ctl->cur != 0) {
    for (int k = 0; k < 3; ++k) {
      double* const* buf = k == 0 ? d.h : (k == 1 ? d.qx : d.qy);
      CK(cudaMemcpyAsync(buf[0], buf[1], sizeof(double) * d.C, cudaMemcpyDeviceToDevice,
                         x->stream));
    }
    x->h_ctl->cur = 0;
  }
  if (d.streak) CK(cudaMemsetAsync(d.streak, 0, sizeof(int2) * d.ntiles, x->stream));
  x->h_ctl->xseq = 0;  // (a context is linked once; nothing has posted to it yet)
  x->h_ctl->cfl_valid = 0;
  x->cfl_host_valid = false;
  CK(cudaMemcpyAsync(x->ctl, x->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, x->stream));
  if (x->exec) {
    CK(cudaGraphExecDestroy(x->exec));
    CK(cudaGraphDestroy(x->graph));
    x->exec = nullptr;
    x->graph = nullptr;
    if (int rc = build_graph(x)) return rc;
  }
  CK(cudaStreamSynchronize(x->stream));
  return SWE_OK;
}

// One phase of a linked step, enqueued without waiting, so that a single
// host thread can drive several linked contexts sharing one device in
// lockstep (every rank's post is enqueued before any rank's wait):
//   0 open (local CFL bound + post if stale)  1 CFL wait + gate
//   2 step kernel(s) + halo push               3 post the step outcome
//   4 wait, combine, commit
int swe_dev_link_phase(swe_dev_ctx* x, int phase, double t_end) {
  if (!x) return fail_invalid("null context");
  if (!x->linked) return fail_invalid("swe_dev_link_phase: context is not linked");
  switch (phase) {
    case 0: {
      if (int rc = sync_ctl(x)) return rc;
      x->cfl_posted = !x->h_ctl->cfl_valid;
      if (x->cfl_posted) {
        k_cfl<<<x->grid_cell, kBlock, 0, x->stream>>>(x->d);
        ++g_launches;
        if (int rc = launch_post(x, x->grid_cell, 1)) return rc;
      }
      return write_params(x, t_end, LLONG_MAX, INFINITY, 1, 0, 1);
    }
    case 1:
      if (x->cfl_posted)
        if (int rc = launch_wait(x, 1, cudaGraphConditionalHandle{}, 0)) return rc;
      x->cfl_posted = false;
      return launch_gate(x);
    case 2: return launch_update(x);
    case 3: return launch_post(x, x->n_step_parts(), 0);
    case 4: return launch_wait(x, 0, cudaGraphConditionalHandle{}, 0);
  }
  return fail_invalid("swe_dev_link_phase: phase must be 0..4");
}

// P linked contexts sharing ONE device stepped by one cooperative launch of
// the persistent kernel (k_run_ranks): the ranks' CTAs run concurrently and
// exchange through the mailboxes exactly as on P GPUs.  Test path: separate
// launches that wait on each other must not share a device.
int swe_dev_run_ranks(swe_dev_ctx* const* xs, int n, long long nsteps, double t_end, int grid) {
  if (!xs || n < 1 || nsteps < 1) return fail_invalid("swe_dev_run_ranks: bad argument");
  int G = grid > 0 ? grid : INT_MAX;
  for (int r = 0; r < n; ++r) {
    swe_dev_ctx* x = xs[r];
    if (!x || !x->linked || !x->persistent || x->device != xs[0]->device ||
        x->tile_threads != xs[0]->tile_threads || x->d.L.rank != r || x->d.L.nranks != n)
      return fail_invalid("swe_dev_run_ranks: contexts must be persistent, linked as ranks "
                          "0..n-1 of n, on one device");
    G = std::min(G, std::min(x->d.ntiles + 1, x->grid_run));  // workers + a control block
  }
  const int NT = xs[0]->tile_threads;
  size_t smem = 0;
  for (int r = 0; r < n; ++r) smem = std::max(smem, xs[r]->tile_smem);
  const void* kr = NT == 128 ? (const void*)k_run_ranks<128> : (const void*)k_run_ranks<256>;
  CK(cudaSetDevice(xs[0]->device));
  CK(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0, sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, xs[0]->device));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kr, NT, smem));
  G = std::min(G, sms * occ / n);
  if (G < 2) return fail_invalid("swe_dev_run_ranks: too many ranks for one device");
  // CFL bound of the current state: every rank posts, then every rank waits
  // (phases, so no waiting kernel runs before all posts are done)
  std::vector<bool> posted(n, false);
  for (int r = 0; r < n; ++r) {
    swe_dev_ctx* x = xs[r];
    if (int rc = sync_ctl(x)) return rc;
    if (!x->h_ctl->cfl_valid) {
      k_cfl<<<x->grid_cell, kBlock, 0, x->stream>>>(x->d);
      ++g_launches;
      if (int rc = launch_post(x, x->grid_cell, 1)) return rc;
      posted[r] = true;
    }
  }
  for (int r = 0; r < n; ++r) CK(cudaStreamSynchronize(xs[r]->stream));
  for (int r = 0; r < n; ++r)
    if (posted[r])
      if (int rc = launch_wait(xs[r], 1, cudaGraphConditionalHandle{}, 0)) return rc;
  for (int r = 0; r < n; ++r) {
    swe_dev_ctx* x = xs[r];
    x->cfl_host_valid = true;
    if (int rc = write_params(x, t_end, LLONG_MAX, INFINITY, x->rec_cap, 1, 0, nsteps)) return rc;
    if (int rc = launch_gate(x)) return rc;
  }
  std::vector<Dev> devs(n);
  for (int r = 0; r < n; ++r) devs[r] = xs[r]->d;
  Dev* ddevs = nullptr;
  CK(cudaMalloc(&ddevs, sizeof(Dev) * n));
  struct Free {
    void* p;
    ~Free() { cudaFree(p); }
  } guard{ddevs};
  CK(cudaMemcpy(ddevs, devs.data(), sizeof(Dev) * n, cudaMemcpyHostToDevice));
  for (int r = 0; r < n; ++r) CK(cudaStreamSynchronize(xs[r]->stream));
  const Dev* dp = ddevs;
  void* args[] = {&dp, &G};
  CK(cudaLaunchCooperativeKernel(kr, dim3(G * n), dim3(NT), args, smem, xs[0]->stream));
  ++g_launches;
  CK(cudaStreamSynchronize(xs[0]->stream));
  int worst = SWE_OK;
  for (int r = 0; r < n; ++r) {
    const int code = read_status(xs[r], nullptr);
    if (code != SWE_OK && worst == SWE_OK) worst = code;
  }
  return worst;
}

// experiment builds (SWE_RUN_TIMING=1): the persistent loop's phase-time
// sums [work ns, epoch-wait ns, arrival-wait ns, commit ns, CTA-steps,
// commits]; read and cleared
int swe_dev_run_timing(swe_dev_ctx* x, long long* out, int n) {
  if (!x || !out || !x->d.sync) return fail_invalid("swe_dev_run_timing: no persistent context");
  Sync h;
  CK(cudaStreamSynchronize(x->stream));
  CK(cudaMemcpy(&h, x->d.sync, sizeof(Sync), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < 12; ++i) out[i] = (long long)h.timing[i];
  CK(cudaMemset(x->d.sync, 0, sizeof(Sync)));
  return SWE_OK;
}

int swe_dev_last_record(swe_dev_ctx* x, swe_step_record* rec, swe_status* st) {
  if (!x) return fail_invalid("null context");
  const int code = read_status(x, st);
  if (code == SWE_OK && rec && x->h_ctl->n_rec > 0)
    CK(cudaMemcpy(rec, x->rec, sizeof(swe_step_record), cudaMemcpyDeviceToHost));
  return code;
}

// ---------------------------------------------------------------------------
// asynchronous snapshots (reference run() on_snapshot, engine.hpp:347-379)
// ---------------------------------------------------------------------------
int swe_dev_snapshot_async(swe_dev_ctx* x, int slot, double* h, double* qx, double* qy) {
  if (!x || slot < 0 || slot > 1 || !h || !qx || !qy)
    return fail_invalid("swe_dev_snapshot_async: bad argument");
  const int C = x->d.C;
  CK(cudaSetDevice(x->device));
  if (!x->copy_stream) {
    CK(cudaStreamCreateWithFlags(&x->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&x->snap_ready[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&x->snap_done[i], cudaEventDisableTiming));
    }
  }
  if (!x->snap[slot][0])
    for (int k = 0; k < 3; ++k) CK(cudaMalloc(&x->snap[slot][k], sizeof(double) * C));
  // the slot's previous copy must be done before it is overwritten
  CK(cudaStreamWaitEvent(x->stream, x->snap_done[slot], 0));
  k_snapshot<<<blocks_for(C), kBlock, 0, x->stream>>>(x->d, x->snap[slot][0], x->snap[slot][1],
                                                      x->snap[slot][2]);
  ++g_launches;
  CK(cudaGetLastError());
  CK(cudaEventRecord(x->snap_ready[slot], x->stream));
  CK(cudaStreamWaitEvent(x->copy_stream, x->snap_ready[slot], 0));
  double* dst[3] = {h, qx, qy};
  for (int k = 0; k < 3; ++k)
    CK(cudaMemcpyAsync(dst[k], x->snap[slot][k], sizeof(double) * C, cudaMemcpyDeviceToHost,
                       x->copy_stream));
  CK(cudaEventRecord(x->snap_done[slot], x->copy_stream));
  return SWE_OK;
}

int swe_dev_snapshot_wait(swe_dev_ctx* x, int slot) {
  if (!x || slot < 0 || slot > 1) return fail_invalid("swe_dev_snapshot_wait: bad argument");
  if (!x->snap_done[slot]) return SWE_OK;
  CK(cudaEventSynchronize(x->snap_done[slot]));
  return SWE_OK;
}

void* swe_dev_host_alloc(long long bytes) {
  void* p = nullptr;
  if (bytes <= 0 || cudaMallocHost(&p, (size_t)bytes) != cudaSuccess) return nullptr;
  return p;
}

void swe_dev_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int swe_dev_host_register(void* p, long long bytes) {
  if (!p || bytes <= 0) return fail_invalid("swe_dev_host_register: bad argument");
  CK(cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault));
  return SWE_OK;
}

int swe_dev_host_unregister(void* p) {
  if (!p) return SWE_OK;
  CK(cudaHostUnregister(p));
  return SWE_OK;
}

// ---------------------------------------------------------------------------
// build_mesh on the device (swe_build.cuh; reference mesh.hpp:121-240)
// ---------------------------------------------------------------------------
}  // extern "C"

struct swe_built_mesh {
  int device = 0, nn = 0, nc = 0, ne = 0;
  std::vector<void*> allocs;
  int *cn = nullptr, *ce = nullptr, *cs = nullptr, *en = nullptr, *el = nullptr, *er = nullptr;
  double *area = nullptr, *cx = nullptr, *cy = nullptr, *inr = nullptr;
  double *nx = nullptr, *ny = nullptr, *len = nullptr;
  template <class V>
  V* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(V)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return static_cast<V*>(p);
  }
  ~swe_built_mesh() {
    for (void* p : allocs) cudaFree(p);
  }
};

namespace {
void put_err(const std::string& m, char* err, int errlen) {
  g_last_error = m;
  if (err && errlen > 0) {
    std::strncpy(err, m.c_str(), (size_t)errlen - 1);
    err[errlen - 1] = 0;
  }
}
double hnorm(double x, double y) { return std::sqrt(x * x + y * y); }
}  // namespace

extern "C" {

int swe_dev_build_mesh(int device, int nn, const double* xy, int nc, const int* tris,
                       swe_built_mesh** out, char* err, int errlen) {
  if (!out || nn < 0 || nc < 0 || (nn && !xy) || (nc && !tris))
    return fail_invalid("swe_dev_build_mesh: bad argument");
  *out = nullptr;
  const bool timing = std::getenv("SWE_BUILD_TIMING") != nullptr;
  auto tick = [t0 = std::chrono::steady_clock::now(), timing](const char* what) mutable {
    if (!timing) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[build_mesh_device] %-10s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  CK(cudaSetDevice(device));
  tick("set_device");
  auto* b = new swe_built_mesh();
  b->device = device;
  b->nn = nn;
  b->nc = nc;
  auto bail = [&](int rc) {
    delete b;
    return rc;
  };
  cudaStream_t s = nullptr;
  if (!cuda_ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream")) return bail(SWE_CUDA);
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{s};
  Temps tmp;
  const long long n3 = 3LL * nc;
  double* dxy = (double*)tmp.get(sizeof(double) * 2 * (size_t)std::max(1, nn));
  int* dtri = (int*)tmp.get(sizeof(int) * (size_t)std::max(1LL, n3));
  BuildErr* derr = (BuildErr*)tmp.get(sizeof(BuildErr));
  b->cn = b->alloc<int>(n3);
  b->area = b->alloc<double>(nc);
  b->cx = b->alloc<double>(nc);
  b->cy = b->alloc<double>(nc);
  b->inr = b->alloc<double>(nc);
  b->ce = b->alloc<int>(n3);
  b->cs = b->alloc<int>(n3);
  if (!dxy || !dtri || !derr || !b->cn || !b->inr || !b->cs) {
    g_last_error = "swe_dev_build_mesh: cudaMalloc failed";
    return bail(SWE_CUDA);
  }
  BuildErr h_err{INT_MAX, INT_MAX, INT_MAX, 0};
  bool ok = (!nn || cuda_ok(cudaMemcpyAsync(dxy, xy, sizeof(double) * 2 * (size_t)nn,
                                            cudaMemcpyHostToDevice, s), "upload")) &&
            (!nc || cuda_ok(cudaMemcpyAsync(dtri, tris, sizeof(int) * (size_t)n3,
                                            cudaMemcpyHostToDevice, s), "upload")) &&
            cuda_ok(cudaMemcpyAsync(derr, &h_err, sizeof(h_err), cudaMemcpyHostToDevice, s), "upload");
  if (!ok) return bail(SWE_CUDA);
  tick("alloc+h2d");
  // loop 1: cells (mesh.hpp:189-212)
  if (nc) kb_cells<<<blocks_for(nc), kBlock, 0, s>>>(nn, nc, dxy, dtri, b->cn, b->area, b->cx, b->cy,
                                                     b->inr, derr);
  if (!cuda_ok(cudaMemcpyAsync(&h_err, derr, sizeof(h_err), cudaMemcpyDeviceToHost, s), "d2h") ||
      !cuda_ok(cudaStreamSynchronize(s), "build cells"))
    return bail(SWE_CUDA);
  tick("cells");
  if (h_err.cell != INT_MAX) {  // the reference's text for the first bad triangle
    const int c = h_err.cell;
    int t[3] = {tris[3 * (size_t)c], tris[3 * (size_t)c + 1], tris[3 * (size_t)c + 2]};
    std::string m;
    for (int k = 0; k < 3 && m.empty(); ++k)
      if (t[k] < 0 || t[k] >= nn)
        m = "build_mesh: node index " + std::to_string(t[k]) + " out of range in triangle " +
            std::to_string(c);
    if (m.empty() && (t[0] == t[1] || t[1] == t[2] || t[0] == t[2]))
      m = "build_mesh: degenerate triangle " + std::to_string(c) + " repeats a node index";
    if (m.empty()) m = "build_mesh: triangle " + std::to_string(c) + " has zero area";
    put_err(m, err, errlen);
    return bail(SWE_INVALID);
  }
  // incidences in (lower node, upper node, cell, local) order (mesh.hpp:214-246)
  unsigned long long* k0 = (unsigned long long*)tmp.get(8 * (size_t)std::max(1LL, n3));
  unsigned long long* k1 = (unsigned long long*)tmp.get(8 * (size_t)std::max(1LL, n3));
  int* v0 = (int*)tmp.get(4 * (size_t)std::max(1LL, n3));
  int* v1 = (int*)tmp.get(4 * (size_t)std::max(1LL, n3));
  int* head = (int*)tmp.get(4 * (size_t)std::max(1LL, n3));
  int* eid = (int*)tmp.get(4 * (size_t)std::max(1LL, n3));
  if (!k0 || !k1 || !v0 || !v1 || !head || !eid) {
    g_last_error = "swe_dev_build_mesh: cudaMalloc failed";
    return bail(SWE_CUDA);
  }
  int ne = 0;
  if (n3) {
    kb_keys<<<blocks_for(n3), kBlock, 0, s>>>(nc, b->cn, k0, v0);
    if (!radix_sort(tmp, k0, k1, v0, v1, (int)n3, 32 + bits_for(nn), s)) return bail(SWE_CUDA);
    kb_heads<<<blocks_for(n3), kBlock, 0, s>>>(n3, k1, head);
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, head, eid, (int)n3, s);
    void* store = tmp.get(tb);
    if (!store || !cuda_ok(cub::DeviceScan::InclusiveSum(store, tb, head, eid, (int)n3, s), "scan"))
      return bail(SWE_CUDA);
    if (!cuda_ok(cudaMemcpyAsync(&ne, eid + n3 - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h") ||
        !cuda_ok(cudaStreamSynchronize(s), "build keys"))
      return bail(SWE_CUDA);
  }
  tick("sort+scan");
  b->ne = ne;
  b->en = b->alloc<int>(2 * (size_t)ne);
  b->el = b->alloc<int>(ne);
  b->er = b->alloc<int>(ne);
  b->nx = b->alloc<double>(ne);
  b->ny = b->alloc<double>(ne);
  b->len = b->alloc<double>(ne);
  if (!b->en || !b->len) {
    g_last_error = "swe_dev_build_mesh: cudaMalloc failed";
    return bail(SWE_CUDA);
  }
  if (n3) {
    kb_edges<<<blocks_for(n3), kBlock, 0, s>>>(n3, k1, v1, head, eid, b->cn, dxy, b->en, b->el, b->er,
                                               b->nx, b->ny, b->len, b->ce, b->cs, derr);
    if (!cuda_ok(cudaMemcpyAsync(&h_err, derr, sizeof(h_err), cudaMemcpyDeviceToHost, s), "d2h") ||
        !cuda_ok(cudaStreamSynchronize(s), "build edges"))
      return bail(SWE_CUDA);
  }
  tick("edges");
  if (h_err.run != INT_MAX) {  // the first bad run in sorted order (mesh.hpp:252-272)
    const long long i = h_err.run;
    const int w = (int)std::min<long long>(64, n3 - i);
    std::vector<unsigned long long> kk(w);
    std::vector<int> vv(w);
    cudaMemcpy(kk.data(), k1 + i, 8 * (size_t)w, cudaMemcpyDeviceToHost);
    cudaMemcpy(vv.data(), v1 + i, 4 * (size_t)w, cudaMemcpyDeviceToHost);
    int cnt = 1;
    while (cnt < w && kk[cnt] == kk[0]) ++cnt;
    auto directed = [&](int v, int& a0, int& a1) {
      int t[3];
      cudaMemcpy(t, b->cn + 3 * (size_t)(v / 3), sizeof(t), cudaMemcpyDeviceToHost);
      a0 = t[v % 3];
      a1 = t[(v % 3 + 1) % 3];
    };
    int a0, a1;
    directed(vv[0], a0, a1);
    std::string m = "build_mesh: non-manifold edge (" + std::to_string(a0) + "," + std::to_string(a1) + ")";
    if (cnt > 2)
      m += " shared by " + std::to_string(cnt) + " triangles";
    else
      m += " traversed twice in the same direction; triangles " + std::to_string(vv[0] / 3) +
           " and " + std::to_string(vv[1] / 3) + " overlap or are inconsistently oriented";
    put_err(m, err, errlen);
    return bail(SWE_INVALID);
  }
  if (nc) {  // closed-polygon identity (mesh.hpp:280-291)
    kb_closure<<<blocks_for(nc), kBlock, 0, s>>>(nc, b->ce, b->cs, b->nx, b->ny, b->len, derr);
    if (!cuda_ok(cudaMemcpyAsync(&h_err, derr, sizeof(h_err), cudaMemcpyDeviceToHost, s), "d2h") ||
        !cuda_ok(cudaStreamSynchronize(s), "build closure"))
      return bail(SWE_CUDA);
  }
  tick("closure");
  if (h_err.closure != INT_MAX) {
    const int c = h_err.closure;
    int ce[3], cs[3];
    cudaMemcpy(ce, b->ce + 3 * (size_t)c, sizeof(ce), cudaMemcpyDeviceToHost);
    cudaMemcpy(cs, b->cs + 3 * (size_t)c, sizeof(cs), cudaMemcpyDeviceToHost);
    double sx = 0.0, sy = 0.0;
    for (int k = 0; k < 3; ++k) {
      double l, nxv, nyv;
      cudaMemcpy(&l, b->len + ce[k], 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&nxv, b->nx + ce[k], 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&nyv, b->ny + ce[k], 8, cudaMemcpyDeviceToHost);
      const double t = cs[k] * l;
      sx = sx + t * nxv;
      sy = sy + t * nyv;
    }
    put_err("build_mesh: cell " + std::to_string(c) +
                " fails the closed-polygon identity (residual " + std::to_string(hnorm(sx, sy)) + ")",
            err, errlen);
    return bail(SWE_INVALID);
  }
  *out = b;
  return SWE_OK;
}

int swe_dev_built_sizes(swe_built_mesh* b, int* n_nodes, int* n_cells, int* n_edges) {
  if (!b) return fail_invalid("null mesh");
  if (n_nodes) *n_nodes = b->nn;
  if (n_cells) *n_cells = b->nc;
  if (n_edges) *n_edges = b->ne;
  return SWE_OK;
}

int swe_dev_built_export(swe_built_mesh* b, int* cell_nodes, double* area, double* cx, double* cy,
                         double* inradius, int* cell_edge, int* cell_sign, int* edge_nodes,
                         int* edge_left, int* edge_right, double* nx, double* ny, double* len) {
  if (!b) return fail_invalid("null mesh");
  CK(cudaSetDevice(b->device));
  const size_t C = (size_t)b->nc, E = (size_t)b->ne;
  auto get = [&](void* dst, const void* src, size_t bytes) {
    return !dst || !bytes || cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) == cudaSuccess;
  };
  const bool ok = get(cell_nodes, b->cn, 12 * C) && get(area, b->area, 8 * C) &&
                  get(cx, b->cx, 8 * C) && get(cy, b->cy, 8 * C) && get(inradius, b->inr, 8 * C) &&
                  get(cell_edge, b->ce, 12 * C) && get(cell_sign, b->cs, 12 * C) &&
                  get(edge_nodes, b->en, 8 * E) && get(edge_left, b->el, 4 * E) &&
                  get(edge_right, b->er, 4 * E) && get(nx, b->nx, 8 * E) && get(ny, b->ny, 8 * E) &&
                  get(len, b->len, 8 * E);
  if (!ok) return cuda_ok(cudaGetLastError(), "swe_dev_built_export") ? SWE_CUDA : SWE_CUDA;
  return SWE_OK;
}

void swe_dev_built_free(swe_built_mesh* b) { delete b; }

int swe_dev_cell_order(swe_dev_ctx* x, int* order) {
  if (!x || !order) return fail_invalid("swe_dev_cell_order: null argument");
  CK(cudaMemcpy(order, x->d.c_orig, sizeof(int) * (size_t)x->d.C, cudaMemcpyDeviceToHost));
  return SWE_OK;
}

int swe_dev_cell_skip(swe_dev_ctx* x, unsigned char* skipped) {
  if (!x || !skipped) return fail_invalid("swe_dev_cell_skip: null argument");
  const int C = x->d.C;
  if (int rc = sync_ctl(x)) return rc;
  unsigned char* dv = nullptr;
  CK(cudaMalloc(&dv, (size_t)C));
  if (x->d.skip && x->persistent) {
    k_cell_skip_run<<<blocks_for(C), kBlock, 0, x->stream>>>(x->d, x->h_ctl->step, dv);
    ++g_launches;
  } else if (x->d.skip) {
    k_cell_skip<<<blocks_for(C), kBlock, 0, x->stream>>>(x->d, (int)(x->h_ctl->step + 1), dv);
    ++g_launches;
  } else {
    CK(cudaMemsetAsync(dv, 0, (size_t)C, x->stream));
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(skipped, dv, (size_t)C, cudaMemcpyDeviceToHost, x->stream));
  CK(cudaStreamSynchronize(x->stream));
  cudaFree(dv);
  return SWE_OK;
}

void* swe_dev_stream(swe_dev_ctx* x) { return x ? (void*)x->stream : nullptr; }

long long swe_dev_memory_bytes(swe_dev_ctx* x) { return x ? x->bytes : 0; }

int swe_dev_point_eval(int kind, long long n, const swe_params* p, const double* l,
                       const double* r, const double* z, const double* nrm, double* out) {
  if (n <= 0) return SWE_OK;
  if (!p || !l || !out) return fail_invalid("swe_dev_point_eval: null argument");
  if (kind < 0 || kind > 9) return fail_invalid("swe_dev_point_eval: unknown kind");
  static const size_t kOutW[10] = {3, 3, 6, 3, 1, 3, 3, 12, 1, 5};
  const size_t outw = kOutW[kind];
  // one packed staging buffer (pinned host + device, grown on demand, reused):
  // a call is one copy in, one kernel, one copy out -- the drop-in
  // kernels.hpp entry points are called per point by the reference's tests
  struct Scratch {
    double* host = nullptr;
    double* dev = nullptr;
    size_t cap = 0;  // doubles
    cudaStream_t s = nullptr;
  };
  static thread_local Scratch sc;
  const size_t in_n = 10 * (size_t)n, need = in_n + outw * (size_t)n;
  if (need > sc.cap) {
    if (sc.host) cudaFreeHost(sc.host);
    if (sc.dev) cudaFree(sc.dev);
    sc.host = nullptr;
    sc.dev = nullptr;
    sc.cap = 0;
    const size_t cap = std::max<size_t>(need, 4096);
    CK(cudaMallocHost(&sc.host, sizeof(double) * cap));
    CK(cudaMalloc(&sc.dev, sizeof(double) * cap));
    sc.cap = cap;
  }
  if (!sc.s) CK(cudaStreamCreateWithFlags(&sc.s, cudaStreamNonBlocking));
  double* h = sc.host;
  std::memcpy(h, l, sizeof(double) * 3 * n);
  if (r) std::memcpy(h + 3 * n, r, sizeof(double) * 3 * n);
  if (z) std::memcpy(h + 6 * n, z, sizeof(double) * 2 * n);
  if (nrm) std::memcpy(h + 8 * n, nrm, sizeof(double) * 2 * n);
  double* d = sc.dev;
  CK(cudaMemcpyAsync(d, h, sizeof(double) * in_n, cudaMemcpyHostToDevice, sc.s));
  const Phys P{p->g, p->h_dry, p->cfl, p->dt_max, p->h_ref};
  k_point<<<blocks_for(n), kBlock, 0, sc.s>>>(kind, n, P, d, d + 3 * n, d + 6 * n, d + 8 * n,
                                              d + in_n);
  ++g_launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(h + in_n, d + in_n, sizeof(double) * outw * n, cudaMemcpyDeviceToHost, sc.s));
  CK(cudaStreamSynchronize(sc.s));
  std::memcpy(out, h + in_n, sizeof(double) * outw * n);
  return SWE_OK;
}

int swe_dev_stable_dt(int device, long long n, const swe_params* p, const double* h,
                      const double* qx, const double* qy, const double* inradius, double* dt,
                      long long* bad_cell) {
  if (!p || !dt || (n > 0 && (!h || !qx || !qy || !inradius)))
    return fail_invalid("swe_dev_stable_dt: null argument");
  if (bad_cell) *bad_cell = -1;
  const Phys P{p->g, p->h_dry, p->cfl, p->dt_max, p->h_ref};
  if (n <= 0) {
    *dt = P.dt_max;
    return SWE_OK;
  }
  CK(cudaSetDevice(device));
  double* buf = nullptr;
  CK(cudaMalloc(&buf, sizeof(double) * (4 * (size_t)n + 2)));
  struct Free {
    void* q;
    ~Free() { cudaFree(q); }
  } guard{buf};
  const double* in[4] = {h, qx, qy, inradius};
  for (int k = 0; k < 4; ++k)
    CK(cudaMemcpy(buf + k * (size_t)n, in[k], sizeof(double) * n, cudaMemcpyHostToDevice));
  double* lo = buf + 4 * (size_t)n;
  auto* bad = reinterpret_cast<unsigned long long*>(lo + 1);
  double init[2] = {INFINITY, 0.0};
  const unsigned long long none = ~0ULL;  // bad = ULLONG_MAX
  std::memcpy(&init[1], &none, sizeof(none));
  CK(cudaMemcpy(lo, init, sizeof(init), cudaMemcpyHostToDevice));
  const int grid = (int)std::min<long long>(blocks_for(n), 148 * 8);
  k_stable_dt<<<grid, kBlock>>>(n, P, buf, buf + n, buf + 2 * (size_t)n, buf + 3 * (size_t)n, lo, bad);
  ++g_launches;
  CK(cudaGetLastError());
  double out[2];
  CK(cudaMemcpy(out, lo, sizeof(out), cudaMemcpyDeviceToHost));
  unsigned long long b;
  std::memcpy(&b, &out[1], sizeof(b));
  if (b != ~0ULL) {  // kernels.hpp:182-183
    if (bad_cell) *bad_cell = (long long)b;
    return SWE_NONFINITE_SPEED;
  }
  *dt = std::isfinite(out[0]) ? P.cfl * out[0] : P.dt_max;  // kernels.hpp:185
  return SWE_OK;
}

int swe_dev_mass(int device, long long n, const double* h, const double* area, double* mass) {
  if (!mass || (n > 0 && (!h || !area))) return fail_invalid("swe_dev_mass: null argument");
  *mass = 0.0;
  if (n <= 0) return SWE_OK;
  CK(cudaSetDevice(device));
  constexpr int kParts = 1024;
  double* buf = nullptr;
  CK(cudaMalloc(&buf, sizeof(double) * (2 * (size_t)n + kParts + 1)));
  struct Free {
    void* q;
    ~Free() { cudaFree(q); }
  } guard{buf};
  CK(cudaMemcpy(buf, h, sizeof(double) * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(buf + n, area, sizeof(double) * n, cudaMemcpyHostToDevice));
  double* part = buf + 2 * (size_t)n;
  k_mass_parts<<<kParts, kBlock>>>(n, buf, buf + n, part);
  k_mass_final<<<1, kBlock>>>(kParts, part, part + kParts);
  g_launches += 2;
  CK(cudaGetLastError());
  CK(cudaMemcpy(mass, part + kParts, sizeof(double), cudaMemcpyDeviceToHost));
  return SWE_OK;
}

int swe_dev_step_timed(swe_dev_ctx* x, double t_end, swe_step_record* rec, swe_status* st,
                       double* flux_ms, double* update_ms) {
  if (!x) return fail_invalid("null context");
  if (x->linked) return fail_invalid("swe_dev_step_timed: not available on a linked context");
  Dev& d = x->d;
  if (!d.TM) {  // per-incidence contribution slots of the two-phase kernels
    d.TM = x->alloc<double>(3 * (size_t)d.C);
    d.TX = x->alloc<double>(3 * (size_t)d.C);
    d.TY = x->alloc<double>(3 * (size_t)d.C);
    if (!d.TY) return fail_invalid("swe_dev_step_timed: cudaMalloc failed"), SWE_CUDA;
    // (the run graph holds a copy of Dev without these slots: it never uses them)
  }
  if (int rc = ensure_cfl(x)) return rc;
  if (int rc = write_params(x, t_end, LLONG_MAX, INFINITY, 1, 0, 1)) return rc;
  if (int rc = launch_gate(x)) return rc;
  cudaEvent_t ev[3];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  struct Destroy {
    cudaEvent_t* e;
    ~Destroy() {
      for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  // the two-phase kernels (bit-identical to the fused step) so the flux and
  // update phases are timed apart, as the reference's StepStats timers
  // (engine.hpp:314-317); the CFL bound is fused into the previous update
  CK(cudaEventRecord(ev[0], x->stream));
  k_face_c<<<x->grid_face, kBlock, 0, x->stream>>>(d);
  CK(cudaEventRecord(ev[1], x->stream));
  k_cell_c<<<x->grid_cell, kBlock, 0, x->stream>>>(d);
  g_launches += 2;
  CK(cudaGetLastError());
  // k_cell_c wrote grid_cell partials: finalize reduces those
  k_finalize<<<1, kBlock, 0, x->stream>>>(d, x->grid_cell, cudaGraphConditionalHandle{}, 0);
  ++g_launches;
  CK(cudaGetLastError());
  CK(cudaEventRecord(ev[2], x->stream));
  const int code = read_status(x, st);
  float a = 0.f, b = 0.f;
  CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
  CK(cudaEventElapsedTime(&b, ev[1], ev[2]));
  if (flux_ms) *flux_ms = a;
  if (update_ms) *update_ms = b;
  if (code == SWE_OK && rec)
    CK(cudaMemcpy(rec, x->rec, sizeof(swe_step_record), cudaMemcpyDeviceToHost));
  return code;
}

}  // extern "C"
