/*
 * swe_dev.h -- C-ABI of the B200 explicit HLLC shallow-water step.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/swe/engine.hpp).  Plain pointers and sizes,
 * no C++ or torch types; every entry point returns an int status (SWE_OK = 0)
 * and never throws.  Host C++ (include/swe/engine.hpp) maps the codes back to
 * the reference's exception types and message texts; Python reaches the same
 * symbols through ctypes (paper_1807_00672_b200/_lib.py).
 *
 * Numbering: every array crossing this boundary is in the REFERENCE numbering
 * (the cell/edge order build_mesh produces, mesh.hpp:121-240).  The device
 * renumbers cells and edges internally for locality (Morton order of
 * centroids) and permutes state on upload/download; error indices are mapped
 * back to reference numbering (lowest index wins, as the sequential backend).
 *
 * Threading: one context is driven from one host thread (the reference's
 * Simulation is not re-entrant either, SPEC.md "Concurrency Model").
 */
#ifndef SWE_DEV_H
#define SWE_DEV_H

#ifndef SWE_API
#if defined(__GNUC__)
#define SWE_API __attribute__((visibility("default")))
#else
#define SWE_API
#endif
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct swe_dev_ctx swe_dev_ctx;

/* swe::PhysParams (core.hpp:36-42) */
typedef struct {
  double g, h_dry, cfl, dt_max, h_ref;
} swe_params;

/* The arrays of swe::Mesh the step consumes (mesh.hpp:33-61), as SoA views
 * in reference numbering.  cx/cy (cell centroids) drive the locality
 * renumbering; pass NULL to keep the reference order. */
typedef struct {
  int n_cells, n_edges;
  const double* area;     /* [C] cell_area */
  const double* inradius; /* [C] cell_inradius */
  const double* bed;      /* [C] cell_bed */
  const double* manning;  /* [C] cell_manning */
  const double* cx;       /* [C] cell_centroid.x (optional) */
  const double* cy;       /* [C] cell_centroid.y (optional) */
  const int* cell_edge;   /* [3C] cell_edges[c][k].edge, CCW local order */
  const int* cell_sign;   /* [3C] cell_edges[c][k].sign (+1 left, -1 right) */
  const int* edge_left;   /* [E] */
  const int* edge_right;  /* [E] -1 (kBoundary) for reflective walls */
  const double* nx;       /* [E] edge_normal.x */
  const double* ny;       /* [E] edge_normal.y */
  const double* len;      /* [E] edge_length */
  /* multi-device runs: cells [0, n_owned) are owned and updated, the rest
   * are ghosts (read-only copies of neighbours, refreshed by the halo
   * exchange); every edge must touch an owned cell.  0 = all owned. */
  int n_owned;
} swe_mesh_view;

enum {
  SWE_OK = 0,
  SWE_NONFINITE_SPEED = 1, /* stable_dt: non-finite velocity in cell N (engine.hpp:205-206) */
  SWE_NEGATIVE_DEPTH = 2,  /* compute_fluxes: negative depth at edge N (engine.hpp:168-169) */
  SWE_BLOWUP = 3,          /* advance_step: numeric blowup (engine.hpp:292-297) */
  SWE_CUDA = 4,            /* CUDA runtime failure (message via swe_dev_last_error) */
  SWE_NCCL = 5,            /* multi-device exchange failure (a peer did not post in time) */
  SWE_INVALID = 6          /* bad argument / inconsistent mesh view */
};

/* Outcome of a step call.  index is a reference-numbered cell or edge; on
 * SWE_BLOWUP, step/dt/h carry the values the reference prints. */
typedef struct {
  int code;
  long long index;
  long long step;
  double dt;
  double h;
} swe_status;

/* One row of RunStats::series (engine.hpp:99-107, without wall clocks). */
typedef struct {
  long long step;
  double t, dt, max_speed, mass;
} swe_step_record;

/* create flags */
#define SWE_FLAG_IDENTITY_ORDER 1u /* skip the Morton renumbering */
#define SWE_FLAG_NO_GRAPH 2u       /* advance with plain launches: no CUDA graph and no
                                      persistent step kernel */
#define SWE_FLAG_TWO_PHASE 4u      /* face kernel + cell kernel (records through HBM)
                                      instead of the fused tile kernel */

/* Uploads the mesh, renumbers it on the device, allocates the double-buffered
 * state and edge records.  device = CUDA ordinal.  One context drives one GPU
 * (SURVEY.md §8(b) sketched one context over n_gpus driven from one thread);
 * a multi-GPU run is one context per GPU and process, joined by
 * swe_dev_link (below), so every rank keeps its own stream and graph. */
SWE_API int swe_dev_create(const swe_mesh_view* mesh, const swe_params* params, int device,
                   unsigned flags, swe_dev_ctx** out);
SWE_API int swe_dev_destroy(swe_dev_ctx* ctx);

/* Host state in/out (reference numbering); copies are synchronous.  set_state
 * also resets the CFL cache so the next step recomputes it from this state. */
SWE_API int swe_dev_set_state(swe_dev_ctx* ctx, const double* h, const double* qx, const double* qy,
                      double t, long long step);
SWE_API int swe_dev_get_state(swe_dev_ctx* ctx, double* h, double* qx, double* qy, double* t,
                      long long* step);
/* Same, with DEVICE pointers (reference numbering) -- no host copies. */
SWE_API int swe_dev_set_state_device(swe_dev_ctx* ctx, const double* d_h, const double* d_qx,
                             const double* d_qy, double t, long long step);
SWE_API int swe_dev_get_state_device(swe_dev_ctx* ctx, double* d_h, double* d_qx, double* d_qy);

/* The clip ledger (engine.hpp:85-89). */
SWE_API int swe_dev_get_ledger(swe_dev_ctx* ctx, double* clipped_volume, long long* clip_events);
SWE_API int swe_dev_set_ledger(swe_dev_ctx* ctx, double clipped_volume, long long clip_events);

/* One advance_step (engine.hpp:226-319): CFL from the current state, truncated
 * to land on t_end, flux, update, friction, clamp.  rec may be NULL. */
SWE_API int swe_dev_step(swe_dev_ctx* ctx, double t_end, swe_step_record* rec, swe_status* st);

/* The run() time loop body (engine.hpp:355-380) on the device: steps while
 * t < t_end, step < max_steps and t < next_snapshot - 1e-12, at most
 * max_records steps; one record per step into series (host array, may be
 * NULL when max_records is given only as a bound).  The whole loop is one
 * CUDA graph launch (conditional WHILE node).  *n_done = steps taken. */
SWE_API int swe_dev_advance(swe_dev_ctx* ctx, double t_end, long long max_steps, double next_snapshot,
                    swe_step_record* series, long long max_records, long long* n_done,
                    swe_status* st);

/* Exactly n steps (t_end = +inf semantics of the bench harness,
 * bench.hpp:91-110), asynchronous on the context stream: no host sync, no
 * record download.  Status is checked by the next synchronous call. */
SWE_API int swe_dev_advance_n_async(swe_dev_ctx* ctx, long long n, double t_end);
/* swe_dev_advance split in two: enqueue the graph launch (no host sync when
 * the CFL cache is known valid), then collect status + records. */
SWE_API int swe_dev_advance_async(swe_dev_ctx* ctx, double t_end, long long max_steps,
                                  double next_snapshot, long long max_records);
SWE_API int swe_dev_records(swe_dev_ctx* ctx, swe_step_record* series, long long max_records,
                            long long* n_done, swe_status* st);
SWE_API int swe_dev_synchronize(swe_dev_ctx* ctx, swe_status* st);

/* Asynchronous snapshot of the current state (as of this point in the
 * context's stream) into host arrays h/qx/qy [C] (reference numbering; pinned
 * memory -- swe_dev_host_alloc -- lets the copy overlap later steps).  Two
 * slots: a slot's previous copy is waited for before it is reused.
 * swe_dev_snapshot_wait blocks until the slot's copy has landed. */
SWE_API int swe_dev_snapshot_async(swe_dev_ctx* ctx, int slot, double* h, double* qx, double* qy);
SWE_API int swe_dev_snapshot_wait(swe_dev_ctx* ctx, int slot);
/* Page-locked host memory (cudaMallocHost) for callers without CUDA headers. */
SWE_API void* swe_dev_host_alloc(long long bytes);
SWE_API void swe_dev_host_free(void* p);
/* Page-lock (cudaHostRegister) / release existing host memory, e.g. the
 * caller's state vectors, so snapshot copies land in them at full speed. */
SWE_API int swe_dev_host_register(void* p, long long bytes);
SWE_API int swe_dev_host_unregister(void* p);

/* compute_fluxes (engine.hpp:138-170) on the current state; left/right are
 * [3E] Flux3 arrays in reference numbering. */
SWE_API int swe_dev_compute_fluxes(swe_dev_ctx* ctx, double* left, double* right, swe_status* st);

/* total_mass (engine.hpp:128-132) of the current state (fixed-order tree sum). */
SWE_API int swe_dev_total_mass(swe_dev_ctx* ctx, double* mass);

/* ---- multi-device (domain decomposition, include/swe/partition.hpp) ----
 * One context per part.  Per step the driver (1) exchanges ghost states --
 * pack the owned cells peers need into a device buffer, move it (NCCL or a
 * peer copy), unpack into the ghosts -- (2) reduces the parts' local CFL
 * bounds (min dts, max max_speed), (3) steps every part with the global
 * bound.  Cell lists are in the context's reference (local) numbering;
 * buffers are DEVICE pointers of 3 doubles (h, qx, qy) per cell.  Pack /
 * unpack complete before returning. */
SWE_API int swe_dev_set_halo_plan(swe_dev_ctx* ctx, int n_send, const int* send_cells, int n_recv,
                                  const int* recv_cells);
SWE_API int swe_dev_pack_halo(swe_dev_ctx* ctx, double* d_buf);
SWE_API int swe_dev_unpack_halo(swe_dev_ctx* ctx, const double* d_buf);
/* CFL bound of the owned cells' current state: cfl * min(r / speed) (or
 * dt_max), max signal speed, owned mass.  Status SWE_NONFINITE_SPEED (with
 * st->index) if an owned cell has a non-finite speed. */
SWE_API int swe_dev_local_cfl(swe_dev_ctx* ctx, double* dts, double* max_speed, double* mass,
                              swe_status* st);
/* advance_step with the globally reduced bound (engine.hpp:235-237 applied to
 * dts; max_speed is recorded); rec->mass is the owned mass after the step. */
SWE_API int swe_dev_step_global(swe_dev_ctx* ctx, double t_end, double dts, double max_speed,
                                swe_step_record* rec, swe_status* st);

/* ---- linked contexts: the device-resident multi-device step ----
 * The production multi-GPU path: no host round trip per step.
 * Each rank's state buffers and a mailbox live in one device allocation (the
 * arena) that every peer maps.  The step kernel stores the new state of the
 * owned cells a peer holds as ghosts directly into that peer's next state
 * buffer over NVLink; the step outcome (CFL bound, max speed, mass, clip
 * ledger, error) is posted to every rank's mailbox and combined in rank
 * order, so all ranks commit the same dt sequence, records and ledger, and
 * the results are bit-identical to one device (the mass is a rank-ordered
 * sum).  After linking, swe_dev_advance / swe_dev_advance_n_async run the
 * whole exchange inside the CUDA graph; every rank must make the same calls
 * (advance, set_state, total_mass are collective).  Error indices of a linked
 * context are GLOBAL ids (gcell / gedge).  A peer that does not post within
 * timeout_s yields SWE_NCCL instead of a hang. */
/* This rank's arena (device pointer) and its CUDA IPC handle (64 bytes). */
SWE_API int swe_dev_link_export(swe_dev_ctx* ctx, void** arena, unsigned char* ipc_handle);
/* Link the context as `rank` of `nranks`.  Peers' arenas come either as
 * pointers valid in this process (arenas[q], contexts of this process, same
 * or peer-enabled devices) or as IPC handles (ipc_handles[64*q], other
 * processes; a NULL arenas[q] falls back to ipc_handles for that rank).
 * peer_cells[q] = n_cells of rank q.  Push entry j sends owned
 * cell push_cell[j] (reference-local id) to ghost push_ghost[j] (local id on
 * rank push_rank[j]).  gcell[C] / gedge[E]: local -> global ids (NULL =
 * identity). */
SWE_API int swe_dev_link(swe_dev_ctx* ctx, int rank, int nranks, void* const* arenas,
                         const unsigned char* ipc_handles, const long long* peer_cells, int n_push,
                         const int* push_cell, const int* push_rank, const int* push_ghost,
                         const int* gcell, const int* gedge, double timeout_s);
/* One phase of a linked single step, enqueued only (lockstep driving of
 * several linked contexts from one thread, e.g. parts sharing one device):
 * 0 open, 1 CFL wait + gate, 2 step kernel + halo push, 3 post, 4 wait +
 * commit.  Run phase k on every context before phase k+1 on any. */
SWE_API int swe_dev_link_phase(swe_dev_ctx* ctx, int phase, double t_end);
/* P linked contexts (ranks 0..P-1, persistent kernel, all on ONE device)
 * stepped nsteps steps by ONE cooperative launch of the persistent step
 * kernel: the ranks' CTAs run concurrently and exchange through the device
 * mailboxes as on P GPUs (separate launches that wait on each other must not
 * share a device).  grid: CTAs per rank, one of them the rank's control block
 * (0 = as many as fit).  Test path for
 * the concurrent exchange protocol; returns the first rank's error status. */
SWE_API int swe_dev_run_ranks(swe_dev_ctx* const* ctxs, int n, long long nsteps, double t_end,
                              int grid);
/* Experiment builds (-DSWE_RUN_TIMING=1): phase-time sums of the persistent
 * step kernel [worker work ns, worker epoch-wait ns, control wait for the
 * arrivals ns, commit ns, worker CTA-steps, commits, worker arrival-wait ns],
 * read and cleared (zeros in normal builds). */
SWE_API int swe_dev_run_timing(swe_dev_ctx* ctx, long long* out, int n);
/* Status and record of the last single step (after phase 4). */
SWE_API int swe_dev_last_record(swe_dev_ctx* ctx, swe_step_record* rec, swe_status* st);

/* Kernel-level timing: when enabled, swe_dev_advance_n_async launches without
 * a graph and brackets every kernel with CUDA events; times accumulate per
 * kernel (ms): [0] face, [1] cell, [2] finalize, [3] cfl. */
SWE_API int swe_dev_set_profiling(swe_dev_ctx* ctx, int on);
SWE_API int swe_dev_kernel_times(swe_dev_ctx* ctx, double* ms, long long* launches, int n);

/* Layout facts: [0] fused?, [1] cells per tile, [2] tiles, [3] max slots per
 * tile, [4] halo edges, [5] tile grid, [6] face grid, [7] cell grid,
 * [8] tile shared-memory bytes, [9] edges, [10] dry-tile skipping on?,
 * [11] dry tiles skipped so far (n > 11 synchronises the context),
 * [12] steps per WHILE iteration of the run graph, [13] run loop is the
 * persistent kernel?, [14] its CTAs, [15] of the skipped tiles, those whose
 * next state was already in place (no writes). */
SWE_API int swe_dev_info(swe_dev_ctx* ctx, long long* out, int n);

/* Per cell (reference numbering): 1 if dry-tile skipping will skip the cell's
 * tile in the next step (the measured cost pattern behind cost-weighted
 * partitions, paper_1807_00672_b200/dist.py measured_cost_weights). */
SWE_API int swe_dev_cell_skip(swe_dev_ctx* ctx, unsigned char* skipped);

/* The device cell order: order[i] = reference cell stored at device position
 * i (the blocked-Hilbert renumbering; ghosts of a part keep their place). */
SWE_API int swe_dev_cell_order(swe_dev_ctx* ctx, int* order);

/* cudaStream_t of the context (as void*), for events on the launching stream. */
SWE_API void* swe_dev_stream(swe_dev_ctx* ctx);
/* Device bytes held by the context. */
SWE_API long long swe_dev_memory_bytes(swe_dev_ctx* ctx);
/* Kernels launched by this process through any context. */
SWE_API long long swe_dev_launch_count(void);

/* Point physics on the device over arrays (kernel-level parity and the
 * drop-in kernels.hpp entry points, reference kernels.hpp:15-216):
 * kind 0 hllc_flux(l,r,n), 1 wall_flux(l,n), 2 edge combine(l,r,z,n) -> out[6],
 * 3 apply_friction(l, z[0]=n_manning, z[1]=dt), 4 pow(h, 4/3) (l[0]=h),
 * 5 physical_flux_normal(l,n), 6 wave_speed_estimates(hL=l[0], uL=l[1],
 * hR=r[0], uR=r[1]) -> {SL, S*, SR}, 7 hydrostatic_reconstruct(l, z[0], r,
 * z[1], n) -> out[12] = {left, right, corr_left, corr_right},
 * 8 cell_signal_speed(l) -> out[1], 9 clamp_dry(l) -> out[5] = {h, qx, qy,
 * clipped depth, 1 if it throws}.
 * l, r: [3n]; z: [2n]; nrm: [2n]; out: [w n], w = 3 except as noted. */
SWE_API int swe_dev_point_eval(int kind, long long n, const swe_params* params, const double* l,
                       const double* r, const double* z, const double* nrm, double* out);
/* stable_dt (kernels.hpp:174-186) of host arrays [n] on the device: *dt =
 * cfl * min over wet cells of inradius / signal speed, or dt_max when all are
 * dry; SWE_NONFINITE_SPEED with *bad_cell = the lowest offending cell. */
SWE_API int swe_dev_stable_dt(int device, long long n, const swe_params* params, const double* h,
                              const double* qx, const double* qy, const double* inradius,
                              double* dt, long long* bad_cell);
/* total_mass (engine.hpp:128-132) of host arrays [n] on the device, a
 * fixed-order tree sum of h * area; stateless (touches no context). */
SWE_API int swe_dev_mass(int device, long long n, const double* h, const double* area,
                         double* mass);
/* One advance_step like swe_dev_step, through the two-phase kernels with the
 * flux and update phases timed apart by CUDA events (StepStats timers,
 * engine.hpp:314-317); results are the fused step's, bit for bit. */
SWE_API int swe_dev_step_timed(swe_dev_ctx* ctx, double t_end, swe_step_record* rec,
                               swe_status* st, double* flux_ms, double* update_ms);

/* build_mesh (mesh.hpp:121-240) on the device: same numbering, geometry and
 * error texts as the host build_mesh (include/swe/mesh.hpp).  xy [2*n_nodes],
 * tris [3*n_cells].  SWE_INVALID with the reference's mesh_error text in err.
 * Export arrays (any may be NULL): cell_nodes/cell_edge/cell_sign [3C],
 * area/cx/cy/inradius [C], edge_nodes [2E], edge_left/right, nx/ny/len [E]. */
typedef struct swe_built_mesh swe_built_mesh;
SWE_API int swe_dev_build_mesh(int device, int n_nodes, const double* xy, int n_cells,
                               const int* tris, swe_built_mesh** out, char* err, int errlen);
SWE_API int swe_dev_built_sizes(swe_built_mesh* mesh, int* n_nodes, int* n_cells, int* n_edges);
SWE_API int swe_dev_built_export(swe_built_mesh* mesh, int* cell_nodes, double* area, double* cx,
                                 double* cy, double* inradius, int* cell_edge, int* cell_sign,
                                 int* edge_nodes, int* edge_left, int* edge_right, double* nx,
                                 double* ny, double* len);
SWE_API void swe_dev_built_free(swe_built_mesh* mesh);

SWE_API const char* swe_dev_strerror(int code);
/* Last CUDA/argument error message of this thread. */
SWE_API const char* swe_dev_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
