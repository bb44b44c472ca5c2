/*
 * swe_host.h -- C-ABI of the host-side input producers of the drop-in API
 * (include/swe/mesh.hpp, include/swe/cases.hpp): raw triangulations, the
 * reference's build_mesh (mesh.hpp:121-240) and the case/scenario field
 * initialisers (cases.hpp:114-193).  Not on the step path; these feed
 * swe_dev_create / swe_dev_set_state from Python (ctypes) and C callers.
 * Handles are opaque; errors return NULL / non-zero with the reference's
 * exception text in err.
 */
#ifndef SWE_HOST_H
#define SWE_HOST_H

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

SWE_API void* swe_host_raw_square(int nx, int ny, double lx, double ly, char* err, int errlen);
SWE_API void* swe_host_raw_unstructured(int nx, int ny, double lx, double ly, double jitter,
                                unsigned long long seed, char* err, int errlen);
SWE_API void* swe_host_raw_arrays(int n_nodes, const double* xy, int n_cells, const int* tris);
SWE_API void swe_host_raw_sizes(void* raw, int* n_nodes, int* n_cells);
SWE_API void swe_host_raw_export(void* raw, double* xy, int* tris);
SWE_API void swe_host_raw_free(void* raw);

/* reference case by name ("water_drop", "three_mounds", "lake_at_rest",
 * "dam_break_1d"); spec = {lx, ly, eta0, amplitude, sigma, manning, h_left,
 * h_right, x_dam, t_end} or NULL for make_case defaults.  Returns 0 or an
 * error kind (1 numeric, 2 config, 3 mesh, 4 case). */
SWE_API int swe_host_case_defaults(const char* name, double* spec);
SWE_API int swe_host_init_case(void* raw, const char* name, const double* spec, double* bed,
                       double* manning, double* h, double* qx, double* qy, char* err, int errlen);

/* benchmark configuration (cases.hpp make_scenario): returns a handle that
 * owns a raw mesh and its fields */
SWE_API void* swe_host_scenario(const char* name, double scale, int unstructured, unsigned long long seed,
                        int weak_nx, double* t_end, char* err, int errlen);
SWE_API void* swe_host_scenario_raw(void* scenario); /* borrowed */
SWE_API void swe_host_scenario_fields(void* scenario, double* bed, double* manning, double* h, double* qx,
                              double* qy);
SWE_API void swe_host_scenario_free(void* scenario);

/* build_mesh; bed/manning sized to the triangle count */
SWE_API void* swe_host_build_mesh(void* raw, const double* bed, const double* manning, char* err,
                          int errlen);
SWE_API void swe_host_mesh_sizes(void* mesh, int* n_cells, int* n_edges, int* n_boundary);
/* any output may be NULL; layouts as swe_mesh_view (cell_edge/sign [3C],
 * edge_nodes [2E], cell_nodes [3C]) */
SWE_API void swe_host_mesh_export(void* mesh, int* cell_nodes, double* area, double* cx, double* cy,
                          double* inradius, int* cell_edge, int* cell_sign, int* edge_nodes,
                          int* edge_left, int* edge_right, double* nx, double* ny, double* len);
SWE_API void swe_host_mesh_free(void* mesh);

/* domain decomposition (include/swe/partition.hpp): part id per cell by
 * recursive coordinate bisection */
SWE_API int swe_host_partition(void* mesh, int nparts, int* part_out);
/* the same with per-cell weights (equal weight per part; include/swe/partition.hpp
 * cost_weights gives the step's measured cost of wet vs dry cells) */
SWE_API int swe_host_partition_weighted(void* mesh, int nparts, const double* weights, int* part_out);
/* RCB of a RAW mesh's triangle centroids (weights may be NULL) */
SWE_API int swe_host_partition_raw(void* raw, int nparts, const double* weights, int* part_out);
/* part p's local mesh built from the raw mesh alone (include/swe/multigpu.hpp
 * build_rank_mesh: owned triangles + ghost layer; edge ids part-local);
 * the same handle type as swe_host_local_mesh */
SWE_API void* swe_host_rank_mesh(void* raw, const double* bed, const double* manning,
                                 const int* part, int p, char* err, int errlen);
/* part p's local mesh (owned cells first, then ghosts) and exchange plan */
SWE_API void* swe_host_local_mesh(void* mesh, const int* part, int p, char* err, int errlen);
SWE_API void swe_host_local_sizes(void* local, int* n_cells, int* n_owned, int* n_edges,
                                  int* n_peers, int* n_send, int* n_recv);
/* arrays in the layout of swe_mesh_view; any output may be NULL */
SWE_API void swe_host_local_export(void* local, int* cells, int* edges, double* area,
                                   double* inradius, double* bed, double* manning, double* cx,
                                   double* cy, int* cell_edge, int* cell_sign, int* edge_left,
                                   int* edge_right, double* nx, double* ny, double* len);
/* peers [n_peers]; per peer send/recv counts; flattened cell lists */
SWE_API void swe_host_local_plan(void* local, int* peers, int* send_counts, int* recv_counts,
                                 int* send_cells, int* recv_cells);
SWE_API void swe_host_local_free(void* local);

/* build_mesh on the GPU (include/swe/engine.hpp build_mesh_device): the same
 * Mesh handle as swe_host_build_mesh, computed by swe_dev_build_mesh. */
SWE_API void* swe_host_build_mesh_device(void* raw, const double* bed, const double* manning,
                                         int device, char* err, int errlen);

/* SWEMESH 1 mesh files (include/swe/swemesh.hpp; reference io.hpp:80-165):
 * parallel parse / format, the reference's values and error texts.  A file
 * handle owns a raw mesh (borrowed by swe_host_swemesh_raw, usable with
 * swe_host_raw_* and swe_host_build_mesh) + bed + manning.  threads <= 0:
 * all cores.  NULL / 7 (io error) with the message in err. */
SWE_API void* swe_host_swemesh_read(const char* path, int threads, char* err, int errlen);
SWE_API void* swe_host_swemesh_parse(const char* text, long long size, int threads, char* err,
                                     int errlen);
SWE_API void* swe_host_swemesh_raw(void* file);
SWE_API void swe_host_swemesh_fields(void* file, double* bed, double* manning);
SWE_API void swe_host_swemesh_free(void* file);
SWE_API int swe_host_swemesh_write(const char* path, void* raw, const double* bed,
                                   const double* manning, int threads, char* err, int errlen);

#ifdef __cplusplus
}
#endif
#endif
