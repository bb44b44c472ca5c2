// swe_prep.cuh -- device mesh preprocessor (run once per swe_dev_create):
// space-filling-curve renumbering of cells (blocked Hilbert),
// edge ordering by owner tile, the tile tables of the fused kernel, and the reference<->device permutation kernels.
// The reference layout it consumes is build_mesh's (mesh.hpp:121-240);
// orientation (left = reference left cell) and each cell's local edge order
// are preserved so every sum is formed in the reference's order.
#pragma once

#include "swe_ctl.cuh"

namespace swe_b200 {

// cell order: a blocked Hilbert curve (k_hilbert_blocks).  Measured on B200
// against Morton and one Hilbert curve over the bounding square (both
// removed): 1M three-mound -16%, 10M dry bed -2.5%, 10M channel +0.8% step
// time vs Morton

// 32-bit Hilbert index of (x, y) on a 65536^2 grid
__device__ __forceinline__ unsigned hilbert16(unsigned x, unsigned y) {
  unsigned d = 0;
  for (unsigned s = 1u << 15; s > 0; s >>= 1) {
    const unsigned rx = (x & s) ? 1u : 0u, ry = (y & s) ? 1u : 0u;
    d += s * s * ((3u * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = 65535u - x;
        y = 65535u - y;
      }
      const unsigned t = x;
      x = y;
      y = t;
    }
  }
  return d;
}

// The bounding box cut into squares along its long axis, each
// traversed by a 65536^2 Hilbert curve (a curve ends at the corner where the
// next square's begins); key = square index << 32 | Hilbert index (40 bits)
__global__ void k_hilbert_blocks(int C, const double* cx, const double* cy, double x0, double y0,
                                 double side, int long_is_y, unsigned long long* key, int* idx) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double a = (cx[c] - x0) / side, b = (cy[c] - y0) / side;
  if (long_is_y) {
    const double t = a;
    a = b;
    b = t;
  }
  const double blk = fmin(fmax(floor(a), 0.0), 255.0);
  const double fx = fmin(fmax((a - blk) * 65536.0, 0.0), 65535.0);
  const double fy = fmin(fmax(b * 65536.0, 0.0), 65535.0);
  key[c] = ((unsigned long long)blk << 32) | hilbert16((unsigned)fx, (unsigned)fy);
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

// edge order key: (owner tile, wall?, lower device cell); the owner tile is
// the tile of the edge's lower device cell (its only cell for a wall)
__global__ void k_edge_keys(int E, const int* el, const int* er, const int* c_new, int T,
                            unsigned long long* key, int* idx) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int l = c_new[el[e]];
  const int r = er[e] < 0 ? -1 : c_new[er[e]];
  const int lo = r < 0 ? l : min(l, r);
  key[e] = ((unsigned long long)(lo / T) << 33) | ((unsigned long long)(r < 0) << 32) |
           (unsigned long long)lo;
  idx[e] = e;
}

template <class V>
__global__ void k_gather(int n, const int* perm, const V* src, V* dst) {
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

__device__ __forceinline__ int owner_tile(const int* el, const int* er, int e, int T) {
  const int l = el[e], r = er[e];
  return (r < 0 ? l : min(l, r)) / T;
}

// eoff[t] = first edge owned by tile t (edges sorted by owner tile)
__global__ void k_tile_bounds(int E, const int* el, const int* er, int T, int ntiles, int* eoff) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int ow = owner_tile(el, er, e, T);
  const int prev = e == 0 ? -1 : owner_tile(el, er, e - 1, T);
  for (int t = prev + 1; t <= ow; ++t) eoff[t] = e;
  if (e == E - 1)
    for (int t = ow + 1; t <= ntiles; ++t) eoff[t] = E;
}

// interior edges between owned cells of different tiles -> (tile of the
// upper cell, edge).  Edges to a ghost cell (device id >= C_own) belong to
// the owned cell's tile alone.
__global__ void k_halo_keys(int E, const int* el, const int* er, int T, int C_own,
                            unsigned long long* key, int* count) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int r = er[e];
  if (r < 0 || r >= C_own || el[e] >= C_own) return;
  const int a = el[e] / T, b = r / T;
  if (a == b) return;
  const int slot = atomicAdd(count, 1);
  key[slot] = ((unsigned long long)max(a, b) << 32) | (unsigned)e;
}

__global__ void k_halo_bounds(int nh, const unsigned long long* key, int ntiles, int* hoff,
                              int* halo) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nh) return;
  const int t = (int)(key[j] >> 32);
  halo[j] = (int)(key[j] & 0xffffffffu);
  const int prev = j == 0 ? -1 : (int)(key[j - 1] >> 32);
  for (int u = prev + 1; u <= t; ++u) hoff[u] = j;
  if (j == nh - 1)
    for (int u = t + 1; u <= ntiles; ++u) hoff[u] = nh;
}

// staged tiles: slot arrays in tile order (one warp per tile)
__global__ void k_slots(Dev d, int* soff, int* sel, int* ser, int* skk, int* sedge, double* snx,
                        double* sny, double* slen) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= d.ntiles) return;
  const int e0 = d.eoff[t], no = d.eoff[t + 1] - e0;
  const int h0 = d.hoff[t], ns = no + d.hoff[t + 1] - h0;
  const int s0 = e0 + h0;  // slots before tile t: owned edges + halo edges before it
  if (lane == 0) {
    soff[t] = s0;
    if (t == d.ntiles - 1) soff[t + 1] = s0 + ns;
  }
  for (int j = lane; j < ns; j += 32) {
    const int e = j < no ? e0 + j : d.halo[h0 + (j - no)];
    sel[s0 + j] = d.el[e];
    ser[s0 + j] = d.er[e];
    skk[s0 + j] = d.kl[e] | (d.kr[e] << 8);
    sedge[s0 + j] = e;
    snx[s0 + j] = d.nx[e];
    sny[s0 + j] = d.ny[e];
    slen[s0 + j] = d.len[e];
  }
}

// dry-tile skipping: (tile, neighbour tile) pairs from every slot's two
// cells; slot j of tile t writes keys[2 (s0 + j) + side] (t << 32 | t when the
// cell is inside t or a wall)
__global__ void k_tile_pairs(Dev d, unsigned long long* keys) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= d.ntiles) return;
  const int e0 = d.eoff[t], no = d.eoff[t + 1] - e0;
  const int h0 = d.hoff[t], ns = no + d.hoff[t + 1] - h0;
  const int s0 = e0 + h0, c0 = t * d.T, c1 = min(c0 + d.T, d.C_own);
  for (int j = lane; j < ns; j += 32) {
    const int e = j < no ? e0 + j : d.halo[h0 + (j - no)];
    const int cs[2] = {d.el[e], d.er[e]};
    for (int k = 0; k < 2; ++k) {
      const int c = cs[k];
      unsigned long long nb = (unsigned)t;
      if (c >= 0 && (c < c0 || c >= c1)) nb = c >= d.C_own ? (unsigned)d.ntiles : (unsigned)(c / d.T);
      keys[2 * (size_t)(s0 + j) + k] = ((unsigned long long)t << 32) | nb;
    }
  }
}

__global__ void k_pair_bounds(int n, const unsigned long long* key, int ntiles, int* off, int* nbr) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int t = (int)(key[j] >> 32);
  nbr[j] = (int)(key[j] & 0xffffffffu);
  const int prev = j == 0 ? -1 : (int)(key[j - 1] >> 32);
  for (int u = prev + 1; u <= t; ++u) off[u] = j;
  if (j == n - 1)
    for (int u = t + 1; u <= ntiles; ++u) off[u] = n;
}

// per reference cell: 1 if its tile is skipped in the next step (dry-tile
// skipping), for cost-weighted partitions
__global__ void k_cell_skip(Dev d, int tag, unsigned char* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d.C) return;
  out[d.c_orig[c]] = (c < d.C_own && d.skipmask[c / d.T] == tag) ? 1 : 0;
}

__global__ void k_fill_int(int n, int* v, int value) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = value;
}

// local index k (0..2, the reference's CCW order) of each edge in its left
// and right cell; every (edge, side) has exactly one writer.  kr of a wall
// stays 0xff.
__global__ void k_local_index(int C, const int* i0, const int* i1, const int* i2,
                              unsigned char* kl, unsigned char* kr) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int inc[3] = {i0[c], i1[c], i2[c]};
  for (int k = 0; k < 3; ++k) (inc[k] & 1 ? kr : kl)[inc[k] >> 1] = (unsigned char)k;
}

__global__ void k_local_check(int E, const int* er, const unsigned char* kl,
                              const unsigned char* kr, int* bad) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  if (kl[e] > 2 || (er[e] >= 0 && kr[e] > 2)) atomicExch(bad, 2);
}

// k_tile's packed edge records (Dev::ek, Dev::enxy); cells < 2^30 (checked)
__global__ void k_pack_edges(int E, const int* el, const int* er, const unsigned char* kl,
                             const unsigned char* kr, const double* nx, const double* ny,
                             int2* ek, double2* enxy) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int r = er[e];
  ek[e] = make_int2(el[e] | ((int)kl[e] << 30), r < 0 ? -1 : (r | ((int)kr[e] << 30)));
  enxy[e] = make_double2(nx[e], ny[e]);
}

// k_tile's cell records (Dev::cg)
__global__ void k_pack_cells(int C, const double* z, const double* area, const double* man,
                             const double* inr, CellGeo* cg) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  cg[c] = CellGeo{z[c], area[c], man[c], inr[c]};
}

// multi-device halo exchange: owned cells' current state -> buffer (h, qx, qy
// interleaved), buffer -> ghost cells' current state
__global__ void k_halo_pack(Dev d, double* buf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n_send) return;
  const int cur = d.ctl->cur, c = d.send_cells[i];
  buf[3 * (size_t)i] = d.h[cur][c];
  buf[3 * (size_t)i + 1] = d.qx[cur][c];
  buf[3 * (size_t)i + 2] = d.qy[cur][c];
}

__global__ void k_halo_unpack(Dev d, const double* buf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n_recv) return;
  const int cur = d.ctl->cur, c = d.recv_cells[i];
  d.h[cur][c] = buf[3 * (size_t)i];
  d.qx[cur][c] = buf[3 * (size_t)i + 1];
  d.qy[cur][c] = buf[3 * (size_t)i + 2];
}

__global__ void k_map_cells(int n, const int* c_new, int* cells) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cells[i] = c_new[cells[i]];
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

// current state (buffer chosen on the device, for snapshots enqueued behind
// asynchronous launches) -> reference order
__global__ void k_snapshot(Dev d, double* h, double* qx, double* qy) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= d.C) return;
  const int cur = d.ctl->cur, c = d.c_new[o];
  h[o] = d.h[cur][c];
  qx[o] = d.qx[cur][c];
  qy[o] = d.qy[cur][c];
}

// edge records -> reference left/right Flux3 arrays (compute_fluxes layout)
__global__ void k_flux_out(Dev d, double* left, double* right) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= d.E) return;
  const int o = d.e_orig[e];
  const bool wall_e = d.er[e] < 0;
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
  } else if (kind == 5) {  // physical_flux_normal, kernels.hpp:21-27
    const Flux f = normal_flux(a, nrm[2 * i], nrm[2 * i + 1], P);
    out[3 * i] = f.m;
    out[3 * i + 1] = f.fx;
    out[3 * i + 2] = f.fy;
  } else if (kind == 6) {  // wave_speed_estimates(l[0], l[1], r[0], r[1]), kernels.hpp:38-66
    double SL, Ss, SR;
    wave_speeds(a.h, a.qx, r[3 * i], r[3 * i + 1], P, SL, Ss, SR);
    out[3 * i] = SL;
    out[3 * i + 1] = Ss;
    out[3 * i + 2] = SR;
  } else if (kind == 7) {  // hydrostatic_reconstruct, kernels.hpp:126-152 -> out[12]
    const Cons b{r[3 * i], r[3 * i + 1], r[3 * i + 2]};
    reconstruct(a, z[2 * i], b, z[2 * i + 1], nrm[2 * i], nrm[2 * i + 1], P, out + 12 * i);
  } else if (kind == 8) {  // cell_signal_speed, kernels.hpp:167-170
    out[i] = signal_speed(a, P);
  } else if (kind == 9) {  // clamp_dry, kernels.hpp:205-216 -> {h, qx, qy, clipped, throws}
    const bool bad = a.h < -1e-14 * P.h_ref;
    const bool neg = !bad && a.h < 0.0;
    const bool dry = !bad && !neg && a.h < P.h_dry;
    out[5 * i] = neg ? 0.0 : a.h;
    out[5 * i + 1] = (neg || dry) ? 0.0 : a.qx;
    out[5 * i + 2] = (neg || dry) ? 0.0 : a.qy;
    out[5 * i + 3] = neg ? -a.h : 0.0;
    out[5 * i + 4] = bad ? 1.0 : 0.0;
  }
}

// linked contexts: tiles with an edge on a ghost cell (they read peers' pushes)
__global__ void k_tile_ghost(Dev d, unsigned char* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.ntiles) return;
  int g = 0;
  auto touch = [&](int e) {
    const int r = d.er[e];
    g |= d.el[e] >= d.C_own || r >= d.C_own;
  };
  for (int e = d.eoff[t]; e < d.eoff[t + 1]; ++e) touch(e);
  for (int k = d.hoff[t]; k < d.hoff[t + 1]; ++k) touch(d.halo[k]);
  out[t] = (unsigned char)g;
}

// total_mass (engine.hpp:128-132) of host arrays: a fixed-order tree sum
// (gridDim.x partials, each a fixed strided walk + shuffle tree; then one
// block folds the partials), independent of the device it runs on
__global__ void k_mass_parts(long long n, const double* h, const double* area, double* part) {
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m += h[i] * area[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  __shared__ double s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    part[blockIdx.x] = t;
  }
}

__global__ void k_mass_final(int n, const double* part, double* out) {
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  __shared__ double s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    *out = t;
  }
}

// stable_dt (kernels.hpp:174-186) over arrays: the minimum of r / speed over
// wet cells (an order-independent select-min, so the grid's order cannot
// change it) and the lowest cell with a non-finite speed
__device__ __forceinline__ void atomic_sel_min(double* p, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(p);
  unsigned long long old = *a;
  while (true) {
    const double cur = __longlong_as_double((long long)old);
    const double nv = sel_min(cur, v);
    if (__double_as_longlong(nv) == __double_as_longlong(cur)) return;
    const unsigned long long prev = atomicCAS(a, old, (unsigned long long)__double_as_longlong(nv));
    if (prev == old) return;
    old = prev;
  }
}

__global__ void k_stable_dt(long long n, Phys P, const double* h, const double* qx,
                            const double* qy, const double* inr, double* lo_out,
                            unsigned long long* bad) {
  double lo = INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const Cons u{h[i], qx[i], qy[i]};
    if (u.h < P.h_dry) continue;
    const double s = signal_speed(u, P);
    if (!isfinite(s)) {
      atomicMin(bad, (unsigned long long)i);
      continue;
    }
    lo = sel_min(lo, inr[i] / s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lo = sel_min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
  if ((threadIdx.x & 31) == 0 && lo < INFINITY) atomic_sel_min(lo_out, lo);
}

}  // namespace swe_b200
