/*
 * swe_oracle.c -- TEST INFRASTRUCTURE ONLY (see swe_oracle.h).
 *
 * A plain-C restatement of the reference's explicit HLLC step.  Every
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/include/swe/).  Expression trees follow the reference
 * exactly (C evaluates a*b*c as (a*b)*c); std::min/std::max are restated as
 * (b<a)?b:a and (a<b)?b:a so signed zeros and NaNs behave identically.
 * Build with -ffp-contract=off (reference CMakeLists.txt:17-18).
 */
#include "swe_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline double so_min(double a, double b) { return (b < a) ? b : a; } /* std::min */
static inline double so_max(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* kernels.hpp:15-18 */
static inline void so_velocity(so_state u, double h_dry, double* vx, double* vy) {
  if (u.h < h_dry) {
    *vx = 0.0;
    *vy = 0.0;
    return;
  }
  *vx = u.qx / u.h;
  *vy = u.qy / u.h;
}

/* kernels.hpp:21-27 */
so_flux so_physical_flux_normal(so_state u, double nx, double ny, const so_params* p) {
  so_flux f = {0.0, 0.0, 0.0};
  if (u.h < p->h_dry) return f;
  double vx, vy;
  so_velocity(u, p->h_dry, &vx, &vy);
  const double un = vx * nx + vy * ny;
  const double pressure = 0.5 * p->g * u.h * u.h;
  f.mass = u.h * un;
  f.momx = u.h * vx * un + pressure * nx;
  f.momy = u.h * vy * un + pressure * ny;
  return f;
}

/* kernels.hpp:38-66 */
so_speeds so_wave_speed_estimates(double hL, double uL, double hR, double uR, const so_params* p) {
  const double g = p->g;
  const int dryL = hL < p->h_dry;
  const int dryR = hR < p->h_dry;
  double SL, SR;
  if (dryR && !dryL) {
    const double cL = sqrt(g * hL);
    SL = uL - cL;
    SR = uL + 2.0 * cL;
  } else if (dryL && !dryR) {
    const double cR = sqrt(g * hR);
    SL = uR - 2.0 * cR;
    SR = uR + cR;
  } else {
    const double cL = sqrt(g * hL);
    const double cR = sqrt(g * hR);
    const double ustar = 0.5 * (uL + uR) + cL - cR;
    const double cstar = fabs(0.5 * (cL + cR) + 0.25 * (uL - uR));
    SL = so_min(uL - cL, ustar - cstar);
    SR = so_max(uR + cR, ustar + cstar);
  }
  const double num = SL * hR * (uR - SR) - SR * hL * (uL - SL);
  const double den = hR * (uR - SR) - hL * (uL - SL);
  so_speeds s;
  s.SL = SL;
  s.SR = SR;
  s.Sstar = fabs(den) < 1e-14 ? 0.5 * (uL + uR) : num / den;
  return s;
}

/* kernels.hpp:72-114 */
int so_hllc_flux(so_state l, so_state r, double nx, double ny, const so_params* p, so_flux* out) {
  so_flux z = {0.0, 0.0, 0.0};
  if (l.h < 0.0 || r.h < 0.0) return -1; /* :74-76 throws numeric_error */
  const int dryL = l.h < p->h_dry;
  const int dryR = r.h < p->h_dry;
  if (dryL && dryR) {
    *out = z;
    return 0;
  }
  if (l.h == r.h && l.qx == r.qx && l.qy == r.qy) { /* :83-84 */
    *out = so_physical_flux_normal(l, nx, ny, p);
    return 0;
  }
  double vLx, vLy, vRx, vRy;
  so_velocity(l, p->h_dry, &vLx, &vLy);
  so_velocity(r, p->h_dry, &vRx, &vRy);
  const double unL = vLx * nx + vLy * ny, utL = -vLx * ny + vLy * nx;
  const double unR = vRx * nx + vRy * ny, utR = -vRx * ny + vRy * nx;
  const double hL = l.h, hR = r.h;
  const so_speeds s = so_wave_speed_estimates(hL, unL, hR, unR, p);
  const double FL0 = hL * unL, FL1 = hL * unL * unL + 0.5 * p->g * hL * hL;
  const double FR0 = hR * unR, FR1 = hR * unR * unR + 0.5 * p->g * hR * hR;
  double f0, f1, ft;
  if (s.SL >= 0.0) {
    f0 = FL0;
    f1 = FL1;
    ft = f0 * utL;
  } else if (s.SR <= 0.0) {
    f0 = FR0;
    f1 = FR1;
    ft = f0 * utR;
  } else {
    const double inv = 1.0 / (s.SR - s.SL);
    f0 = (s.SR * FL0 - s.SL * FR0 + s.SL * s.SR * (hR - hL)) * inv;
    f1 = (s.SR * FL1 - s.SL * FR1 + s.SL * s.SR * (hR * unR - hL * unL)) * inv;
    ft = f0 * (s.Sstar >= 0.0 ? utL : utR);
  }
  out->mass = f0;
  out->momx = f1 * nx - ft * ny;
  out->momy = f1 * ny + ft * nx;
  return 0;
}

/* kernels.hpp:126-152 */
void so_hydrostatic_reconstruct(so_state ul, double zl, so_state ur, double zr, double nx, double ny,
                                const so_params* p, so_state* l_out, so_state* r_out,
                                so_flux* corr_l, so_flux* corr_r) {
  const double hl_star = zl >= zr ? ul.h : so_max(0.0, ul.h + (zl - zr));
  const double hr_star = zr >= zl ? ur.h : so_max(0.0, ur.h + (zr - zl));
  if (hl_star == ul.h) {
    *l_out = ul;
  } else {
    double vx, vy;
    so_velocity(ul, p->h_dry, &vx, &vy);
    l_out->h = hl_star;
    l_out->qx = hl_star * vx;
    l_out->qy = hl_star * vy;
  }
  if (hr_star == ur.h) {
    *r_out = ur;
  } else {
    double vx, vy;
    so_velocity(ur, p->h_dry, &vx, &vy);
    r_out->h = hr_star;
    r_out->qx = hr_star * vx;
    r_out->qy = hr_star * vy;
  }
  const double pl = 0.5 * p->g * (ul.h * ul.h - hl_star * hl_star);
  const double pr = 0.5 * p->g * (ur.h * ur.h - hr_star * hr_star);
  corr_l->mass = 0.0;
  corr_l->momx = pl * nx;
  corr_l->momy = pl * ny;
  corr_r->mass = 0.0;
  corr_r->momx = pr * nx;
  corr_r->momy = pr * ny;
}

/* kernels.hpp:156-164 */
so_flux so_wall_flux(so_state u, double nx, double ny, const so_params* p) {
  double vx, vy;
  so_velocity(u, p->h_dry, &vx, &vy);
  const double un = vx * nx + vy * ny;
  const double vmx = vx - 2.0 * un * nx;
  const double vmy = vy - 2.0 * un * ny;
  so_state mirror;
  mirror.h = u.h;
  mirror.qx = u.h * vmx;
  mirror.qy = u.h * vmy;
  so_flux f;
  so_hllc_flux(u, mirror, nx, ny, p, &f); /* u.h >= 0 checked by the caller */
  f.mass = 0.0;
  return f;
}

/* kernels.hpp:167-170 */
double so_cell_signal_speed(so_state u, const so_params* p) {
  double vx, vy;
  so_velocity(u, p->h_dry, &vx, &vy);
  return sqrt(vx * vx + vy * vy) + sqrt(p->g * u.h);
}

/* kernels.hpp:174-186 */
int so_stable_dt(int n, const double* h, const double* qx, const double* qy, const double* r,
                 const so_params* p, double* dt_out) {
  double dt = INFINITY;
  for (int i = 0; i < n; ++i) {
    if (h[i] < p->h_dry) continue;
    so_state u = {h[i], qx[i], qy[i]};
    const double speed = so_cell_signal_speed(u, p);
    if (!isfinite(speed)) return i;
    dt = so_min(dt, r[i] / speed);
  }
  *dt_out = isfinite(dt) ? p->cfl * dt : p->dt_max;
  return -1;
}

/* kernels.hpp:191-199 */
so_state so_apply_friction(so_state u, double n_manning, double dt, const so_params* p) {
  if (u.h < p->h_dry || n_manning == 0.0) return u;
  double vx, vy;
  so_velocity(u, p->h_dry, &vx, &vy);
  const double speed = sqrt(vx * vx + vy * vy);
  if (speed == 0.0) return u;
  const double denom = 1.0 + dt * p->g * n_manning * n_manning * speed / pow(u.h, 4.0 / 3.0);
  so_state o = {u.h, u.qx / denom, u.qy / denom};
  return o;
}

/* kernels.hpp:205-216 */
int so_clamp_dry(so_state u, const so_params* p, double* clipped, so_state* out) {
  if (u.h < -1e-14 * p->h_ref) return -1;
  if (u.h < 0.0) {
    if (clipped) *clipped += -u.h;
    so_state z = {0.0, 0.0, 0.0};
    *out = z;
    return 0;
  }
  if (u.h < p->h_dry) {
    so_state d = {u.h, 0.0, 0.0};
    *out = d;
    return 0;
  }
  *out = u;
  return 0;
}

/* engine.hpp:128-132 */
double so_total_mass(const so_mesh* m, const double* h) {
  double s = 0.0;
  for (int c = 0; c < m->n_cells; ++c) s += h[c] * m->area[c];
  return s;
}

/* engine.hpp:138-170 */
int so_compute_fluxes(const so_mesh* m, const so_params* p, const double* h, const double* qx,
                      const double* qy, double* left, double* right) {
  int bad = -1;
  for (int e = 0; e < m->n_edges; ++e) {
    const int cl = m->edge_left[e];
    const int cr = m->edge_right[e];
    const double nx = m->nx[e], ny = m->ny[e];
    so_state ul = {h[cl], qx[cl], qy[cl]};
    double* L = left + 3 * (size_t)e;
    double* R = right + 3 * (size_t)e;
    if (ul.h < 0.0 || (cr != -1 && h[cr] < 0.0)) { /* :147-153 */
      if (bad < 0) bad = e;
      L[0] = L[1] = L[2] = 0.0;
      R[0] = R[1] = R[2] = 0.0;
      continue;
    }
    if (cr == -1) { /* :155-159 */
      so_flux f = so_wall_flux(ul, nx, ny, p);
      L[0] = f.mass;
      L[1] = f.momx;
      L[2] = f.momy;
      R[0] = R[1] = R[2] = 0.0;
      continue;
    }
    so_state ur = {h[cr], qx[cr], qy[cr]};
    so_state rl, rr;
    so_flux cl_, cr_, f;
    so_hydrostatic_reconstruct(ul, m->bed[cl], ur, m->bed[cr], nx, ny, p, &rl, &rr, &cl_, &cr_);
    so_hllc_flux(rl, rr, nx, ny, p, &f);
    L[0] = f.mass; /* :165-166 */
    L[1] = f.momx + cl_.momx;
    L[2] = f.momy + cl_.momy;
    R[0] = -f.mass;
    R[1] = -(f.momx + cr_.momx);
    R[2] = -(f.momy + cr_.momy);
  }
  return bad;
}

/* engine.hpp:179-216 (block decomposition irrelevant: min/max are exact) */
int so_stable_dt_blocks(const so_mesh* m, const so_params* p, const double* h, const double* qx,
                        const double* qy, double* dt_stable, double* max_speed) {
  double lo = INFINITY, hi = 0.0;
  for (int c = 0; c < m->n_cells; ++c) {
    if (h[c] < p->h_dry) continue;
    so_state u = {h[c], qx[c], qy[c]};
    const double speed = so_cell_signal_speed(u, p);
    if (!isfinite(speed)) return c;
    lo = so_min(lo, m->inradius[c] / speed);
    hi = so_max(hi, speed);
  }
  *dt_stable = isfinite(lo) ? p->cfl * lo : p->dt_max;
  *max_speed = hi;
  return -1;
}

#define SO_REDUCE_BLOCK 4096 /* engine.hpp:47 */

/* engine.hpp:226-319 */
int so_advance_step(const so_mesh* m, const so_params* p, double t_end, const double* h,
                    const double* qx, const double* qy, double* nh, double* nqx, double* nqy,
                    double* scratch, so_clock* clk, so_step_stats* st, int* err_index,
                    double* err_h) {
  double dt_stable, max_speed;
  int bad = so_stable_dt_blocks(m, p, h, qx, qy, &dt_stable, &max_speed); /* :235 */
  if (bad >= 0) {
    *err_index = bad;
    return SO_NONFINITE_SPEED;
  }
  const int last = clk->t + dt_stable >= t_end; /* :236-237 */
  const double dt = last ? t_end - clk->t : dt_stable;

  double* left = scratch;
  double* right = scratch + 3 * (size_t)m->n_edges;
  bad = so_compute_fluxes(m, p, h, qx, qy, left, right); /* :240 */
  if (bad >= 0) {
    *err_index = bad;
    return SO_NEGATIVE_DEPTH;
  }

  const int C = m->n_cells;
  const int nb = (C + SO_REDUCE_BLOCK - 1) / SO_REDUCE_BLOCK;
  double* block_clip = (double*)calloc(nb > 0 ? nb : 1, sizeof(double));
  long* block_events = (long*)calloc(nb > 0 ? nb : 1, sizeof(long));
  int bad_cell = -1;
  for (int b = 0; b < nb; ++b) { /* :248-290 */
    const int b0 = b * SO_REDUCE_BLOCK;
    const int b1 = b0 + SO_REDUCE_BLOCK < C ? b0 + SO_REDUCE_BLOCK : C;
    double clip = 0.0;
    long events = 0;
    for (int c = b0; c < b1; ++c) {
      const double own_pressure = 0.5 * p->g * h[c] * h[c]; /* :254 */
      double am = 0.0, ax = 0.0, ay = 0.0;
      for (int k = 0; k < 3; ++k) { /* :256-264 */
        const int e = m->cell_edge[3 * (size_t)c + k];
        const int sg = m->cell_sign[3 * (size_t)c + k];
        const double* f = sg > 0 ? left + 3 * (size_t)e : right + 3 * (size_t)e;
        const double l = m->len[e];
        const double ox = sg * m->nx[e];
        const double oy = sg * m->ny[e];
        am += f[0] * l;
        ax += (f[1] - own_pressure * ox) * l;
        ay += (f[2] - own_pressure * oy) * l;
      }
      const double scale = dt / m->area[c]; /* :265-268 */
      so_state u = {h[c] - scale * am, qx[c] - scale * ax, qy[c] - scale * ay};
      u = so_apply_friction(u, m->manning[c], dt, p); /* :269 */
      if (u.h < -1e-14 * p->h_ref || !isfinite(u.h) || !isfinite(u.qx) || !isfinite(u.qy)) {
        if (bad_cell < 0) bad_cell = c; /* :273-279 */
        nh[c] = u.h;
        nqx[c] = u.qx;
        nqy[c] = u.qy;
        continue;
      }
      double clipped = 0.0; /* :280-286 */
      so_clamp_dry(u, p, &clipped, &u);
      if (clipped > 0.0) {
        clip += clipped * m->area[c];
        ++events;
      }
      nh[c] = u.h;
      nqx[c] = u.qx;
      nqy[c] = u.qy;
    }
    block_clip[b] = clip;
    block_events[b] = events;
  }
  if (bad_cell >= 0) { /* :292-297 */
    *err_index = bad_cell;
    *err_h = nh[bad_cell];
    free(block_clip);
    free(block_events);
    return SO_BLOWUP;
  }
  for (int b = 0; b < nb; ++b) { /* :300-303 */
    clk->clipped_volume += block_clip[b];
    clk->clip_events += block_events[b];
  }
  free(block_clip);
  free(block_events);
  clk->t = last ? t_end : clk->t + dt; /* :306-307 */
  clk->step += 1;
  st->step = clk->step;
  st->t = clk->t;
  st->dt = dt;
  st->max_speed = max_speed;
  return SO_OK;
}

/* ---- mesh.hpp:121-240 restated ---------------------------------------- */

typedef struct {
  uint64_t key;
  int cell, local;
} so_incidence;

static int so_inc_cmp(const void* a, const void* b) { /* mesh.hpp:187-189 */
  const so_incidence* x = (const so_incidence*)a;
  const so_incidence* y = (const so_incidence*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  if (x->cell != y->cell) return x->cell < y->cell ? -1 : 1;
  return 0;
}

static inline double so_norm(double x, double y) { return sqrt(x * x + y * y); } /* core.hpp:19 */

int so_build_mesh(int nn, const double* xy, int nc, const int* tris, int* cell_nodes, double* area,
                  double* cx, double* cy, double* inradius, int* cell_edge, int* cell_sign,
                  int* edge_nodes, int* edge_left, int* edge_right, double* nx, double* ny,
                  double* len) {
  for (int c = 0; c < nc; ++c) { /* :143-168 */
    int t0 = tris[3 * c], t1 = tris[3 * c + 1], t2 = tris[3 * c + 2];
    if (t0 < 0 || t0 >= nn || t1 < 0 || t1 >= nn || t2 < 0 || t2 >= nn) return -1;
    if (t0 == t1 || t1 == t2 || t0 == t2) return -2;
    /* signed_area = 0.5 * cross(b - a, c - a), mesh.hpp:112-114 */
    const double bax = xy[2 * t1] - xy[2 * t0], bay = xy[2 * t1 + 1] - xy[2 * t0 + 1];
    const double cax = xy[2 * t2] - xy[2 * t0], cay = xy[2 * t2 + 1] - xy[2 * t0 + 1];
    double a = 0.5 * (bax * cay - bay * cax);
    if (a < 0.0) {
      int tmp = t1;
      t1 = t2;
      t2 = tmp;
      a = -a;
    }
    if (!(a > 0.0)) return -3;
    const double p0x = xy[2 * t0], p0y = xy[2 * t0 + 1];
    const double p1x = xy[2 * t1], p1y = xy[2 * t1 + 1];
    const double p2x = xy[2 * t2], p2y = xy[2 * t2 + 1];
    const double perim = so_norm(p1x - p0x, p1y - p0y) + so_norm(p2x - p1x, p2y - p1y) +
                         so_norm(p0x - p2x, p0y - p2y);
    cell_nodes[3 * c] = t0;
    cell_nodes[3 * c + 1] = t1;
    cell_nodes[3 * c + 2] = t2;
    area[c] = a;
    cx[c] = (p0x + p1x + p2x) / 3.0;
    cy[c] = (p0y + p1y + p2y) / 3.0;
    inradius[c] = 2.0 * a / perim;
  }
  so_incidence* inc = (so_incidence*)malloc(sizeof(so_incidence) * (size_t)(3 * (size_t)nc + 1));
  for (int c = 0; c < nc; ++c) /* :177-186 */
    for (int k = 0; k < 3; ++k) {
      const int a = cell_nodes[3 * c + k];
      const int b = cell_nodes[3 * c + (k + 1) % 3];
      const uint64_t lo = (uint64_t)(a < b ? a : b);
      const uint64_t hi = (uint64_t)(a < b ? b : a);
      inc[3 * (size_t)c + k].key = lo * (uint64_t)nn + hi;
      inc[3 * (size_t)c + k].cell = c;
      inc[3 * (size_t)c + k].local = k;
    }
  const size_t ni = 3 * (size_t)nc;
  qsort(inc, ni, sizeof(so_incidence), so_inc_cmp);
  int ne = 0;
  for (size_t i = 0; i < ni;) { /* :195-225 */
    size_t j = i;
    while (j < ni && inc[j].key == inc[i].key) ++j;
    const int a0 = cell_nodes[3 * inc[i].cell + inc[i].local];
    const int a1 = cell_nodes[3 * inc[i].cell + (inc[i].local + 1) % 3];
    if (j - i > 2) {
      free(inc);
      return -4;
    }
    const int e = ne++;
    const double dx = xy[2 * a1] - xy[2 * a0], dy = xy[2 * a1 + 1] - xy[2 * a0 + 1];
    const double l = so_norm(dx, dy);
    edge_nodes[2 * e] = a0;
    edge_nodes[2 * e + 1] = a1;
    nx[e] = dy / l; /* :208 */
    ny[e] = -dx / l;
    len[e] = l;
    edge_left[e] = inc[i].cell;
    edge_right[e] = -1;
    cell_edge[3 * inc[i].cell + inc[i].local] = e;
    cell_sign[3 * inc[i].cell + inc[i].local] = +1;
    if (j - i == 2) {
      const int b0 = cell_nodes[3 * inc[i + 1].cell + inc[i + 1].local];
      const int b1 = cell_nodes[3 * inc[i + 1].cell + (inc[i + 1].local + 1) % 3];
      if (b0 != a1 || b1 != a0) {
        free(inc);
        return -5;
      }
      edge_right[e] = inc[i + 1].cell;
      cell_edge[3 * inc[i + 1].cell + inc[i + 1].local] = e;
      cell_sign[3 * inc[i + 1].cell + inc[i + 1].local] = -1;
    }
    i = j;
  }
  free(inc);
  for (int c = 0; c < nc; ++c) { /* :228-238 closed-polygon check */
    double sx = 0.0, sy = 0.0, perim = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int e = cell_edge[3 * c + k];
      const double s = cell_sign[3 * c + k] * len[e];
      sx = sx + s * nx[e];
      sy = sy + s * ny[e];
      perim += len[e];
    }
    if (so_norm(sx, sy) > 1e-10 * perim) return -6;
  }
  return ne;
}

/* ---- batch point physics over arrays (kernel-level parity tests) ------- */

void so_batch(int kind, long n, const so_params* p, const double* l, const double* r,
              const double* z, const double* nrm, double* out) {
  for (long i = 0; i < n; ++i) {
    so_state a = {l[3 * i], l[3 * i + 1], l[3 * i + 2]};
    if (kind == 0) { /* hllc_flux, kernels.hpp:72-114 */
      so_state b = {r[3 * i], r[3 * i + 1], r[3 * i + 2]};
      so_flux f;
      so_hllc_flux(a, b, nrm[2 * i], nrm[2 * i + 1], p, &f);
      out[3 * i] = f.mass;
      out[3 * i + 1] = f.momx;
      out[3 * i + 2] = f.momy;
    } else if (kind == 1) { /* wall_flux, kernels.hpp:156-164 */
      so_flux f = so_wall_flux(a, nrm[2 * i], nrm[2 * i + 1], p);
      out[3 * i] = f.mass;
      out[3 * i + 1] = f.momx;
      out[3 * i + 2] = f.momy;
    } else if (kind == 2) { /* interior edge of compute_fluxes, engine.hpp:161-166 */
      so_state b = {r[3 * i], r[3 * i + 1], r[3 * i + 2]};
      so_state rl, rr;
      so_flux cl, cr, f;
      so_hydrostatic_reconstruct(a, z[2 * i], b, z[2 * i + 1], nrm[2 * i], nrm[2 * i + 1], p, &rl,
                                 &rr, &cl, &cr);
      so_hllc_flux(rl, rr, nrm[2 * i], nrm[2 * i + 1], p, &f);
      out[6 * i] = f.mass;
      out[6 * i + 1] = f.momx + cl.momx;
      out[6 * i + 2] = f.momy + cl.momy;
      out[6 * i + 3] = -f.mass;
      out[6 * i + 4] = -(f.momx + cr.momx);
      out[6 * i + 5] = -(f.momy + cr.momy);
    } else if (kind == 3) { /* apply_friction, kernels.hpp:191-199 */
      so_state o = so_apply_friction(a, z[2 * i], z[2 * i + 1], p);
      out[3 * i] = o.h;
      out[3 * i + 1] = o.qx;
      out[3 * i + 2] = o.qy;
    } else if (kind == 4) { /* libm pow(h, 4/3), kernels.hpp:197 */
      out[i] = pow(a.h, 4.0 / 3.0);
    }
  }
}

/* ---- decomposed-domain stepping (test infrastructure for the multi-rank
 * path, include/swe/partition.hpp): cells [0, n_owned) are owned, the rest
 * ghosts; the CFL bound is reduced across parts by the caller. ---------- */

int so_local_cfl(const so_mesh* m, int n_owned, const so_params* p, const double* h,
                 const double* qx, const double* qy, double* dts, double* max_speed) {
  so_mesh part = *m;
  part.n_cells = n_owned; /* stable_dt_blocks over the owned cells only */
  return so_stable_dt_blocks(&part, p, h, qx, qy, dts, max_speed);
}

/* engine.hpp:236-307 with the given bound; ghosts are left untouched */
int so_step_owned(const so_mesh* m, int n_owned, const so_params* p, double t_end, double dts,
                  double max_speed, const double* h, const double* qx, const double* qy,
                  double* nh, double* nqx, double* nqy, double* scratch, so_clock* clk,
                  so_step_stats* st, int* err_index) {
  const int last = clk->t + dts >= t_end;
  const double dt = last ? t_end - clk->t : dts;
  double* left = scratch;
  double* right = scratch + 3 * (size_t)m->n_edges;
  int bad = so_compute_fluxes(m, p, h, qx, qy, left, right);
  if (bad >= 0) {
    *err_index = bad;
    return SO_NEGATIVE_DEPTH;
  }
  for (int c = n_owned; c < m->n_cells; ++c) { /* ghosts carry over */
    nh[c] = h[c];
    nqx[c] = qx[c];
    nqy[c] = qy[c];
  }
  for (int c = 0; c < n_owned; ++c) {
    const double own_pressure = 0.5 * p->g * h[c] * h[c];
    double am = 0.0, ax = 0.0, ay = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int e = m->cell_edge[3 * (size_t)c + k];
      const int sg = m->cell_sign[3 * (size_t)c + k];
      const double* f = sg > 0 ? left + 3 * (size_t)e : right + 3 * (size_t)e;
      const double l = m->len[e];
      am += f[0] * l;
      ax += (f[1] - own_pressure * (sg * m->nx[e])) * l;
      ay += (f[2] - own_pressure * (sg * m->ny[e])) * l;
    }
    const double scale = dt / m->area[c];
    so_state u = {h[c] - scale * am, qx[c] - scale * ax, qy[c] - scale * ay};
    u = so_apply_friction(u, m->manning[c], dt, p);
    if (u.h < -1e-14 * p->h_ref || !isfinite(u.h) || !isfinite(u.qx) || !isfinite(u.qy)) {
      *err_index = c;
      return SO_BLOWUP;
    }
    double clipped = 0.0;
    so_clamp_dry(u, p, &clipped, &u);
    if (clipped > 0.0) {
      clk->clipped_volume += clipped * m->area[c];
      ++clk->clip_events;
    }
    nh[c] = u.h;
    nqx[c] = u.qx;
    nqy[c] = u.qy;
  }
  clk->t = last ? t_end : clk->t + dt;
  clk->step += 1;
  st->step = clk->step;
  st->t = clk->t;
  st->dt = dt;
  st->max_speed = max_speed;
  return SO_OK;
}
