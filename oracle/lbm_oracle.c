/* TEST INFRASTRUCTURE ONLY — CPU oracle (plain-C restatement of the reference).
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj). All node physics is written once
 * over forward-mode dual numbers (dual.hpp:14-71): the value part of every
 * dual operation is the plain IEEE operation, so running with d = 0 gives the
 * reference's double-precision results bit for bit, and seeding d gives the
 * reference's Jacobian columns (adjoint.cpp:21-42). Operation order mirrors
 * the reference expression trees exactly (left-to-right C++ evaluation), and
 * this file is compiled without FMA contraction (oracle/Makefile: no -march).
 * Pinned against oracle/_ref by tests/test_oracle.py.
 */
#include "lbm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- dual numbers (dual.hpp:14-71) ---------------- */
typedef struct {
  double v, d;
} D;

static inline D dc(double v) { D r = {v, 0.0}; return r; }
static inline D dadd(D a, D b) { D r = {a.v + b.v, a.d + b.d}; return r; }
static inline D dsub(D a, D b) { D r = {a.v - b.v, a.d - b.d}; return r; }
static inline D dmul(D a, D b) { D r = {a.v * b.v, a.d * b.v + a.v * b.d}; return r; }
static inline D ddiv(D a, D b) {
  const double q = a.v / b.v;
  D r = {q, (a.d - q * b.d) / b.v};
  return r;
}
static inline D dneg(D a) { D r = {-a.v, -a.d}; return r; }
static inline D dabs(D a) { return a.v < 0.0 ? dneg(a) : a; }
static inline D dpow(D x, double p) {
  const double pv = pow(x.v, p);
  const double dv = p * pow(x.v, p - 1.0);
  D r = {pv, dv * x.d};
  return r;
}

/* ---------------- descriptors (lattice.cpp:83-136) ---------------- */
static const int V_D2Q9[9][3] = {{0, 0, 0},  {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                                 {1, 1, 0},  {-1, 1, 0}, {1, -1, 0}, {-1, -1, 0}};
static const int V_D3Q19[19][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0},  {0, 1, 0},  {0, -1, 0},
                                   {0, 0, 1},  {0, 0, -1},  {1, 1, 0},   {-1, 1, 0}, {1, -1, 0},
                                   {-1, -1, 0}, {1, 0, 1},  {-1, 0, 1},  {1, 0, -1}, {-1, 0, -1},
                                   {0, 1, 1},  {0, -1, 1},  {0, 1, -1},  {0, -1, -1}};
static const int V_D3Q7[7][3] = {{0, 0, 0}, {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},
                                 {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};

static void find_opp(const int (*v)[3], int q, int* opp) { /* lattice.cpp:15-26 */
  for (int j = 0; j < q; ++j) {
    opp[j] = -1;
    for (int k = 0; k < q; ++k)
      if (v[k][0] == -v[j][0] && v[k][1] == -v[j][1] && v[k][2] == -v[j][2]) {
        opp[j] = k;
        break;
      }
  }
}

/* Moment bases (lattice.cpp:31-81). */
static void moment_d2q9(double* U) {
  for (int j = 0; j < 9; ++j) {
    const double ex = V_D2Q9[j][0], ey = V_D2Q9[j][1];
    const double n2 = ex * ex + ey * ey;
    const double rows[9] = {1.0, 3.0 * n2 - 4.0, 4.0 - 10.5 * n2 + 4.5 * n2 * n2, ex,
                            (3.0 * n2 - 5.0) * ex, ey, (3.0 * n2 - 5.0) * ey,
                            ex * ex - ey * ey, ex * ey};
    for (int i = 0; i < 9; ++i) U[i * 9 + j] = rows[i];
  }
}
static void moment_d3q19(double* U) {
  for (int j = 0; j < 19; ++j) {
    const double ex = V_D3Q19[j][0], ey = V_D3Q19[j][1], ez = V_D3Q19[j][2];
    const double n2 = ex * ex + ey * ey + ez * ez;
    const double rows[19] = {1.0,
                             19.0 * n2 - 30.0,
                             (21.0 * n2 * n2 - 53.0 * n2 + 24.0) / 2,
                             ex,
                             (5.0 * n2 - 9.0) * ex,
                             ey,
                             (5.0 * n2 - 9.0) * ey,
                             ez,
                             (5.0 * n2 - 9.0) * ez,
                             3.0 * ex * ex - n2,
                             (3.0 * n2 - 5.0) * (3.0 * ex * ex - n2),
                             ey * ey - ez * ez,
                             (3.0 * n2 - 5.0) * (ey * ey - ez * ez),
                             ex * ey,
                             ey * ez,
                             ex * ez,
                             ex * (ey * ey - ez * ez),
                             ey * (ez * ez - ex * ex),
                             ez * (ex * ex - ey * ey)};
    for (int i = 0; i < 19; ++i) U[i * 19 + j] = rows[i];
  }
}

/* Full-pivot Gauss-Jordan inverse: the stand-in for Eigen::FullPivLU that the
 * oracle/_ref build also uses (oracle/eigen_standin/Eigen/Dense), so the two
 * oracles agree bit for bit on U^-1 (matrix.cpp:51-67). */
static int invert(const double* m, int n, double* out) {
  double a[19 * 19], inv[19 * 19];
  int colperm[19];
  memcpy(a, m, sizeof(double) * n * n);
  memset(inv, 0, sizeof(double) * n * n);
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0, colperm[i] = i;
  double det = 1.0;
  for (int k = 0; k < n; ++k) {
    int pr = k, pc = k;
    double best = -1.0;
    for (int i = k; i < n; ++i)
      for (int j = k; j < n; ++j)
        if (fabs(a[i * n + j]) > best) best = fabs(a[i * n + j]), pr = i, pc = j;
    if (!(best > 0.0)) return 2;
    if (pr != k) {
      for (int j = 0; j < n; ++j) {
        double t = a[pr * n + j]; a[pr * n + j] = a[k * n + j]; a[k * n + j] = t;
        t = inv[pr * n + j]; inv[pr * n + j] = inv[k * n + j]; inv[k * n + j] = t;
      }
      det = -det;
    }
    if (pc != k) {
      for (int i = 0; i < n; ++i) {
        double t = a[i * n + pc]; a[i * n + pc] = a[i * n + k]; a[i * n + k] = t;
      }
      int t = colperm[pc]; colperm[pc] = colperm[k]; colperm[k] = t;
      det = -det;
    }
    const double p = a[k * n + k];
    det *= p;
    for (int j = 0; j < n; ++j) a[k * n + j] /= p, inv[k * n + j] /= p;
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = a[i * n + k];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) a[i * n + j] -= f * a[k * n + j], inv[i * n + j] -= f * inv[k * n + j];
    }
  }
  if (!(fabs(det) > 1e-12)) return 2;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j) out[colperm[k] * n + j] = inv[k * n + j];
  return 0;
}

/* Dense product with the reference's loop order and zero skip (matrix.cpp:24-33). */
static void matmul(const double* l, const double* r, int n, double* out) {
  memset(out, 0, sizeof(double) * n * n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const double v = l[i * n + k];
      if (v == 0.0) continue;
      for (int j = 0; j < n; ++j) out[i * n + j] += v * r[k * n + j];
    }
}

/* mt19937_64 (the C++ standard engine used by config.cpp:360-369). */
typedef struct {
  uint64_t mt[312];
  int i;
} mt64;
static void mt_seed(mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
}
static uint64_t mt_next(mt64* g) {
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t y = (g->mt[k] & 0xFFFFFFFF80000000ULL) | (g->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
      g->mt[k] = g->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    g->i = 0;
  }
  uint64_t x = g->mt[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static long fidx(const lbo_system* s, int x, int y, int z) {
  return x + (long)s->nx * (y + (long)s->ny * z);
}

/* ---------------- system build (config.cpp:302-427, collision.cpp:31-102) ---------------- */
int lbo_build(const lbo_params* p, lbo_system* s) {
  memset(s, 0, sizeof *s);
  s->nx = p->nx, s->ny = p->ny, s->nz = p->nz;
  s->n = (long)p->nx * p->ny * p->nz;
  const int is3d = p->nz > 1;
  const int(*vf)[3] = is3d ? V_D3Q19 : V_D2Q9;
  const int(*vt)[3] = is3d ? V_D3Q7 : V_D2Q9;
  s->mf = is3d ? 19 : 9;
  s->mt = is3d ? 7 : 9;
  s->m = s->mf + s->mt;
  int of[19], ot[9];
  find_opp(vf, s->mf, of);
  find_opp(vt, s->mt, ot);
  for (int j = 0; j < s->mf; ++j) {
    for (int a = 0; a < 3; ++a) s->vel[j][a] = vf[j][a];
    s->opp[j] = of[j];
  }
  for (int j = 0; j < s->mt; ++j) {
    for (int a = 0; a < 3; ++a) s->vel[s->mf + j][a] = vt[j][a];
    s->opp[s->mf + j] = s->mf + ot[j];
  }
  if (is3d) {
    s->wf[0] = 1.0 / 3;
    for (int j = 1; j < 19; ++j) s->wf[j] = j <= 6 ? 1.0 / 18 : 1.0 / 36;
    s->wt[0] = 0.0;
    for (int j = 1; j < 7; ++j) s->wt[j] = 1.0 / 6;
  } else {
    const double w9[9] = {4.0 / 9, 1.0 / 9, 1.0 / 9, 1.0 / 9, 1.0 / 9,
                          1.0 / 36, 1.0 / 36, 1.0 / 36, 1.0 / 36};
    memcpy(s->wf, w9, sizeof w9);
    memcpy(s->wt, w9, sizeof w9);
  }
  s->nu = p->nu, s->beta_fluid = p->beta_fluid, s->beta_solid = p->beta_solid;
  s->inlet_dp = p->inlet_dp, s->u_clamp = p->u_clamp, s->omega_nonhydro = p->omega_nonhydro;
  s->theta = p->theta, s->bgk = p->bgk, s->fluid_power = p->fluid_power;

  /* ModelTables::build (collision.cpp:46-71) */
  const int mf = s->mf;
  const double om = 1.0 / (0.5 + 3.0 * s->nu);
  double U[361], Uinv[361], imt[361], tmp[361];
  memset(U, 0, sizeof U);
  memset(Uinv, 0, sizeof Uinv);
  if (s->bgk) {
    for (int i = 0; i < mf; ++i) U[i * mf + i] = 1.0, Uinv[i * mf + i] = 1.0, s->relax[i] = om;
  } else {
    if (is3d) moment_d3q19(U); else moment_d2q9(U);
    if (invert(U, mf, Uinv)) return 2;
    for (int i = 0; i < mf; ++i) s->relax[i] = s->omega_nonhydro;
    if (is3d) {
      const int sh[5] = {9, 11, 13, 14, 15}, co[4] = {0, 3, 5, 7};
      for (int k = 0; k < 5; ++k) s->relax[sh[k]] = om;
      for (int k = 0; k < 4; ++k) s->relax[co[k]] = 1.0;
    } else {
      const int sh[2] = {7, 8}, co[3] = {0, 3, 5};
      for (int k = 0; k < 2; ++k) s->relax[sh[k]] = om;
      for (int k = 0; k < 3; ++k) s->relax[co[k]] = 1.0;
    }
  }
  memset(imt, 0, sizeof imt);
  for (int i = 0; i < mf; ++i) imt[i * mf + i] = 1.0 - s->relax[i];
  matmul(imt, U, mf, tmp);
  matmul(Uinv, tmp, mf, s->A);
  for (int i = 0; i < mf; ++i)
    for (int j = 0; j < mf; ++j) s->At[j * mf + i] = s->A[i * mf + j];

  /* build_tags (config.cpp:302-343) */
  const long n = s->n;
  s->tag = calloc(n, 1);
  s->bc_T = calloc(n, sizeof(double));
  s->bc_axis = calloc(n, 1);
  s->bc_sign = calloc(n, 1);
  s->w = malloc(n * sizeof(double));
  s->mask = calloc(n, 1);
  s->on_support = calloc(n, 1);
  if (!p->periodic) {
    for (int z = 0; z < p->nz; ++z)
      for (int y = 0; y < p->ny; ++y)
        for (int x = 0; x < p->nx; ++x) {
          const long i = fidx(s, x, y, z);
          const int wall = y == 0 || y == p->ny - 1 || (is3d && (z == 0 || z == p->nz - 1));
          if (wall) {
            s->tag[i] = LBO_WALL;
          } else if (x == 0) {
            s->tag[i] = LBO_INLET;
            s->bc_axis[i] = 0;
            s->bc_sign[i] = 1;
            s->bc_T[i] = p->split_inlet ? (y < p->ny / 2 ? -1.0 : 1.0) : p->inlet_T;
          } else if (x == p->nx - 1) {
            s->tag[i] = LBO_OUTLET;
            s->bc_axis[i] = 0;
            s->bc_sign[i] = -1;
          }
        }
    if (p->heater_x0 >= 0) {
      const int width = p->heater_x1 - p->heater_x0 + 1;
      const int z0 = is3d ? (p->nz - width) / 2 : 0;
      const int z1 = is3d ? z0 + width - 1 : 0;
      for (int z = z0; z <= z1; ++z)
        for (int x = p->heater_x0; x <= p->heater_x1; ++x) {
          const long i = fidx(s, x, 0, z);
          s->tag[i] = LBO_HEATER;
          s->bc_T[i] = 1.0;
        }
    }
  }
  /* build_design (config.cpp:347-371) + DesignField ctor (topology.cpp:14-20) */
  for (long i = 0; i < n; ++i) s->w[i] = 1.0;
  if (p->design_x0 >= 0)
    for (int z = 0; z < p->nz; ++z)
      for (int y = 0; y < p->ny; ++y)
        for (int x = p->design_x0; x <= p->design_x1; ++x) {
          const long i = fidx(s, x, y, z);
          if (s->tag[i] == LBO_INTERIOR) s->mask[i] = 1;
        }
  long nd = 0;
  for (long i = 0; i < n; ++i) nd += s->mask[i];
  s->design = malloc((nd ? nd : 1) * sizeof(long));
  s->n_design = 0;
  for (long i = 0; i < n; ++i)
    if (s->mask[i]) s->design[s->n_design++] = i;
  mt64 g;
  mt_seed(&g, p->seed);
  for (long k = 0; k < s->n_design; ++k) {
    double w = p->initial_w;
    if (p->init_noise > 0) {
      const double u = (double)(mt_next(&g) >> 11) * 0x1p-53;
      w += p->init_noise * (2.0 * u - 1.0);
    }
    s->w[s->design[k]] = w < 0.0 ? 0.0 : (1.0 < w ? 1.0 : w);
  }
  /* build_objective (config.cpp:373-395) */
  s->obj_kind = p->obj_kind;
  s->flux_axis = 0;
  s->flux_sign = 1;
  const int xp = p->nx - 1 - p->plane_offset;
  s->support = malloc(sizeof(long) * (size_t)p->ny * p->nz);
  s->n_support = 0;
  for (int z = 0; z < p->nz; ++z)
    for (int y = 0; y < p->ny; ++y) {
      const long i = fidx(s, xp, y, z);
      if (s->tag[i] == LBO_INTERIOR) s->support[s->n_support++] = i, s->on_support[i] = 1;
    }
  if (s->n_support == 0) return 2;
  return 0;
}

void lbo_free(lbo_system* s) {
  free(s->tag); free(s->bc_T); free(s->bc_axis); free(s->bc_sign); free(s->w);
  free(s->mask); free(s->design); free(s->on_support); free(s->support);
  memset(s, 0, sizeof *s);
}

/* ---------------- node physics (collision.hpp:92-134, collision.cpp:104-294) ---------------- */
static int flow_moments(const lbo_system* s, const D* f, D* rho, D* u) {
  D r = dc(0.0), q[3] = {dc(0.0), dc(0.0), dc(0.0)};
  for (int j = 0; j < s->mf; ++j) {
    r = dadd(r, f[j]);
    for (int a = 0; a < 3; ++a)
      if (s->vel[j][a]) q[a] = dadd(q[a], dmul(dc((double)s->vel[j][a]), f[j]));
  }
  *rho = r;
  if (!(r.v > 0)) return 3;
  for (int a = 0; a < 3; ++a) u[a] = ddiv(q[a], r);
  return 0;
}

static D edot(const int* e, const D* u) {
  return dadd(dadd(dmul(dc((double)e[0]), u[0]), dmul(dc((double)e[1]), u[1])),
              dmul(dc((double)e[2]), u[2]));
}

static void flow_eq(const lbo_system* s, D rho, const D* u, D* feq) {
  const D usq = dadd(dadd(dmul(u[0], u[0]), dmul(u[1], u[1])), dmul(u[2], u[2]));
  for (int j = 0; j < s->mf; ++j) {
    const D eu = edot(s->vel[j], u);
    const D in = dsub(dadd(dadd(dc(1.0), dmul(dc(3.0), eu)), dmul(dmul(dc(4.5), eu), eu)),
                      dmul(dc(1.5), usq));
    feq[j] = dmul(dmul(dc(s->wf[j]), rho), in);
  }
}

static void therm_eq(const lbo_system* s, D temp, const D* u, D* geq) {
  for (int j = 0; j < s->mt; ++j) {
    const D eu = edot(s->vel[s->mf + j], u);
    geq[j] = dmul(dmul(dc(s->wt[j]), temp), dadd(dc(1.0), dmul(dc(3.0), eu)));
  }
}

static D switching(const lbo_system* s, D w) { /* topology.hpp:42-46 */
  if (!s->fluid_power) return dsub(dc(1.0), dpow(dsub(dc(1.0), w), s->theta));
  return dpow(w, s->theta);
}
static double switching_derivative(const lbo_system* s, double w) { /* topology.cpp:34-38 */
  if (!s->fluid_power) return s->theta * pow(1.0 - w, s->theta - 1.0);
  return s->theta * pow(w, s->theta - 1.0);
}
static D diffusivity(const lbo_system* s, D w) { /* topology.hpp:51-54 */
  return dadd(dmul(w, dc(s->beta_fluid)), dmul(dsub(dc(1.0), w), dc(s->beta_solid)));
}

/* interior_collide (collision.cpp:181-215) */
static int interior_collide(const lbo_system* s, const D* f, const D* g, D w, D* of, D* og) {
  D rho, u[3];
  if (flow_moments(s, f, &rho, u)) return 3;
  const D G = switching(s, w);
  const D up[3] = {dmul(G, u[0]), dmul(G, u[1]), dmul(G, u[2])};
  D fpre[19], fpost[19], df[19];
  flow_eq(s, rho, u, fpre);
  flow_eq(s, rho, up, fpost);
  for (int j = 0; j < s->mf; ++j) df[j] = dsub(f[j], fpre[j]);
  for (int i = 0; i < s->mf; ++i) {
    D acc = fpost[i];
    for (int j = 0; j < s->mf; ++j) acc = dadd(acc, dmul(dc(s->A[i * s->mf + j]), df[j]));
    of[i] = acc;
  }
  D temp = dc(0.0);
  for (int j = 0; j < s->mt; ++j) temp = dadd(temp, g[j]);
  const D beta = diffusivity(s, w);
  const D om = ddiv(dc(1.0), dadd(dc(0.5), dmul(dc(3.0), beta)));
  D geq[9];
  therm_eq(s, temp, up, geq);
  for (int j = 0; j < s->mt; ++j) og[j] = dadd(g[j], dmul(om, dsub(geq[j], g[j])));
  return 0;
}

/* zou_he_pressure (collision.cpp:122-177) */
static void zou_he(const lbo_system* s, const D* fin, D rho_t, int axis, int sign, D* fout, D* ua_out) {
  const int m = s->mf;
  D k0 = dc(0.0), km = dc(0.0);
  for (int j = 0; j < m; ++j) {
    const int ea = s->vel[j][axis];
    if (ea == 0) k0 = dadd(k0, fin[j]);
    else if (ea == -sign) km = dadd(km, fin[j]);
  }
  const D sg = dc((double)sign);
  D ua = dmul(sg, dsub(dc(1.0), ddiv(dadd(k0, dmul(dc(2.0), km)), rho_t)));
  D rho = rho_t;
  if (dabs(ua).v > s->u_clamp) {
    ua = ua.v > 0 ? dc(s->u_clamp) : dc(-s->u_clamp);
    rho = ddiv(dadd(k0, dmul(dc(2.0), km)), dsub(dc(1.0), dmul(sg, ua)));
  }
  D u[3] = {dc(0.0), dc(0.0), dc(0.0)};
  u[axis] = ua;
  D feq[19];
  flow_eq(s, rho, u, feq);
  D nb[3] = {dc(0.0), dc(0.0), dc(0.0)};
  for (int j = 0; j < m; ++j) {
    if (s->vel[j][axis] != 0) continue;
    for (int b = 0; b < 3; ++b)
      if (b != axis && s->vel[j][b]) nb[b] = dadd(nb[b], dmul(dc(0.5 * s->vel[j][b]), fin[j]));
  }
  for (int j = 0; j < m; ++j) fout[j] = fin[j];
  for (int j = 0; j < m; ++j) {
    if (s->vel[j][axis] != sign) continue;
    const int o = s->opp[j];
    D corr = dc(0.0);
    for (int b = 0; b < 3; ++b)
      if (b != axis && s->vel[j][b]) corr = dadd(corr, dmul(dc((double)s->vel[j][b]), nb[b]));
    fout[j] = dsub(dadd(fin[o], dsub(feq[j], feq[o])), corr);
  }
  *ua_out = ua;
}

/* collide_node (collision.cpp:219-294) */
static int collide_node_d(const lbo_system* s, int tag, int axis, int sign, double bcT,
                          const D* fin, D w, D rho_t, D* fout) {
  const int mf = s->mf, mt = s->mt;
  const D* f = fin;
  const D* g = fin + mf;
  D* of = fout;
  D* og = fout + mf;
  switch (tag) {
    case LBO_INTERIOR:
      return interior_collide(s, f, g, w, of, og);
    case LBO_WALL:
      for (int j = 0; j < mf; ++j) of[j] = f[s->opp[j]];
      for (int j = 0; j < mt; ++j) og[j] = g[s->opp[mf + j] - mf];
      return 0;
    case LBO_HEATER: {
      for (int j = 0; j < mf; ++j) of[j] = f[s->opp[j]];
      const D u0[3] = {dc(0.0), dc(0.0), dc(0.0)};
      therm_eq(s, dc(bcT), u0, og);
      return 0;
    }
    case LBO_INLET: {
      D frec[19], grec[9], ua;
      zou_he(s, f, rho_t, axis, sign, frec, &ua);
      D u[3] = {dc(0.0), dc(0.0), dc(0.0)};
      u[axis] = ua;
      therm_eq(s, dc(bcT), u, grec);
      return interior_collide(s, frec, grec, w, of, og);
    }
    default: { /* outlet */
      D frec[19], grec[9], ua;
      zou_he(s, f, dc(1.0), axis, sign, frec, &ua);
      D u[3] = {dc(0.0), dc(0.0), dc(0.0)};
      u[axis] = ua;
      D tnum = dc(0.0), tden = dc(0.0);
      for (int j = 0; j < mt; ++j) {
        const int* e = s->vel[mf + j];
        if (e[axis] == sign) continue;
        const D eu = edot(e, u);
        tnum = dadd(tnum, g[j]);
        tden = dadd(tden, dmul(dc(s->wt[j]), dadd(dc(1.0), dmul(dc(3.0), eu))));
      }
      therm_eq(s, ddiv(tnum, tden), u, grec);
      return interior_collide(s, frec, grec, w, of, og);
    }
  }
}

static double rho_inlet(const lbo_system* s) { return 1.0 + 3.0 * s->inlet_dp; }

int lbo_collide_node(const lbo_system* s, int tag, int axis, int sign, double bcT,
                     const double* fin, double w, double* fout) {
  D in[28], out[28];
  for (int p = 0; p < s->m; ++p) in[p] = dc(fin[p]);
  const int rc = collide_node_d(s, tag, axis, sign, bcT, in, dc(w), dc(rho_inlet(s)), out);
  for (int p = 0; p < s->m; ++p) fout[p] = out[p].v;
  return rc;
}

void lbo_init_state(const lbo_system* s, double* f) { /* collision.cpp:296-306 */
  for (int p = 0; p < s->m; ++p)
    for (long i = 0; i < s->n; ++i) f[p * s->n + i] = p < s->mf ? s->wf[p] : 0.0;
}

/* primal_step (collision.cpp:308-363): collide, push along +e with periodic wrap. */
int lbo_primal_step(const lbo_system* s, const double* fc, double* fn, long* bad) {
  const long n = s->n;
  D in[28], out[28];
  const D rt = dc(rho_inlet(s));
  for (int z = 0; z < s->nz; ++z)
    for (int y = 0; y < s->ny; ++y)
      for (int x = 0; x < s->nx; ++x) {
        const long idx = fidx(s, x, y, z);
        for (int p = 0; p < s->m; ++p) in[p] = dc(fc[p * n + idx]);
        if (collide_node_d(s, s->tag[idx], s->bc_axis[idx], s->bc_sign[idx], s->bc_T[idx], in,
                           dc(s->w[idx]), rt, out)) {
          if (bad) *bad = idx;
          return 3;
        }
        for (int p = 0; p < s->m; ++p) {
          const int xt = (x + s->vel[p][0] + s->nx) % s->nx;
          const int yt = (y + s->vel[p][1] + s->ny) % s->ny;
          const int zt = (z + s->vel[p][2] + s->nz) % s->nz;
          fn[p * n + fidx(s, xt, yt, zt)] = out[p].v;
        }
      }
  return 0;
}

/* step_residual (collision.cpp:365-375): NaN-propagating max norm. */
double lbo_residual(const double* a, const double* b, long count) {
  double r = 0.0;
  for (long i = 0; i < count; ++i) {
    const double d = fabs(a[i] - b[i]);
    if (!(d <= r)) r = d;
  }
  return r;
}

/* ---------------- objective (objective.cpp:19-72) ---------------- */
static int node_partial(const lbo_system* s, const D* fin, D* out) {
  if (s->obj_kind == 2) {
    for (int p = 0; p < s->m; ++p) out[p] = fin[p];
    return 0;
  }
  D rho, u[3];
  if (flow_moments(s, fin, &rho, u)) return 3;
  D temp = dc(0.0);
  for (int j = 0; j < s->mt; ++j) temp = dadd(temp, fin[s->mf + j]);
  const int a = s->flux_axis;
  const D sgn = dc((double)s->flux_sign);
  const D un = dmul(sgn, u[a]);
  const D du = s->obj_kind == 0 ? dmul(dsub(dc(1.0), dmul(temp, temp)), sgn) : dmul(temp, sgn);
  for (int k = 0; k < s->mf; ++k)
    out[k] = ddiv(dmul(du, dsub(dc((double)s->vel[k][a]), u[a])), rho);
  const D dT = s->obj_kind == 0 ? dmul(dmul(dc(-2.0), temp), un) : un;
  for (int k = 0; k < s->mt; ++k) out[s->mf + k] = dT;
  return 0;
}

static double node_term(const lbo_system* s, const D* fin) {
  if (s->obj_kind == 2) {
    D acc = dc(0.0);
    for (int p = 0; p < s->m; ++p) acc = dadd(acc, dmul(fin[p], fin[p]));
    return dmul(dc(0.5), acc).v;
  }
  D rho, u[3];
  if (flow_moments(s, fin, &rho, u)) return NAN;
  D temp = dc(0.0);
  for (int j = 0; j < s->mt; ++j) temp = dadd(temp, fin[s->mf + j]);
  const D un = dmul(dc((double)s->flux_sign), u[s->flux_axis]);
  if (s->obj_kind == 0) return dmul(un, dsub(dc(1.0), dmul(temp, temp))).v;
  return dmul(un, temp).v;
}

/* pairwise_sum_fn (reduce.hpp:43-52), leaf 16 */
static double pw(const double* t, long lo, long hi) {
  if (hi - lo <= 16) {
    double acc = 0.0;
    for (long i = lo; i < hi; ++i) acc += t[i];
    return acc;
  }
  const long mid = lo + (hi - lo) / 2;
  return pw(t, lo, mid) + pw(t, mid, hi);
}
double lbo_pairwise_sum(const double* x, long n) { return pw(x, 0, n); }

double lbo_objective(const lbo_system* s, const double* f) {
  double* t = malloc(sizeof(double) * (s->n_support ? s->n_support : 1));
  D in[28];
  for (long i = 0; i < s->n_support; ++i) {
    const long idx = s->support[i];
    for (int p = 0; p < s->m; ++p) in[p] = dc(f[p * s->n + idx]);
    t[i] = node_term(s, in);
  }
  const double r = pw(t, 0, s->n_support);
  free(t);
  return r;
}

double lbo_penalty(const lbo_system* s) { /* topology.cpp:40-50 */
  double* t = malloc(sizeof(double) * (s->n_design ? s->n_design : 1));
  for (long i = 0; i < s->n_design; ++i) {
    const double wi = s->w[s->design[i]];
    t[i] = wi * (1.0 - wi);
  }
  const double r = pw(t, 0, s->n_design);
  free(t);
  return r;
}

/* ---------------- adjoint (adjoint.cpp:21-254) ---------------- */
/* interior_vjp (adjoint.cpp:50-121); all values are plain (d = 0). */
static int interior_vjp(const lbo_system* s, const D* f, const D* g, D w, const D* vf,
                        const D* vg, D* outf, D* outg) {
  const int mf = s->mf, mt = s->mt;
  D rho, u[3];
  if (flow_moments(s, f, &rho, u)) return 3;
  const D G = switching(s, w);
  const D up[3] = {dmul(G, u[0]), dmul(G, u[1]), dmul(G, u[2])};
  D fpre[19], fpost[19], r[19];
  flow_eq(s, rho, u, fpre);
  flow_eq(s, rho, up, fpost);
  for (int k = 0; k < mf; ++k) {
    D acc = dc(0.0);
    for (int j = 0; j < mf; ++j) acc = dadd(acc, dmul(dc(s->At[k * mf + j]), vf[j]));
    r[k] = acc;
  }
  D Pr = dc(0.0), Rr = dc(0.0), Pu[3] = {dc(0), dc(0), dc(0)}, Ru[3] = {dc(0), dc(0), dc(0)};
  for (int j = 0; j < mf; ++j) {
    Pr = dadd(Pr, dmul(vf[j], fpost[j]));
    Rr = dadd(Rr, dmul(r[j], fpre[j]));
    const D e[3] = {dc((double)s->vel[j][0]), dc((double)s->vel[j][1]), dc((double)s->vel[j][2])};
    const D wjrho = dmul(dc(s->wf[j]), rho);
    const D eup = dadd(dadd(dmul(e[0], up[0]), dmul(e[1], up[1])), dmul(e[2], up[2]));
    const D eu = dadd(dadd(dmul(e[0], u[0]), dmul(e[1], u[1])), dmul(e[2], u[2]));
    const D cp = dmul(vf[j], wjrho), cr = dmul(r[j], wjrho);
    for (int a = 0; a < 3; ++a) {
      Pu[a] = dadd(Pu[a], dmul(cp, dsub(dadd(dmul(dc(3), e[a]), dmul(dmul(dc(9), eup), e[a])),
                                        dmul(dc(3), up[a]))));
      Ru[a] = dadd(Ru[a], dmul(cr, dsub(dadd(dmul(dc(3), e[a]), dmul(dmul(dc(9), eu), e[a])),
                                        dmul(dc(3), u[a]))));
    }
  }
  Pr = ddiv(Pr, rho);
  Rr = ddiv(Rr, rho);
  D temp = dc(0.0);
  for (int j = 0; j < mt; ++j) temp = dadd(temp, g[j]);
  const D beta = diffusivity(s, w);
  const D om = ddiv(dc(1), dadd(dc(0.5), dmul(dc(3), beta)));
  D sigma = dc(0.0), S[3] = {dc(0), dc(0), dc(0)};
  for (int j = 0; j < mt; ++j) {
    const int* e = s->vel[mf + j];
    const D tw = dc(s->wt[j]);
    const D eup = dadd(dadd(dmul(dc((double)e[0]), up[0]), dmul(dc((double)e[1]), up[1])),
                       dmul(dc((double)e[2]), up[2]));
    sigma = dadd(sigma, dmul(dmul(vg[j], tw), dadd(dc(1), dmul(dc(3), eup))));
    const D c = dmul(dmul(dmul(dmul(dc(3), om), temp), vg[j]), tw);
    for (int a = 0; a < 3; ++a) S[a] = dadd(S[a], dmul(c, dc((double)e[a])));
  }
  D c[3];
  for (int a = 0; a < 3; ++a) c[a] = dsub(dmul(G, dadd(Pu[a], S[a])), Ru[a]);
  const D s0 = dsub(dsub(Pr, Rr),
                    ddiv(dadd(dadd(dmul(c[0], u[0]), dmul(c[1], u[1])), dmul(c[2], u[2])), rho));
  for (int k = 0; k < mf; ++k) {
    const int* e = s->vel[k];
    outf[k] = dadd(dadd(r[k], s0),
                   ddiv(dadd(dadd(dmul(c[0], dc((double)e[0])), dmul(c[1], dc((double)e[1]))),
                             dmul(c[2], dc((double)e[2]))),
                        rho));
  }
  for (int k = 0; k < mt; ++k) outg[k] = dadd(dmul(dsub(dc(1), om), vg[k]), dmul(om, sigma));
  return 0;
}

/* vjp_dual (adjoint.cpp:21-42) */
static int vjp_dual(const lbo_system* s, int tag, int axis, int sign, double bcT, const double* fin,
                    double w, const double* vin, double* vout) {
  D din[28], col[28];
  for (int k = 0; k < s->m; ++k) {
    for (int p = 0; p < s->m; ++p) din[p].v = fin[p], din[p].d = p == k ? 1.0 : 0.0;
    if (collide_node_d(s, tag, axis, sign, bcT, din, dc(w), dc(rho_inlet(s)), col)) return 3;
    double acc = 0.0;
    for (int j = 0; j < s->m; ++j) acc += vin[j] * col[j].d;
    vout[k] = acc;
  }
  return 0;
}

/* adjoint_collide_node (adjoint.cpp:156-204) without a Jacobian cache. */
static int adjoint_node(const lbo_system* s, long idx, const double* fin, const double* vin,
                        double* vout, int kernel) {
  const int tag = s->tag[idx], axis = s->bc_axis[idx], sign = s->bc_sign[idx];
  const double bcT = s->bc_T[idx], w = s->w[idx];
  const int mf = s->mf, mt = s->mt;
  if (kernel == 1) {
    if (vjp_dual(s, tag, axis, sign, bcT, fin, w, vin, vout)) return 3;
  } else if (tag == LBO_INTERIOR) {
    D f[28], v[28], o[28];
    for (int p = 0; p < s->m; ++p) f[p] = dc(fin[p]), v[p] = dc(vin[p]);
    if (interior_vjp(s, f, f + mf, dc(w), v, v + mf, o, o + mf)) return 3;
    for (int p = 0; p < s->m; ++p) vout[p] = o[p].v;
  } else if (tag == LBO_WALL) {
    for (int k = 0; k < mf; ++k) vout[k] = vin[s->opp[k]];
    for (int k = 0; k < mt; ++k) vout[mf + k] = vin[s->opp[mf + k]];
  } else if (tag == LBO_HEATER) {
    for (int k = 0; k < mf; ++k) vout[k] = vin[s->opp[k]];
    for (int k = 0; k < mt; ++k) vout[mf + k] = 0.0;
  } else {
    if (vjp_dual(s, tag, axis, sign, bcT, fin, w, vin, vout)) return 3;
  }
  if (s->on_support[idx]) {
    D f[28], b[28];
    for (int p = 0; p < s->m; ++p) f[p] = dc(fin[p]);
    if (node_partial(s, f, b)) return 3;
    for (int k = 0; k < s->m; ++k) vout[k] += b[k].v;
  }
  return 0;
}

/* adjoint_step (adjoint.cpp:206-254): reverse push along -e with wrap. */
int lbo_adjoint_step(const lbo_system* s, const double* base, const double* vc, double* vn,
                     int kernel) {
  const long n = s->n;
  double fin[28], vin[28], vout[28];
  for (int z = 0; z < s->nz; ++z)
    for (int y = 0; y < s->ny; ++y)
      for (int x = 0; x < s->nx; ++x) {
        const long idx = fidx(s, x, y, z);
        for (int p = 0; p < s->m; ++p) fin[p] = base[p * n + idx], vin[p] = vc[p * n + idx];
        if (adjoint_node(s, idx, fin, vin, vout, kernel)) return 3;
        for (int p = 0; p < s->m; ++p) {
          const int xt = (x - s->vel[p][0] + s->nx) % s->nx;
          const int yt = (y - s->vel[p][1] + s->ny) % s->ny;
          const int zt = (z - s->vel[p][2] + s->nz) % s->nz;
          vn[p * n + fidx(s, xt, yt, zt)] = vout[p];
        }
      }
  return 0;
}

/* design_gradient_node (adjoint.cpp:311-358) */
static double design_grad(const lbo_system* s, const D* f, const D* g, D w, const D* vf, const D* vg,
                          int* err) {
  const int mf = s->mf, mt = s->mt;
  D rho, u[3];
  if (flow_moments(s, f, &rho, u)) { *err = 3; return 0.0; }
  const D G = switching(s, w);
  const D up[3] = {dmul(G, u[0]), dmul(G, u[1]), dmul(G, u[2])};
  const D dG = dc(switching_derivative(s, w.v));
  D fpost[19];
  flow_eq(s, rho, up, fpost);
  D Pu[3] = {dc(0), dc(0), dc(0)};
  for (int j = 0; j < mf; ++j) {
    const D e[3] = {dc((double)s->vel[j][0]), dc((double)s->vel[j][1]), dc((double)s->vel[j][2])};
    const D eup = dadd(dadd(dmul(e[0], up[0]), dmul(e[1], up[1])), dmul(e[2], up[2]));
    const D cp = dmul(dmul(vf[j], dc(s->wf[j])), rho);
    for (int a = 0; a < 3; ++a)
      Pu[a] = dadd(Pu[a], dmul(cp, dsub(dadd(dmul(dc(3), e[a]), dmul(dmul(dc(9), eup), e[a])),
                                        dmul(dc(3), up[a]))));
  }
  D temp = dc(0.0);
  for (int j = 0; j < mt; ++j) temp = dadd(temp, g[j]);
  const D beta = diffusivity(s, w);
  const D om = ddiv(dc(1), dadd(dc(0.5), dmul(dc(3), beta)));
  const D dom = dmul(dmul(dmul(dc(-3), dsub(dc(s->beta_fluid), dc(s->beta_solid))), om), om);
  D geq[9];
  therm_eq(s, temp, up, geq);
  D S[3] = {dc(0), dc(0), dc(0)}, relax = dc(0);
  for (int j = 0; j < mt; ++j) {
    const int* e = s->vel[mf + j];
    const D c = dmul(dmul(dmul(dmul(dc(3), om), temp), vg[j]), dc(s->wt[j]));
    for (int a = 0; a < 3; ++a) S[a] = dadd(S[a], dmul(c, dc((double)e[a])));
    relax = dadd(relax, dmul(vg[j], dsub(geq[j], g[j])));
  }
  D acc = dc(0);
  for (int a = 0; a < 3; ++a) acc = dadd(acc, dmul(u[a], dadd(Pu[a], S[a])));
  return dadd(dmul(dG, acc), dmul(dom, relax)).v;
}

/* param_gradient (adjoint.cpp:377-420) */
int lbo_param_gradient(const lbo_system* s, const double* v, const double* base, int kernel,
                       double* g_design, double* g_inlet_dp) {
  const long n = s->n;
  D f[28], vv[28], din[28], dout[28];
  for (long i = 0; i < s->n_design; ++i) {
    const long idx = s->design[i];
    for (int p = 0; p < s->m; ++p) f[p] = dc(base[p * n + idx]), vv[p] = dc(v[p * n + idx]);
    if (kernel == 0 && s->tag[idx] == LBO_INTERIOR) {
      int err = 0;
      g_design[i] = design_grad(s, f, f + s->mf, dc(s->w[idx]), vv, vv + s->mf, &err);
      if (err) return err;
    } else { /* design_gradient_node_dual (adjoint.cpp:361-373) */
      for (int p = 0; p < s->m; ++p) din[p] = f[p];
      const D wd = {s->w[idx], 1.0};
      if (collide_node_d(s, s->tag[idx], s->bc_axis[idx], s->bc_sign[idx], s->bc_T[idx], din, wd,
                         dc(rho_inlet(s)), dout))
        return 3;
      double acc = 0.0;
      for (int j = 0; j < s->m; ++j) acc += v[j * n + idx] * dout[j].d;
      g_design[i] = acc;
    }
  }
  if (g_inlet_dp) {
    long ni = 0;
    for (long idx = 0; idx < n; ++idx) ni += s->tag[idx] == LBO_INLET;
    double* t = malloc(sizeof(double) * (ni ? ni : 1));
    long k = 0;
    for (long idx = 0; idx < n; ++idx) {
      if (s->tag[idx] != LBO_INLET) continue;
      for (int p = 0; p < s->m; ++p) din[p] = dc(base[p * n + idx]);
      const D rt = {rho_inlet(s), 3.0};
      if (collide_node_d(s, s->tag[idx], s->bc_axis[idx], s->bc_sign[idx], s->bc_T[idx], din,
                         dc(s->w[idx]), rt, dout)) {
        free(t);
        return 3;
      }
      double acc = 0.0;
      for (int j = 0; j < s->m; ++j) acc += v[j * n + idx] * dout[j].d;
      t[k++] = acc;
    }
    *g_inlet_dp = pw(t, 0, ni);
    free(t);
  }
  return 0;
}

/* One one_shot_run iteration (optimizer.cpp:31-46) with descent_update (:8-16). */
int lbo_one_shot_iter(lbo_system* s, const double* fc, double* fnx, const double* vc, double* vn,
                      double zeta, double lambda, double* comp_max) {
  long bad;
  if (lbo_primal_step(s, fc, fnx, &bad)) return 3;
  if (lbo_adjoint_step(s, fnx, vc, vn, 0)) return 3;
  double* g = malloc(sizeof(double) * (s->n_design ? s->n_design : 1));
  if (lbo_param_gradient(s, vn, fnx, 0, g, NULL)) {
    free(g);
    return 3;
  }
  double gm = 0.0;
  for (long i = 0; i < s->n_design; ++i) {
    const long idx = s->design[i];
    double c = g[i];
    if (lambda != 0.0) c -= lambda * (1.0 - 2.0 * s->w[idx]);
    gm = fmax(gm, fabs(c));
    double w = s->w[idx] + zeta * c;
    s->w[idx] = w < 0.0 ? 0.0 : (1.0 < w ? 1.0 : w);
  }
  if (comp_max) *comp_max = gm;
  free(g);
  return 0;
}
