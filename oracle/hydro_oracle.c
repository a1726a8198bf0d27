/*
 * hydro_oracle.c -- TEST INFRASTRUCTURE ONLY (see hydro_oracle.h).
 *
 * CPU restatement of the reference hydro2d step, written in C for the
 * checker.  Every routine cites the reference routine it restates
 * (paths relative to /root/reference/).  Compiled with -ffp-contract=off,
 * exactly like the reference (proj/CMakeLists.txt:10-14), so results are
 * bitwise comparable.
 *
 * Pinned against: proj/README.md:98-101 (48x48 blast, 5 steps ->
 * b4593af8ee8e4e25), proj/README.md:104-109 (64x64 blast, 5 steps ->
 * bac3a9796ee2e8d5), acceptance_tests.cpp:111-112 digests and the compiled
 * reference itself (tests/test_oracle.py).
 */
#include "hydro_oracle.h"

#include <math.h>
#include <stdio.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define KGHOST 2 /* proj/include/hydro/types.hpp:50 */

typedef struct { double r, ma, mb, e; } ocons;  /* ConservedState types.hpp:11-16 */
typedef struct { double r, va, vb, p; } oprim;  /* PrimitiveState types.hpp:20-25 */
typedef struct { double m, ma, mb, e; } oflux;  /* FluxVector types.hpp:29-34 */

/* std::min / std::max semantics ((b<a)?b:a, (a<b)?b:a), not fmin/fmax. */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

static const char* kFieldName[3] = {"rho", "pres", "internal energy"};

size_t oracle_grid_doubles(int nx, int ny) {
  return (size_t)4 * (size_t)(nx + 4) * (size_t)(ny + 4);
}

/* Grid2D::index (grid.hpp:54-57) plus the plane offset. */
static inline size_t gidx(int nx, int ny, int v, int i, int j) {
  const size_t plane = (size_t)(nx + 4) * (size_t)(ny + 4);
  return (size_t)v * plane + (size_t)(i + 1) * (size_t)(ny + 4) + (size_t)(j + 1);
}
#define AT(u, v, i, j) (u)[gidx(nx, ny, (v), (i), (j))]

static void set_error(oracle_error* err, int category, const char* msg) {
  if (!err) return;
  err->category = category;
  snprintf(err->message, sizeof(err->message), "%s", msg);
}

static void set_positivity(oracle_error* err, int phase, int strip, int loop,
                           int cell, int field, const char* where) {
  if (!err) return;
  err->category = OR_ERR_POSITIVITY;
  err->phase = phase;
  err->strip = strip;
  err->loop = loop;
  err->cell = cell;
  err->field = field;
  snprintf(err->message, sizeof(err->message), "%s non-positive at %s",
           kFieldName[field], where);
}

/* Prefixes context the way rethrow_with_context does (schedulers.cpp:23-26). */
static void prefix_error(oracle_error* err, const char* ctx) {
  if (!err) return;
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", ctx, err->message);
  memcpy(err->message, buf, sizeof(buf));
}

/* ---- conversions, euler_kernel.cpp:11-55 ------------------------------ */

static int to_prim_checked(ocons u, double gamma, oprim* w) {
  /* cons_to_prim, euler_kernel.cpp:11-20 */
  if (!(u.r > 0.0)) return 0;
  const double va = u.ma / u.r;
  const double vb = u.mb / u.r;
  const double p = (gamma - 1.0) * (u.e - 0.5 * u.r * (va * va + vb * vb));
  if (!(p > 0.0)) return 1;
  w->r = u.r; w->va = va; w->vb = vb; w->p = p;
  return 2;
}

static ocons prim_to_cons_nocheck(oprim w, double gamma) {
  /* prim_to_cons / to_cons_unchecked, euler_kernel.cpp:22-28, 51-55 */
  ocons u;
  u.e = w.p / (gamma - 1.0) + 0.5 * w.r * (w.va * w.va + w.vb * w.vb);
  u.r = w.r;
  u.ma = w.r * w.va;
  u.mb = w.r * w.vb;
  return u;
}

static double sound_speed(oprim w, double gamma) {
  /* euler_kernel.cpp:30-32 */
  return sqrt(gamma * w.p / w.r);
}

static oflux phys_flux(oprim w, double gamma) {
  /* physical_flux, euler_kernel.cpp:34-39 */
  const double e = w.p / (gamma - 1.0) + 0.5 * w.r * (w.va * w.va + w.vb * w.vb);
  oflux f;
  f.m = w.r * w.va;
  f.ma = w.r * w.va * w.va + w.p;
  f.mb = w.r * w.va * w.vb;
  f.e = (e + w.p) * w.va;
  return f;
}

static double minmod(double a, double b, double c) {
  /* slope_minmod, euler_kernel.cpp:41-47 */
  const double dl = b - a;
  const double dr = c - b;
  if (dl > 0.0 && dr > 0.0) return smin(dl, dr);
  if (dl < 0.0 && dr < 0.0) return smax(dl, dr);
  return 0.0;
}

/* ---- exact-10 flux mode (BASELINE "exact Riemann, 10 Newton iterations") --
 * Restates the reference's exact solver (proj/src/exact_riemann.cpp:17-95,
 * 139-241) as an interface flux: Newton on the pressure function for exactly
 * 10 iterations from initial_guess with the p_min floor (closed-form root when
 * both waves are rarefactions), the wave structure sampled at x/t = 0, then
 * physical_flux.  std::pow is replaced by or_pow = or_exp(y * or_log(x)),
 * fdlibm-style argument reduction + polynomials in plain IEEE arithmetic --
 * the same operation sequence as csrc/hydro_exact.cuh, so CPU and GPU agree
 * bitwise.  tests/test_exact_flux.py pins it against the reference's own
 * exact_riemann/sample_riemann (tolerance: pow). */

static int g_flux = 0; /* 0 = HLLC (the reference hot path), 1 = exact-10 */

void oracle_set_flux(int flux) { g_flux = flux; }

static double or_from_bits(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t or_to_bits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }

static double or_log(double x) {
  const uint64_t bits = or_to_bits(x);
  uint32_t hx = (uint32_t)(bits >> 32);
  int k = (int)(hx >> 20) - 1023;
  hx &= 0x000fffffu;
  const uint32_t i = (hx + 0x95f64u) & 0x100000u;
  const double m = or_from_bits(((uint64_t)(hx | (i ^ 0x3ff00000u)) << 32) | (bits & 0xffffffffull));
  k += (int)(i >> 20);
  const double f = m - 1.0;
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double w = z * z;
  const double t1 = w * (3.999999999940941908e-01 + w * (2.222219843214978396e-01 + w * 1.531383769920937332e-01));
  const double t2 = z * (6.666666666666735130e-01 + w * (2.857142874366239149e-01 +
                         w * (1.818357216161805012e-01 + w * 1.479819860511658591e-01)));
  const double R = t2 + t1;
  const double hfsq = 0.5 * f * f;
  const double dk = (double)k;
  return dk * 6.93147180369123816490e-01 - ((hfsq - (s * (hfsq + R) + dk * 1.90821492927058770002e-10)) - f);
}

static double or_exp(double x) {
  const double half = (x < 0.0) ? -0.5 : 0.5;
  const int k = (int)(1.44269504088896338700e+00 * x + half);
  const double t = (double)k;
  const double hi = x - t * 6.93147180369123816490e-01;
  const double lo = t * 1.90821492927058770002e-10;
  const double r = hi - lo;
  const double r2 = r * r;
  const double c = r - r2 * (1.66666666666666019037e-01 + r2 * (-2.77777777770155933842e-03 +
                   r2 * (6.61375632143793436117e-05 + r2 * (-1.65339022054652515390e-06 +
                   r2 * 4.13813679705723846039e-08))));
  const double y = 1.0 - ((lo - (r * c) / (2.0 - c)) - hi);
  return or_from_bits(or_to_bits(y) + ((uint64_t)(int64_t)k << 52));
}

static double or_pow(double x, double y) { return or_exp(y * or_log(x)); }

typedef struct { double rho, u, p, c; } xside;

static double side_f(double p, const xside* s, double g) { /* side_fn :26-35 */
  if (p > s->p) {
    const double a = 2.0 / ((g + 1.0) * s->rho);
    const double b = (g - 1.0) / (g + 1.0) * s->p;
    return (p - s->p) * sqrt(a / (p + b));
  }
  return 2.0 * s->c / (g - 1.0) * (or_pow(p / s->p, (g - 1.0) / (2.0 * g)) - 1.0);
}

static void side_fdf(double p, const xside* s, double g, double* f, double* df) { /* :26-45 */
  if (p > s->p) {
    const double a = 2.0 / ((g + 1.0) * s->rho);
    const double b = (g - 1.0) / (g + 1.0) * s->p;
    const double root = sqrt(a / (p + b));
    *f = (p - s->p) * root;
    *df = root * (1.0 - 0.5 * (p - s->p) / (p + b));
  } else {
    const double l = or_log(p / s->p);
    *f = 2.0 * s->c / (g - 1.0) * (or_exp((g - 1.0) / (2.0 * g) * l) - 1.0);
    *df = 1.0 / (s->rho * s->c) * or_exp(-(g + 1.0) / (2.0 * g) * l);
  }
}

/* State at x/t = 0 of the Riemann problem (wl, wr); 0 on vacuum (:52-59). */
static int sample_xi0(oprim wl, oprim wr, double g, oprim* out) {
  const xside l = {wl.r, wl.va, wl.p, sqrt(g * wl.p / wl.r)}; /* make_side :17-22 */
  const xside r = {wr.r, wr.va, wr.p, sqrt(g * wr.p / wr.r)};
  const double du = wr.va - wl.va;
  if (2.0 * (l.c + r.c) / (g - 1.0) <= du) return 0;
  const double p_min = smin(l.p, r.p);
  double p;
  if (side_f(p_min, &l, g) + side_f(p_min, &r, g) + du >= 0.0) { /* :63-69 */
    const double z = (g - 1.0) / (2.0 * g);
    const double numer = l.c + r.c - 0.5 * (g - 1.0) * du;
    const double denom = l.c / or_pow(l.p, z) + r.c / or_pow(r.p, z);
    p = or_pow(numer / denom, 1.0 / z);
  } else { /* newton_root :80-95, exactly 10 iterations */
    const double guess = 0.5 * (l.p + r.p) - 0.125 * du * (l.rho + r.rho) * (l.c + r.c);
    p = smax(guess, p_min);
    for (int it = 0; it < 10; ++it) {
      double fl, dfl, fr, dfr;
      side_fdf(p, &l, g, &fl, &dfl);
      side_fdf(p, &r, g, &fr, &dfr);
      const double f = fl + fr + du;
      const double df = dfl + dfr;
      double next = p - f / df;
      if (next < p_min) next = p_min;
      p = next;
    }
  }
  const double u_star = 0.5 * (wl.va + wr.va) + 0.5 * (side_f(p, &r, g) - side_f(p, &l, g));
  const double gm = (g - 1.0) / (g + 1.0);
  const double xi = 0.0;
  if (xi <= u_star) { /* sample_riemann :208-223 */
    if (p > l.p) {
      const double ratio = p / l.p;
      const double head = l.u - l.c * sqrt((g + 1.0) / (2.0 * g) * ratio + (g - 1.0) / (2.0 * g));
      if (xi <= head) { *out = wl; return 1; }
      out->r = l.rho * (ratio + gm) / (gm * ratio + 1.0); out->va = u_star; out->vb = wl.vb; out->p = p;
      return 1;
    }
    const double head = l.u - l.c;
    if (xi <= head) { *out = wl; return 1; }
    const double c_star = l.c * or_pow(p / l.p, (g - 1.0) / (2.0 * g));
    const double tail = u_star - c_star;
    if (xi >= tail) {
      out->r = l.rho * or_pow(p / l.p, 1.0 / g); out->va = u_star; out->vb = wl.vb; out->p = p;
      return 1;
    }
    const double u = 2.0 / (g + 1.0) * (l.c + 0.5 * (g - 1.0) * l.u + xi);
    const double c = 2.0 / (g + 1.0) * (l.c + 0.5 * (g - 1.0) * (l.u - xi));
    out->r = l.rho * or_pow(c / l.c, 2.0 / (g - 1.0)); out->va = u; out->vb = wl.vb;
    out->p = l.p * or_pow(c / l.c, 2.0 * g / (g - 1.0));
    return 1;
  }
  if (p > r.p) { /* :225-240 */
    const double ratio = p / r.p;
    const double head = r.u + r.c * sqrt((g + 1.0) / (2.0 * g) * ratio + (g - 1.0) / (2.0 * g));
    if (xi >= head) { *out = wr; return 1; }
    out->r = r.rho * (ratio + gm) / (gm * ratio + 1.0); out->va = u_star; out->vb = wr.vb; out->p = p;
    return 1;
  }
  const double head = r.u + r.c;
  if (xi >= head) { *out = wr; return 1; }
  const double c_star = r.c * or_pow(p / r.p, (g - 1.0) / (2.0 * g));
  const double tail = u_star + c_star;
  if (xi <= tail) {
    out->r = r.rho * or_pow(p / r.p, 1.0 / g); out->va = u_star; out->vb = wr.vb; out->p = p;
    return 1;
  }
  const double u = 2.0 / (g + 1.0) * (-r.c + 0.5 * (g - 1.0) * r.u + xi);
  const double c = 2.0 / (g + 1.0) * (r.c - 0.5 * (g - 1.0) * (r.u - xi));
  out->r = r.rho * or_pow(c / r.c, 2.0 / (g - 1.0)); out->va = u; out->vb = wr.vb;
  out->p = r.p * or_pow(c / r.c, 2.0 * g / (g - 1.0));
  return 1;
}

/* 1 on success, 0 on vacuum. */
static int exact10(oprim wl, oprim wr, double gamma, oflux* out) {
  oprim w;
  if (!sample_xi0(wl, wr, gamma, &w)) return 0;
  *out = phys_flux(w, gamma);
  return 1;
}

int oracle_exact10_flux(const double* wl, const double* wr, double gamma, double* flux) {
  oprim a = {wl[0], wl[1], wl[2], wl[3]};
  oprim b = {wr[0], wr[1], wr[2], wr[3]};
  oflux f;
  if (!exact10(a, b, gamma, &f)) return OR_ERR_VALIDATION;
  flux[0] = f.m; flux[1] = f.ma; flux[2] = f.mb; flux[3] = f.e;
  return OR_OK;
}

/* HLLC, euler_kernel.cpp:59-109.  Returns 0 on a positivity failure. */
static int hllc(oprim wl, oprim wr, double gamma, oflux* out, int* field) {
  if (!(wl.r > 0.0)) { *field = 0; return 0; }
  if (!(wl.p > 0.0)) { *field = 1; return 0; }
  if (!(wr.r > 0.0)) { *field = 0; return 0; }
  if (!(wr.p > 0.0)) { *field = 1; return 0; }
  if (wl.r == wr.r && wl.va == wr.va && wl.vb == wr.vb && wl.p == wr.p) {
    *out = phys_flux(wl, gamma); /* equal-state shortcut :70-73 */
    return 1;
  }
  const double cl = sound_speed(wl, gamma);
  const double cr = sound_speed(wr, gamma);
  const double sl = smin(wl.va - cl, wr.va - cr); /* Davis bounds :75-78 */
  const double sr = smax(wl.va + cl, wr.va + cr);
  if (sl >= 0.0) { *out = phys_flux(wl, gamma); return 1; }
  if (sr <= 0.0) { *out = phys_flux(wr, gamma); return 1; }
  const double ql = wl.r * (sl - wl.va);
  const double qr = wr.r * (sr - wr.va);
  const double ss = (wr.p - wl.p + wl.va * ql - wr.va * qr) / (ql - qr);
  /* star flux of the upwind side (:88-108); both branches share a form */
  const oprim w = (ss >= 0.0) ? wl : wr;
  const double s = (ss >= 0.0) ? sl : sr;
  const double q = (ss >= 0.0) ? ql : qr;
  const ocons u = prim_to_cons_nocheck(w, gamma);
  const oflux f = phys_flux(w, gamma);
  const double factor = q / (s - ss);
  const double es = u.e / w.r + (ss - w.va) * (ss + w.p / q);
  out->m = f.m + s * (factor - u.r);
  out->ma = f.ma + s * (factor * ss - u.ma);
  out->mb = f.mb + s * (factor * w.vb - u.mb);
  out->e = f.e + s * (factor * es - u.e);
  return 1;
}

int oracle_riemann_flux(const double* wl, const double* wr, double gamma,
                        double* flux, oracle_error* err) {
  oprim a = {wl[0], wl[1], wl[2], wl[3]};
  oprim b = {wr[0], wr[1], wr[2], wr[3]};
  oflux f;
  int field = 0;
  if (!hllc(a, b, gamma, &f, &field)) {
    set_positivity(err, 0, 0, 0, 0, field, "riemann state");
    return OR_ERR_POSITIVITY;
  }
  flux[0] = f.m; flux[1] = f.ma; flux[2] = f.mb; flux[3] = f.e;
  return OR_OK;
}

/* ---- strip kernel, euler_kernel.cpp:111-223 ---------------------------- */

typedef struct {
  size_t cap;
  oprim* w;
  oprim* fl;
  oprim* fr;
  oflux* f;
} scratch_t;

static void scratch_reserve(scratch_t* s, int total) {
  if ((size_t)total <= s->cap) return;
  free(s->w); free(s->fl); free(s->fr); free(s->f);
  s->cap = (size_t)total;
  s->w = (oprim*)malloc(sizeof(oprim) * s->cap);
  s->fl = (oprim*)malloc(sizeof(oprim) * s->cap);
  s->fr = (oprim*)malloc(sizeof(oprim) * s->cap);
  s->f = (oflux*)malloc(sizeof(oflux) * s->cap);
}

static void scratch_free(scratch_t* s) {
  free(s->w); free(s->fl); free(s->fr); free(s->f);
  memset(s, 0, sizeof(*s));
}

/* Advances one AoS strip in place.  Returns 0 or OR_ERR_POSITIVITY with the
 * location filled in (phase/strip left for the caller). */
static int strip_update(ocons* c, int n, double dx, double dt, double gamma,
                        scratch_t* s, oflux* first, oflux* last,
                        oracle_error* err) {
  const int total = n + 2 * KGHOST;
  const double dtdx = dt / dx;
  char where[64];
  scratch_reserve(s, total);

  /* loop 1: primitives with positivity (:124-139) */
  for (int k = 0; k < total; ++k) {
    const int st = to_prim_checked(c[k], gamma, &s->w[k]);
    if (st != 2) {
      snprintf(where, sizeof(where), "strip cell %d", k - KGHOST);
      set_positivity(err, 0, 0, 0, k - KGHOST, st == 0 ? 0 : 1, where);
      return OR_ERR_POSITIVITY;
    }
  }

  /* loop 2: slopes, Hancock predictor, evolved faces (:145-191) */
  const double half = 0.5 * dtdx;
  for (int k = 1; k < total - 1; ++k) {
    const oprim a = s->w[k - 1], m = s->w[k], b = s->w[k + 1];
    const oprim sl = {minmod(a.r, m.r, b.r), minmod(a.va, m.va, b.va),
                      minmod(a.vb, m.vb, b.vb), minmod(a.p, m.p, b.p)};
    oprim lo = {m.r - 0.5 * sl.r, m.va - 0.5 * sl.va, m.vb - 0.5 * sl.vb,
                m.p - 0.5 * sl.p};
    oprim hi = {m.r + 0.5 * sl.r, m.va + 0.5 * sl.va, m.vb + 0.5 * sl.vb,
                m.p + 0.5 * sl.p};
    if (!(lo.r > 0.0 && lo.p > 0.0 && hi.r > 0.0 && hi.p > 0.0)) {
      lo = m; /* first-order fallback (:158-161) */
      hi = m;
    }
    const oflux flo = phys_flux(lo, gamma);
    const oflux fhi = phys_flux(hi, gamma);
    const ocons ulo = prim_to_cons_nocheck(lo, gamma);
    const ocons uhi = prim_to_cons_nocheck(hi, gamma);
    const ocons d = {half * (flo.m - fhi.m), half * (flo.ma - fhi.ma),
                     half * (flo.mb - fhi.mb), half * (flo.e - fhi.e)};
    const ocons ev[2] = {{ulo.r + d.r, ulo.ma + d.ma, ulo.mb + d.mb, ulo.e + d.e},
                         {uhi.r + d.r, uhi.ma + d.ma, uhi.mb + d.mb, uhi.e + d.e}};
    oprim face[2];
    for (int side = 0; side < 2; ++side) {
      /* face_prim with fallback to the cell state (:179-190) */
      const ocons u = ev[side];
      face[side] = m;
      if (u.r > 0.0) {
        const double va = u.ma / u.r;
        const double vb = u.mb / u.r;
        const double p = (gamma - 1.0) * (u.e - 0.5 * u.r * (va * va + vb * vb));
        if (p > 0.0) {
          face[side].r = u.r; face[side].va = va; face[side].vb = vb;
          face[side].p = p;
        }
      }
    }
    s->fl[k] = face[0];
    s->fr[k] = face[1];
  }

  /* loop 3: one Riemann problem per interface (:195-198) */
  for (int k = 1; k <= n + 1; ++k) {
    int field = 0;
    if (g_flux == 1) {
      if (!exact10(s->fr[k], s->fl[k + 1], gamma, &s->f[k])) {
        /* exact_riemann.cpp:55-57 */
        set_error(err, OR_ERR_VALIDATION, "vacuum-generating Riemann states are out of scope");
        if (err) { err->loop = 1; err->cell = k - KGHOST; err->field = 3; }
        return OR_ERR_VALIDATION;
      }
    } else if (!hllc(s->fr[k], s->fl[k + 1], gamma, &s->f[k], &field)) {
      set_positivity(err, 0, 0, 0, k - KGHOST, field, "riemann state");
      return OR_ERR_POSITIVITY;
    }
  }

  /* loop 4: conservative update + positivity (:200-220) */
  for (int k = KGHOST; k < KGHOST + n; ++k) {
    ocons* u = &c[k];
    const oflux fr = s->f[k];
    const oflux fl = s->f[k - 1];
    u->r -= dtdx * (fr.m - fl.m);
    u->ma -= dtdx * (fr.ma - fl.ma);
    u->mb -= dtdx * (fr.mb - fl.mb);
    u->e -= dtdx * (fr.e - fl.e);
    if (!(u->r > 0.0)) {
      snprintf(where, sizeof(where), "updated strip cell %d", k - KGHOST);
      set_positivity(err, 0, 0, 2, k - KGHOST, 0, where);
      return OR_ERR_POSITIVITY;
    }
    const double eint = u->e - 0.5 * (u->ma * u->ma + u->mb * u->mb) / u->r;
    if (!(eint > 0.0)) {
      snprintf(where, sizeof(where), "updated strip cell %d", k - KGHOST);
      set_positivity(err, 0, 0, 2, k - KGHOST, 2, where);
      return OR_ERR_POSITIVITY;
    }
  }
  if (first) *first = s->f[1];
  if (last) *last = s->f[n + 1];
  return OR_OK;
}

int oracle_sweep_strip(double* cells, int n, double dx, double dt, double gamma,
                       double* first, double* last, oracle_error* err) {
  scratch_t s = {0};
  oflux a, b;
  const int rc = strip_update((ocons*)cells, n, dx, dt, gamma, &s, &a, &b, err);
  scratch_free(&s);
  if (rc == OR_OK) {
    if (first) { first[0] = a.m; first[1] = a.ma; first[2] = a.mb; first[3] = a.e; }
    if (last) { last[0] = b.m; last[1] = b.ma; last[2] = b.mb; last[3] = b.e; }
  }
  return rc;
}

/* ---- grid-level pieces ------------------------------------------------- */

/* apply_boundary (grid.cpp:23-60), generalised with a BC kind and a wall
 * mask.  Reflective layer L mirrors interior layer L with the wall-normal
 * momentum negated; transmissive copies the adjacent interior cell into both
 * layers.  Corners are never touched. */
void oracle_apply_boundary(double* u, int nx, int ny, int bc, int wall_mask) {
  const int refl = (bc == OR_BC_REFLECT);
  for (int layer = 1; layer <= KGHOST; ++layer) {
    const int glo = 1 - layer, ghi = nx + layer;
    const int slo = refl ? layer : 1, shi = refl ? nx + 1 - layer : nx;
    for (int j = 1; j <= ny; ++j) {
      for (int v = 0; v < 4; ++v) {
        const int neg = refl && v == 1;
        if (wall_mask & OR_WALL_XLO)
          AT(u, v, glo, j) = neg ? -AT(u, v, slo, j) : AT(u, v, slo, j);
        if (wall_mask & OR_WALL_XHI)
          AT(u, v, ghi, j) = neg ? -AT(u, v, shi, j) : AT(u, v, shi, j);
      }
    }
  }
  if (!(wall_mask & OR_WALL_Y)) return;
  for (int layer = 1; layer <= KGHOST; ++layer) {
    const int glo = 1 - layer, ghi = ny + layer;
    const int slo = refl ? layer : 1, shi = refl ? ny + 1 - layer : ny;
    for (int i = 1; i <= nx; ++i) {
      for (int v = 0; v < 4; ++v) {
        const int neg = refl && v == 2;
        AT(u, v, i, glo) = neg ? -AT(u, v, i, slo) : AT(u, v, i, slo);
        AT(u, v, i, ghi) = neg ? -AT(u, v, i, shi) : AT(u, v, i, shi);
      }
    }
  }
}

/* cell_dt_limit + compute_dt (euler_kernel.cpp:225-242), minus the cfl. */
int oracle_compute_limit(const double* u, int nx, int ny, double dx, double dy,
                         double gamma, double* limit, oracle_error* err) {
  const double spacing = smin(dx, dy);
  double lim = 0.0;
  for (int i = 1; i <= nx; ++i) {
    for (int j = 1; j <= ny; ++j) {
      const ocons c = {AT(u, 0, i, j), AT(u, 1, i, j), AT(u, 2, i, j), AT(u, 3, i, j)};
      oprim w;
      const int st = to_prim_checked(c, gamma, &w);
      if (st != 2) {
        set_positivity(err, 0, i, 0, j, st == 0 ? 0 : 1, "cons_to_prim input");
        return OR_ERR_POSITIVITY;
      }
      const double speed = smax(fabs(w.va), fabs(w.vb)) + sound_speed(w, gamma);
      const double cell = spacing / speed;
      lim = (i == 1 && j == 1) ? cell : smin(lim, cell);
    }
  }
  *limit = lim;
  return OR_OK;
}

/* sweep_axis_serial + process_strip + read_strip/write_strip
 * (schedulers.cpp:68-87, grid.cpp:62-141).  The Row axis swaps the momenta
 * so mom_a is along the sweep (grid.cpp:88-94, 131-139). */
typedef struct {
  double* u;
  int nx, ny, axis, st_lo, st_hi;
  double dx, dy, gamma, dt;
  int rc, fail_strip;
  oracle_error err;
} sweep_job;

static void sweep_strips(sweep_job* jb) {
  double* u = jb->u;
  const int nx = jb->nx, ny = jb->ny, axis = jb->axis;
  const int n = (axis == 0) ? nx : ny;
  const int total = n + 2 * KGHOST;
  const int ia = (axis == 0) ? 1 : 2; /* plane holding mom_a */
  const int ib = (axis == 0) ? 2 : 1;
  ocons* c = (ocons*)malloc(sizeof(ocons) * (size_t)total);
  scratch_t s = {0};
  jb->rc = OR_OK;
  for (int st = jb->st_lo; st <= jb->st_hi; ++st) {
    for (int k = 0; k < total; ++k) {
      const int i = (axis == 0) ? k - 1 : st;
      const int j = (axis == 0) ? st : k - 1;
      c[k].r = AT(u, 0, i, j);
      c[k].ma = AT(u, ia, i, j);
      c[k].mb = AT(u, ib, i, j);
      c[k].e = AT(u, 3, i, j);
    }
    jb->rc = strip_update(c, n, (axis == 0) ? jb->dx : jb->dy, jb->dt, jb->gamma, &s, NULL, NULL,
                          &jb->err);
    if (jb->rc != OR_OK) {
      jb->fail_strip = st;
      break;
    }
    /* write_strip's validation gate (grid.cpp:106-120) repeats loop 4's
     * test on the same values, so it cannot fire here. */
    for (int k = KGHOST; k < KGHOST + n; ++k) {
      const int i = (axis == 0) ? k - 1 : st;
      const int j = (axis == 0) ? st : k - 1;
      AT(u, 0, i, j) = c[k].r;
      AT(u, ia, i, j) = c[k].ma;
      AT(u, ib, i, j) = c[k].mb;
      AT(u, 3, i, j) = c[k].e;
    }
  }
  scratch_free(&s);
  free(c);
}

static void* sweep_thread(void* arg) {
  sweep_strips((sweep_job*)arg);
  return NULL;
}

/* Strip-parallel sweeps for long golden runs (oracle_set_threads): strips of
 * a sweep read and write disjoint cells (read_strip / write_strip,
 * grid.cpp:62-141), so the result is the sequential one.  On an error the
 * lowest failing strip is reported, but the strips after it may already be
 * updated (the sequential sweep stops there) -- error-path parity uses one
 * thread. */
static int g_threads = 1;
void oracle_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

/* sweep_axis_serial: read_strip -> sweep_strip -> write_strip per strip
 * (schedulers.cpp:68-87, grid.cpp:62-141).  The Row axis swaps the momenta
 * so mom_a is along the sweep (grid.cpp:88-94, 131-139). */
int oracle_sweep_axis(double* u, int nx, int ny, double dx, double dy,
                      double gamma, int axis, double dt, oracle_error* err) {
  const int strips = (axis == 0) ? ny : nx;
  int nt = g_threads < strips ? g_threads : strips;
  if (nt < 1) nt = 1;
  sweep_job* jobs = (sweep_job*)calloc((size_t)nt, sizeof(sweep_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nt, sizeof(pthread_t));
  for (int t = 0; t < nt; ++t) {
    sweep_job* jb = &jobs[t];
    jb->u = u; jb->nx = nx; jb->ny = ny; jb->axis = axis;
    jb->dx = dx; jb->dy = dy; jb->gamma = gamma; jb->dt = dt;
    jb->st_lo = 1 + (int)((long long)strips * t / nt);
    jb->st_hi = (int)((long long)strips * (t + 1) / nt);
    if (nt > 1) pthread_create(&th[t], NULL, sweep_thread, jb);
    else sweep_strips(jb);
  }
  int rc = OR_OK;
  for (int t = 0; t < nt; ++t) {
    if (nt > 1) pthread_join(th[t], NULL);
    if (rc == OR_OK && jobs[t].rc != OR_OK) {
      rc = jobs[t].rc;
      if (err) *err = jobs[t].err;
      char ctx[64];
      snprintf(ctx, sizeof(ctx), "%s strip %d", axis == 0 ? "column sweep" : "row sweep",
               jobs[t].fail_strip);
      if (err) { err->phase = axis + 1; err->strip = jobs[t].fail_strip; }
      prefix_error(err, ctx);
    }
  }
  free(th);
  free(jobs);
  return rc;
}

static int step_error(oracle_error* err, int rc, int step) {
  if (rc != OR_OK && err) {
    char ctx[32];
    snprintf(ctx, sizeof(ctx), "step %d", step);
    err->step = step;
    prefix_error(err, ctx);
  }
  return rc;
}

/* run_sequential, schedulers.cpp:103-116. */
int oracle_run_sequential(double* u, int nx, int ny, double dx, double dy,
                          double gamma, double cfl, int bc, int steps,
                          double* last_dt, oracle_error* err) {
  if (err) memset(err, 0, sizeof(*err));
  for (int step = 0; step < steps; ++step) {
    oracle_apply_boundary(u, nx, ny, bc, OR_WALL_ALL);
    double limit = 0.0;
    int rc = oracle_compute_limit(u, nx, ny, dx, dy, gamma, &limit, err);
    if (rc != OR_OK) return step_error(err, rc, step);
    const double dt = cfl * limit;
    if (last_dt) *last_dt = dt;
    rc = oracle_sweep_axis(u, nx, ny, dx, dy, gamma, 0, dt, err);
    if (rc != OR_OK) return step_error(err, rc, step);
    oracle_apply_boundary(u, nx, ny, bc, OR_WALL_ALL);
    rc = oracle_sweep_axis(u, nx, ny, dx, dy, gamma, 1, dt, err);
    if (rc != OR_OK) return step_error(err, rc, step);
  }
  return OR_OK;
}

/* advance_sequential, schedulers.cpp:95-101 (no step context). */
int oracle_advance(double* u, int nx, int ny, double dx, double dy,
                   double gamma, int bc, double dt, oracle_error* err) {
  if (err) memset(err, 0, sizeof(*err));
  oracle_apply_boundary(u, nx, ny, bc, OR_WALL_ALL);
  int rc = oracle_sweep_axis(u, nx, ny, dx, dy, gamma, 0, dt, err);
  if (rc != OR_OK) return rc;
  oracle_apply_boundary(u, nx, ny, bc, OR_WALL_ALL);
  return oracle_sweep_axis(u, nx, ny, dx, dy, gamma, 1, dt, err);
}

/* run_until, schedulers.cpp:118-138. */
int oracle_run_until(double* u, int nx, int ny, double dx, double dy,
                     double gamma, double cfl, int bc, double t_end,
                     int* steps_out, oracle_error* err) {
  if (err) memset(err, 0, sizeof(*err));
  double t = 0.0;
  int steps = 0;
  while (t < t_end) {
    oracle_apply_boundary(u, nx, ny, bc, OR_WALL_ALL);
    double limit = 0.0;
    int rc = oracle_compute_limit(u, nx, ny, dx, dy, gamma, &limit, err);
    if (rc != OR_OK) { *steps_out = steps; return step_error(err, rc, steps); }
    double dt = cfl * limit;
    if (t + dt > t_end) dt = t_end - t;
    if (!(dt > 0.0) || t + dt == t) break;
    rc = oracle_sweep_axis(u, nx, ny, dx, dy, gamma, 0, dt, err);
    if (rc == OR_OK) {
      oracle_apply_boundary(u, nx, ny, bc, OR_WALL_ALL);
      rc = oracle_sweep_axis(u, nx, ny, dx, dy, gamma, 1, dt, err);
    }
    if (rc != OR_OK) { *steps_out = steps; return step_error(err, rc, steps); }
    t += dt;
    ++steps;
  }
  *steps_out = steps;
  return OR_OK;
}

/* ---- cases, cases.cpp:11-69 plus the BASELINE initialisers ------------- */

uint64_t oracle_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* U[-1,1) variate of (seed, cell, var): (h>>11)*2^-53 mapped by 2u-1. */
static double rnd_sym(uint64_t seed, uint64_t cell, int var) {
  const uint64_t h = oracle_splitmix64(seed ^ (4ull * cell + (uint64_t)var));
  const double unit = (double)(h >> 11) * 0x1.0p-53;
  return 2.0 * unit - 1.0;
}

static void set_cell(double* u, int nx, int ny, int i, int j, ocons c) {
  AT(u, 0, i, j) = c.r;
  AT(u, 1, i, j) = c.ma;
  AT(u, 2, i, j) = c.mb;
  AT(u, 3, i, j) = c.e;
}

static int check_prim(oprim w, oracle_error* err) {
  /* prim_to_cons's checks, euler_kernel.cpp:23-24 */
  if (!(w.r > 0.0)) { set_error(err, OR_ERR_POSITIVITY, "rho non-positive at prim_to_cons input"); return 0; }
  if (!(w.p > 0.0)) { set_error(err, OR_ERR_POSITIVITY, "pres non-positive at prim_to_cons input"); return 0; }
  return 1;
}

int oracle_init_random_rows(double* u, int nx, int ny, int row0, int global_nx,
                            double gamma, uint64_t seed, oracle_error* err) {
  (void)global_nx;
  for (int i = 1; i <= nx; ++i) {
    for (int j = 1; j <= ny; ++j) {
      const uint64_t cell = (uint64_t)(row0 + i - 1) * (uint64_t)ny + (uint64_t)(j - 1);
      oprim w;
      w.r = 1.0 + 0.1 * rnd_sym(seed, cell, 0);
      w.p = 1.0 + 0.1 * rnd_sym(seed, cell, 1);
      w.va = 0.1 * rnd_sym(seed, cell, 2);
      w.vb = 0.1 * rnd_sym(seed, cell, 3);
      if (!check_prim(w, err)) return OR_ERR_POSITIVITY;
      set_cell(u, nx, ny, i, j, prim_to_cons_nocheck(w, gamma));
    }
  }
  return OR_OK;
}

int oracle_init_case(double* u, int nx, int ny, int case_id, double gamma,
                     uint64_t seed, double* dx, double* dy, oracle_error* err) {
  if (err) memset(err, 0, sizeof(*err));
  if (nx < 4 || ny < 4) { /* Grid2D ctor, grid.cpp:11-14 */
    set_error(err, OR_ERR_CONFIG, "grid interior must be at least 4x4");
    return OR_ERR_CONFIG;
  }
  memset(u, 0, sizeof(double) * oracle_grid_doubles(nx, ny));
  *dx = 1.0 / nx;
  *dy = 1.0 / ny;
  oprim amb = {1.0, 0.0, 0.0, 1.0};
  switch (case_id) {
    case OR_CASE_UNIFORM: break;
    case OR_CASE_BLAST: amb.p = 1e-5 * (gamma - 1.0); break;  /* cases.cpp:39 */
    case OR_CASE_CORNER_BLAST: amb.p = 1e-5; break;          /* BASELINE cfg 0 */
    case OR_CASE_SOD_J:
    case OR_CASE_SOD_X:
    case OR_CASE_RANDOM: break;
    default: set_error(err, OR_ERR_CONFIG, "unknown case"); return OR_ERR_CONFIG;
  }
  if (case_id == OR_CASE_RANDOM)
    return oracle_init_random_rows(u, nx, ny, 0, nx, gamma, seed, err);
  if (case_id == OR_CASE_SOD_J || case_id == OR_CASE_SOD_X) {
    const oprim L = {1.0, 0.0, 0.0, 1.0}, R = {0.125, 0.0, 0.0, 0.1};
    const ocons cl = prim_to_cons_nocheck(L, gamma), cr = prim_to_cons_nocheck(R, gamma);
    if (case_id == OR_CASE_SOD_J) { /* cases.cpp:54-69: n = ny, dx = dy = 1/n */
      if (nx != 4 || ny < 8) {
        set_error(err, OR_ERR_CONFIG, "shock tube needs a 4 x n grid with n >= 8");
        return OR_ERR_CONFIG;
      }
      *dx = 1.0 / ny;
      *dy = 1.0 / ny;
    }
    for (int i = 1; i <= nx; ++i)
      for (int j = 1; j <= ny; ++j) {
        const int left = (case_id == OR_CASE_SOD_J) ? (j <= ny / 2) : (i <= nx / 2);
        set_cell(u, nx, ny, i, j, left ? cl : cr);
      }
    return OR_OK;
  }
  if (!check_prim(amb, err)) return OR_ERR_POSITIVITY;
  const ocons c = prim_to_cons_nocheck(amb, gamma);
  for (int i = 1; i <= nx; ++i)
    for (int j = 1; j <= ny; ++j) set_cell(u, nx, ny, i, j, c);
  if (case_id == OR_CASE_BLAST) { /* centre cells share 1.0, cases.cpp:34-52 */
    int ci[2], cj[2], ni, nj;
    if (nx % 2) { ci[0] = (nx + 1) / 2; ni = 1; } else { ci[0] = nx / 2; ci[1] = nx / 2 + 1; ni = 2; }
    if (ny % 2) { cj[0] = (ny + 1) / 2; nj = 1; } else { cj[0] = ny / 2; cj[1] = ny / 2 + 1; nj = 2; }
    const double share = 1.0 / ((double)ni * nj);
    const double volume = *dx * *dy;
    for (int a = 0; a < ni; ++a)
      for (int b = 0; b < nj; ++b) AT(u, 3, ci[a], cj[b]) = share / volume;
  }
  if (case_id == OR_CASE_CORNER_BLAST) AT(u, 3, 1, 1) = 1.0 / (*dx * *dy);
  return OR_OK;
}

/* ---- audit, audit.cpp:16-76, 137-154 ----------------------------------- */

static double pairwise(const double* v, size_t n) {
  if (n <= 8) {
    double s = 0.0;
    for (size_t k = 0; k < n; ++k) s += v[k];
    return s;
  }
  const size_t h = n / 2;
  return pairwise(v, h) + pairwise(v + h, n - h);
}

void oracle_sums(const double* u, int nx, int ny, double sums[4]) {
  double* tmp = (double*)malloc(sizeof(double) * (size_t)nx * (size_t)ny);
  for (int v = 0; v < 4; ++v) {
    size_t n = 0;
    for (int i = 1; i <= nx; ++i)
      for (int j = 1; j <= ny; ++j) tmp[n++] = AT(u, v, i, j);
    sums[v] = pairwise(tmp, n);
  }
  free(tmp);
}

uint64_t oracle_digest(const double* u, int nx, int ny) {
  uint64_t h = 14695981039346656037ull;
  for (int v = 0; v < 4; ++v)
    for (int i = 1; i <= nx; ++i)
      for (int j = 1; j <= ny; ++j) {
        uint64_t bits;
        memcpy(&bits, &AT(u, v, i, j), 8);
        for (int b = 0; b < 8; ++b) {
          h ^= (bits >> (8 * b)) & 0xffu;
          h *= 1099511628211ull;
        }
      }
  return h;
}

void oracle_compare_tolerance(const double* a, const double* b, int nx, int ny,
                              double* max_rel, double* l1_rel) {
  double mx = 0.0, abs_sum = 0.0, scale_sum = 0.0;
  for (int v = 0; v < 4; ++v)
    for (int i = 1; i <= nx; ++i)
      for (int j = 1; j <= ny; ++j) {
        const double x = AT(a, v, i, j), y = AT(b, v, i, j);
        const double scale = smax(smax(fabs(x), fabs(y)), 1.0);
        mx = smax(mx, fabs(x - y) / scale);
        abs_sum += fabs(x - y);
        scale_sum += scale;
      }
  *max_rel = mx;
  *l1_rel = abs_sum / scale_sum;
}
