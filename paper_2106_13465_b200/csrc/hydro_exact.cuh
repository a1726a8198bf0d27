// hydro_exact.cuh -- the exact-Riemann interface flux ("exact-10" mode).
//
// BASELINE.json specifies "exact Riemann solver with 10 Newton iterations".
// The reference keeps its exact solver as a validation oracle
// (proj/src/exact_riemann.cpp, paths relative to /root/reference/); this
// mode puts that algorithm on the hot path in place of HLLC
// (euler_kernel.cpp:196-197):
//
//   make_side (:17-22), side_fn / side_fn_deriv (:26-45), the vacuum check
//   (:52-59), the closed-form two-rarefaction root (:63-69), the
//   initial_guess (:72-74) and Newton with the p_min floor (:80-95) -- run for
//   exactly 10 iterations, no early exit, no residual throw -- then the wave
//   structure (:139-193) sampled at xi = x/t = 0 (sample_riemann, :204-241)
//   and physical_flux of that state (euler_kernel.cpp:34-39).
//
// std::pow is replaced by hb_pow(x, y) = hb_exp(y * hb_log(x)), fdlibm-style
// argument reduction + polynomials using only IEEE +, -, *, / and integer
// bit operations (no FMA: --fmad=false), so the C oracle's restatement
// (oracle/hydro_oracle.c) produces identical bits.  Against the reference's
// std::pow-based solver the mode agrees to a floored relative 1e-12
// (tests/test_exact_flux.py).  Divisions and square roots go through the
// walker's math policy M: FastMath (bitwise the IEEE result in its proven
// range, else the work item is redone) or ExactMath (the compiler's IEEE
// operations); in the tolerance TU the loose TolFast / TolExact policies
// (hydro_physics_tol.cuh), whose results are tolerance-checked, not bitwise.
#pragma once

#include <cstdint>

#include "hydro_physics.cuh"



namespace hb {

namespace exact {

__device__ __forceinline__ double from_bits(unsigned long long b) {
  return __longlong_as_double((long long)b);
}
__device__ __forceinline__ unsigned long long to_bits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

// Polynomial coefficients and ln2 split in constant memory: the FP64
// instructions read them as constant-bank operands instead of
// re-materialising 64-bit immediates in registers on every call.
__constant__ double kLg[7] = {6.666666666666735130e-01, 3.999999999940941908e-01,
                              2.857142874366239149e-01, 2.222219843214978396e-01,
                              1.818357216161805012e-01, 1.531383769920937332e-01,
                              1.479819860511658591e-01};
__constant__ double kEp[5] = {1.66666666666666019037e-01, -2.77777777770155933842e-03,
                              6.61375632143793436117e-05, -1.65339022054652515390e-06,
                              4.13813679705723846039e-08};
__constant__ double kLn2Hi = 6.93147180369123816490e-01;
__constant__ double kLn2Lo = 1.90821492927058770002e-10;
__constant__ double kInvLn2 = 1.44269504088896338700e+00;

// log(x), x positive normal: x = 2^k (1+f), sqrt(2)/2 < 1+f < sqrt(2);
// log(1+f) = f - (hfsq - s*(hfsq + R(s^2))), s = f/(2+f).  The division's
// range is proven for every input: 2+f lies in [1.70, 2.42] and f = m - 1
// is 0 or at least 2^-53 in magnitude.
template <class M>
__device__ __forceinline__ double log_(M& m, double x) {
  const unsigned long long bits = to_bits(x);
  unsigned hx = (unsigned)(bits >> 32);
  int k = (int)(hx >> 20) - 1023;
  hx &= 0x000fffffu;
  const unsigned i = (hx + 0x95f64u) & 0x100000u;  // mantissa above sqrt(2)?
  const double mt = from_bits(((unsigned long long)(hx | (i ^ 0x3ff00000u)) << 32) |
                              (bits & 0xffffffffull));
  k += (int)(i >> 20);
  const double f = mt - 1.0;
  const double s = m.divr(f, 2.0 + f);
  const double z = s * s;
  const double w = z * z;
  const double t1 = w * (kLg[1] + w * (kLg[3] + w * kLg[5]));
  const double t2 = z * (kLg[0] + w * (kLg[2] + w * (kLg[4] + w * kLg[6])));
  const double R = t2 + t1;
  const double hfsq = 0.5 * f * f;
  const double dk = (double)k;
  return dk * kLn2Hi - ((hfsq - (s * (hfsq + R) + dk * kLn2Lo)) - f);
}

// exp(x), |x| < 700: x = k ln2 + r, |r| <= ln2/2; exp(r) from the
// rational form 1 - ((lo - r c/(2-c)) - hi), c = r - r^2 P(r^2); 2^k by
// exponent arithmetic.  The division's range is proven for the solver's
// arguments: 2-c lies in [1.6, 2.4], and r c is 0 (x = 0) or about r^2 >=
// 1e-34 (every argument is 0 or a constant >= 0.14 times a log of a double
// other than 1, hence |x| >= 1.5e-17, and r cancels at most to ulp scale).
template <class M>
__device__ __forceinline__ double exp_(M& m, double x) {
  const double half = (x < 0.0) ? -0.5 : 0.5;
  const int k = (int)(kInvLn2 * x + half);  // truncation
  const double t = (double)k;
  const double hi = x - t * kLn2Hi;
  const double lo = t * kLn2Lo;
  const double r = hi - lo;
  const double r2 = r * r;
  const double c = r - r2 * (kEp[0] + r2 * (kEp[1] + r2 * (kEp[2] + r2 * (kEp[3] + r2 * kEp[4]))));
  const double y = 1.0 - ((lo - m.divr(r * c, 2.0 - c)) - hi);
  return from_bits(to_bits(y) + ((unsigned long long)(long long)k << 52));
}

template <class M>
__device__ __forceinline__ double pow_(M& m, double x, double y) {
  return exp_(m, y * log_(m, x));
}

struct Side {
  double rho, u, p, c;
};

using K = ExactK;

// Divisions: every numerator below is nonzero in a valid state (pressures,
// densities, sound speeds, constants), so they take FastMath's plain range
// test (divn/divnf; a zero or tiny numerator just redoes the item); only the
// Newton step f/df, whose f vanishes at convergence, keeps the signed-zero
// form (divf, over df > 0).

// make_side (exact_riemann.cpp:17-22) of a face, whose 1/rho is at hand
template <class M>
__device__ __forceinline__ Side make_side(M& m, const Face& f, double gamma) {
  return {f.w.r, f.w.va, f.w.p, m.sqrt(m.divn(gamma * f.w.p, f.rr))};
}

// Per-side constants of f_K / f_K' (exact_riemann.cpp:26-45): the same
// subexpressions the oracle evaluates on every Newton step, hoisted.
struct SideK {
  double a;   // 2 / ((g + 1) rho)
  double b;   // (g - 1) / (g + 1) p
  double cf;  // 2 c / (g - 1)
  double dn;  // 1 / (rho c)
  Recip rp;   // for p / p_K
};
template <class M>
__device__ __forceinline__ SideK side_k(M& m, const Side& s, const K& k) {
  return {m.divnf(2.0, k.gp1 * s.rho), k.gm * s.p, m.divnf(2.0 * s.c, k.gm1),
          m.divnf(1.0, s.rho * s.c), m.recip(s.p)};
}

// side_fn (exact_riemann.cpp:26-35) keeping, on the rarefaction branch,
// L = log(p/p_K) and E = (p/p_K)^z = exp(z L) for the sampling below.
struct SideEval {
  double f, L, E;
};
template <class M>
__device__ __forceinline__ SideEval side_eval(M& m, double p, const Side& s, const K& k) {
  SideEval e;
  if (p > s.p) {
    const double a = m.divnf(2.0, k.gp1 * s.rho);
    const double b = k.gm * s.p;
    e.f = (p - s.p) * m.sqrt(m.divnf(a, p + b));
    e.L = e.E = 0.0;
  } else {
    e.L = log_(m, m.divnf(p, s.p));
    e.E = exp_(m, k.z * e.L);
    e.f = m.divnf(2.0 * s.c, k.gm1) * (e.E - 1.0);
  }
  return e;
}

__device__ __forceinline__ bool same_bits(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

// Primitive state at xi = 0 of the Riemann problem (wl, wr); false if the
// states generate vacuum (exact_riemann.cpp:52-59).  Value-preserving
// rearrangement of the oracle's sample_xi0 (oracle/hydro_oracle.c):
//  * side_fn(p_min, K) is exactly +0 for the side whose pressure is p_min
//    (pow(1, z) = exp(z log 1) = 1 bit for bit), so only the other side's
//    term is evaluated;
//  * the sampling reuses the rarefaction side's (p/p_K)^z from u_star and
//    its log for (p/p_K)^(1/g); the fan's two powers share log(c/c_K);
//  * for bitwise-identical side states (uniform flow), each side quantity
//    is evaluated once.
template <class M>
__device__ __forceinline__ bool sample0(M& m, const Face& fl, const Face& fr, const K& k,
                                        Prim& out) {
  const Prim& wl = fl.w;
  const Prim& wr = fr.w;
  const double g = k.g;
  const bool same = same_bits(wl.r, wr.r) & same_bits(wl.va, wr.va) & same_bits(wl.p, wr.p);
  // The two sides ordered by pressure: at p > p_min the low side is on the
  // shock branch of f_K in every lane and only the high side's branch varies
  // across the warp, so a warp evaluates three side branches per pressure
  // instead of four.  Every use of the pair below is a sum (f_L + f_R, the
  // derivatives, l.c + r.c, ...), and IEEE addition commutes bit for bit.
  bool rmin;
  Side lo, hi;
  {
    const Side l = make_side(m, fl, g);
    Side r;
    if (same) r = l;
    else r = make_side(m, fr, g);
    rmin = r.p < l.p;
    lo = rmin ? r : l;
    hi = rmin ? l : r;
  }
  const double du = wr.va - wl.va;
  if (m.divnf(2.0 * (lo.c + hi.c), k.gm1) <= du) return false;  // l.c + r.c

  const double p_min = lo.p;  // smin(l.p, r.p)
  double fo = 0.0;                        // + the min side's +0
  if (!same) fo = side_eval(m, p_min, hi, k).f;
  double p;
  if (fo + du >= 0.0) {
    // both rarefactions: closed-form root (:63-69)
    const double numer = lo.c + hi.c - k.hg * du;
    const double qlo = m.divnf(lo.c, pow_(m, lo.p, k.z));
    double qhi = qlo;
    if (!same) qhi = m.divnf(hi.c, pow_(m, hi.p, k.z));
    const double denom = qlo + qhi;
    p = pow_(m, m.divnf(numer, denom), k.iz);
  } else {
    // Newton from the linearised guess with the p_min floor, 10 iterations
    const double guess =
        0.5 * (lo.p + hi.p) - 0.125 * du * (lo.rho + hi.rho) * (lo.c + hi.c);  // :72-74
    p = smax(guess, p_min);
    const SideK klo = side_k(m, lo, k), khi = side_k(m, hi, k);
    // The step is a fixed map p -> N(p) (same inputs, same arithmetic), so
    // once an iterate repeats one of the last T the sequence is periodic
    // with period T from there and the 10th iterate is known: leaving the
    // loop then is bitwise identical to running all 10 iterations.  In
    // rounding, Newton ends on a fixed point (T = 1) or on a 2-, 3- or
    // 4-cycle of neighbouring doubles about equally often; catching the
    // cycles too matters because a warp runs until its last lane leaves
    // (random states: every warp ran all 10 iterations with T = 1 only,
    // ~6.7 with T <= 4).  pK = p_{j-1-K} for the new iterate p_j.
    double p1 = -1.0, p2 = -1.0, p3 = -1.0;  // never an iterate (p >= p_min > 0)
#pragma unroll 1
    for (int j = 1; j <= 10; ++j) {
      double fA, dfA, fB, dfB;
      // f_K(p), f_K'(p) of both sides (exact_riemann.cpp:26-45); the
      // rarefaction branch shares log(p/p_K) between its two powers.
      // Low side without a branch: p >= p_min = lo.p, and at p == lo.p the
      // shock form's f = (p - lo.p) * root = +0 is the rarefaction
      // branch's cf * (exp(z log 1) - 1) = +0 bit for bit, while f' is the
      // rarefaction's dn * exp(0) = dn.  It is evaluated inside both arms
      // of the high side's branch, so each arm holds two independent chains.
      auto low = [&] {
        const Recip d = m.recip(p + klo.b);
        const double root = m.sqrt(m.divn(klo.a, d));
        fA = (p - lo.p) * root;
        const double dq = root * (1.0 - m.div(0.5 * (p - lo.p), d));  // zero-safe at p == lo.p
        dfA = (p > lo.p) ? dq : klo.dn;
      };
      if (p > hi.p) {
        low();
        const Recip d = m.recip(p + khi.b);
        const double root = m.sqrt(m.divn(khi.a, d));
        fB = (p - hi.p) * root;
        dfB = root * (1.0 - m.divn(0.5 * (p - hi.p), d));
      } else {
        low();
        const double x = m.divn(p, khi.rp);
        const double l = log_(m, x);
#ifdef HB_TOLERANCE
        // tolerance mode: x^(z-1) = x^z / x, one exp fewer per step
        const double xz = exp_(m, k.z * l);
        fB = khi.cf * (xz - 1.0);
        dfB = khi.dn * m.divnf(xz, x);
#else
        fB = khi.cf * (exp_(m, k.z * l) - 1.0);
        dfB = khi.dn * exp_(m, k.zn * l);
#endif
      }
      const double f = fA + fB + du;  // = f_L + f_R + du
      const double df = dfA + dfB;
      double next = p - m.divf(f, df);
      if (next < p_min) next = p_min;
#ifdef HB_TOLERANCE
      // tolerance mode: a Newton step below 2^-26 relative leaves an error
      // of order its square, under one ulp -- stop there instead of at the
      // rounding cycle the bitwise mode waits for
      if (fabs(next - p) <= 0x1p-26 * next) { p = next; break; }
#endif
      // p_10 = p_{j-T+((10-j) mod T)}; p_j itself equals p_{j-T}
      if (next == p) break;
      if (next == p1) { p = ((10 - j) & 1) ? p : next; break; }
      if (next == p2) {
        const int q = (10 - j) % 3;
        p = q == 0 ? next : (q == 1 ? p1 : p);
        break;
      }
      if (next == p3) {
        const int q = (10 - j) & 3;
        p = q == 0 ? next : (q == 1 ? p2 : (q == 2 ? p1 : p));
        break;
      }
      p3 = p2;
      p2 = p1;
      p1 = p;
      p = next;
    }
  }
  const SideEval elo = side_eval(m, p, lo, k);
  SideEval ehi = elo;
  if (!same) ehi = side_eval(m, p, hi, k);
  const SideEval el = rmin ? ehi : elo;
  const SideEval er = rmin ? elo : ehi;
  const Side l = rmin ? hi : lo;
  const Side r = rmin ? lo : hi;
  const double u_star = 0.5 * (wl.va + wr.va) + 0.5 * (er.f - el.f);
  const double xi = 0.0;
  // sample_riemann's right half (:225-240) is the left half (:208-223)
  // mirrored, u -> -u, xi -> -xi: every right-side expression is the exact
  // negation of the left-side one on negated operands (IEEE negation and
  // round-to-nearest are sign-symmetric), and each comparison flips with it.
  // One mirrored evaluation keeps a warp whose lanes sample both sides of
  // the contact in one branch family; va is negated back at the end.
  const bool lft = xi <= u_star;
  const Side& S = lft ? l : r;
  const SideEval& E = lft ? el : er;
  const Prim& wS = lft ? wl : wr;
  const double su = lft ? S.u : -S.u;
  const double sus = lft ? u_star : -u_star;
  const double sx = lft ? xi : -xi;
  double va;
  if (p > S.p) {  // shock
    const double ratio = m.divnf(p, S.p);
    const double head = su - S.c * m.sqrt(k.zp * ratio + k.z);
    if (sx <= head) { out = wS; return true; }
    out = {m.divnf(S.rho * (ratio + k.gm), k.gm * ratio + 1.0), u_star, wS.vb, p};
    return true;
  }
  const double head = su - S.c;  // rarefaction
  if (sx <= head) { out = wS; return true; }
  const double c_star = S.c * E.E;
  const double tail = sus - c_star;
  if (sx >= tail) {
    out = {S.rho * exp_(m, k.ig * E.L), u_star, wS.vb, p};
    return true;
  }
  va = k.a2 * (S.c + k.hg * su + sx);
  const double c = k.a2 * (S.c + k.hg * (su - sx));
  const double lc = log_(m, m.divnf(c, S.c));
  out.r = S.rho * exp_(m, k.er * lc);
  out.va = lft ? va : -va;
  out.vb = wS.vb;
  out.p = S.p * exp_(m, k.ep * lc);
  return true;
}

}  // namespace exact

// Interface flux of the exact-10 mode; vacuum -> `vacuum` set, flux unused.
template <class M>
__device__ __forceinline__ Flux exact10_flux(M& m, const Face& fl, const Face& fr, const Gas& g,
                                             bool& vacuum) {
  Prim w;
  vacuum = !exact::sample0(m, fl, fr, g.ek, w);
  // physical_flux (euler_kernel.cpp:34-39)
  const double ener = m.divn(w.p, g.rgm1) + (0.5 * w.r) * (w.va * w.va + w.vb * w.vb);
  const double rva = w.r * w.va;
  return {rva, rva * w.va + w.p, rva * w.vb, (ener + w.p) * w.va};
}

}  // namespace hb
