// Gas-kinetic BGK fluxes for DG-HGKS on sm_100a, fp64.
//
// Same physics as the reference (proj/include/hgks/{core,moments,microslope,
// flux}.hpp), restructured for the FP64 pipe:
//
//  * Maxwellian moments factor per axis, so a slope moment
//      S_m = < a u^i v^j w^k psi_m >,  a = c1 + c2 u + c3 v + c4 w + c5 |c|^2/2
//    (microslope.hpp:14-24: 8 psi_moments = 253 flops) is evaluated from three
//    a-weighted 1-D sequences
//      alpha_p = (c1 + c5/2 xi2) U_p + c2 U_{p+1} + c5/2 U_{p+2}
//      beta_q  = c3 V_{q+1} + c5/2 V_{q+2},   gamma_r = c4 W_{r+1} + c5/2 W_{r+2}
//    as G(p,q,r) = V_q W_r alpha_p + U_p (beta_q W_r + V_q gamma_r), with
//      S0..S3 = G at (i,j,k),(i+1,..),(..,j+1,..),(..,k+1)
//      S4 = 1/2 [G(i+2,j,k)+G(i,j+2,k)+G(i,j,k+2) + xi2 G(i,j,k)
//                + c5/2 (xi4 - xi2^2) U_i V_j W_k]
//    (~40 flops; indices are template constants so everything unrolls).
//  * The [0,dt] / [0,dt/2] window integrals followed by flux_linearize
//    (flux.hpp:26-48, :180-189) are folded into closed-form (F, Ft) weights per
//    time-coefficient term, removing the If - 2 Ih cancellation.
//  * Only the half-space table a side actually uses is built (one erfc per
//    side instead of two per table, moments.hpp:35-46).
// Results agree with the reference to rounding (tests: 1e-10 norm-relative
// after N steps; ~1e-13 on a residual).
#pragma once

#include <cuda_runtime.h>
#include <math.h>

#define HD __host__ __device__ __forceinline__

namespace hgks_dev {

struct GasC {
    double gamma, gm1;  // gamma, gamma - 1
    double K;           // internal dof (core.hpp:38)
    double D;           // K + 3
    double mu;          // 1/Re (0 = Euler)
    double four_D;      // 4 / D
};

// Maxwellian parameters; il = 1/(2 lam) = p/rho is carried so no kernel
// divides by lam again (2 FP64 divisions per state: 1/rho and 1/p)
struct Prim {
    double rho, U, V, W, lam;
    double inv_rho, il;
};

// error codes reported through the device error key (core.hpp:58-70)
enum : int { ERR_NONE = 0, ERR_DENSITY = 1, ERR_PRESSURE = 2 };

// pressure from conserved (core.hpp:72-74)
HD double pressure_q(const double* q, const GasC& g) {
    return g.gm1 * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
}

// primitive_from_conserved with the reference's checks (core.hpp:76-82)
HD int prim_from_q(const double* q, const GasC& g, Prim& w, double& bad) {
    if (!(q[0] > 0.0)) {
        bad = q[0];
        return ERR_DENSITY;
    }
    // one reciprocal per state: with P = rho p = (gamma-1)(rho E - |m|^2/2)
    // and r = 1/(rho P): 1/rho = P r, p/rho = P (1/rho)^2, lam = rho^3 r / 2
    // (p > 0 <=> P > 0 for rho > 0; the division for the reported p is on
    // the error path only)
    const double P = g.gm1 * (q[4] * q[0] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]));
    if (!(P > 0.0)) {
        bad = P / q[0];
        return ERR_PRESSURE;
    }
    const double r = 1.0 / (q[0] * P);
    const double inv = P * r;
    w.rho = q[0];
    w.inv_rho = inv;
    w.U = q[1] * inv;
    w.V = q[2] * inv;
    w.W = q[3] * inv;
    w.lam = 0.5 * (q[0] * q[0]) * (q[0] * r);
    w.il = P * (inv * inv);  // p / rho = 1/(2 lam)
    return ERR_NONE;
}

// The same without an early exit: the state is formed unconditionally and
// the checks become selects, so callers can keep one basic block (the
// compiler then overlaps the division chain with independent work) and test
// the code once at the end. Same codes and reported values as prim_from_q.
HD int prim_from_q_nb(const double* q, const GasC& g, Prim& w, double& bad) {
    const double P = g.gm1 * (q[4] * q[0] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]));
    const double r = 1.0 / (q[0] * P);
    const double inv = P * r;
    w.rho = q[0];
    w.inv_rho = inv;
    w.U = q[1] * inv;
    w.V = q[2] * inv;
    w.W = q[3] * inv;
    w.lam = 0.5 * (q[0] * q[0]) * (q[0] * r);
    w.il = P * (inv * inv);
    const bool okr = q[0] > 0.0, okp = P > 0.0;
    bad = okr ? (P != 0.0 ? P * inv : 0.0) : q[0];
    return okr ? (okp ? ERR_NONE : ERR_PRESSURE) : ERR_DENSITY;
}

// Per-state constants of the closed-form 5x5 micro-slope solve
// (microslope.hpp:29-44).
struct SolveC {
    double U, V, W, two_lam, c5f2, hqs, k1;  // hqs = (q2 + sbar)/2, c5f2 = 8 lam^2 / D, k1 = (q2 - sbar)/2
};

HD SolveC solve_consts(const Prim& w, const GasC& g) {
    SolveC s;
    s.U = w.U;
    s.V = w.V;
    s.W = w.W;
    const double q2 = w.U * w.U + w.V * w.V + w.W * w.W;
    const double sbar = g.D * w.il;  // 0.5 D / lam
    s.hqs = 0.5 * (q2 + sbar);
    s.k1 = 0.5 * (q2 - sbar);
    s.two_lam = 2.0 * w.lam;
    s.c5f2 = 2.0 * ((w.lam * w.lam) * g.four_D);  // 8 lam^2 / D
    return s;
}

struct Slope {
    double c1, c2, c3, c4, c5;
};

// solve <a psi> = r (r already divided by rho)
HD Slope solve_unit(const SolveC& s, double r0, double r1, double r2, double r3, double r4) {
    // B/2 and the factor 2 moved into c5f2: power-of-two rescalings, so the
    // same roundings as B = 2 r4 - qs r0, c5 = c5f (B - 2 (U R2 + V R3 + W R4))
    const double hB = r4 - s.hqs * r0;
    const double R2 = r1 - s.U * r0;
    const double R3 = r2 - s.V * r0;
    const double R4 = r3 - s.W * r0;
    Slope a;
    const double X = s.U * R2 + s.V * R3 + s.W * R4;
    a.c5 = s.c5f2 * (hB - X);
    a.c2 = s.two_lam * R2 - s.U * a.c5;
    a.c3 = s.two_lam * R3 - s.V * a.c5;
    a.c4 = s.two_lam * R4 - s.W * a.c5;
    // r0 - U c2 - V c3 - W c4 - c5 qs/2 with c2..c4 substituted:
    // r0 - 2 lam X + c5 (q2 - qs/2)
    a.c1 = (r0 - s.two_lam * X) + a.c5 * s.k1;
    return a;
}

// micro_slope (microslope.hpp:49-52): dq scaled by 1/rho
HD Slope micro_slope(const SolveC& s, double inv_rho, const double* dq) {
    return solve_unit(s, inv_rho * dq[0], inv_rho * dq[1], inv_rho * dq[2], inv_rho * dq[3],
                      inv_rho * dq[4]);
}

// rho * micro_slope: the solve is linear, so the flux passes carry slopes
// pre-scaled by the state's density (a' = rho a) and drop both the 1/rho on
// the way in and the rho on every slope-moment accumulation (the time
// coefficient of a' slopes is rho A, also linear)
HD Slope micro_slope_rho(const SolveC& s, const double* dq) {
    return solve_unit(s, dq[0], dq[1], dq[2], dq[3], dq[4]);
}

// 1-D Gaussian moment recursion (moments.hpp:49-56)
template <int NMAX>
HD void full_seq(double us, double il, double* U) {
    U[0] = 1.0;
    U[1] = us;
#pragma unroll
    for (int n = 2; n <= NMAX; ++n) U[n] = us * U[n - 1] + ((n - 1) * il) * U[n - 2];
}

// Maclaurin coefficients of erf(x) / (2x/sqrt(pi)) in z = x^2:
// (-1)^n / (n! (2n+1)), each correctly rounded (n! (2n+1) < 2^53 is exact)
struct ErfSeries {
    double a[16];
};
constexpr ErfSeries make_erf_series() {
    ErfSeries s{};
    double f = 1.0;
    for (int n = 0; n < 16; ++n) {
        if (n) f *= n;
        s.a[n] = ((n & 1) ? -1.0 : 1.0) / (f * (2 * n + 1));
    }
    return s;
}
#ifdef __CUDA_ARCH__
__device__ constexpr ErfSeries kErfSeries = make_erf_series();
#else
constexpr ErfSeries kErfSeries = make_erf_series();
#endif

// erfc(x). Near the Maxwellian's mean (|x| < 0.75, the subsonic case) a
// 16-term series of erf (last term < 5e-18 relative, no cancellation:
// erfc in (0.28, 1.72)) replaces the library's range-reduced rational + exp
// chain; elsewhere the library erfc. Agrees with erfc to ~2 ulp.
#ifndef HGKS_ERFC_NOINLINE
#define HGKS_ERFC_NOINLINE 1
#endif
#if defined(__CUDA_ARCH__) && HGKS_ERFC_NOINLINE
// the library erfc out of line: the slow path (|x| >= 0.75, supersonic
// half-space moments) then costs no registers in the face point's one block
__device__ __noinline__ double erfc_far(double x) { return erfc(x); }
#else
HD double erfc_far(double x) { return erfc(x); }
#endif
HD double erfc_near0(double x) {
    if (fabs(x) < 0.75) {
        const double z = x * x;
        double s = kErfSeries.a[15];
#pragma unroll
        for (int n = 14; n >= 0; --n) s = fma(s, z, kErfSeries.a[n]);
        return 1.0 - (1.1283791670955125739 * x) * s;  // 2/sqrt(pi)
    }
    return erfc_far(x);
}

// Half-space table for u>0 (sign=+1) or u<0 (sign=-1) (moments.hpp:35,43-46).
// erfc is evaluated once on the non-cancelling side.
template <int NMAX>
HD void half_seq(double us, double lam, double il, int sign, double* U) {
#ifdef __CUDA_ARCH__
    const double rs = rsqrt(lam);  // 1/sqrt(lam): no sqrt + division on the chain
#else
    const double rs = 1.0 / sqrt(lam);
#endif
    const double sql = lam * rs;
    const double beta = (0.28209479177387814347 * rs) * exp(-lam * us * us);  // 1/(2 sqrt(pi))
    const double x = sign > 0 ? -sql * us : sql * us;
    U[0] = 0.5 * erfc_near0(x);
    U[1] = sign > 0 ? us * U[0] + beta : us * U[0] - beta;
#pragma unroll
    for (int n = 2; n <= NMAX; ++n) U[n] = us * U[n - 1] + ((n - 1) * il) * U[n - 2];
}

// Moment sequences of one Maxwellian. Ut is the u-axis table in use (full or
// half); V, W always full.
template <int NU, int NV>
struct Tab {
    double U[NU + 1];
    double V[NV + 1];
    double W[NV + 1];
    double xi2;   // K/(2 lam)
    double dxi;   // xi4 - xi2^2 = 2 K/(2 lam)^2
};

template <int NU, int NV>
HD void make_tab(const Prim& w, const GasC& g, Tab<NU, NV>& t) {
    const double il = w.il;
    full_seq<NU>(w.U, il, t.U);
    full_seq<NV>(w.V, il, t.V);
    full_seq<NV>(w.W, il, t.W);
    t.xi2 = g.K * il;
    t.dxi = 2.0 * g.K * il * il;
}

// psi moment <u^i v^j w^k psi> (moments.hpp:79-91, s = 0)
template <int I, int J, int K, class T>
HD void psi_moment(const double* Ut, const T& t, double* r) {
    const double vw = t.V[J] * t.W[K];
    const double base = Ut[I] * vw;
    r[0] = base;
    r[1] = Ut[I + 1] * vw;
    r[2] = Ut[I] * (t.V[J + 1] * t.W[K]);
    r[3] = Ut[I] * (t.V[J] * t.W[K + 1]);
    r[4] = 0.5 * ((Ut[I + 2] * vw + Ut[I] * (t.V[J + 2] * t.W[K] + t.V[J] * t.W[K + 2])) +
                  base * t.xi2);
}

// slope moment <a u^i v^j w^k psi> via the factorised sequences (see header)
template <int I, int J, int K, class T>
HD void slope_moment(const double* Ut, const T& t, const Slope& a, double* r) {
    const double h5 = 0.5 * a.c5;
    const double c1x = a.c1 + h5 * t.xi2;
#define AL(p) (c1x * Ut[p] + a.c2 * Ut[(p) + 1] + h5 * Ut[(p) + 2])
#define BE(q) (a.c3 * t.V[(q) + 1] + h5 * t.V[(q) + 2])
#define GA(r) (a.c4 * t.W[(r) + 1] + h5 * t.W[(r) + 2])
#define GG(p, q, r) ((t.V[q] * t.W[r]) * AL(p) + Ut[p] * (BE(q) * t.W[r] + t.V[q] * GA(r)))
#define XT(q, r) (BE(q) * t.W[r] + t.V[q] * GA(r))
    // G(I,J,K) and G(I+1,J,K) share the transverse part; in the energy
    // moment the three second-order G's are regrouped by their common
    // factors AL(I) and U_I (the V_q W_r sums depend on the table only)
    const double vw = t.V[J] * t.W[K];
    const double x0 = XT(J, K);
    const double al0 = AL(I);
    const double g0 = vw * al0 + Ut[I] * x0;
    r[0] = g0;
    r[1] = vw * AL(I + 1) + Ut[I + 1] * x0;
    r[2] = GG(I, J + 1, K);
    r[3] = GG(I, J, K + 1);
    r[4] = 0.5 * (vw * AL(I + 2) + Ut[I + 2] * x0 +
                  al0 * (t.V[J + 2] * t.W[K] + t.V[J] * t.W[K + 2]) +
                  Ut[I] * ((XT(J + 2, K) + XT(J, K + 2)) + (h5 * t.dxi) * vw) + t.xi2 * g0);
#undef XT
#undef AL
#undef BE
#undef GA
#undef GG
}

HD void axpy5(double s, const double* x, double* y) {
#pragma unroll
    for (int i = 0; i < 5; ++i) y[i] += s * x[i];
}

// time_coefficient (microslope.hpp:56-61) with the full table of w
template <class T>
HD Slope time_coefficient(const SolveC& sc, const T& t, const Slope* a) {
    double s[5], r[5];
    slope_moment<1, 0, 0>(t.U, t, a[0], s);
    slope_moment<0, 1, 0>(t.U, t, a[1], r);
#pragma unroll
    for (int m = 0; m < 5; ++m) s[m] += r[m];
    slope_moment<0, 0, 1>(t.U, t, a[2], r);
#pragma unroll
    for (int m = 0; m < 5; ++m) s[m] = -(s[m] + r[m]);
    return solve_unit(sc, s[0], s[1], s[2], s[3], s[4]);
}

// Closed-form (F, Ft) weights of the six BGK time-coefficient terms
// (flux.hpp:26-48 integrated over [0,dt], [0,dt/2], then flux.hpp:180-189).
struct TimeW {
    double g0F, g0Ft, abF, abFt, AbF, AbFt;  // equilibrium: g0, abar, Abar
    double f0F, f0Ft, anF, anFt, AnF, AnFt;  // non-equilibrium: f0, aneq, Aneq
};

// rh = dt / (2 tau) and inv_dt = 1/dt are passed in so callers can form them
// without a division (the face kernel has tau = 2 mu / (p_l + p_r))
HD TimeW time_weights_r(double tau, double inv_dt, double rh) {
    // branch-free: the general weights are formed and the tau = 0 limits
    // (flux.hpp:32-38) selected, so the face point stays one basic block
    TimeW w;
    // s = 1 - e^{-dt/(2 tau)}; for rh > 54 ln 2 = 37.43, e^{-rh} < 2^-54 and s
    // rounds to 1 exactly (this also covers the reference's e^{-r} -> 0 clamp
    // for r > 700, flux.hpp:40) — no expm1 on the chain at TGV 128^3 (rh ~ 38)
    const double s = rh > 37.5 ? 1.0 : -expm1(-rh);
    const double x = tau * inv_dt;
    const double t3 = s * (2.0 + s);
    const double ss = s * s;
    const double q4 = 4.0 * x * inv_dt;
    w.g0F = 1.0 - x * t3;
    w.g0Ft = q4 * ss;
    w.f0F = x * t3;
    w.f0Ft = -q4 * ss;
    w.AbF = tau * (x * t3 - 1.0);
    w.AbFt = 1.0 - 4.0 * x * x * ss;
    w.AnF = -tau * x * t3;
    w.AnFt = 4.0 * x * x * ss;
    const double ab_t = 4.0 * x * (1.0 - s) * s - 8.0 * x * x * ss;
    w.abF = tau * (ss - 2.0) + 2.0 * tau * x * t3;
    w.abFt = ab_t;
    w.anF = tau * (1.0 - ss) - 2.0 * tau * x * t3;
    w.anFt = -ab_t;
    if (!(tau > 0.0)) {  // tau = 0 limits (flux.hpp:32-38), as selects
        w.g0F = 1.0;
        w.g0Ft = 0.0;
        w.abF = w.abFt = 0.0;
        w.AbF = 0.0;
        w.AbFt = 1.0;
        w.f0F = w.f0Ft = w.anF = w.anFt = w.AnF = w.AnFt = 0.0;
    }
    return w;
}

HD TimeW time_weights(double tau, double dt) {
    return time_weights_r(tau, 1.0 / dt, tau > 0.0 ? 0.5 * dt / tau : 0.0);
}

// Second-order BGK interface flux at one face point, already linearised in
// time: F and dF/dt at t_n (flux.hpp:71-124 + :180-189), split into one pass
// per side plus a merge so a kernel can build each trace just in time.
// Traces are in the face-local frame: q[5], dq_n[5], dq_t1[5], dq_t2[5].
// A side pass accumulates its half-space moments of the merged state and
// slopes and its UNWEIGHTED non-equilibrium moments, and reports its pressure:
// tau = mu / mean trace pressure (dg.hpp:378-383) needs both sides, so the
// time weights enter once, in the merge.
struct FluxAcc {
    double q0_[5];      // rho_l <psi>_+ + rho_r <psi>_-              (flux.hpp:85-86)
    double dq0_[3][5];  // rho_l <a_l psi>_+ + rho_r <a_r psi>_-       (flux.hpp:92-93)
    double nq_[3][5];   // sum_sides rho <u psi>_h, <u (a.u) psi>_h, <u A psi>_h (flux.hpp:112-121)
    HD double& q0(int m) { return q0_[m]; }
    HD double& dq0(int d, int m) { return dq0_[d][m]; }
    HD double& nq(int k, int m) { return nq_[k][m]; }
};

// the same accumulator as a per-thread shared-memory column ([slot][thread]:
// consecutive lanes hit consecutive 8-byte words)
struct SmemAcc {
    double* p;   // &base[tid]
    int stride;  // threads per CTA
    HD double& q0(int m) { return p[m * stride]; }
    HD double& dq0(int d, int m) { return p[(5 + 5 * d + m) * stride]; }
    HD double& nq(int k, int m) { return p[(20 + 5 * k + m) * stride]; }
};

template <class Acc>
HD void flux_init(Acc& acc) {
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        acc.q0(m) = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            acc.dq0(d, m) = 0.0;
            acc.nq(d, m) = 0.0;
        }
    }
}

// <u (a1 u + a2 v + a3 w) psi> (flux.hpp:59-64)
template <class T>
HD void directional_flux(const double* Ut, const T& t, const Slope* a, double* out) {
    double r[5];
    slope_moment<2, 0, 0>(Ut, t, a[0], out);
    slope_moment<1, 1, 0>(Ut, t, a[1], r);
#pragma unroll
    for (int m = 0; m < 5; ++m) out[m] += r[m];
    slope_moment<1, 0, 1>(Ut, t, a[2], r);
#pragma unroll
    for (int m = 0; m < 5; ++m) out[m] += r[m];
}

// side 0 = left (u>0 half), 1 = right (u<0 half). Returns ERR_*; p_side is the
// trace pressure (core.hpp:72-74) for tau.
template <bool VISCOUS, class Acc>
HD int flux_side(const double* t, int side, const GasC& g, Acc& acc, double& p_side, double& bad) {
    Prim w;
    const int rc = prim_from_q_nb(t, g, w, bad);  // checked at the end (one basic block)
    p_side = w.rho * w.il;
    const SolveC sc = solve_consts(w, g);
    // One table object: V, W full; U first full (for A), then overwritten by
    // this side's half table, so the two U sequences are never live together
    // (the side pass peaks below 168 registers less often).
    Tab<6, 5> tb;
    const double il = w.il;
    full_seq<5>(w.V, il, tb.V);
    full_seq<5>(w.W, il, tb.W);
    tb.xi2 = g.K * il;
    tb.dxi = 2.0 * g.K * il * il;
    Slope a[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) a[d] = micro_slope_rho(sc, t + 5 + 5 * d);  // rho a
    Slope A{};  // rho A
    if (VISCOUS) {
        // A from compatibility with the full table (flux.hpp:109-110)
        full_seq<5>(w.U, il, tb.U);
        A = time_coefficient(sc, tb, a);
    }
    half_seq<6>(w.U, w.lam, il, side == 0 ? +1 : -1, tb.U);
    double r[5];
    psi_moment<0, 0, 0>(tb.U, tb, r);
#pragma unroll
    for (int m = 0; m < 5; ++m) acc.q0(m) += w.rho * r[m];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        slope_moment<0, 0, 0>(tb.U, tb, a[d], r);
#pragma unroll
        for (int m = 0; m < 5; ++m) acc.dq0(d, m) += r[m];
    }
    if (VISCOUS) {
        // free-streaming moments of this side (flux.hpp:112-121), unweighted
        psi_moment<1, 0, 0>(tb.U, tb, r);
#pragma unroll
        for (int m = 0; m < 5; ++m) acc.nq(0, m) += w.rho * r[m];
        directional_flux(tb.U, tb, a, r);
#pragma unroll
        for (int m = 0; m < 5; ++m) acc.nq(1, m) += r[m];
        slope_moment<1, 0, 0>(tb.U, tb, A, r);
#pragma unroll
        for (int m = 0; m < 5; ++m) acc.nq(2, m) += r[m];
    }
    return rc;
}

// The merge split in two halves for two cooperating threads: both build the
// merged state (setup), then part A adds g0 + Abar terms (time coefficient +
// 2 moments) and part B the abar term (3 slope moments); the halves' F/Ft
// sum to flux_merge's.
struct MergeState {
    Prim w0;
    SolveC s0;
    Tab<6, 5> t0;
    Slope ab[3];  // rho0 abar
};

HD int merge_setup(const GasC& g, const double* q0, const double* dq0 /*[3][5]*/, MergeState& M,
                   double& bad) {
    const int rc = prim_from_q_nb(q0, g, M.w0, bad);  // checked at the end
    M.s0 = solve_consts(M.w0, g);
    const double il = M.w0.il;
    full_seq<6>(M.w0.U, il, M.t0.U);
    full_seq<5>(M.w0.V, il, M.t0.V);
    full_seq<5>(M.w0.W, il, M.t0.W);
    M.t0.xi2 = g.K * il;
    M.t0.dxi = 2.0 * g.K * il * il;
#pragma unroll
    for (int d = 0; d < 3; ++d) M.ab[d] = micro_slope_rho(M.s0, dq0 + 5 * d);
    return rc;
}

HD void merge_part_a(const MergeState& M, const TimeW& tw, double* F, double* Ft) {
    const Slope Ab = time_coefficient(M.s0, M.t0, M.ab);  // rho0 Abar
    double r[5];
    psi_moment<1, 0, 0>(M.t0.U, M.t0, r);
    const double sF = M.w0.rho * tw.g0F, sFt = M.w0.rho * tw.g0Ft;
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        F[m] = sF * r[m];
        Ft[m] = sFt * r[m];
    }
    slope_moment<1, 0, 0>(M.t0.U, M.t0, Ab, r);
    const double aF = tw.AbF, aFt = tw.AbFt;
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        F[m] += aF * r[m];
        Ft[m] += aFt * r[m];
    }
}

template <bool VISCOUS>
HD void merge_part_b(const MergeState& M, const TimeW& tw, double* F, double* Ft) {
#pragma unroll
    for (int m = 0; m < 5; ++m) F[m] = Ft[m] = 0.0;
    if (VISCOUS) {  // abar's weight vanishes at tau = 0 (flux.hpp:32-37)
        double r[5];
        directional_flux(M.t0.U, M.t0, M.ab, r);
        const double sF = tw.abF, sFt = tw.abFt;
#pragma unroll
        for (int m = 0; m < 5; ++m) {
            F[m] = sF * r[m];
            Ft[m] = sFt * r[m];
        }
    }
}

// Merged-state equilibrium terms (flux.hpp:87-106) plus the time-weighted
// non-equilibrium moments (flux.hpp:112-121): F, Ft final.
template <bool VISCOUS, class Acc>
HD int flux_merge(const GasC& g, const TimeW& tw, Acc& acc, double* F, double* Ft, double& bad) {
    double q0[5], dq0[15];
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        q0[m] = acc.q0(m);
#pragma unroll
        for (int d = 0; d < 3; ++d) dq0[5 * d + m] = acc.dq0(d, m);
    }
    MergeState M;
    const int rc = merge_setup(g, q0, dq0, M, bad);  // checked at the end
    merge_part_a(M, tw, F, Ft);
    double Fb[5], Ftb[5];
    merge_part_b<VISCOUS>(M, tw, Fb, Ftb);
#pragma unroll
    for (int m = 0; m < 5; ++m) {
        F[m] += Fb[m];
        Ft[m] += Ftb[m];
        if (VISCOUS) {
            F[m] += tw.f0F * acc.nq(0, m) + tw.anF * acc.nq(1, m) + tw.AnF * acc.nq(2, m);
            Ft[m] += tw.f0Ft * acc.nq(0, m) + tw.anFt * acc.nq(1, m) + tw.AnFt * acc.nq(2, m);
        }
    }
    return rc;
}

// Whole interface flux from two traces at a given tau; stage = 0 left,
// 1 right, 2 merged on failure (the reference's check order, flux.hpp:73-87).
template <bool VISCOUS>
HD int interface_flux(const double* tl, const double* tr, const GasC& g, const TimeW& tw,
                      double* F, double* Ft, int& stage, double& bad) {
    FluxAcc acc;
    flux_init(acc);
    double pl = 0.0, pr = 0.0;
    int rc = flux_side<VISCOUS>(tl, 0, g, acc, pl, bad);
    if (rc) {
        stage = 0;
        return rc;
    }
    rc = flux_side<VISCOUS>(tr, 1, g, acc, pr, bad);
    if (rc) {
        stage = 1;
        return rc;
    }
    rc = flux_merge<VISCOUS>(g, tw, acc, F, Ft, bad);
    if (rc) {
        stage = 2;
        return rc;
    }
    return ERR_NONE;
}

// Smooth in-cell flux along all three axes at one volume point, linearised:
// F_a = rho <u_a psi> - tau (rho sum_i <a_i u_i u_a psi> + FA_a), Ft_a = FA_a
// (flux.hpp:128-165 + :180-189 in closed form). t = q[5], dq_x, dq_y, dq_z.
// out[a][0..4] = F_a, out[a][5..9] = Ft_a.
// FT_ONLY (the S2O4 second stage, which uses only Lt): skip F, i.e. the
// psi moments and the 9 viscous slope moments; out[a][5..9] only.
template <bool VISCOUS, int NAXES, bool FT_ONLY = false>
HD int smooth_flux(const double* t, const GasC& g, double* out, double& bad) {
    Prim w;
    const int rc = prim_from_q_nb(t, g, w, bad);  // checked at the end
    const double tau = VISCOUS ? g.mu * (2.0 * w.lam * w.inv_rho) : 0.0;  // tau = mu/p (dg.hpp:433)
    const SolveC sc = solve_consts(w, g);
    Tab<6, 6> tb;
    make_tab(w, g, tb);
    Slope a[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) a[d] = micro_slope_rho(sc, t + 5 + 5 * d);  // rho a
    const Slope A = time_coefficient(sc, tb, a);                                 // rho A
    double F0[5], FA[5], r[5], v[5];
#pragma unroll
    for (int ax = 0; ax < NAXES; ++ax) {
        if (FT_ONLY) {
            if (ax == 0) slope_moment<1, 0, 0>(tb.U, tb, A, FA);
            else if (ax == 1) slope_moment<0, 1, 0>(tb.U, tb, A, FA);
            else slope_moment<0, 0, 1>(tb.U, tb, A, FA);
            double* o = out + 10 * ax;
#pragma unroll
            for (int m = 0; m < 5; ++m) o[5 + m] = FA[m];
            continue;
        }
        if (ax == 0) {
            psi_moment<1, 0, 0>(tb.U, tb, F0);
            slope_moment<1, 0, 0>(tb.U, tb, A, FA);
        } else if (ax == 1) {
            psi_moment<0, 1, 0>(tb.U, tb, F0);
            slope_moment<0, 1, 0>(tb.U, tb, A, FA);
        } else {
            psi_moment<0, 0, 1>(tb.U, tb, F0);
            slope_moment<0, 0, 1>(tb.U, tb, A, FA);
        }
        double* o = out + 10 * ax;
        if (VISCOUS) {
            if (ax == 0) {
                slope_moment<2, 0, 0>(tb.U, tb, a[0], v);
                slope_moment<1, 1, 0>(tb.U, tb, a[1], r);
#pragma unroll
                for (int m = 0; m < 5; ++m) v[m] += r[m];
                slope_moment<1, 0, 1>(tb.U, tb, a[2], r);
            } else if (ax == 1) {
                slope_moment<1, 1, 0>(tb.U, tb, a[0], v);
                slope_moment<0, 2, 0>(tb.U, tb, a[1], r);
#pragma unroll
                for (int m = 0; m < 5; ++m) v[m] += r[m];
                slope_moment<0, 1, 1>(tb.U, tb, a[2], r);
            } else {
                slope_moment<1, 0, 1>(tb.U, tb, a[0], v);
                slope_moment<0, 1, 1>(tb.U, tb, a[1], r);
#pragma unroll
                for (int m = 0; m < 5; ++m) v[m] += r[m];
                slope_moment<0, 0, 2>(tb.U, tb, a[2], r);
            }
#pragma unroll
            for (int m = 0; m < 5; ++m) {
                const double fvis = (v[m] + r[m]) + FA[m];
                o[m] = w.rho * F0[m] - tau * fvis;
                o[5 + m] = FA[m];
            }
        } else {
#pragma unroll
            for (int m = 0; m < 5; ++m) {
                o[m] = w.rho * F0[m];
                o[5 + m] = FA[m];
            }
        }
    }
    return rc;
}

}  // namespace hgks_dev
