/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference DG-HGKS
 * time step, the CPU oracle for the CUDA path. See hgks_oracle.h for the
 * parity pin. Every routine cites the reference lines it restates
 * (paths relative to /root/reference/proj/include/hgks/). Floating-point
 * operation order follows the reference expression by expression so the two
 * agree to the last bit when built with the same contraction setting.
 * Single-threaded: the reference's worker partition (runtime.hpp:47-77) is
 * bitwise neutral, so sequential order is the reference result for every W.
 */
#include "hgks_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define MAXN 20   /* P3 in 3D */
#define MAXPTS 125

/* ------------------------------------------------------------------ state */
typedef struct { double v[5]; } V5;

static V5 v5_add(V5 a, V5 b) { V5 r; for (int i = 0; i < 5; ++i) r.v[i] = a.v[i] + b.v[i]; return r; }
static V5 v5_sub(V5 a, V5 b) { V5 r; for (int i = 0; i < 5; ++i) r.v[i] = a.v[i] - b.v[i]; return r; }
static V5 v5_scale(double s, V5 a) { V5 r; for (int i = 0; i < 5; ++i) r.v[i] = s * a.v[i]; return r; }
static void v5_acc(V5* a, V5 b) { for (int i = 0; i < 5; ++i) a->v[i] += b.v[i]; }

typedef struct { double gamma, K, mu; } Gas;           /* core.hpp:29-43 */
typedef struct { double rho, U, V, W, lam; } Prim;      /* core.hpp:52-54 */

static Gas gas_make(double gamma, double mu) {          /* core.hpp:35-42 */
    Gas g; g.gamma = gamma; g.K = (5.0 - 3.0 * gamma) / (gamma - 1.0); g.mu = mu; return g;
}

/* core.hpp:72-74 */
static double pressure_q(const double* q, const Gas* g) {
    return (g->gamma - 1.0) * (q[4] - 0.5 * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) / q[0]);
}

/* core.hpp:76-82; returns ORC_OK or the failing code with *bad = value */
static int prim_from_q(const double* q, const Gas* g, Prim* w, double* bad) {
    if (!(q[0] > 0.0)) { *bad = q[0]; return ORC_NONPOS_DENSITY; }
    const double p = pressure_q(q, g);
    if (!(p > 0.0)) { *bad = p; return ORC_NONPOS_PRESSURE; }
    const double inv = 1.0 / q[0];
    w->rho = q[0]; w->U = q[1] * inv; w->V = q[2] * inv; w->W = q[3] * inv; w->lam = 0.5 * q[0] / p;
    return ORC_OK;
}

static double pressure_w(const Prim* w) { return 0.5 * w->rho / w->lam; }      /* core.hpp:90 */
static double sound_speed(const Prim* w, const Gas* g) {                        /* core.hpp:92-94 */
    return sqrt(g->gamma * pressure_w(w) / w->rho);
}

static void fill_msg(orc_error* e, int code, int item, double value, int wrap) {
    if (!e) return;
    e->code = code; e->item = item; e->value = value;
    char inner[160];
    if (code == ORC_NONPOS_DENSITY) snprintf(inner, sizeof inner, "non-positive density: rho=%f", value);
    else if (code == ORC_NONPOS_PRESSURE) snprintf(inner, sizeof inner, "non-positive pressure: p=%f", value);
    else if (code == ORC_NONPOS_DT) snprintf(inner, sizeof inner, "compute_dt: nonpositive dt");
    else snprintf(inner, sizeof inner, "configuration error");
    if (wrap) snprintf(e->msg, sizeof e->msg, "item %d: %s", item, inner); /* runtime.hpp:37-41 */
    else snprintf(e->msg, sizeof e->msg, "%s", inner);
}

/* ---------------------------------------------------------------- moments */
/* MomentTable, moments.hpp:16-25 */
typedef struct { double u[9], upos[9], uneg[9], v[9], w[9], xi2, xi4; } Mom;
enum { H_NONE = 0, H_POS = 1, H_NEG = 2 };

/* maxwellian_moments, moments.hpp:27-60 */
static void moments(const Prim* p, const Gas* g, Mom* m) {
    const double us = p->U, vs = p->V, ws = p->W;
    const double il = 0.5 / p->lam;
    const double sql = sqrt(p->lam);
    const double beta = 0.5 * exp(-p->lam * us * us) / sqrt(M_PI * p->lam);
    m->u[0] = 1.0; m->u[1] = us;
    m->v[0] = 1.0; m->v[1] = vs;
    m->w[0] = 1.0; m->w[1] = ws;
    m->upos[0] = 0.5 * erfc(-sql * us);
    m->upos[1] = us * m->upos[0] + beta;
    m->uneg[0] = 0.5 * erfc(sql * us);
    m->uneg[1] = us * m->uneg[0] - beta;
    for (int n = 2; n <= 8; ++n) {
        const double c = (n - 1) * il;
        m->u[n] = us * m->u[n - 1] + c * m->u[n - 2];
        m->v[n] = vs * m->v[n - 1] + c * m->v[n - 2];
        m->w[n] = ws * m->w[n - 1] + c * m->w[n - 2];
        m->upos[n] = us * m->upos[n - 1] + c * m->upos[n - 2];
        m->uneg[n] = us * m->uneg[n - 1] + c * m->uneg[n - 2];
    }
    m->xi2 = g->K * il;
    m->xi4 = g->K * (g->K + 2.0) * il * il;
}

static const double* utab(const Mom* m, int h) { return h == H_POS ? m->upos : h == H_NEG ? m->uneg : m->u; }
static double xif(const Mom* m, int s) { return s == 0 ? 1.0 : s == 1 ? m->xi2 : m->xi4; }

/* psi_moment, moments.hpp:79-91 */
static V5 psi(const Mom* m, int i, int j, int k, int s, int h) {
    const double* mu = utab(m, h);
    const double x0 = xif(m, s), x1 = xif(m, s + 1);
    const double vj = m->v[j], wk = m->w[k];
    const double base = mu[i] * vj * wk;
    V5 r;
    r.v[0] = base * x0;
    r.v[1] = mu[i + 1] * vj * wk * x0;
    r.v[2] = mu[i] * m->v[j + 1] * wk * x0;
    r.v[3] = mu[i] * vj * m->w[k + 1] * x0;
    r.v[4] = 0.5 * ((mu[i + 2] * vj * wk + mu[i] * m->v[j + 2] * wk + mu[i] * vj * m->w[k + 2]) * x0 +
                    base * x1);
    return r;
}

/* MicroSlope, microslope.hpp:9-11 */
typedef struct { double c1, c2, c3, c4, c5; } Slope;

/* slope_moment, microslope.hpp:14-24 */
static V5 slope_moment(const Mom* m, const Slope* a, int i, int j, int k, int h) {
    V5 r = v5_scale(a->c1, psi(m, i, j, k, 0, h));
    v5_acc(&r, v5_scale(a->c2, psi(m, i + 1, j, k, 0, h)));
    v5_acc(&r, v5_scale(a->c3, psi(m, i, j + 1, k, 0, h)));
    v5_acc(&r, v5_scale(a->c4, psi(m, i, j, k + 1, 0, h)));
    V5 q = v5_add(v5_add(v5_add(psi(m, i + 2, j, k, 0, h), psi(m, i, j + 2, k, 0, h)),
                         psi(m, i, j, k + 2, 0, h)),
                  psi(m, i, j, k, 1, h));
    v5_acc(&r, v5_scale(0.5 * a->c5, q));
    return r;
}

/* detail::solve_slope_unit, microslope.hpp:29-44 */
static Slope solve_slope_unit(const Prim* w, V5 r, const Gas* g) {
    const double D = g->K + 3.0;
    const double q2 = w->U * w->U + w->V * w->V + w->W * w->W;
    const double sbar = 0.5 * D / w->lam;
    const double B = 2.0 * r.v[4] - (q2 + sbar) * r.v[0];
    const double R2 = r.v[1] - w->U * r.v[0];
    const double R3 = r.v[2] - w->V * r.v[0];
    const double R4 = r.v[3] - w->W * r.v[0];
    Slope a;
    a.c5 = 4.0 * w->lam * w->lam / D * (B - 2.0 * (w->U * R2 + w->V * R3 + w->W * R4));
    a.c2 = 2.0 * w->lam * R2 - w->U * a.c5;
    a.c3 = 2.0 * w->lam * R3 - w->V * a.c5;
    a.c4 = 2.0 * w->lam * R4 - w->W * a.c5;
    a.c1 = r.v[0] - w->U * a.c2 - w->V * a.c3 - w->W * a.c4 - 0.5 * a.c5 * (q2 + sbar);
    return a;
}

/* micro_slope, microslope.hpp:49-52 */
static Slope micro_slope(const Prim* w, V5 dq, const Gas* g) {
    const double inv = 1.0 / w->rho;
    return solve_slope_unit(w, v5_scale(inv, dq), g);
}

/* time_coefficient, microslope.hpp:56-61 */
static Slope time_coefficient(const Prim* w, const Mom* m, const Slope* ax, const Slope* ay,
                              const Slope* az, const Gas* g) {
    V5 s = v5_add(v5_add(slope_moment(m, ax, 1, 0, 0, H_NONE), slope_moment(m, ay, 0, 1, 0, H_NONE)),
                  slope_moment(m, az, 0, 0, 1, H_NONE));
    return solve_slope_unit(w, v5_scale(-1.0, s), g);
}

/* ------------------------------------------------------------------ fluxes */
typedef struct { double g0, abar, Abar, f0, aneq, Aneq; } TCoef;

/* flux_time_integrals, flux.hpp:26-48 */
static TCoef time_integrals(double tau, double dt) {
    TCoef c;
    if (tau <= 0.0) {
        c.g0 = dt; c.abar = 0.0; c.Abar = 0.5 * dt * dt; c.f0 = c.aneq = c.Aneq = 0.0;
        return c;
    }
    const double r = dt / tau;
    const double E = r > 700.0 ? 0.0 : exp(-r);
    c.g0 = dt - tau * (1.0 - E);
    c.abar = 2.0 * tau * tau - tau * dt - tau * (dt + 2.0 * tau) * E;
    c.Abar = 0.5 * dt * dt - tau * dt + tau * tau * (1.0 - E);
    c.f0 = tau * (1.0 - E);
    c.aneq = -2.0 * tau * tau + tau * (dt + 2.0 * tau) * E;
    c.Aneq = -tau * tau * (1.0 - E);
    return c;
}

/* detail::directional_slope_flux, flux.hpp:59-64 */
static V5 dir_flux(const Mom* m, const Slope* a, int h) {
    return v5_add(v5_add(slope_moment(m, &a[0], 2, 0, 0, h), slope_moment(m, &a[1], 1, 1, 0, h)),
                  slope_moment(m, &a[2], 1, 0, 1, h));
}

static V5 q5(const double* t) { V5 r; memcpy(r.v, t, sizeof r.v); return r; }

/* interface_flux_integrals, flux.hpp:71-124. Traces t = q[5], dq[3][5] in
 * the face-local frame. fail = which state failed (0 left, 1 right, 2 merged). */
static int interface_flux(const double* tl, const double* tr, const Gas* g, double tau, double dt,
                          V5* full, V5* half, double* bad) {
    Prim wl, wr, w0;
    int rc;
    if ((rc = prim_from_q(tl, g, &wl, bad))) return rc;
    if ((rc = prim_from_q(tr, g, &wr, bad))) return rc;
    Mom ml, mr, m0;
    moments(&wl, g, &ml);
    moments(&wr, g, &mr);
    Slope al[3], ar[3], abar[3];
    for (int i = 0; i < 3; ++i) {
        al[i] = micro_slope(&wl, q5(tl + 5 + 5 * i), g);
        ar[i] = micro_slope(&wr, q5(tr + 5 + 5 * i), g);
    }
    const V5 q0 = v5_add(v5_scale(wl.rho, psi(&ml, 0, 0, 0, 0, H_POS)),
                         v5_scale(wr.rho, psi(&mr, 0, 0, 0, 0, H_NEG)));
    if ((rc = prim_from_q(q0.v, g, &w0, bad))) return rc;
    moments(&w0, g, &m0);
    for (int i = 0; i < 3; ++i) {
        const V5 dq0 = v5_add(v5_scale(wl.rho, slope_moment(&ml, &al[i], 0, 0, 0, H_POS)),
                              v5_scale(wr.rho, slope_moment(&mr, &ar[i], 0, 0, 0, H_NEG)));
        abar[i] = micro_slope(&w0, dq0, g);
    }
    const Slope Abar = time_coefficient(&w0, &m0, &abar[0], &abar[1], &abar[2], g);
    const V5 Fg0 = v5_scale(w0.rho, psi(&m0, 1, 0, 0, 0, H_NONE));
    const V5 Fabar = v5_scale(w0.rho, dir_flux(&m0, abar, H_NONE));
    const V5 FAbar = v5_scale(w0.rho, slope_moment(&m0, &Abar, 1, 0, 0, H_NONE));
    const TCoef cf = time_integrals(tau, dt);
    const TCoef ch = time_integrals(tau, 0.5 * dt);
    *full = v5_add(v5_add(v5_scale(cf.g0, Fg0), v5_scale(cf.abar, Fabar)), v5_scale(cf.Abar, FAbar));
    *half = v5_add(v5_add(v5_scale(ch.g0, Fg0), v5_scale(ch.abar, Fabar)), v5_scale(ch.Abar, FAbar));
    if (tau > 0.0) {
        const Slope Al = time_coefficient(&wl, &ml, &al[0], &al[1], &al[2], g);
        const Slope Ar = time_coefficient(&wr, &mr, &ar[0], &ar[1], &ar[2], g);
        const V5 Ff0 = v5_add(v5_scale(wl.rho, psi(&ml, 1, 0, 0, 0, H_POS)),
                              v5_scale(wr.rho, psi(&mr, 1, 0, 0, 0, H_NEG)));
        const V5 Faneq = v5_add(v5_scale(wl.rho, dir_flux(&ml, al, H_POS)),
                                v5_scale(wr.rho, dir_flux(&mr, ar, H_NEG)));
        const V5 FAneq = v5_add(v5_scale(wl.rho, slope_moment(&ml, &Al, 1, 0, 0, H_POS)),
                                v5_scale(wr.rho, slope_moment(&mr, &Ar, 1, 0, 0, H_NEG)));
        v5_acc(full, v5_add(v5_add(v5_scale(cf.f0, Ff0), v5_scale(cf.aneq, Faneq)), v5_scale(cf.Aneq, FAneq)));
        v5_acc(half, v5_add(v5_add(v5_scale(ch.f0, Ff0), v5_scale(ch.aneq, Faneq)), v5_scale(ch.Aneq, FAneq)));
    }
    return ORC_OK;
}

/* SmoothPoint / make_smooth_point, flux.hpp:128-143 */
typedef struct { Prim w; Mom m; Slope a[3]; Slope A; } Smooth;

static int make_smooth(const double* t, const Gas* g, Smooth* p, double* bad) {
    int rc = prim_from_q(t, g, &p->w, bad);
    if (rc) return rc;
    moments(&p->w, g, &p->m);
    for (int i = 0; i < 3; ++i) p->a[i] = micro_slope(&p->w, q5(t + 5 + 5 * i), g);
    p->A = time_coefficient(&p->w, &p->m, &p->a[0], &p->a[1], &p->a[2], g);
    return ORC_OK;
}

/* smooth_flux_integrals, flux.hpp:148-165 */
static void smooth_flux(const Smooth* p, double tau, double dt, int axis, V5* full, V5* half) {
    const int iu = axis == 0, iv = axis == 1, iw = axis == 2;
    const V5 F0 = v5_scale(p->w.rho, psi(&p->m, iu, iv, iw, 0, H_NONE));
    const V5 FA = v5_scale(p->w.rho, slope_moment(&p->m, &p->A, iu, iv, iw, H_NONE));
    V5 Fvis = {{0, 0, 0, 0, 0}};
    if (tau > 0.0) {
        Fvis = v5_add(v5_add(slope_moment(&p->m, &p->a[0], iu + 1, iv, iw, H_NONE),
                             slope_moment(&p->m, &p->a[1], iu, iv + 1, iw, H_NONE)),
                      slope_moment(&p->m, &p->a[2], iu, iv, iw + 1, H_NONE));
        Fvis = v5_add(v5_scale(p->w.rho, Fvis), FA);
    }
    const double ds[2] = {dt, 0.5 * dt};
    for (int q = 0; q < 2; ++q) {
        const double d = ds[q];
        const V5 r = v5_add(v5_scale(d, v5_sub(F0, v5_scale(tau, Fvis))), v5_scale(0.5 * d * d, FA));
        if (q == 0) *full = r; else *half = r;
    }
}

/* flux_linearize, flux.hpp:180-189 */
static void linearize(V5 If, V5 Ih, double dt, double* F, double* Ft) {
    const double a = 1.0 / dt;
    const double b = 4.0 / (dt * dt);
    for (int i = 0; i < 5; ++i) {
        F[i] = (4.0 * Ih.v[i] - If.v[i]) * a;
        Ft[i] = (If.v[i] - 2.0 * Ih.v[i]) * b;
    }
}

/* ------------------------------------------------------ quadrature & basis */
/* QuadRule::gauss, quadrature.hpp:15-58 */
static int gauss(int m, double* x, double* w) {
    switch (m) {
        case 1: x[0] = 0.0; w[0] = 2.0; return 1;
        case 2: { const double a = 1.0 / sqrt(3.0); x[0] = -a; x[1] = a; w[0] = w[1] = 1.0; return 2; }
        case 3: { const double a = sqrt(3.0 / 5.0);
                  x[0] = -a; x[1] = 0.0; x[2] = a; w[0] = 5.0 / 9.0; w[1] = 8.0 / 9.0; w[2] = 5.0 / 9.0; return 3; }
        case 4: { const double s = sqrt(6.0 / 5.0);
                  const double a = sqrt((3.0 - 2.0 * s) / 7.0), b = sqrt((3.0 + 2.0 * s) / 7.0);
                  const double wa = (18.0 + sqrt(30.0)) / 36.0, wb = (18.0 - sqrt(30.0)) / 36.0;
                  x[0] = -b; x[1] = -a; x[2] = a; x[3] = b; w[0] = wb; w[1] = wa; w[2] = wa; w[3] = wb; return 4; }
        case 5: { const double s = sqrt(10.0 / 7.0);
                  const double a = sqrt(5.0 - 2.0 * s) / 3.0, b = sqrt(5.0 + 2.0 * s) / 3.0;
                  const double wa = (322.0 + 13.0 * sqrt(70.0)) / 900.0, wb = (322.0 - 13.0 * sqrt(70.0)) / 900.0;
                  x[0] = -b; x[1] = -a; x[2] = 0.0; x[3] = a; x[4] = b;
                  w[0] = wb; w[1] = wa; w[2] = 128.0 / 225.0; w[3] = wa; w[4] = wb; return 5; }
    }
    return 0;
}

/* legendre / legendre_deriv, basis.hpp:11-34 */
static double legendre(int l, double x) {
    if (l == 0) return 1.0;
    double pm = 1.0, p = x;
    for (int n = 1; n < l; ++n) {
        const double pn = ((2.0 * n + 1.0) * x * p - n * pm) / (n + 1.0);
        pm = p; p = pn;
    }
    return p;
}
static double legendre_d(int l, double x) {
    if (l == 0) return 0.0;
    double pm = 1.0, p = x, dm = 0.0, d = 1.0;
    for (int n = 1; n < l; ++n) {
        const double pn = ((2.0 * n + 1.0) * x * p - n * pm) / (n + 1.0);
        const double dn = ((2.0 * n + 1.0) * (p + x * d) - n * dm) / (n + 1.0);
        pm = p; p = pn; dm = d; d = dn;
    }
    return d;
}

typedef struct { int degree, dim, N; int idx[MAXN][3]; } Basis;

static int idx_less(const int* a, const int* c) {  /* graded, then lexicographic (basis.hpp:71-75) */
    const int da = a[0] + a[1] + a[2], dc = c[0] + c[1] + c[2];
    if (da != dc) return da < dc;
    for (int i = 0; i < 3; ++i) if (a[i] != c[i]) return a[i] < c[i];
    return 0;
}

/* build_basis, basis.hpp:64-82 (degree 1 accepted here as the documented
 * P1 extension; the reference rejects it) */
static int build_basis(int k, int dim, Basis* b) {
    if (k < 1 || k > 3 || (dim != 2 && dim != 3)) return ORC_CONFIG;
    b->degree = k; b->dim = dim; b->N = 0;
    const int zmax = dim == 3 ? k : 0;
    for (int nx = 0; nx <= k; ++nx)
        for (int ny = 0; ny <= k; ++ny)
            for (int nz = 0; nz <= zmax; ++nz)
                if (nx + ny + nz <= k) { b->idx[b->N][0] = nx; b->idx[b->N][1] = ny; b->idx[b->N][2] = nz; ++b->N; }
    for (int i = 1; i < b->N; ++i)  /* insertion sort: same order as std::sort with a strict key */
        for (int j = i; j > 0 && idx_less(b->idx[j], b->idx[j - 1]); --j) {
            int t[3]; memcpy(t, b->idx[j], sizeof t); memcpy(b->idx[j], b->idx[j - 1], sizeof t); memcpy(b->idx[j - 1], t, sizeof t);
        }
    return ORC_OK;
}

static double basis_eval(const Basis* b, int n, double x, double y, double z) {     /* basis.hpp:43-47 */
    return legendre(b->idx[n][0], x) * legendre(b->idx[n][1], y) * legendre(b->idx[n][2], z);
}
static double basis_deriv(const Basis* b, int n, int a, double x, double y, double z) { /* :50-55 */
    const double fx = a == 0 ? legendre_d(b->idx[n][0], x) : legendre(b->idx[n][0], x);
    const double fy = a == 1 ? legendre_d(b->idx[n][1], y) : legendre(b->idx[n][1], y);
    const double fz = a == 2 ? legendre_d(b->idx[n][2], z) : legendre(b->idx[n][2], z);
    return fx * fy * fz;
}

/* PointBasis, dg.hpp:54-74 */
typedef struct {
    int npts;
    double B[MAXPTS][MAXN];
    double dB[MAXPTS][3][MAXN];
    double w[MAXPTS];
    double ref[MAXPTS][3];
} PB;

static void pb_add(PB* pb, const Basis* b, double x, double y, double z, double w) {
    const int p = pb->npts++;
    pb->ref[p][0] = x; pb->ref[p][1] = y; pb->ref[p][2] = z; pb->w[p] = w;
    for (int n = 0; n < b->N; ++n) pb->B[p][n] = basis_eval(b, n, x, y, z);
    for (int a = 0; a < 3; ++a)
        for (int n = 0; n < b->N; ++n) pb->dB[p][a][n] = basis_deriv(b, n, a, x, y, z);
}

/* DGTables::make, dg.hpp:91-128. P1 uses a 2-point flux rule (extension). */
typedef struct { Basis basis; int nq_flux, nq_proj; PB vol, proj, fm[3], fp[3]; } Tables;

static void tables_make(Tables* t, const Basis* b) {
    memset(t, 0, sizeof *t);
    t->basis = *b;
    t->nq_flux = b->degree <= 2 ? 2 : 3;
    t->nq_proj = b->degree + 2;
    double xf[5], wf[5], xp[5], wp[5], x1[1], w1[1];
    const int nf = gauss(t->nq_flux, xf, wf), np = gauss(t->nq_proj, xp, wp);
    gauss(1, x1, w1);
    const int nfz = b->dim == 3 ? nf : 1, npz = b->dim == 3 ? np : 1;
    const double *xfz = b->dim == 3 ? xf : x1, *wfz = b->dim == 3 ? wf : w1;
    const double *xpz = b->dim == 3 ? xp : x1, *wpz = b->dim == 3 ? wp : w1;
    for (int i = 0; i < nf; ++i)
        for (int j = 0; j < nf; ++j)
            for (int k = 0; k < nfz; ++k) pb_add(&t->vol, b, xf[i], xf[j], xfz[k], wf[i] * wf[j] * wfz[k]);
    for (int i = 0; i < np; ++i)
        for (int j = 0; j < np; ++j)
            for (int k = 0; k < npz; ++k) pb_add(&t->proj, b, xp[i], xp[j], xpz[k], wp[i] * wp[j] * wpz[k]);
    for (int a = 0; a < 3; ++a) {
        const int bb = (a + 1) % 3, c = (a + 2) % 3;
        const int use1b = bb == 2 && b->dim == 2, use1c = c == 2 && b->dim == 2;
        const int nb = use1b ? 1 : nf, nc = use1c ? 1 : nf;
        const double *xb = use1b ? x1 : xf, *wb = use1b ? w1 : wf;
        const double *xc = use1c ? x1 : xf, *wc = use1c ? w1 : wf;
        for (int ib = 0; ib < nb; ++ib)
            for (int ic = 0; ic < nc; ++ic) {
                double r[3] = {0, 0, 0};
                r[bb] = xb[ib]; r[c] = xc[ic];
                const double w = wb[ib] * wc[ic];
                r[a] = -1.0; pb_add(&t->fm[a], b, r[0], r[1], r[2], w);
                r[a] = 1.0;  pb_add(&t->fp[a], b, r[0], r[1], r[2], w);
            }
    }
}

/* eval_tabulated, dg.hpp:139-161: out = q[5], dq[3][5] (global frame) */
static void eval_tab(const double* coeffs, int N, const PB* pb, int p, const double* h, double* out) {
    double val[5] = {0, 0, 0, 0, 0};
    for (int n = 0; n < N; ++n) {
        const double b = pb->B[p][n];
        for (int v = 0; v < 5; ++v) val[v] += b * coeffs[n * 5 + v];
    }
    memcpy(out, val, sizeof val);
    for (int a = 0; a < 3; ++a) {
        const double scale = 2.0 / h[a];
        double d[5] = {0, 0, 0, 0, 0};
        for (int n = 0; n < N; ++n) {
            const double b = pb->dB[p][a][n];
            for (int v = 0; v < 5; ++v) d[v] += b * coeffs[n * 5 + v];
        }
        for (int v = 0; v < 5; ++v) out[5 + 5 * a + v] = scale * d[v];
    }
}

/* detail::to_face_local / from_face_local, dg.hpp:323-345 */
static void to_face_local(const double* e, int axis, double* t) {
    const int c1 = (axis + 1) % 3, c2 = (axis + 2) % 3;
    for (int d = 0; d < 4; ++d) {
        const double* s = d == 0 ? e : e + 5 + 5 * (d == 1 ? axis : d == 2 ? c1 : c2);
        double* o = t + 5 * d;
        o[0] = s[0]; o[1] = s[1 + axis]; o[2] = s[1 + c1]; o[3] = s[1 + c2]; o[4] = s[4];
    }
}
static void from_face_local(const double* f, int axis, double* g) {
    const int c1 = (axis + 1) % 3, c2 = (axis + 2) % 3;
    g[0] = f[0]; g[4] = f[4]; g[1 + axis] = f[1]; g[1 + c1] = f[2]; g[1 + c2] = f[3];
}

/* ------------------------------------------------------------------ solver */
typedef enum { CASE_NONE, CASE_ADV2D, CASE_ADV3D, CASE_VORTEX2D, CASE_TGV } CaseId;

struct orc_solver {
    int nx, ny, nz, ncells;
    double *xs, *ys, *zs;
    Gas gas;
    Basis basis;
    Tables* tab;
    double* q;           /* AoS state */
    double *R, *Rt, *face[3];
    double *L1, *Lt1, *L2, *Lt2, *qs;
    CaseId cid;
    double mach0, eps;
};

static void widths(const orc_solver* s, int c, double* h) {   /* mesh.hpp:34-56 */
    const int i = c % s->nx, j = (c / s->nx) % s->ny, k = c / (s->nx * s->ny);
    h[0] = s->xs[i + 1] - s->xs[i]; h[1] = s->ys[j + 1] - s->ys[j]; h[2] = s->zs[k + 1] - s->zs[k];
}
static void center(const orc_solver* s, int c, double* x) {   /* mesh.hpp:49-61 */
    const int i = c % s->nx, j = (c / s->nx) % s->ny, k = c / (s->nx * s->ny);
    x[0] = 0.5 * (s->xs[i] + s->xs[i + 1]); x[1] = 0.5 * (s->ys[j] + s->ys[j + 1]); x[2] = 0.5 * (s->zs[k] + s->zs[k + 1]);
}
static int neighbor(const orc_solver* s, int c, int axis, int dir) {  /* dg.hpp:307-319 */
    int ijk[3] = {c % s->nx, (c / s->nx) % s->ny, c / (s->nx * s->ny)};
    const int n = axis == 0 ? s->nx : axis == 1 ? s->ny : s->nz;
    ijk[axis] = (ijk[axis] + (dir < 0 ? n - 1 : 1)) % n;
    return ijk[0] + s->nx * (ijk[1] + s->ny * ijk[2]);
}

orc_solver* orc_create(int nx, int ny, int nz, const double* xs, const double* ys, const double* zs,
                       int degree, int dim, double gamma, double mu, orc_error* err) {
    Basis b;
    if (build_basis(degree, dim, &b) != ORC_OK || nx < 1 || ny < 1 || nz < 1) {
        if (err) { err->code = ORC_CONFIG; err->item = -1; snprintf(err->msg, sizeof err->msg, "invalid configuration"); }
        return NULL;
    }
    orc_solver* s = calloc(1, sizeof *s);
    s->nx = nx; s->ny = ny; s->nz = nz; s->ncells = nx * ny * nz;
    s->xs = malloc((nx + 1) * sizeof(double)); memcpy(s->xs, xs, (nx + 1) * sizeof(double));
    s->ys = malloc((ny + 1) * sizeof(double)); memcpy(s->ys, ys, (ny + 1) * sizeof(double));
    s->zs = malloc((nz + 1) * sizeof(double)); memcpy(s->zs, zs, (nz + 1) * sizeof(double));
    s->gas = gas_make(gamma, mu);
    s->basis = b;
    s->tab = malloc(sizeof(Tables));
    tables_make(s->tab, &b);
    const size_t nc = (size_t)s->ncells * b.N * 5;
    s->q = calloc(nc, sizeof(double));
    s->R = calloc(nc, sizeof(double)); s->Rt = calloc(nc, sizeof(double));
    s->L1 = calloc(nc, sizeof(double)); s->Lt1 = calloc(nc, sizeof(double));
    s->L2 = calloc(nc, sizeof(double)); s->Lt2 = calloc(nc, sizeof(double));
    s->qs = calloc(nc, sizeof(double));
    for (int a = 0; a < 3; ++a) s->face[a] = calloc((size_t)s->ncells * s->tab->fm[a].npts * 10, sizeof(double));
    s->cid = CASE_NONE;
    return s;
}

void orc_free(orc_solver* s) {
    if (!s) return;
    free(s->xs); free(s->ys); free(s->zs); free(s->tab); free(s->q); free(s->R); free(s->Rt);
    free(s->L1); free(s->Lt1); free(s->L2); free(s->Lt2); free(s->qs);
    for (int a = 0; a < 3; ++a) free(s->face[a]);
    free(s);
}

int orc_N(const orc_solver* s) { return s->basis.N; }
int orc_ncells(const orc_solver* s) { return s->ncells; }
long orc_ncoeffs(const orc_solver* s) { return (long)s->ncells * s->basis.N * 5; }
double* orc_state(orc_solver* s) { return s->q; }
int orc_face_npts(const orc_solver* s, int axis) { return s->tab->fm[axis].npts; }

/* residual, dg.hpp:354-450 */
int orc_residual(orc_solver* s, const double* coeffs, double dt, double* R, double* Rt,
                 double* face0, double* face1, double* face2, long* flux_evals, orc_error* err) {
    const int N = s->basis.N, nc = s->ncells;
    const double mu = s->gas.mu;
    const Tables* tab = s->tab;
    double* faces[3] = {face0 ? face0 : s->face[0], face1 ? face1 : s->face[1], face2 ? face2 : s->face[2]};
    if (!coeffs) coeffs = s->q;
    if (!R) R = s->R;
    if (!Rt) Rt = s->Rt;
    /* phase 1: face f of axis a is the minus-a face of cell f (dg.hpp:362-394) */
    for (int fa = 0; fa < 3 * nc; ++fa) {
        const int axis = fa / nc, f = fa % nc;
        const int cm = neighbor(s, f, axis, -1);
        const PB* pbL = &tab->fp[axis];
        const PB* pbR = &tab->fm[axis];
        double hL[3], hR[3];
        widths(s, cm, hL); widths(s, f, hR);
        double* out = faces[axis] + (size_t)f * pbL->npts * 10;
        for (int p = 0; p < pbL->npts; ++p) {
            double eL[20], eR[20], tl[20], tr[20];
            eval_tab(coeffs + (size_t)cm * N * 5, N, pbL, p, hL, eL);
            eval_tab(coeffs + (size_t)f * N * 5, N, pbR, p, hR, eR);
            to_face_local(eL, axis, tl);
            to_face_local(eR, axis, tr);
            double tau = 0.0;
            if (mu > 0.0) {
                const double pl = pressure_q(tl, &s->gas), pr = pressure_q(tr, &s->gas);
                tau = mu / (0.5 * (pl + pr));
            }
            V5 If, Ih;
            double bad = 0;
            const int rc = interface_flux(tl, tr, &s->gas, tau, dt, &If, &Ih, &bad);
            if (rc) { fill_msg(err, rc, fa, bad, 1); return rc; }
            double F[5], Ft[5];
            linearize(If, Ih, dt, F, Ft);
            from_face_local(F, axis, out + p * 10);
            from_face_local(Ft, axis, out + p * 10 + 5);
        }
        if (flux_evals) *flux_evals += pbL->npts;
    }
    /* phase 2: gather faces + volume fluxes per cell (dg.hpp:396-449) */
    for (int c = 0; c < nc; ++c) {
        double h[3];
        widths(s, c, h);
        double* Rc = R + (size_t)c * N * 5;
        double* Rtc = Rt + (size_t)c * N * 5;
        for (int i = 0; i < N * 5; ++i) Rc[i] = Rtc[i] = 0.0;
        for (int axis = 0; axis < 3; ++axis) {
            const int b = (axis + 1) % 3, cc = (axis + 2) % 3;
            const double jac = h[b] * h[cc] / 4.0;
            const PB* pbm = &tab->fm[axis];
            const PB* pbp = &tab->fp[axis];
            const int fplus = neighbor(s, c, axis, +1);
            const double* Fm = faces[axis] + (size_t)c * pbm->npts * 10;
            const double* Fp = faces[axis] + (size_t)fplus * pbm->npts * 10;
            for (int p = 0; p < pbm->npts; ++p) {
                const double wj = pbm->w[p] * jac;
                for (int n = 0; n < N; ++n) {
                    const double wm = wj * pbm->B[p][n], wp = wj * pbp->B[p][n];
                    for (int v = 0; v < 5; ++v) {
                        Rc[n * 5 + v] += wm * Fm[p * 10 + v] - wp * Fp[p * 10 + v];
                        Rtc[n * 5 + v] += wm * Fm[p * 10 + 5 + v] - wp * Fp[p * 10 + 5 + v];
                    }
                }
            }
        }
        const double vjac = h[0] * h[1] * h[2] / 8.0;
        const int naxes = s->basis.dim == 3 ? 3 : 2;
        const PB* pv = &tab->vol;
        for (int p = 0; p < pv->npts; ++p) {
            double e[20];
            eval_tab(coeffs + (size_t)c * N * 5, N, pv, p, h, e);
            Smooth sp;
            double bad = 0;
            const int rc = make_smooth(e, &s->gas, &sp, &bad);
            if (rc) { fill_msg(err, rc, c, bad, 1); return rc; }
            const double tau = mu > 0.0 ? mu / pressure_w(&sp.w) : 0.0;
            const double wj = pv->w[p] * vjac;
            for (int axis = 0; axis < naxes; ++axis) {
                V5 If, Ih;
                smooth_flux(&sp, tau, dt, axis, &If, &Ih);
                double F[5], Ft[5];
                linearize(If, Ih, dt, F, Ft);
                const double scale = 2.0 / h[axis];
                for (int n = 0; n < N; ++n) {
                    const double w = wj * pv->dB[p][axis][n] * scale;
                    for (int v = 0; v < 5; ++v) {
                        Rc[n * 5 + v] += w * F[v];
                        Rtc[n * 5 + v] += w * Ft[v];
                    }
                }
            }
        }
    }
    return ORC_OK;
}

/* mass_diag (dg.hpp:42-50) + apply_inverse_mass (solver.hpp:42-54) */
void orc_apply_inverse_mass(const orc_solver* s, const double* R, double* L) {
    const int N = s->basis.N;
    for (int c = 0; c < s->ncells; ++c) {
        double h[3];
        widths(s, c, h);
        const double vol = h[0] * h[1] * h[2];
        for (int n = 0; n < N; ++n) {
            const int* ix = s->basis.idx[n];
            const double m = vol / ((2.0 * ix[0] + 1.0) * (2.0 * ix[1] + 1.0) * (2.0 * ix[2] + 1.0));
            const double inv = 1.0 / m;
            for (int v = 0; v < 5; ++v) L[((size_t)c * N + n) * 5 + v] = R[((size_t)c * N + n) * 5 + v] * inv;
        }
    }
}

/* compute_dt, integrator.hpp:27-45 (cfl-based; dt_fixed handled by callers) */
int orc_compute_dt(const orc_solver* s, double cfl, double* dt_out, orc_error* err) {
    double dt = INFINITY;
    const int N = s->basis.N;
    for (int c = 0; c < s->ncells; ++c) {
        const double* avg = s->q + (size_t)c * N * 5;
        Prim w;
        double bad = 0;
        const int rc = prim_from_q(avg, &s->gas, &w, &bad);
        if (rc) { fill_msg(err, rc, c, bad, 0); return rc; }
        double hw[3];
        widths(s, c, hw);
        double h = hw[0];
        if (hw[1] < h) h = hw[1];
        if (hw[2] < h) h = hw[2];
        const double speed = fabs(w.U) + fabs(w.V) + fabs(w.W) + sound_speed(&w, &s->gas);
        const double cand = cfl * h / speed;
        if (cand < dt) dt = cand;
        if (s->gas.mu > 0.0) {
            const double vis = cfl * h * h * w.rho / (2.0 * s->gas.mu * (2.0 * s->basis.degree + 1.0));
            if (vis < dt) dt = vis;
        }
    }
    if (!(dt > 0.0) || !isfinite(dt)) { fill_msg(err, ORC_NONPOS_DT, -1, dt, 0); return ORC_NONPOS_DT; }
    *dt_out = dt;
    return ORC_OK;
}

/* two_stage_step (integrator.hpp:64-75) with eval = residual + inverse mass
 * (solver.hpp:81-88); the same full dt drives both residuals (solver.hpp:85) */
int orc_step(orc_solver* s, double dt, orc_error* err) {
    const size_t n = (size_t)orc_ncoeffs(s);
    int rc = orc_residual(s, s->q, dt, s->R, s->Rt, NULL, NULL, NULL, NULL, err);
    if (rc) return rc;
    orc_apply_inverse_mass(s, s->R, s->L1);
    orc_apply_inverse_mass(s, s->Rt, s->Lt1);
    for (size_t i = 0; i < n; ++i) s->qs[i] = s->q[i] + 0.5 * dt * s->L1[i] + 0.125 * dt * dt * s->Lt1[i];
    rc = orc_residual(s, s->qs, dt, s->R, s->Rt, NULL, NULL, NULL, NULL, err);
    if (rc) return rc;
    orc_apply_inverse_mass(s, s->R, s->L2);
    orc_apply_inverse_mass(s, s->Rt, s->Lt2);
    const double c = dt * dt / 6.0;
    for (size_t i = 0; i < n; ++i) s->q[i] += dt * s->L1[i] + c * (s->Lt1[i] + 2.0 * s->Lt2[i]);
    return ORC_OK;
}

/* ------------------------------------------------------------------- cases */
/* density_wave, cases.hpp:78-87 */
static void density_wave(int dim, const double* x, double t, double gamma, double* q) {
    double s = x[0] + x[1] - 2.0 * t;
    if (dim == 3) s = x[0] + x[1] + x[2] - 3.0 * t;
    const double rho = 1.0 + 0.2 * sin(M_PI * s);
    const double W = dim == 3 ? 1.0 : 0.0;
    const double p = 1.0;
    const double E = p / (gamma - 1.0) + 0.5 * rho * (1.0 + 1.0 + W * W);
    q[0] = rho; q[1] = rho; q[2] = rho; q[3] = rho * W; q[4] = E;
}

static double wrap10(double v) {
    v = fmod(v, 10.0);
    if (v < -5.0) v += 10.0;
    if (v >= 5.0) v -= 10.0;
    return v;
}

/* isotropic_vortex, cases.hpp:91-111 */
static void isotropic_vortex(const double* x, double t, double eps, double gamma, double* q) {
    const double dx = wrap10(x[0] - 5.0 - t), dy = wrap10(x[1] - 5.0 - t);
    const double r2 = dx * dx + dy * dy;
    const double g = eps / (2.0 * M_PI) * exp(0.5 * (1.0 - r2));
    const double U = 1.0 - g * dy, V = 1.0 + g * dx;
    const double T = 1.0 - (gamma - 1.0) * eps * eps / (8.0 * gamma * M_PI * M_PI) * exp(1.0 - r2);
    const double rho = pow(T, 1.0 / (gamma - 1.0));
    const double p = rho * T;
    const double E = p / (gamma - 1.0) + 0.5 * rho * (U * U + V * V);
    q[0] = rho; q[1] = rho * U; q[2] = rho * V; q[3] = 0.0; q[4] = E;
}

/* taylor_green_init, cases.hpp:115-124 */
static void taylor_green(const double* x, double gamma, double mach0, double* q) {
    const double p0 = 1.0 / (gamma * mach0 * mach0);
    const double U = sin(x[0]) * cos(x[1]) * cos(x[2]);
    const double V = -cos(x[0]) * sin(x[1]) * cos(x[2]);
    const double p = p0 + (cos(2.0 * x[0]) + cos(2.0 * x[1])) * (cos(2.0 * x[2]) + 2.0) / 16.0;
    const double rho = p / p0;
    const double E = p / (gamma - 1.0) + 0.5 * rho * (U * U + V * V);
    q[0] = rho; q[1] = rho * U; q[2] = rho * V; q[3] = 0.0; q[4] = E;
}

static void field_at(const orc_solver* s, const double* x, double t, double* q) {  /* cases.hpp:127-151 */
    switch (s->cid) {
        case CASE_ADV2D: density_wave(2, x, t, s->gas.gamma, q); break;
        case CASE_ADV3D: density_wave(3, x, t, s->gas.gamma, q); break;
        case CASE_VORTEX2D: isotropic_vortex(x, t, s->eps, s->gas.gamma, q); break;
        default: taylor_green(x, s->gas.gamma, s->mach0, q); break;
    }
}

/* project, dg.hpp:193-220 */
static void project_field(orc_solver* s, double t) {
    const int N = s->basis.N;
    const PB* pp = &s->tab->proj;
    double bn[MAXN];
    for (int n = 0; n < N; ++n) {
        const int* ix = s->basis.idx[n];
        bn[n] = (2.0 * ix[0] + 1.0) * (2.0 * ix[1] + 1.0) * (2.0 * ix[2] + 1.0) / 8.0;
    }
    for (int c = 0; c < s->ncells; ++c) {
        double ctr[3], h[3];
        center(s, c, ctr); widths(s, c, h);
        double* out = s->q + (size_t)c * N * 5;
        for (int i = 0; i < N * 5; ++i) out[i] = 0.0;
        for (int p = 0; p < pp->npts; ++p) {
            const double x[3] = {ctr[0] + 0.5 * h[0] * pp->ref[p][0], ctr[1] + 0.5 * h[1] * pp->ref[p][1],
                                 ctr[2] + 0.5 * h[2] * pp->ref[p][2]};
            double f[5];
            field_at(s, x, t, f);
            const double wq = pp->w[p];
            for (int n = 0; n < N; ++n)
                for (int v = 0; v < 5; ++v) out[n * 5 + v] += wq * pp->B[p][n] * f[v];
        }
        for (int n = 0; n < N; ++n)
            for (int v = 0; v < 5; ++v) out[n * 5 + v] *= bn[n];
    }
}

/* case_axis_nodes / build_mesh / CaseConfig::named, cases.hpp:12-73;
 * setup_run, solver.hpp:29-37 */
orc_solver* orc_setup(const char* name, int n, int degree, int nonuniform, orc_error* err) {
    CaseId cid;
    int dim;
    double lo = 0.0, hi = 2.0, mu = 0.0;
    if (!strcmp(name, "adv2d")) { cid = CASE_ADV2D; dim = 2; }
    else if (!strcmp(name, "adv3d")) { cid = CASE_ADV3D; dim = 3; }
    else if (!strcmp(name, "vortex2d")) { cid = CASE_VORTEX2D; dim = 2; hi = 10.0; }
    else if (!strcmp(name, "tgv")) { cid = CASE_TGV; dim = 3; lo = -M_PI; hi = M_PI; mu = 1.0 / 1600.0; }
    else {
        if (err) { err->code = ORC_CONFIG; err->item = -1; snprintf(err->msg, sizeof err->msg, "unknown case: %s", name); }
        return NULL;
    }
    if (n < 4) {
        if (err) { err->code = ORC_CONFIG; err->item = -1; snprintf(err->msg, sizeof err->msg, "build_mesh: need at least 4 cells per axis"); }
        return NULL;
    }
    double* nodes = malloc((n + 1) * sizeof(double));
    for (int i = 0; i <= n; ++i) {
        const double xi = lo + (hi - lo) * i / n;
        nodes[i] = nonuniform ? xi + 0.05 * sin(M_PI * xi) : xi;
    }
    const double zn[2] = {lo, hi};
    orc_solver* s = dim == 2 ? orc_create(n, n, 1, nodes, nodes, zn, degree, 2, 1.4, mu, err)
                             : orc_create(n, n, n, nodes, nodes, nodes, degree, 3, 1.4, mu, err);
    free(nodes);
    if (!s) return NULL;
    s->cid = cid; s->mach0 = 0.1; s->eps = 5.0;
    project_field(s, 0.0);
    return s;
}

/* tgv_diagnostics, cases.hpp:165-204 */
void orc_tgv_diagnostics(const orc_solver* s, double* out) {
    const int N = s->basis.N;
    const PB* pp = &s->tab->proj;
    double ek = 0, ens = 0, vol = 0;
    for (int c = 0; c < s->ncells; ++c) {
        double h[3];
        widths(s, c, h);
        const double vjac = h[0] * h[1] * h[2] / 8.0;
        double cek = 0, cens = 0;
        for (int p = 0; p < pp->npts; ++p) {
            double e[20];
            eval_tab(s->q + (size_t)c * N * 5, N, pp, p, h, e);
            const double inv = 1.0 / e[0];
            const double U = e[1] * inv, V = e[2] * inv, W = e[3] * inv;
            const double vel[4] = {0, U, V, W};
            cek += pp->w[p] * 0.5 * (e[1] * U + e[2] * V + e[3] * W);
#define DVEL(comp, ax) ((e[5 + 5 * (ax) + (comp)] - vel[comp] * e[5 + 5 * (ax)]) * inv)
            const double wx = DVEL(3, 1) - DVEL(2, 2);
            const double wy = DVEL(1, 2) - DVEL(3, 0);
            const double wz = DVEL(2, 0) - DVEL(1, 1);
#undef DVEL
            cens += pp->w[p] * 0.5 * e[0] * (wx * wx + wy * wy + wz * wz);
        }
        ek += vjac * cek;
        ens += vjac * cens;
    }
    for (int c = 0; c < s->ncells; ++c) {
        double h[3];
        widths(s, c, h);
        vol += h[0] * h[1] * h[2];
    }
    out[0] = ek / vol;
    out[1] = 2.0 * s->gas.mu * ens / vol;
}

/* error_norms, dg.hpp:228-266 */
int orc_error_norms(const orc_solver* s, double t, double* out) {
    if (s->cid == CASE_TGV || s->cid == CASE_NONE) return ORC_CONFIG;
    const int N = s->basis.N;
    const PB* pp = &s->tab->proj;
    double l1 = 0, l2 = 0, ec = 0;
    for (int c = 0; c < s->ncells; ++c) {
        double ctr[3], h[3];
        center(s, c, ctr); widths(s, c, h);
        const double vol = h[0] * h[1] * h[2];
        const double* co = s->q + (size_t)c * N * 5;
        double cl1 = 0, cl2 = 0, avg = 0;
        for (int p = 0; p < pp->npts; ++p) {
            const double x[3] = {ctr[0] + 0.5 * h[0] * pp->ref[p][0], ctr[1] + 0.5 * h[1] * pp->ref[p][1],
                                 ctr[2] + 0.5 * h[2] * pp->ref[p][2]};
            double f[5];
            field_at(s, x, t, f);
            double rh = 0;
            for (int n = 0; n < N; ++n) rh += pp->B[p][n] * co[n * 5];
            const double d = fabs(f[0] - rh);
            cl1 += pp->w[p] * d;
            cl2 += pp->w[p] * d * d;
            avg += pp->w[p] * f[0];
        }
        avg /= 8.0;
        const double davg = avg - co[0];
        l1 += vol / 8.0 * cl1;
        l2 += vol / 8.0 * cl2;
        ec += vol * davg * davg;
    }
    out[0] = l1; out[1] = sqrt(l2); out[2] = sqrt(ec);
    return ORC_OK;
}

/* -------------------------------------------------------- kinetics exports */
int orc_interface_flux(const double* tl, const double* tr, double gamma, double tau, double dt,
                       double* full, double* half, orc_error* err) {
    const Gas g = gas_make(gamma, 0.0);
    V5 If, Ih;
    double bad = 0;
    const int rc = interface_flux(tl, tr, &g, tau, dt, &If, &Ih, &bad);
    if (rc) { fill_msg(err, rc, -1, bad, 0); return rc; }
    memcpy(full, If.v, sizeof If.v);
    memcpy(half, Ih.v, sizeof Ih.v);
    return ORC_OK;
}

int orc_smooth_flux(const double* t, double gamma, double tau, double dt, int axis, double* full,
                    double* half, orc_error* err) {
    const Gas g = gas_make(gamma, 0.0);
    Smooth sp;
    double bad = 0;
    const int rc = make_smooth(t, &g, &sp, &bad);
    if (rc) { fill_msg(err, rc, -1, bad, 0); return rc; }
    V5 If, Ih;
    smooth_flux(&sp, tau, dt, axis, &If, &Ih);
    memcpy(full, If.v, sizeof If.v);
    memcpy(half, Ih.v, sizeof Ih.v);
    return ORC_OK;
}

void orc_maxwellian_moments(const double* prim, double gamma, double* out) {
    const Gas g = gas_make(gamma, 0.0);
    const Prim w = {prim[0], prim[1], prim[2], prim[3], prim[4]};
    Mom m;
    moments(&w, &g, &m);
    for (int n = 0; n < 9; ++n) {
        out[n] = m.u[n]; out[9 + n] = m.upos[n]; out[18 + n] = m.uneg[n]; out[27 + n] = m.v[n]; out[36 + n] = m.w[n];
    }
    out[45] = m.xi2; out[46] = m.xi4;
}
