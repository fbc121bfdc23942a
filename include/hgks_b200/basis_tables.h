// Host-side discretisation tables for the device kernels: Gauss-Legendre
// rules (quadrature.hpp:15-58), the graded tensor-Legendre basis
// (basis.hpp:11-82) and the tabulated point bases (dg.hpp:54-128), flattened
// into one device array. Degree 1 is the documented P1 extension (2-point
// flux rule, as DGTables would pick for k <= 2).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <stdexcept>
#include <vector>

namespace hgks_host {

struct Rule {
    std::vector<double> x, w;
};

inline Rule gauss_rule(int m) {
    Rule r;
    switch (m) {
        case 1: r.x = {0.0}; r.w = {2.0}; break;
        case 2: {
            const double a = 1.0 / std::sqrt(3.0);
            r.x = {-a, a};
            r.w = {1.0, 1.0};
        } break;
        case 3: {
            const double a = std::sqrt(0.6);
            r.x = {-a, 0.0, a};
            r.w = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
        } break;
        case 4: {
            const double s = std::sqrt(1.2);
            const double a = std::sqrt((3.0 - 2.0 * s) / 7.0), b = std::sqrt((3.0 + 2.0 * s) / 7.0);
            const double wa = (18.0 + std::sqrt(30.0)) / 36.0, wb = (18.0 - std::sqrt(30.0)) / 36.0;
            r.x = {-b, -a, a, b};
            r.w = {wb, wa, wa, wb};
        } break;
        case 5: {
            const double s = std::sqrt(10.0 / 7.0);
            const double a = std::sqrt(5.0 - 2.0 * s) / 3.0, b = std::sqrt(5.0 + 2.0 * s) / 3.0;
            const double wa = (322.0 + 13.0 * std::sqrt(70.0)) / 900.0;
            const double wb = (322.0 - 13.0 * std::sqrt(70.0)) / 900.0;
            r.x = {-b, -a, 0.0, a, b};
            r.w = {wb, wa, 128.0 / 225.0, wa, wb};
        } break;
        default: throw std::invalid_argument("gauss_rule: unsupported point count");
    }
    return r;
}

// P_l and P_l' by the three-term recursion
inline void legendre_pd(int l, double x, double& p, double& d) {
    if (l == 0) {
        p = 1.0;
        d = 0.0;
        return;
    }
    double pm = 1.0, pc = x, dm = 0.0, dc = 1.0;
    for (int n = 1; n < l; ++n) {
        const double pn = ((2.0 * n + 1.0) * x * pc - n * pm) / (n + 1.0);
        const double dn = ((2.0 * n + 1.0) * (pc + x * dc) - n * dm) / (n + 1.0);
        pm = pc;
        pc = pn;
        dm = dc;
        dc = dn;
    }
    p = pc;
    d = dc;
}

struct Basis {
    int degree = 0, dim = 3, N = 0;
    std::vector<std::array<int, 3>> idx;

    double eval(int n, const double* r) const {
        double v = 1.0;
        for (int a = 0; a < 3; ++a) {
            double p, d;
            legendre_pd(idx[n][a], r[a], p, d);
            v *= p;
        }
        return v;
    }
    double deriv(int n, int axis, const double* r) const {
        double v = 1.0;
        for (int a = 0; a < 3; ++a) {
            double p, d;
            legendre_pd(idx[n][a], r[a], p, d);
            v *= (a == axis ? d : p);
        }
        return v;
    }
};

inline Basis make_basis(int k, int dim) {
    if (k < 1 || k > 3) throw std::invalid_argument("basis: degree must be 1, 2 or 3");
    if (dim != 2 && dim != 3) throw std::invalid_argument("basis: dim must be 2 or 3");
    Basis b;
    b.degree = k;
    b.dim = dim;
    const int zmax = dim == 3 ? k : 0;
    for (int a = 0; a <= k; ++a)
        for (int c = 0; c <= k; ++c)
            for (int e = 0; e <= zmax; ++e)
                if (a + c + e <= k) b.idx.push_back({a, c, e});
    // graded (total degree), then lexicographic on (nx, ny, nz)
    std::stable_sort(b.idx.begin(), b.idx.end(), [](const auto& u, const auto& v) {
        const int du = u[0] + u[1] + u[2], dv = v[0] + v[1] + v[2];
        return du != dv ? du < dv : u < v;
    });
    b.N = static_cast<int>(b.idx.size());
    return b;
}

struct PointSet {
    int npts = 0;
    std::vector<double> B, dB, w, ref;  // B[p][N], dB[p][3][N], w[p], ref[p][3]
    void add(const Basis& b, const double* r, double wt) {
        ++npts;
        w.push_back(wt);
        for (int a = 0; a < 3; ++a) ref.push_back(r[a]);
        for (int n = 0; n < b.N; ++n) B.push_back(b.eval(n, r));
        for (int a = 0; a < 3; ++a)
            for (int n = 0; n < b.N; ++n) dB.push_back(b.deriv(n, a, r));
    }
};

struct Tables {
    Basis basis;
    int nq_flux = 0, nq_proj = 0;
    PointSet vol, proj, face[3][2];  // face[a][0] = minus face (ref coord -1), [1] = plus face

    // flattened device image and section offsets (in doubles)
    std::vector<double> img;
    long off_fB[3][2], off_fdB[3][2], off_fw[3], off_vB, off_vdB, off_vw, off_pB, off_pdB, off_pw,
        off_pref, off_massf;
};

inline Tables make_tables(int degree, int dim) {
    Tables t;
    t.basis = make_basis(degree, dim);
    const Basis& b = t.basis;
    t.nq_flux = degree <= 2 ? 2 : 3;
    t.nq_proj = degree + 2;
    const Rule qf = gauss_rule(t.nq_flux), qp = gauss_rule(t.nq_proj), q1 = gauss_rule(1);
    const Rule& qfz = dim == 3 ? qf : q1;
    const Rule& qpz = dim == 3 ? qp : q1;
    // volume points, k fastest (dg.hpp:102-105)
    for (size_t i = 0; i < qf.x.size(); ++i)
        for (size_t j = 0; j < qf.x.size(); ++j)
            for (size_t k = 0; k < qfz.x.size(); ++k) {
                const double r[3] = {qf.x[i], qf.x[j], qfz.x[k]};
                t.vol.add(b, r, qf.w[i] * qf.w[j] * qfz.w[k]);
            }
    for (size_t i = 0; i < qp.x.size(); ++i)
        for (size_t j = 0; j < qp.x.size(); ++j)
            for (size_t k = 0; k < qpz.x.size(); ++k) {
                const double r[3] = {qp.x[i], qp.x[j], qpz.x[k]};
                t.proj.add(b, r, qp.w[i] * qp.w[j] * qpz.w[k]);
            }
    // face points: p = ib * nc + ic with b = (a+1)%3 outer, c = (a+2)%3 inner (dg.hpp:111-126)
    for (int a = 0; a < 3; ++a) {
        const int bb = (a + 1) % 3, cc = (a + 2) % 3;
        const Rule& rb = (bb == 2 && dim == 2) ? q1 : qf;
        const Rule& rc = (cc == 2 && dim == 2) ? q1 : qf;
        for (size_t ib = 0; ib < rb.x.size(); ++ib)
            for (size_t ic = 0; ic < rc.x.size(); ++ic) {
                double r[3] = {0, 0, 0};
                r[bb] = rb.x[ib];
                r[cc] = rc.x[ic];
                const double wt = rb.w[ib] * rc.w[ic];
                r[a] = -1.0;
                t.face[a][0].add(b, r, wt);
                r[a] = 1.0;
                t.face[a][1].add(b, r, wt);
            }
    }
    auto put = [&](const std::vector<double>& v) {
        const long o = static_cast<long>(t.img.size());
        t.img.insert(t.img.end(), v.begin(), v.end());
        while (t.img.size() % 4) t.img.push_back(0.0);  // 32-byte alignment of sections
        return o;
    };
    for (int a = 0; a < 3; ++a)
        for (int s = 0; s < 2; ++s) {
            t.off_fB[a][s] = put(t.face[a][s].B);
            t.off_fdB[a][s] = put(t.face[a][s].dB);
        }
    for (int a = 0; a < 3; ++a) t.off_fw[a] = put(t.face[a][0].w);
    t.off_vB = put(t.vol.B);
    t.off_vdB = put(t.vol.dB);
    t.off_vw = put(t.vol.w);
    t.off_pB = put(t.proj.B);
    t.off_pdB = put(t.proj.dB);
    t.off_pw = put(t.proj.w);
    t.off_pref = put(t.proj.ref);
    std::vector<double> mf(b.N);
    for (int n = 0; n < b.N; ++n)
        mf[n] = (2.0 * b.idx[n][0] + 1.0) * (2.0 * b.idx[n][1] + 1.0) * (2.0 * b.idx[n][2] + 1.0);
    t.off_massf = put(mf);
    return t;
}

}  // namespace hgks_host
