// hgks_b200/discretization.hpp — mesh, basis, quadrature, state and the
// tabulated point bases of the drop-in (proj/include/hgks/quadrature.hpp,
// basis.hpp, mesh.hpp, dg.hpp:18-190, :307-345). Host-side setup and
// evaluation helpers; the per-step arithmetic runs on the device, which
// builds the same tables from include/hgks_b200/basis_tables.h.
#pragma once

#include <algorithm>
#include <array>
#include <stdexcept>
#include <vector>

#include "basis_tables.h"
#include "core.hpp"

namespace hgks {

// ------------------------------------------------------------- quadrature
/// Gauss-Legendre rule on [-1, 1] (quadrature.hpp:11-58): m points integrate
/// degree 2m-1 exactly; m = 1..5.
struct QuadRule {
    std::vector<double> x;
    std::vector<double> w;
    static QuadRule gauss(int m) {
        if (m < 1 || m > 5) throw std::invalid_argument("QuadRule::gauss: supported point counts are 1..5");
        const hgks_host::Rule r = hgks_host::gauss_rule(m);
        return {r.x, r.w};
    }
    int size() const { return static_cast<int>(x.size()); }
};

// ------------------------------------------------------------------ basis
inline double legendre(int l, double x) {
    double p, d;
    hgks_host::legendre_pd(l, x, p, d);
    return p;
}
inline double legendre_deriv(int l, double x) {
    double p, d;
    hgks_host::legendre_pd(l, x, p, d);
    return d;
}

struct unsupported_degree : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

/// Tensor-Legendre basis of total degree <= k, graded-lex order
/// (basis.hpp:43-82); dim = 2 restricts to nz = 0.
struct BasisSet {
    int degree;
    int dim;
    int N;
    std::vector<std::array<int, 3>> idx;

    double eval(int n, double xi, double eta, double zeta) const {
        const auto& ix = idx[n];
        return legendre(ix[0], xi) * legendre(ix[1], eta) * legendre(ix[2], zeta);
    }
    double eval_deriv(int n, int axis, double xi, double eta, double zeta) const {
        const auto& ix = idx[n];
        const double r[3] = {xi, eta, zeta};
        double f[3];
        for (int a = 0; a < 3; ++a) f[a] = a == axis ? legendre_deriv(ix[a], r[a]) : legendre(ix[a], r[a]);
        return f[0] * f[1] * f[2];
    }
};

/// The reference's degrees only (2, 3): P1 is this library's extension,
/// reached through build_basis_extended / Scheme::make_extended.
inline BasisSet build_basis_extended(int k, int dim) {
    if (dim != 2 && dim != 3) throw std::invalid_argument("build_basis: dim must be 2 or 3");
    const hgks_host::Basis b = hgks_host::make_basis(k, dim);
    return {b.degree, b.dim, b.N, b.idx};
}
inline BasisSet build_basis(int k, int dim) {
    if (k != 2 && k != 3) throw unsupported_degree("build_basis: degree must be 2 or 3");
    return build_basis_extended(k, dim);
}

// ------------------------------------------------------------------- mesh
/// Periodic box with per-axis node coordinates (mesh.hpp:11-64), x fastest.
struct Mesh {
    int nx, ny, nz;
    std::vector<double> xs, ys, zs;
    std::array<bool, 3> periodic = {true, true, true};

    static Mesh make(std::vector<double> xnodes, std::vector<double> ynodes, std::vector<double> znodes) {
        for (const auto* v : {&xnodes, &ynodes, &znodes})
            for (size_t i = 1; i < v->size(); ++i)
                if (!((*v)[i] > (*v)[i - 1]))
                    throw std::invalid_argument("Mesh: node coordinates must be strictly increasing");
        Mesh m;
        m.nx = static_cast<int>(xnodes.size()) - 1;
        m.ny = static_cast<int>(ynodes.size()) - 1;
        m.nz = static_cast<int>(znodes.size()) - 1;
        m.xs = std::move(xnodes);
        m.ys = std::move(ynodes);
        m.zs = std::move(znodes);
        return m;
    }
    int ncells() const { return nx * ny * nz; }
    int cell_index(int i, int j, int k) const { return i + nx * (j + ny * k); }
    std::array<int, 3> cell_ijk(int c) const { return {c % nx, (c / nx) % ny, c / (nx * ny)}; }
    double dx(int i) const { return xs[i + 1] - xs[i]; }
    double dy(int j) const { return ys[j + 1] - ys[j]; }
    double dz(int k) const { return zs[k + 1] - zs[k]; }
    double xc(int i) const { return 0.5 * (xs[i] + xs[i + 1]); }
    double yc(int j) const { return 0.5 * (ys[j] + ys[j + 1]); }
    double zc(int k) const { return 0.5 * (zs[k] + zs[k + 1]); }
    std::array<double, 3> widths(int c) const {
        const auto ijk = cell_ijk(c);
        return {dx(ijk[0]), dy(ijk[1]), dz(ijk[2])};
    }
    std::array<double, 3> center(int c) const {
        const auto ijk = cell_ijk(c);
        return {xc(ijk[0]), yc(ijk[1]), zc(ijk[2])};
    }
    double volume(int c) const {
        const auto h = widths(c);
        return h[0] * h[1] * h[2];
    }
};

// ------------------------------------------------------------------ state
/// Modal coefficients, AoS [(cell*N + n)*5 + var]; n = 0 is the cell mean.
struct DGState {
    int ncells = 0;
    int N = 0;
    double time = 0.0;
    std::vector<double> coeffs;

    static DGState zeros(int ncells, int N) {
        DGState s;
        s.ncells = ncells;
        s.N = N;
        s.coeffs.assign(static_cast<size_t>(ncells) * N * 5, 0.0);
        return s;
    }
    double* cell(int c) { return coeffs.data() + static_cast<size_t>(c) * N * 5; }
    const double* cell(int c) const { return coeffs.data() + static_cast<size_t>(c) * N * 5; }
    double& coeff(int c, int n, int v) { return coeffs[(static_cast<size_t>(c) * N + n) * 5 + v]; }
    double coeff(int c, int n, int v) const { return coeffs[(static_cast<size_t>(c) * N + n) * 5 + v]; }
};

/// Diagonal modal mass matrix of one box cell (dg.hpp:42-50).
inline std::vector<double> mass_diag(const std::array<double, 3>& widths, const BasisSet& basis) {
    const double vol = widths[0] * widths[1] * widths[2];
    std::vector<double> m(basis.N);
    for (int n = 0; n < basis.N; ++n) {
        const auto& ix = basis.idx[n];
        m[n] = vol / ((2.0 * ix[0] + 1.0) * (2.0 * ix[1] + 1.0) * (2.0 * ix[2] + 1.0));
    }
    return m;
}

namespace detail {
/// Basis values / reference derivatives at a point set (dg.hpp:54-79).
struct PointBasis {
    std::vector<double> B;                   // [p*N + n]
    std::vector<double> dB;                  // [(p*3 + axis)*N + n]
    std::vector<double> wq;                  // weight per point
    std::vector<std::array<double, 3>> ref;  // reference coordinates per point
    int npts = 0;

    void add_point(const BasisSet& basis, double xi, double eta, double zeta, double w) {
        ref.push_back({xi, eta, zeta});
        wq.push_back(w);
        for (int n = 0; n < basis.N; ++n) B.push_back(basis.eval(n, xi, eta, zeta));
        for (int a = 0; a < 3; ++a)
            for (int n = 0; n < basis.N; ++n) dB.push_back(basis.eval_deriv(n, a, xi, eta, zeta));
        ++npts;
    }
    const double* Bp(int p, int N) const { return B.data() + static_cast<size_t>(p) * N; }
    const double* dBp(int p, int axis, int N) const { return dB.data() + (static_cast<size_t>(p) * 3 + axis) * N; }
};
}  // namespace detail

/// Flux rule (k points per axis; 2 for k <= 2), projection rule (k+2), and
/// face point sets with the tangential ordering of dg.hpp:111-126.
struct DGTables {
    BasisSet basis;
    int nq_flux;
    int nq_proj;
    detail::PointBasis vol;
    detail::PointBasis proj;
    detail::PointBasis face_minus[3];
    detail::PointBasis face_plus[3];

    static DGTables make(const BasisSet& basis) {
        DGTables t;
        t.basis = basis;
        t.nq_flux = basis.degree <= 2 ? 2 : 3;
        t.nq_proj = basis.degree + 2;
        const QuadRule qf = QuadRule::gauss(t.nq_flux), qp = QuadRule::gauss(t.nq_proj), q1 = QuadRule::gauss(1);
        const QuadRule& qfz = basis.dim == 3 ? qf : q1;
        const QuadRule& qpz = basis.dim == 3 ? qp : q1;
        auto volume_set = [&](detail::PointBasis& pb, const QuadRule& q, const QuadRule& qz) {
            for (int i = 0; i < q.size(); ++i)
                for (int j = 0; j < q.size(); ++j)
                    for (int k = 0; k < qz.size(); ++k)  // k fastest (dg.hpp:102-105)
                        pb.add_point(basis, q.x[i], q.x[j], qz.x[k], q.w[i] * q.w[j] * qz.w[k]);
        };
        volume_set(t.vol, qf, qfz);
        volume_set(t.proj, qp, qpz);
        for (int a = 0; a < 3; ++a) {
            const int b = (a + 1) % 3, c = (a + 2) % 3;
            const QuadRule& rb = (b == 2 && basis.dim == 2) ? q1 : qf;
            const QuadRule& rc = (c == 2 && basis.dim == 2) ? q1 : qf;
            for (int ib = 0; ib < rb.size(); ++ib)
                for (int ic = 0; ic < rc.size(); ++ic) {
                    std::array<double, 3> r{};
                    r[b] = rb.x[ib];
                    r[c] = rc.x[ic];
                    const double w = rb.w[ib] * rc.w[ic];
                    r[a] = -1.0;
                    t.face_minus[a].add_point(basis, r[0], r[1], r[2], w);
                    r[a] = 1.0;
                    t.face_plus[a].add_point(basis, r[0], r[1], r[2], w);
                }
        }
        return t;
    }
};

/// Value and global derivatives of the expansion at a point.
struct EvalPoint {
    Conserved q;
    std::array<Vec5, 3> dq;
};

/// Face-local trace (flux.hpp:53-56): normal along u.
struct FaceTrace {
    Conserved q;
    std::array<Vec5, 3> dq;
};

namespace detail {
inline EvalPoint eval_tabulated(const double* coeffs, int N, const PointBasis& pb, int p,
                                const std::array<double, 3>& widths) {
    Vec5 val{};
    std::array<Vec5, 3> der{};
    const double* B = pb.Bp(p, N);
    for (int n = 0; n < N; ++n)
        for (int v = 0; v < 5; ++v) val[v] += B[n] * coeffs[n * 5 + v];
    for (int a = 0; a < 3; ++a) {
        const double* dB = pb.dBp(p, a, N);
        Vec5 d{};
        for (int n = 0; n < N; ++n)
            for (int v = 0; v < 5; ++v) d[v] += dB[n] * coeffs[n * 5 + v];
        der[a] = (2.0 / widths[a]) * d;
    }
    return {Conserved::from(val), der};
}

/// periodic neighbours along an axis (dg.hpp:307-319)
inline int neighbor_minus(const Mesh& mesh, int c, int axis) {
    auto ijk = mesh.cell_ijk(c);
    const int n = axis == 0 ? mesh.nx : axis == 1 ? mesh.ny : mesh.nz;
    ijk[axis] = (ijk[axis] + n - 1) % n;
    return mesh.cell_index(ijk[0], ijk[1], ijk[2]);
}
inline int neighbor_plus(const Mesh& mesh, int c, int axis) {
    auto ijk = mesh.cell_ijk(c);
    const int n = axis == 0 ? mesh.nx : axis == 1 ? mesh.ny : mesh.nz;
    ijk[axis] = (ijk[axis] + 1) % n;
    return mesh.cell_index(ijk[0], ijk[1], ijk[2]);
}

/// global -> face-local frame: momentum and derivative directions cycled to
/// (axis, axis+1, axis+2) (dg.hpp:323-334); from_face_local undoes it on a flux
inline FaceTrace to_face_local(const EvalPoint& e, int axis) {
    const int g[3] = {axis, (axis + 1) % 3, (axis + 2) % 3};
    const Vec5 q = e.q.vec();
    FaceTrace t;
    t.q = Conserved::from({q[0], q[1 + g[0]], q[1 + g[1]], q[1 + g[2]], q[4]});
    for (int d = 0; d < 3; ++d) {
        const Vec5& s = e.dq[g[d]];
        t.dq[d] = {s[0], s[1 + g[0]], s[1 + g[1]], s[1 + g[2]], s[4]};
    }
    return t;
}
inline Vec5 from_face_local(const Vec5& f, int axis) {
    Vec5 out;
    out[0] = f[0];
    out[4] = f[4];
    out[1 + axis] = f[1];
    out[1 + (axis + 1) % 3] = f[2];
    out[1 + (axis + 2) % 3] = f[3];
    return out;
}
}  // namespace detail

/// Expansion and its global derivatives at an arbitrary reference point
/// (dg.hpp:167-184).
inline EvalPoint eval_at(const DGState& s, const Mesh& mesh, const BasisSet& basis, int cell,
                         const std::array<double, 3>& ref) {
    const auto h = mesh.widths(cell);
    const double* c = s.cell(cell);
    Vec5 val{};
    std::array<Vec5, 3> der{};
    for (int n = 0; n < basis.N; ++n) {
        const double b = basis.eval(n, ref[0], ref[1], ref[2]);
        for (int v = 0; v < 5; ++v) val[v] += b * c[n * 5 + v];
        for (int a = 0; a < 3; ++a) {
            const double db = basis.eval_deriv(n, a, ref[0], ref[1], ref[2]);
            for (int v = 0; v < 5; ++v) der[a][v] += db * c[n * 5 + v] * 2.0 / h[a];
        }
    }
    return {Conserved::from(val), der};
}

/// One-sided trace at face point p of a cell's minus (side < 0) or plus face
/// (dg.hpp:186-190).
inline EvalPoint trace_and_slopes(const DGState& s, const Mesh& mesh, const DGTables& tab, int cell, int axis,
                                  int side, int p) {
    const auto& pb = side < 0 ? tab.face_minus[axis] : tab.face_plus[axis];
    return detail::eval_tabulated(s.cell(cell), tab.basis.N, pb, p, mesh.widths(cell));
}

struct ErrorNorms {
    double l1, l2, cell_avg;
};

}  // namespace hgks
