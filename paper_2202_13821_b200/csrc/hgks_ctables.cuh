// Compile-time basis / quadrature tables (the same values include/hgks_b200/basis_tables.h
// tabulates on the host: graded tensor-Legendre basis, basis.hpp:64-82;
// Gauss-Legendre points, quadrature.hpp:15-58; point order of DGTables::make,
// dg.hpp:91-128). They are built once per (degree, dim) by the front end's
// constexpr evaluator into a __device__ constexpr table; kernels index it with
// unrolled (constant) indices, so every basis value becomes an immediate
// operand and zero entries drop out.
#pragma once

namespace hgks_dev {
namespace ct {

// Gauss-Legendre abscissae / weights (nq = 1, 2, 3)
__host__ __device__ constexpr double gx(int nq, int i) {
    return nq == 1 ? 0.0
         : nq == 2 ? (i == 0 ? -0.57735026918962576451 : 0.57735026918962576451)
                   : (i == 0 ? -0.77459666924148337704 : i == 1 ? 0.0 : 0.77459666924148337704);
}
__host__ __device__ constexpr double gw(int nq, int i) {
    return nq == 1 ? 2.0 : nq == 2 ? 1.0 : (i == 1 ? 8.0 / 9.0 : 5.0 / 9.0);
}

// P_l(x) and P_l'(x), three-term recursion (basis.hpp:11-34)
__host__ __device__ constexpr double leg(int l, double x) {
    if (l == 0) return 1.0;
    double pm = 1.0, p = x;
    for (int n = 1; n < l; ++n) {
        const double pn = ((2.0 * n + 1.0) * x * p - n * pm) / (n + 1.0);
        pm = p;
        p = pn;
    }
    return p;
}
__host__ __device__ constexpr double dleg(int l, double x) {
    if (l == 0) return 0.0;
    double pm = 1.0, p = x, dm = 0.0, d = 1.0;
    for (int n = 1; n < l; ++n) {
        const double pn = ((2.0 * n + 1.0) * x * p - n * pm) / (n + 1.0);
        const double dn = ((2.0 * n + 1.0) * (p + x * d) - n * dm) / (n + 1.0);
        pm = p;
        p = pn;
        dm = d;
        d = dn;
    }
    return d;
}

// n-th multi-index of the graded-lexicographic basis, component `axis`
__host__ __device__ constexpr int bidx(int P, int DIM, int n, int axis) {
    int k = 0;
    for (int d = 0; d <= P; ++d)
        for (int a = 0; a <= d; ++a)
            for (int b = 0; b <= d - a; ++b) {
                const int c = d - a - b;
                if (DIM == 2 && c != 0) continue;
                if (k == n) return axis == 0 ? a : axis == 1 ? b : c;
                ++k;
            }
    return 0;
}

__host__ __device__ constexpr double basis(int P, int DIM, int n, const double* r) {
    return leg(bidx(P, DIM, n, 0), r[0]) * leg(bidx(P, DIM, n, 1), r[1]) * leg(bidx(P, DIM, n, 2), r[2]);
}
__host__ __device__ constexpr double dbasis(int P, int DIM, int n, int a, const double* r) {
    const double fx = a == 0 ? dleg(bidx(P, DIM, n, 0), r[0]) : leg(bidx(P, DIM, n, 0), r[0]);
    const double fy = a == 1 ? dleg(bidx(P, DIM, n, 1), r[1]) : leg(bidx(P, DIM, n, 1), r[1]);
    const double fz = a == 2 ? dleg(bidx(P, DIM, n, 2), r[2]) : leg(bidx(P, DIM, n, 2), r[2]);
    return fx * fy * fz;
}

// one (degree, dim) family; sized for the largest (P3: 20 basis functions,
// 9 face points, 27 volume points). Face side index 0 = reference coordinate
// -1 (a cell's minus face), 1 = +1 (its plus face).
struct Tab {
    int N, NQ, NVP, nfp[3];
    double fB[3][2][9][20];
    double fdB[3][2][9][3][20];
    double fw[3][9];
    double vB[27][20];
    double vdB[27][3][20];
    double vw[27];
    double massf[20];  // (2nx+1)(2ny+1)(2nz+1) (dg.hpp:42-50)
    int par[3][20];    // parity of basis n along each axis: B(+1) = (-1)^par B(-1)
};

template <int P, int DIM>
__host__ __device__ constexpr Tab make_tab() {
    Tab t{};
    const int NQ = P <= 2 ? 2 : 3;
    int N = 0;
    for (int d = 0; d <= P; ++d)
        for (int a = 0; a <= d; ++a)
            for (int b = 0; b <= d - a; ++b)
                if (DIM == 3 || d - a - b == 0) ++N;
    t.N = N;
    t.NQ = NQ;
    const int nqz = DIM == 3 ? NQ : 1;
    t.NVP = NQ * NQ * nqz;
    for (int n = 0; n < N; ++n) {
        t.massf[n] = (2.0 * bidx(P, DIM, n, 0) + 1.0) * (2.0 * bidx(P, DIM, n, 1) + 1.0) *
                     (2.0 * bidx(P, DIM, n, 2) + 1.0);
        for (int a = 0; a < 3; ++a) t.par[a][n] = bidx(P, DIM, n, a) & 1;
    }
    // volume points, k fastest (dg.hpp:102-105)
    for (int i = 0; i < NQ; ++i)
        for (int j = 0; j < NQ; ++j)
            for (int k = 0; k < nqz; ++k) {
                const int p = (i * NQ + j) * nqz + k;
                const double r[3] = {gx(NQ, i), gx(NQ, j), gx(nqz, k)};
                t.vw[p] = gw(NQ, i) * gw(NQ, j) * gw(nqz, k);
                for (int n = 0; n < N; ++n) {
                    t.vB[p][n] = basis(P, DIM, n, r);
                    for (int a = 0; a < 3; ++a) t.vdB[p][a][n] = dbasis(P, DIM, n, a, r);
                }
            }
    // face points: p = ib * nc + ic, b = (a+1)%3 outer, c = (a+2)%3 inner (dg.hpp:111-126)
    for (int a = 0; a < 3; ++a) {
        const int bb = (a + 1) % 3, cc = (a + 2) % 3;
        const int nb = (bb == 2 && DIM == 2) ? 1 : NQ;
        const int nc = (cc == 2 && DIM == 2) ? 1 : NQ;
        t.nfp[a] = nb * nc;
        for (int ib = 0; ib < nb; ++ib)
            for (int ic = 0; ic < nc; ++ic) {
                const int p = ib * nc + ic;
                t.fw[a][p] = gw(nb, ib) * gw(nc, ic);
                for (int s = 0; s < 2; ++s) {
                    double r[3] = {0.0, 0.0, 0.0};
                    r[bb] = gx(nb, ib);
                    r[cc] = gx(nc, ic);
                    r[a] = s == 0 ? -1.0 : 1.0;
                    for (int n = 0; n < N; ++n) {
                        t.fB[a][s][p][n] = basis(P, DIM, n, r);
                        for (int d = 0; d < 3; ++d) t.fdB[a][s][p][d][n] = dbasis(P, DIM, n, d, r);
                    }
                }
            }
    }
    return t;
}

}  // namespace ct

template <int P, int DIM>
__device__ constexpr ct::Tab ctab = ct::make_tab<P, DIM>();

}  // namespace hgks_dev
