// Device kernels of the DG-HGKS S2O4 step (sm_100a, fp64).
//
//   face_kernel<P,DIM,VISC,AXIS>  one kinetic flux per owned face point
//                                 (replaces residual phase 1, dg.hpp:362-394)
//   cell_kernel<P,DIM,VISC,MODE>  volume fluxes + face gather + projection,
//                                 fused with the inverse mass matrix and the
//                                 S2O4 stage combine (dg.hpp:396-449,
//                                 solver.hpp:42-54, integrator.hpp:68-74)
//   dt_kernel, ghost_wrap_kernel, project_kernel, tgv_kernel
//
// HBM layout (SoA, fp64): state q[comp][cell_g], comp = n*5 + var,
// cell_g = i + nx*(j + ny*(k+1)) for local z layers k = -1..nzl (one ghost
// layer each side); face buffers f_a[p*10 + (F|Ft)][i + nx*(j + ny*k)].
#pragma once

#include <stdint.h>

#include "hgks_kinetics.cuh"

namespace hgks_dev {

template <int P>
struct Deg {
    static constexpr int N3 = P == 1 ? 4 : P == 2 ? 10 : 20;  // 3-D basis size
    static constexpr int NQ = P <= 2 ? 2 : 3;                 // flux rule points per axis
};

template <int P, int DIM>
struct Shape {
    static constexpr int N = DIM == 3 ? Deg<P>::N3 : (P == 1 ? 3 : P == 2 ? 6 : 10);
    static constexpr int NC = N * 5;
    static constexpr int NQ = Deg<P>::NQ;
    static constexpr int NVP = DIM == 3 ? NQ * NQ * NQ : NQ * NQ;
    // face points per axis (dg.hpp:111-126): in 2-D the z extent is one point
    template <int AXIS>
    __host__ __device__ static constexpr int nfp() {
        return DIM == 3 ? NQ * NQ : (AXIS == 2 ? NQ * NQ : NQ);
    }
    static constexpr int NAX = DIM == 3 ? 3 : 2;
    // cell tile along x and threads of the cell kernel
    static constexpr int TC = P == 3 ? 8 : 32;
    static constexpr int NT_CELL = P == 3 ? 224 : 256;
};

struct KParams {
    int nx, ny, nzl;       // local cells (nzl owned z layers)
    int S;                 // nx * ny
    long cs;               // state component stride (elements)
    long fs;               // face component stride (elements)
    int zface_layers;      // z-face layers stored: nzl (periodic single slab) or nzl + 1
    int z_wrap;            // 1: single periodic slab, top z-face wraps to layer 0
    long ncells_glob;      // for reference item numbering
    int kglob0;            // global z index of local layer 0
    int stage;             // 0 first residual of a step, 1 second
    int count_fluxes;
    int report;            // re-run in report mode: write err_val for the winning key
    double dt;
    GasC gas;
    const double* dx;      // [nx]
    const double* dy;      // [ny]
    const double* dz;      // [nzl + 2] indexed k + 1
    const double* tab;     // table image (hgks_basis.h)
    long off_fB[3][2], off_fdB[3][2], off_fw[3];
    long off_vB, off_vdB, off_vw, off_pB, off_pdB, off_pw, off_pref, off_massf;
    unsigned long long* err_key;
    double* err_val;
    unsigned long long* flux_count;
};

// error key: lexicographic (stage, phase, item, point, sub) = the reference's
// sequential failure order (runtime.hpp:50-58 lowest item wins; phase 1
// before phase 2; within a point: left, right, merged, flux.hpp:73-87)
__device__ __forceinline__ unsigned long long err_key(int stage, int phase, long item, int point,
                                                      int sub, int code) {
    return ((unsigned long long)stage << 62) | ((unsigned long long)phase << 61) |
           ((unsigned long long)item << 22) | ((unsigned long long)point << 12) |
           ((unsigned long long)sub << 8) | (unsigned long long)code;
}

__device__ __forceinline__ void report_error(const KParams& kp, unsigned long long key,
                                             double bad) {
    if (kp.report) {
        if (*kp.err_key == key) *kp.err_val = bad;
    } else {
        atomicMin(kp.err_key, key);
    }
}

// -------------------------------------------------------------- face kernel
// CTA = 32 consecutive faces along x (one lane each) x NFP warps (one face
// point per warp, so table reads are warp-uniform broadcasts). The two
// neighbour cells' coefficients are staged in shared memory SoA
// [side][comp][lane] with coalesced 256 B row loads.
template <int P, int DIM, bool VISC, int AXIS>
__global__ void __launch_bounds__(32 * Shape<P, DIM>::template nfp<AXIS>())
    face_kernel(KParams kp, const double* __restrict__ q, double* __restrict__ face,
                int tile_x0, int tile_y0, int tile_z0) {
    using SH = Shape<P, DIM>;
    constexpr int N = SH::N, NC = SH::NC;
    constexpr int NFP = SH::template nfp<AXIS>();
    constexpr int NT = 32 * NFP;
    constexpr int C1 = (AXIS + 1) % 3, C2 = (AXIS + 2) % 3;
    extern __shared__ double smem[];
    double* sc = smem;  // [2][NC][32]

    const int tid = threadIdx.x;
    const int i0 = (blockIdx.x + tile_x0) * 32;
    const int j = blockIdx.y + tile_y0;
    const int k = blockIdx.z + tile_z0;  // local z layer of the plus-side cell
    const int nx = kp.nx, ny = kp.ny;

    // stage both neighbours' coefficients: side 0 = minus-side cell, 1 = plus-side
    for (int e = tid; e < 2 * NC * 32; e += NT) {
        const int l = e & 31;
        const int row = e >> 5;
        const int side = row >= NC;
        const int comp = row - side * NC;
        const int i = i0 + l;
        double v = 0.0;
        if (i < nx) {
            int ci = i, cj = j, ck = k;
            if (!side) {
                if (AXIS == 0) ci = (i == 0 ? nx - 1 : i - 1);
                if (AXIS == 1) cj = (j == 0 ? ny - 1 : j - 1);
                if (AXIS == 2) ck = k - 1;
            }
            v = __ldg(q + comp * kp.cs + (long)(ck + 1) * kp.S + (long)cj * nx + ci);
        }
        sc[(side * NC + comp) * 32 + l] = v;
    }
    __syncthreads();

    const int lane = tid & 31;
    const int p = tid >> 5;
    const int i = i0 + lane;
    if (i >= nx) return;

    // widths of the two cells
    const int im = AXIS == 0 ? (i == 0 ? nx - 1 : i - 1) : i;
    const int jm = AXIS == 1 ? (j == 0 ? ny - 1 : j - 1) : j;
    const int km = AXIS == 2 ? k - 1 : k;
    const double hL[3] = {__ldg(kp.dx + im), __ldg(kp.dy + jm), __ldg(kp.dz + km + 1)};
    const double hR[3] = {__ldg(kp.dx + i), __ldg(kp.dy + j), __ldg(kp.dz + k + 1)};

    // left trace = minus-side cell at its plus face; right = plus-side cell at its minus face
    const double* BL = kp.tab + kp.off_fB[AXIS][1] + p * N;
    const double* BR = kp.tab + kp.off_fB[AXIS][0] + p * N;

    // pressures of the two traces for tau = mu / mean p (dg.hpp:378-383)
    double tau = 0.0;
    if (VISC) {
        double ql[5] = {0, 0, 0, 0, 0}, qr[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int n = 0; n < N; ++n) {
            const double bl = __ldg(BL + n), br = __ldg(BR + n);
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                ql[v] += bl * sc[(0 * NC + n * 5 + v) * 32 + lane];
                qr[v] += br * sc[(1 * NC + n * 5 + v) * 32 + lane];
            }
        }
        const double pl = pressure_q(ql, kp.gas), pr = pressure_q(qr, kp.gas);
        tau = kp.gas.mu / (0.5 * (pl + pr));
    }
    const TimeW tw = time_weights(tau, kp.dt);

    FluxAcc acc;
    flux_init(acc);
    const bool owned = k < kp.nzl;
    const long f_glob = (long)i + (long)nx * (j + (long)ny * (k + kp.kglob0));
    const long item = (long)AXIS * kp.ncells_glob + f_glob;
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
        const double* B = side == 0 ? BL : BR;
        const double* dB = kp.tab + kp.off_fdB[AXIS][side == 0 ? 1 : 0] + p * 3 * N;
        const double* h = side == 0 ? hL : hR;
        const double* c = sc + side * NC * 32 + lane;
        double e[20];
#pragma unroll
        for (int m = 0; m < 20; ++m) e[m] = 0.0;
#pragma unroll
        for (int n = 0; n < N; ++n) {
            const double b = __ldg(B + n);
            const double d0 = __ldg(dB + n), d1 = __ldg(dB + N + n), d2 = __ldg(dB + 2 * N + n);
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                const double cv = c[(n * 5 + v) * 32];
                e[v] += b * cv;
                e[5 + v] += d0 * cv;
                e[10 + v] += d1 * cv;
                e[15 + v] += d2 * cv;
            }
        }
        const double s0 = 2.0 / h[0], s1 = 2.0 / h[1], s2 = 2.0 / h[2];
        // global -> face-local frame: momentum and derivative directions cycled
        // to (AXIS, C1, C2) (dg.hpp:323-334)
        double t[20];
        const double sc3[3] = {s0, s1, s2};
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int g = d == 0 ? -1 : (d == 1 ? AXIS : d == 2 ? C1 : C2);
            const double* src = d == 0 ? e : e + 5 + 5 * g;
            const double sf = d == 0 ? 1.0 : sc3[g < 0 ? 0 : g];
            t[5 * d + 0] = sf * src[0];
            t[5 * d + 1] = sf * src[1 + AXIS];
            t[5 * d + 2] = sf * src[1 + C1];
            t[5 * d + 3] = sf * src[1 + C2];
            t[5 * d + 4] = sf * src[4];
        }
        double bad = 0.0;
        const int rc = flux_side<VISC>(t, side, kp.gas, tw, acc, bad);
        if (rc) {
            if (owned) report_error(kp, err_key(kp.stage, 0, item, p, side, rc), bad);
            return;
        }
    }
    double bad = 0.0;
    const int rc = flux_merge<VISC>(kp.gas, tw, acc, bad);
    if (rc) {
        if (owned) report_error(kp, err_key(kp.stage, 0, item, p, 2, rc), bad);
        return;
    }
    if (kp.report) return;
    // face-local -> global (dg.hpp:336-345)
    const long fidx = (long)i + (long)nx * (j + (long)ny * k);
    double* out = face + (long)(p * 10) * kp.fs + fidx;
    const double F[5] = {acc.F[0], acc.F[1], acc.F[2], acc.F[3], acc.F[4]};
    const double Ft[5] = {acc.Ft[0], acc.Ft[1], acc.Ft[2], acc.Ft[3], acc.Ft[4]};
    double G[5], Gt[5];
    G[0] = F[0];
    G[4] = F[4];
    G[1 + AXIS] = F[1];
    G[1 + C1] = F[2];
    G[1 + C2] = F[3];
    Gt[0] = Ft[0];
    Gt[4] = Ft[4];
    Gt[1 + AXIS] = Ft[1];
    Gt[1 + C1] = Ft[2];
    Gt[1 + C2] = Ft[3];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
        out[v * kp.fs] = G[v];
        out[(5 + v) * kp.fs] = Gt[v];
    }
    if (kp.count_fluxes && owned) atomicAdd(kp.flux_count, 1ull);
}

// -------------------------------------------------------------- cell kernel
enum : int { MODE_RESIDUAL = 0, MODE_STAGE1 = 1, MODE_STAGE2 = 2 };

// CTA = TC consecutive cells along x. Phase B: one (cell, volume point) item
// per thread -> smooth fluxes to shared memory. Phase C: one (cell, n, var)
// item per thread -> face gather + volume projection + M^-1 + S2O4 combine.
template <int P, int DIM, bool VISC, int MODE>
__global__ void __launch_bounds__(Shape<P, DIM>::NT_CELL)
    cell_kernel(KParams kp, const double* __restrict__ qin, const double* __restrict__ f0,
                const double* __restrict__ f1, const double* __restrict__ f2,
                const double* __restrict__ qn, const double* __restrict__ L1,
                const double* __restrict__ Lt1, double* __restrict__ out0,
                double* __restrict__ out1, double* __restrict__ out2, int tile_x0, int tile_y0,
                int tile_z0) {
    using SH = Shape<P, DIM>;
    constexpr int N = SH::N, NC = SH::NC, NVP = SH::NVP, TC = SH::TC, NT = SH::NT_CELL;
    constexpr int NAX = SH::NAX;
    extern __shared__ double smem[];
    double* sc = smem;            // [NC][TC]
    double* vf = smem + NC * TC;  // [NVP][30][TC]

    const int tid = threadIdx.x;
    const int i0 = (blockIdx.x + tile_x0) * TC;
    const int j = blockIdx.y + tile_y0;
    const int k = blockIdx.z + tile_z0;
    const int nx = kp.nx, ny = kp.ny;
    const long cbase = (long)(k + 1) * kp.S + (long)j * nx;

    for (int e = tid; e < NC * TC; e += NT) {
        const int l = e % TC, comp = e / TC;
        const int i = i0 + l;
        sc[comp * TC + l] = i < nx ? __ldg(qin + comp * kp.cs + cbase + i) : 0.0;
    }
    __syncthreads();

    const double hy = __ldg(kp.dy + j), hz = __ldg(kp.dz + k + 1);
    const long cglob_row = (long)nx * (j + (long)ny * (k + kp.kglob0));

    // ---- phase B: smooth fluxes at volume points
    for (int it = tid; it < TC * NVP; it += NT) {
        const int l = it % TC, p = it / TC;
        const int i = i0 + l;
        if (i >= nx) continue;
        const double h[3] = {__ldg(kp.dx + i), hy, hz};
        const double* B = kp.tab + kp.off_vB + p * N;
        const double* dB = kp.tab + kp.off_vdB + p * 3 * N;
        double e[20];
#pragma unroll
        for (int m = 0; m < 20; ++m) e[m] = 0.0;
#pragma unroll
        for (int n = 0; n < N; ++n) {
            const double b = __ldg(B + n);
            const double d0 = __ldg(dB + n), d1 = __ldg(dB + N + n), d2 = __ldg(dB + 2 * N + n);
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                const double cv = sc[(n * 5 + v) * TC + l];
                e[v] += b * cv;
                e[5 + v] += d0 * cv;
                e[10 + v] += d1 * cv;
                e[15 + v] += d2 * cv;
            }
        }
        const double s0 = 2.0 / h[0], s1 = 2.0 / h[1], s2 = 2.0 / h[2];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            e[5 + v] *= s0;
            e[10 + v] *= s1;
            e[15 + v] *= s2;
        }
        double o[30];
        double bad = 0.0;
        const int rc = smooth_flux<VISC, NAX>(e, kp.gas, o, bad);
        if (rc) {
            report_error(kp, err_key(kp.stage, 1, cglob_row + i, p, 0, rc), bad);
#pragma unroll
            for (int m = 0; m < 30; ++m) o[m] = 0.0;
        }
#pragma unroll
        for (int m = 0; m < 10 * NAX; ++m) vf[(p * 30 + m) * TC + l] = o[m];
    }
    if (kp.report) return;
    __syncthreads();

    // ---- phase C: gather + projection + inverse mass + stage combine
    const double* tab = kp.tab;
    for (int it = tid; it < TC * NC; it += NT) {
        const int l = it % TC, comp = it / TC;
        const int n = comp / 5, v = comp - 5 * (comp / 5);
        const int i = i0 + l;
        if (i >= nx) continue;
        const double h[3] = {__ldg(kp.dx + i), hy, hz};
        double R = 0.0, Rt = 0.0;
        // faces (dg.hpp:404-425): + w jac B- F(minus face) - w jac B+ F(plus face)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double* fa = a == 0 ? f0 : a == 1 ? f1 : f2;
            const int nfp = a == 0 ? SH::template nfp<0>() : a == 1 ? SH::template nfp<1>()
                                                                    : SH::template nfp<2>();
            const double jac = h[(a + 1) % 3] * h[(a + 2) % 3] / 4.0;
            const long fm = (long)i + (long)nx * (j + (long)ny * k);
            long fp;
            if (a == 0) fp = (long)(i + 1 == nx ? 0 : i + 1) + (long)nx * (j + (long)ny * k);
            else if (a == 1) fp = (long)i + (long)nx * ((j + 1 == ny ? 0 : j + 1) + (long)ny * k);
            else {
                const int kp1 = (k + 1 == kp.zface_layers && kp.z_wrap) ? 0 : k + 1;
                fp = (long)i + (long)nx * (j + (long)ny * kp1);
            }
            const double* Bm = tab + kp.off_fB[a][0];
            const double* Bp = tab + kp.off_fB[a][1];
            const double* w = tab + kp.off_fw[a];
#pragma unroll
            for (int pf = 0; pf < nfp; ++pf) {
                const double wj = __ldg(w + pf) * jac;
                const double wm = wj * __ldg(Bm + pf * N + n), wp = wj * __ldg(Bp + pf * N + n);
                const long r0 = (long)(pf * 10 + v) * kp.fs, r1 = (long)(pf * 10 + 5 + v) * kp.fs;
                R += wm * __ldg(fa + r0 + fm) - wp * __ldg(fa + r0 + fp);
                Rt += wm * __ldg(fa + r1 + fm) - wp * __ldg(fa + r1 + fp);
            }
        }
        // volume (dg.hpp:427-448): + w (h0 h1 h2 / 8) (2/h_a) dB_a F_a
        const double vjac = h[0] * h[1] * h[2] / 8.0;
#pragma unroll
        for (int p = 0; p < NVP; ++p) {
            const double wj = __ldg(tab + kp.off_vw + p) * vjac;
#pragma unroll
            for (int a = 0; a < NAX; ++a) {
                const double wgt = wj * __ldg(tab + kp.off_vdB + (p * 3 + a) * N + n) * (2.0 / h[a]);
                R += wgt * vf[(p * 30 + a * 10 + v) * TC + l];
                Rt += wgt * vf[(p * 30 + a * 10 + 5 + v) * TC + l];
            }
        }
        const long gi = comp * kp.cs + cbase + i;
        if (MODE == MODE_RESIDUAL) {
            out0[gi] = R;
            out1[gi] = Rt;
        } else {
            // mass_diag (dg.hpp:42-50), inverse applied as R * (1/M) (solver.hpp:49-51)
            const double m = h[0] * h[1] * h[2] / __ldg(tab + kp.off_massf + n);
            const double inv = 1.0 / m;
            const double L = R * inv, Lt = Rt * inv;
            const double dt = kp.dt;
            if (MODE == MODE_STAGE1) {
                // q* = q + dt/2 L + dt^2/8 Lt (integrator.hpp:69-70)
                out0[gi] = sc[comp * TC + l] + 0.5 * dt * L + 0.125 * dt * dt * Lt;
                out1[gi] = L;
                out2[gi] = Lt;
            } else {
                // q += dt L1 + dt^2/6 (Lt1 + 2 Lt2) (integrator.hpp:72-74)
                const double c = dt * dt / 6.0;
                out0[gi] = __ldg(qn + gi) + (dt * __ldg(L1 + gi) + c * (__ldg(Lt1 + gi) + 2.0 * Lt));
            }
        }
    }
}

}  // namespace hgks_dev
