// Device kernels of the DG-HGKS S2O4 step (sm_100a, fp64).
//
//   face_kernel<P,DIM,VISC,AXIS>  one kinetic flux per owned face point
//                                 (replaces residual phase 1, dg.hpp:362-394)
//   cell_kernel<P,DIM,VISC,MODE>  volume fluxes + face gather + projection,
//                                 fused with the inverse mass matrix and the
//                                 S2O4 stage combine (dg.hpp:396-449,
//                                 solver.hpp:42-54, integrator.hpp:68-74)
//
// HBM layout (SoA, fp64): state q[comp][cell_g], comp = n*5 + var,
// cell_g = i + nx*(j + ny*(k+1)) for local z layers k = -1..nzl (one ghost
// layer each side); face buffers f_a[p*10 + (F|Ft)][i + nx*(j + ny*k)].
// Basis/quadrature values are compile-time constants (hgks_ctables.cuh).
#pragma once

#include <cuda.h>
#include <stdint.h>

#include <type_traits>

#include "hgks_ctables.cuh"
#include "hgks_kinetics.cuh"

// resident viscous face CTAs per SM the register allocator must allow. 3
// (168 registers, ~110 B of spills, 12 warps/SM) against 2 (242 registers,
// no spills, 8 warps): TGV P2 128^3 10.99 vs 11.15 ms per step, once the
// point keeps its failure codes in scalars and the library erfc is out of
// line (round 1, with ~700 B of spills, 3 measured 14.5 vs 11.6 ms)
#ifndef HGKS_FACE_MINB
#define HGKS_FACE_MINB 3
#endif
// the inviscid flux fits 4 CTAs/SM (128 registers, no spills; 3 CTAs at 166
// registers: adv3d P2 128^3 8.16 vs 8.08 ms per step); shared memory caps it at 4
#ifndef HGKS_FACE_MINB_INV
#define HGKS_FACE_MINB_INV 4
#endif
#define HGKS_FACE_MINB_PV(P, VISC) ((P) == 3 ? 1 : (VISC) ? HGKS_FACE_MINB : HGKS_FACE_MINB_INV)
// face kernel staging buffers (2: double-buffered prefetch, 1: single) and
// where the 35-double flux accumulator lives (0: registers, 1: shared memory)
#ifndef HGKS_FACE_STAGES
#define HGKS_FACE_STAGES 2
#endif
// P1/P2 face point as one basic block (both side passes + merge, codes
// checked afterwards): TGV 9.36 -> 8.85 ms per step, adv3d 6.31 -> 6.04 (the
// inviscid kernel still fits 3 CTAs/SM); P3: see HGKS_FACE_P3_ONE_BLOCK (one block
// only pays once the CTA has one point per warp)
#ifndef HGKS_FACE_ONE_BLOCK
#define HGKS_FACE_ONE_BLOCK 1
#endif
// P3 face CTAs: one point per warp (9-warp CTAs, 1 per SM, 168 registers
// with ~130 B of spills) and the point as one basic block: TGV P3 64^3
// 6.74 -> 5.91 ms per step against 3 points per warp in 3-warp CTAs (2 per
// SM, 255 registers, 6 warps) with sequential side passes
#ifndef HGKS_FACE_P3_PPW
#define HGKS_FACE_P3_PPW 1
#endif
#ifndef HGKS_FACE_P3_ONE_BLOCK
#define HGKS_FACE_P3_ONE_BLOCK 1
#endif
#ifndef HGKS_FACE_ACC_SMEM
#define HGKS_FACE_ACC_SMEM 0
#endif
// face kernel staging: both paths are compiled; KParams::face_tma selects
// TMA (cp.async.bulk.tensor of the two neighbour [NC][32] boxes per tile,
// one elected thread, mbarrier completion) or per-lane cp.async at run time
// threads of the 3-D P1/P2 cell kernel (0: one per (cell, volume point));
// 160 = one per (cell, var, F|Ft) item of the stage-1 projection, 10 warps/SM
#ifndef HGKS_CELL_NT3
#define HGKS_CELL_NT3 160
#endif
// stage-1 cell kernel of 3-D P1/P2 with 128 threads at 3 CTAs/SM and the
// combine by lane-pair shuffles (1) or 160 threads at 2 CTAs/SM (0)
#ifndef HGKS_CELL_S1X
#define HGKS_CELL_S1X 1
#endif
// P3 cell kernels (8-cell tiles, 27 volume points per cell): 6 warps at 2
// CTAs per SM (≤ 168 registers, ~100 B of spills in stage 1), projection
// items split into two basis ranges, one per warp of a pair (80 / 40 whole
// items would leave most warps idle): TGV P3 64^3 5.89 -> 5.44 ms per step
// against 7 warps at 1 CTA per SM with whole items. Per mode: stage 1 and
// the residual (NT, MINB, SPLIT1), stage 2 (NT2, MINB2, SPLIT2).
#ifndef HGKS_CELL_P3_TC
#define HGKS_CELL_P3_TC 8
#endif
#ifndef HGKS_CELL_P3_NT
#define HGKS_CELL_P3_NT 192
#endif
#ifndef HGKS_CELL_P3_MINB
#define HGKS_CELL_P3_MINB 2
#endif
#ifndef HGKS_CELL_P3_NT2
#define HGKS_CELL_P3_NT2 192
#endif
#ifndef HGKS_CELL_P3_MINB2
#define HGKS_CELL_P3_MINB2 2
#endif
#ifndef HGKS_CELL_P3_SPLIT2
#define HGKS_CELL_P3_SPLIT2 1
#endif
#ifndef HGKS_CELL_P3_SPLIT1
#define HGKS_CELL_P3_SPLIT1 1
#endif
// threads of the S1X stage-1 CTA: 160 = one per projection item (phase C in
// one round; 32 idle in phase B), 15 warps/SM at 3 CTAs with ~170 B of
// spills: stage 1 2.22 -> 2.19 ms (adv3d 1.86 -> 1.72) against 128 (one per
// (cell, volume point)); 192: 3.48 ms, 160 at 2 CTAs/SM: 2.54 ms. P2 only:
// P1 (4 basis functions, lighter phase C) stays at 128 (6.06 vs 6.33 ms)
#ifndef HGKS_CELL_S1X_NT
#define HGKS_CELL_S1X_NT 160
#endif
#ifndef HGKS_CELL_S1_MINB
#define HGKS_CELL_S1_MINB 3
#endif
// resident stage-2 CTAs per SM for 3-D P1/P2 (128 threads each)
#ifndef HGKS_CELL_S2_MINB
#define HGKS_CELL_S2_MINB 4
#endif
// P1 (20 coefficients per cell) fits 5 (96 registers): stage 2 2.85 -> 2.77 ms at 192^3
#ifndef HGKS_CELL_S2_MINB_P1
#define HGKS_CELL_S2_MINB_P1 5
#endif
// cells per cell-kernel CTA for P1/P2 (16: 128 threads per CTA in stages 1 and 2)
#ifndef HGKS_CELL_TC
#define HGKS_CELL_TC 16
#endif

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
    // cell tile along x and threads of the cell kernel (one thread per
    // (cell, volume point) in phase B for P1/P2)
    static constexpr int TC = P == 3 ? HGKS_CELL_P3_TC : HGKS_CELL_TC;
    static constexpr int NT_CELL = P == 3 ? HGKS_CELL_P3_NT : (DIM == 3 && HGKS_CELL_NT3 > 0) ? HGKS_CELL_NT3 : HGKS_CELL_TC * NVP;
    static constexpr int MINB_CELL = P == 3 ? HGKS_CELL_P3_MINB : (HGKS_CELL_TC <= 16 ? 2 : 1);
};

enum : int { SC_DT = 0, SC_INV_DT = 1, SC_RH = 2, SC_ACTIVE = 3, SC_SLOT = 8 };

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
    int ft_only;           // face pass of S2O4 stage 2: only Ft is consumed, F is not stored
    // step scalars live in device memory (written by set_scalars_kernel or,
    // in the device-resident advance loop, by dt_finalize_kernel), so a
    // captured step graph is independent of dt:
    //   scal[SC_DT] dt, [SC_INV_DT] 1/dt, [SC_RH] dt / (4 mu), [SC_ACTIVE] 0
    //   = this step is a no-op (the loop halted or reached t_end)
    const double* scal;
    double two_mu;         // 2 mu: face tau = 2 mu / (p_l + p_r)
    int grid_cap;          // > 0: cap on the persistent grids (tests: many tiles per CTA)
    unsigned shake;        // != 0: race shaker seed (tests; see race_shake)
    int face_tma;          // 1: face kernels stage by TMA (the qmap argument is valid)
    int cell_tma;          // 1: cell kernels stage by TMA (the CellMaps argument is valid)
    GasC gas;
    const double* dx;      // [nx] widths
    const double* dy;      // [ny]
    const double* dz;      // [nzl + 2] indexed k + 1
    const double* i2dx;    // 2 / h per axis (same indexing)
    const double* i2dy;
    const double* i2dz;
    const double* tab;     // runtime table image (aux kernels; include/hgks_b200/basis_tables.h)
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

// Race shaker (test hook, KParams::shake != 0): before every cp.async wait
// and barrier, each warp sleeps a pseudo-random 0..4 us keyed by (seed, CTA,
// warp, site, tile), so a missing barrier or a wrong cp.async group count
// shows up as a changed result against the unperturbed run (bitwise). It
// stands in for compute-sanitizer racecheck, which this GPU pool does not run.
__device__ __forceinline__ void race_shake(const KParams& kp, int site, int n) {
    if (kp.shake) {
        unsigned h = kp.shake * 2654435761u ^ (blockIdx.x * 40503u) ^ ((threadIdx.x >> 5) * 9973u) ^
                     ((unsigned)site * 7919u) ^ ((unsigned)n * 104729u);
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        __nanosleep(h & 4095u);
    }
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

// ---- sign symmetry of the tensor Gauss rules
// Per axis the rule's abscissae are symmetric (-g, [0,] +g) and
// P_l(-x) = (-1)^l P_l(x) exactly in floating point. A quadrature point's
// CLASS is its zero pattern (which coordinates are 0: the middle point of the
// 3-point rule, or a collapsed 2-D axis); within a class a table row equals
// the row at the class' canonical point (+g on every non-zero axis) with
// basis n negated by prod over negative axes of (-1)^{par_a(n)} (a derivative
// along a negative axis carries one more sign). The evaluators below flip
// the sign bit of each coefficient (an integer op) and run ONE compile-time
// table per class: 1 class for the 2-point rule, 4 face / 8 volume classes
// for the 3-point rule (instead of one code path per point: 9 / 27 for P3).
// The products and sums are bitwise those of the per-point tables; the
// symmetry of the tables is verified at compile time (gauss_symmetric).
constexpr unsigned kSignBit = 0x80000000u;
__device__ __forceinline__ double flip_sign(double x, unsigned m) {
    return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}
__host__ __device__ constexpr bool g_zero(int nq, int idx) { return (nq & 1) && idx == nq / 2; }
__host__ __device__ constexpr bool g_neg(int nq, int idx) { return !g_zero(nq, idx) && idx < nq / 2; }
__host__ __device__ constexpr int g_canon(int nq, int idx) { return g_zero(nq, idx) ? idx : nq - 1; }

// face-point geometry of axis a: tangential axes (C1, C2) with nb, nc points
template <int P, int DIM, int AXIS>
struct FaceRule {
    static constexpr int NQ = Shape<P, DIM>::NQ;
    static constexpr int C1 = (AXIS + 1) % 3, C2 = (AXIS + 2) % 3;
    static constexpr int NB = (C1 == 2 && DIM == 2) ? 1 : NQ;
    static constexpr int NCC = (C2 == 2 && DIM == 2) ? 1 : NQ;
    // class = (tangential 1 zero, tangential 2 zero) -> canonical point
    static constexpr int canon(int zb, int zc) {
        return (zb ? NB / 2 : NB - 1) * NCC + (zc ? NCC / 2 : NCC - 1);
    }
};

template <int P, int DIM>
constexpr bool gauss_symmetric() {
    constexpr ct::Tab T = ct::make_tab<P, DIM>();
    const int NQ = T.NQ, nqz = DIM == 3 ? NQ : 1;
    auto sg = [](bool neg, int par) { return (neg && par) ? -1.0 : 1.0; };
    for (int p = 0; p < T.NVP; ++p) {
        const int i = p / (NQ * nqz), j = (p / nqz) % NQ, k = p % nqz;
        const bool ni = g_neg(NQ, i), nj = g_neg(NQ, j), nk = g_neg(nqz, k);
        const int pc = (g_canon(NQ, i) * NQ + g_canon(NQ, j)) * nqz + g_canon(nqz, k);
        for (int n = 0; n < T.N; ++n) {
            const double sn = sg(ni, T.par[0][n]) * sg(nj, T.par[1][n]) * sg(nk, T.par[2][n]);
            if (T.vB[p][n] != sn * T.vB[pc][n]) return false;
            const double sa[3] = {ni ? -1.0 : 1.0, nj ? -1.0 : 1.0, nk ? -1.0 : 1.0};
            for (int a = 0; a < 3; ++a)
                if (T.vdB[p][a][n] != sa[a] * sn * T.vdB[pc][a][n]) return false;
        }
    }
    for (int a = 0; a < 3; ++a) {
        const int c1 = (a + 1) % 3, c2 = (a + 2) % 3;
        const int nb = (c1 == 2 && DIM == 2) ? 1 : NQ, nc = (c2 == 2 && DIM == 2) ? 1 : NQ;
        for (int sd = 0; sd < 2; ++sd)
            for (int p = 0; p < nb * nc; ++p) {
                const int ib = p / nc, ic = p % nc;
                const bool n1 = g_neg(nb, ib), n2 = g_neg(nc, ic);
                const int pc = g_canon(nb, ib) * nc + g_canon(nc, ic);
                for (int n = 0; n < T.N; ++n) {
                    const double sn = sg(n1, T.par[c1][n]) * sg(n2, T.par[c2][n]);
                    if (T.fB[a][sd][p][n] != sn * T.fB[a][sd][pc][n]) return false;
                    for (int d = 0; d < 3; ++d) {
                        const double s1 = d == c1 && n1 ? -1.0 : 1.0, s2 = d == c2 && n2 ? -1.0 : 1.0;
                        if (T.fdB[a][sd][p][d][n] != s1 * s2 * sn * T.fdB[a][sd][pc][d][n]) return false;
                    }
                }
            }
    }
    return true;
}

// Trace of one side at a face point of class PS (its canonical index) in the
// face-local frame (eval_tabulated dg.hpp:139-161 + to_face_local
// dg.hpp:323-334); m1, m2: sign masks of the point's tangential axes.
// SIDE 0 = minus-side cell at its plus face (ref coord +1), 1 = plus-side
// cell at its minus face (-1). c = shared-memory coefficients [comp][RS].
template <int P, int DIM, int AXIS, int SIDE, int RS, int PS>
__device__ __forceinline__ void face_trace_canon(unsigned m1, unsigned m2, const double* __restrict__ c,
                                                 const double* i2h, double* t) {
    using SH = Shape<P, DIM>;
    constexpr int N = SH::N;
    constexpr int C1 = (AXIS + 1) % 3, C2 = (AXIS + 2) % 3;
    constexpr int SI = SIDE == 0 ? 1 : 0;
    double e[20];
#pragma unroll
    for (int m = 0; m < 20; ++m) e[m] = 0.0;
#pragma unroll
    for (int n = 0; n < N; ++n) {
        const double b = ctab<P, DIM>.fB[AXIS][SI][PS][n];
        const double d0 = ctab<P, DIM>.fdB[AXIS][SI][PS][0][n];
        const double d1 = ctab<P, DIM>.fdB[AXIS][SI][PS][1][n];
        const double d2 = ctab<P, DIM>.fdB[AXIS][SI][PS][2][n];
        const unsigned mn = (ctab<P, DIM>.par[C1][n] ? m1 : 0u) ^ (ctab<P, DIM>.par[C2][n] ? m2 : 0u);
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            const double cv = flip_sign(c[(n * 5 + v) * RS], mn);
            if (b != 0.0) e[v] += b * cv;
            if (d0 != 0.0) e[5 + v] += d0 * cv;
            if (d1 != 0.0) e[10 + v] += d1 * cv;
            if (d2 != 0.0) e[15 + v] += d2 * cv;
        }
    }
    // global -> face-local: momentum and derivative directions cycled to
    // (AXIS, C1, C2); derivatives scaled by 2/h of their direction (with the
    // point's sign on a tangential axis)
    constexpr int g[3] = {AXIS, C1, C2};
    t[0] = e[0];
    t[1] = e[1 + AXIS];
    t[2] = e[1 + C1];
    t[3] = e[1 + C2];
    t[4] = e[4];
#pragma unroll
    for (int d = 1; d < 4; ++d) {
        const int gd = g[d - 1];
        const double* src = e + 5 + 5 * gd;
        const double sf = flip_sign(i2h[gd], gd == C1 ? m1 : gd == C2 ? m2 : 0u);
        t[5 * d + 0] = sf * src[0];
        t[5 * d + 1] = sf * src[1 + AXIS];
        t[5 * d + 2] = sf * src[1 + C1];
        t[5 * d + 3] = sf * src[1 + C2];
        t[5 * d + 4] = sf * src[4];
    }
}

// face point p -> its class' evaluator (one code path per class)
template <int P, int DIM, int AXIS, int SIDE, int RS>
__device__ __forceinline__ void face_trace_sym(int p, const double* __restrict__ c, const double* i2h,
                                               double* t) {
    static_assert(gauss_symmetric<P, DIM>(), "basis tables are not sign-symmetric");
    using FR = FaceRule<P, DIM, AXIS>;
    const int ib = p / FR::NCC, ic = p % FR::NCC;
    const unsigned m1 = g_neg(FR::NB, ib) ? kSignBit : 0u, m2 = g_neg(FR::NCC, ic) ? kSignBit : 0u;
    const bool zb = g_zero(FR::NB, ib), zc = g_zero(FR::NCC, ic);
    if constexpr (FR::NQ == 2 && FR::NB != 1 && FR::NCC != 1) {
        face_trace_canon<P, DIM, AXIS, SIDE, RS, FR::canon(0, 0)>(m1, m2, c, i2h, t);
    } else {
        if (!zb && !zc) face_trace_canon<P, DIM, AXIS, SIDE, RS, FR::canon(0, 0)>(m1, m2, c, i2h, t);
        else if (!zb) face_trace_canon<P, DIM, AXIS, SIDE, RS, FR::canon(0, 1)>(m1, m2, c, i2h, t);
        else if (!zc) face_trace_canon<P, DIM, AXIS, SIDE, RS, FR::canon(1, 0)>(m1, m2, c, i2h, t);
        else face_trace_canon<P, DIM, AXIS, SIDE, RS, FR::canon(1, 1)>(m1, m2, c, i2h, t);
    }
}

// Tile walk of the persistent kernels: tile t = tx + ntx (j + ny k). The
// stride (gridDim.x tiles) is decomposed once; each step is then a few adds
// with carries instead of two integer divisions on the prefetch's critical path.
struct TileWalk {
    int ntx, ny, W;      // x tiles per row, rows, cells per x tile
    int sx, sj, sk;      // stride in (tx, j, k)
    __device__ __forceinline__ TileWalk(int ntx_, int ny_, int w, int step) : ntx(ntx_), ny(ny_), W(w) {
        const int a = step / ntx;
        sx = step - a * ntx;
        sk = a / ny;
        sj = a - sk * ny;
    }
    struct TI {
        int i0, j, k, tx;
    };
    __device__ __forceinline__ TI of(int t) const {
        const int a = t / ntx;
        TI r;
        r.tx = t - a * ntx;
        r.i0 = r.tx * W;
        r.k = a / ny;
        r.j = a - r.k * ny;
        return r;
    }
    __device__ __forceinline__ TI next(TI r) const {
        r.tx += sx;
        const int cx = r.tx >= ntx;
        r.tx -= cx ? ntx : 0;
        r.j += sj + cx;
        const int cy = r.j >= ny;
        r.j -= cy ? ny : 0;
        r.k += sk + cy;
        r.i0 = r.tx * W;
        return r;
    }
};

// async global->shared copies (cp.async, LDGSTS): the persistent kernels
// prefetch the next tile while computing the current one
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
                 "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
// one [box] of a 3-D tensor map (x, row, comp) into shared memory, completing
// on `bar` (transaction bytes)
__device__ __forceinline__ void tma_load3(double* dst, const CUtensorMap* map, int x, int row, int comp,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(x), "r"(row), "r"(comp), "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

// face-kernel stage layout: y / z faces [side][comp][32]; x faces one shared
// [comp][34] row (x = i0-2 .. i0+31), minus side at column lane+1, plus side
// at lane+2
// x box width (build knob): 34 (x = i0-2 .. i0+31) or 48 (x = i0-16 ..
// i0+31: the plus side's rows then start 128-byte aligned in shared memory)
#ifndef HGKS_FACE_XBOX
#define HGKS_FACE_XBOX 34
#endif
template <int NC, int AXIS>
struct FaceStage {
    static constexpr int XW = HGKS_FACE_XBOX, XOFF = XW - 32;  // x box: x = i0 - XOFF .. i0 + 31
    // stages start 128-byte aligned (TMA destinations)
    static constexpr int STG = AXIS == 0 ? (XW * NC + 15) / 16 * 16 : 2 * NC * 32;
    static constexpr int RSL = AXIS == 0 ? XW : 32, RSR = RSL;
    static constexpr int OFL = AXIS == 0 ? XOFF - 1 : 0, OFR = AXIS == 0 ? XOFF : NC * 32;
};

__device__ __forceinline__ void tma_load4(double* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

// Persistent face kernel. A CTA = NFP warps; each tile is 32 consecutive faces
// along x (one lane each) at one (j, k), one face point per warp, so the
// point index is warp-uniform. The two neighbour cells' coefficients of the
// NEXT tile stream into the other half of a double-buffered shared-memory
// stage (TMA boxes, or cp.async rows when the state has no TMA view) while
// the current tile's fluxes are computed. P3 (9 points) keeps one point per
// warp by default (HGKS_FACE_P3_PPW; 3 gives 3-warp CTAs at 255 registers).
template <int P, int DIM, int AXIS>
struct FaceCTA {
    static constexpr int NFP = Shape<P, DIM>::template nfp<AXIS>();
    static constexpr int PPW = (P == 3 && NFP % HGKS_FACE_P3_PPW == 0) ? HGKS_FACE_P3_PPW : 1;  // points per warp
    static constexpr int NT = 32 * NFP / PPW;
};

// FTO (the S2O4 second stage: only Ft is consumed) is a template argument so
// the F-only arithmetic of the merge drops out of that instantiation
template <int P, int DIM, bool VISC, int AXIS, bool FTO = false>
__global__ void __launch_bounds__(FaceCTA<P, DIM, AXIS>::NT, HGKS_FACE_MINB_PV(P, VISC))
    face_kernel(KParams kp, const double* __restrict__ q, double* __restrict__ face,
                int tile_first, int tile_count, const __grid_constant__ CUtensorMap qmap) {
    using SH = Shape<P, DIM>;
    constexpr int NC = SH::NC;
    constexpr int NFP = SH::template nfp<AXIS>();
    constexpr int PPW = FaceCTA<P, DIM, AXIS>::PPW;
    constexpr int NT = FaceCTA<P, DIM, AXIS>::NT;
    constexpr int C1 = (AXIS + 1) % 3, C2 = (AXIS + 2) % 3;
    // one stage: y / z faces [side][comp][32]; x faces ONE [comp][34] row
    // (x = i0-2 .. i0+31): the minus neighbour of lane l is column l+1, the
    // plus neighbour column l+2 (the two sides overlap in x)
    constexpr int STG = FaceStage<NC, AXIS>::STG;
    constexpr int RSL = FaceStage<NC, AXIS>::RSL, RSR = FaceStage<NC, AXIS>::RSR;
    constexpr int OFL = FaceStage<NC, AXIS>::OFL, OFR = FaceStage<NC, AXIS>::OFR;
    extern __shared__ __align__(128) double smem[];  // 128 B: TMA destinations

    if (kp.scal[SC_ACTIVE] == 0.0) return;  // halted device loop: no-op step
    const double inv_dt = kp.scal[SC_INV_DT], rh_coef = kp.scal[SC_RH];
    const int tid = threadIdx.x;
    const int nx = kp.nx, ny = kp.ny;
    const int ntx = (nx + 31) / 32;
    const int tile_end = tile_first + tile_count;
    const int step = kp.report ? tile_count : gridDim.x;

    const int lane = tid & 31;
    const int warp = tid >> 5;
    // tile t -> (x offset, row j, layer k); computed once per tile
    using TI = TileWalk::TI;
    const TileWalk walk(ntx, ny, 32, step);
    // both neighbours' coefficients of one tile: lane = face, rows = components
    // (each warp streams its share of the 2*NC rows, 256 B per row)
    auto prefetch = [&](const TI& ti, double* dst) {
        constexpr int NW = NT / 32;
        if (AXIS == 0) {
            // column c = x = i0 - XOFF + c (periodic wrap at both ends); the
            // kernel reads columns XOFF-1 .. XOFF+31: lanes fetch XOFF..XOFF+31,
            // lane 0 also column XOFF-1
            constexpr int XW = FaceStage<NC, AXIS>::XW, XOFF = FaceStage<NC, AXIS>::XOFF;
            const long row = (long)(ti.k + 1) * kp.S + (long)ti.j * nx;
            const int xa = ti.i0 + lane, xb = ti.i0 - 1;
            const bool oka = xa < nx;
            const double* sa = q + row + (oka ? xa : 0);
            const double* sb = q + row + (xb < 0 ? xb + nx : xb);
#pragma unroll 4
            for (int c = warp; c < NC; c += NW) {
                cp_async8(dst + c * XW + XOFF + lane, sa + c * kp.cs, oka);
                if (lane == 0) cp_async8(dst + c * XW + XOFF - 1, sb + c * kp.cs, true);
            }
            return;
        }
        const int i = ti.i0 + lane;
        const bool ok = i < nx;
        const int ci = ok ? i : 0;
        int mj = ti.j, mk = ti.k;
        if (AXIS == 1) mj = ti.j == 0 ? ny - 1 : ti.j - 1;
        if (AXIS == 2) mk = ti.k - 1;
        const double* sL = q + (long)(mk + 1) * kp.S + (long)mj * nx + ci;
        const double* sR = q + (long)(ti.k + 1) * kp.S + (long)ti.j * nx + ci;
#pragma unroll 4
        for (int c = warp; c < NC; c += NW) {
            cp_async8(dst + c * 32 + lane, sL + c * kp.cs, ok);
            cp_async8(dst + (NC + c) * 32 + lane, sR + c * kp.cs, ok);
        }
    };

    // TMA staging: both neighbours' [NC][32] boxes of a tile, one elected
    // thread, completion counted in bytes on the stage's mbarrier
    __shared__ uint64_t mbar[2];
    const bool tma = kp.face_tma != 0 && HGKS_FACE_STAGES == 2;
    // (the box start must be 16-byte aligned: x starts at even columns)
    auto tma_tile = [&](const TI& ti, int stage) {
        double* dst = smem + stage * STG;
        const int rowR = ti.j + ny * (ti.k + 1);
        if (AXIS == 0) {
            // one XW-wide box from x = i0 - XOFF (x < 0 at i0 = 0 is
            // zero-filled and patched after the wait: TMA has no periodic wrap)
            mbar_expect_tx(&mbar[stage], (unsigned)FaceStage<NC, AXIS>::XW * NC * 8u);
            tma_load3(dst, &qmap, ti.i0 - FaceStage<NC, AXIS>::XOFF, rowR, 0, &mbar[stage]);
            return;
        }
        const int rowL = AXIS == 1 ? (ti.j == 0 ? ny - 1 : ti.j - 1) + ny * (ti.k + 1) : ti.j + ny * ti.k;
        mbar_expect_tx(&mbar[stage], 2u * NC * 32u * 8u);
        tma_load3(dst, &qmap, ti.i0, rowL, 0, &mbar[stage]);
        tma_load3(dst + NC * 32, &qmap, ti.i0, rowR, 0, &mbar[stage]);
    };
    if (tma) {
        if (tid == 0) {
            mbar_init(&mbar[0], 1);
            mbar_init(&mbar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
    }
    const int t0 = tile_first + (kp.report ? 0 : blockIdx.x);
    TI cur = walk.of(t0);
    if (tma) {
        if (tid == 0 && t0 < tile_end) tma_tile(cur, 0);
    } else {
        if (t0 < tile_end) prefetch(cur, smem);
        cp_async_commit();
    }
    // periodic x with TMA: the minus neighbour of face 0 is cell nx-1, which
    // the box (x = -2 .. 31 at i0 = 0) cannot wrap to; its NC values are
    // loaded into registers a tile ahead (latency hidden) and patched into
    // column 1 after the box lands
    double wrapv[2] = {0.0, 0.0};
    auto load_wrap = [&](const TI& ti) {
        if (AXIS == 0 && tma && ti.i0 == 0) {
            const double* src = q + (long)(ti.k + 1) * kp.S + (long)ti.j * nx + (nx - 1);
#pragma unroll
            for (int r = 0; r < 2; ++r)
                if (tid + r * NT < NC) wrapv[r] = __ldg(src + (long)(tid + r * NT) * kp.cs);
        }
    };
    if (t0 < tile_end) load_wrap(cur);
    int n = 0;
    for (int t = t0; t < tile_end; t += step, ++n) {
        double* sc = smem + (HGKS_FACE_STAGES == 2 ? (n & 1) * STG : 0);
        const bool has_next = t + step < tile_end;
        const TI nxt = walk.next(cur);
        if (tma) {
            if (tid == 0 && has_next) {
                // the other stage was last read in tile n-1 (end-of-tile barrier)
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                tma_tile(nxt, (n + 1) & 1);
            }
        } else if (HGKS_FACE_STAGES == 2) {
            if (has_next) prefetch(nxt, smem + ((n + 1) & 1) * STG);
            cp_async_commit();
        }
        const int i0 = cur.i0, j = cur.j, k = cur.k;
        const int i = i0 + lane;
        race_shake(kp, 0, n);
        if (tma) {
            mbar_wait(&mbar[n & 1], (n >> 1) & 1);  // this tile's stage landed
            if (AXIS == 0 && i0 == 0) {
                // column 1 (x = -1) arrived zero-filled: the wrap values
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    if (tid + r * NT < NC) sc[(tid + r * NT) * RSL + OFL] = wrapv[r];
                __syncthreads();
            }
            if (has_next) load_wrap(nxt);  // the next tile's, a tile ahead
        } else {
            if (HGKS_FACE_STAGES == 2) cp_async_wait<1>();  // this tile's stage
            else cp_async_wait<0>();
            __syncthreads();
        }
#pragma unroll 1
        for (int ip = 0; ip < PPW; ++ip) {
        const int p = warp * PPW + ip;
        if (i < nx) {
            const int im = AXIS == 0 ? (i == 0 ? nx - 1 : i - 1) : i;
            const int jm = AXIS == 1 ? (j == 0 ? ny - 1 : j - 1) : j;
            const int km = AXIS == 2 ? k - 1 : k;
            const double i2hL[3] = {__ldg(kp.i2dx + im), __ldg(kp.i2dy + jm), __ldg(kp.i2dz + km + 1)};
            const double i2hR[3] = {__ldg(kp.i2dx + i), __ldg(kp.i2dy + j), __ldg(kp.i2dz + k + 1)};
            const double* cL = sc + OFL + lane;
            const double* cR = sc + OFR + lane;

#if HGKS_FACE_ACC_SMEM
            SmemAcc acc{smem + HGKS_FACE_STAGES * STG + tid, NT};
#else
            FluxAcc acc;
#endif
            flux_init(acc);
            const bool owned = k < kp.nzl;
            const long item = (long)AXIS * kp.ncells_glob + (long)i + (long)nx * (j + (long)ny * (k + kp.kglob0));
            int fail = 0;
            double psum = 0.0;  // p_l + p_r of the traces
            double F[5], Ft[5];
            if constexpr ((P < 3 || HGKS_FACE_P3_ONE_BLOCK) && HGKS_FACE_ONE_BLOCK) {
            // both side passes and the merge without early exits: one basic
            // block, so the scheduler can overlap their dependency chains; the
            // codes are checked afterwards in the reference's order
            // (left, right, merged state)
            int rc0 = 0, rc1 = 0, rc2 = 0;  // scalars, no runtime-indexed (local) arrays
            double bad0 = 0.0, bad1 = 0.0, bad2 = 0.0;
#ifdef HGKS_FACE_SIDE_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
            for (int side = 0; side < 2; ++side) {
                double tr[20];
                if (side == 0) face_trace_sym<P, DIM, AXIS, 0, RSL>(p, cL, i2hL, tr);
                else face_trace_sym<P, DIM, AXIS, 1, RSR>(p, cR, i2hR, tr);
                double ps = 0.0, bd = 0.0;
                const int rc = flux_side<VISC>(tr, side, kp.gas, acc, ps, bd);
                if (side == 0) { rc0 = rc; bad0 = bd; } else { rc1 = rc; bad1 = bd; }
                psum += ps;
            }
            {
                // tau = mu / mean trace pressure (dg.hpp:378-383); dt/(2 tau) without a division
                const double tau = VISC ? kp.two_mu / psum : 0.0;
                const TimeW tw = time_weights_r(tau, inv_dt, VISC ? psum * rh_coef : 0.0);
                rc2 = flux_merge<VISC>(kp.gas, tw, acc, F, Ft, bad2);
            }
            if (rc0 | rc1 | rc2) {
                // first failing stage in the reference's order (left, right, merged state)
                const int st = rc0 ? 0 : rc1 ? 1 : 2;
                const int rc = rc0 ? rc0 : rc1 ? rc1 : rc2;
                const double bd = rc0 ? bad0 : rc1 ? bad1 : bad2;
                if (owned) report_error(kp, err_key(kp.stage, 0, item, p, st, rc), bd);
                fail = 1;
            }
            } else {
            // P3: sequential passes
#pragma unroll 1
            for (int side = 0; side < 2 && !fail; ++side) {
                double tr[20];
                if (side == 0) face_trace_sym<P, DIM, AXIS, 0, RSL>(p, cL, i2hL, tr);
                else face_trace_sym<P, DIM, AXIS, 1, RSR>(p, cR, i2hR, tr);
                double bad = 0.0, ps = 0.0;
                const int rc = flux_side<VISC>(tr, side, kp.gas, acc, ps, bad);
                psum += ps;
                if (rc) {
                    if (owned) report_error(kp, err_key(kp.stage, 0, item, p, side, rc), bad);
                    fail = 1;
                }
            }
            if (!fail) {
                // tau = mu / mean trace pressure (dg.hpp:378-383); dt/(2 tau) without a division
                const double tau = VISC ? kp.two_mu / psum : 0.0;
                const TimeW tw = time_weights_r(tau, inv_dt, VISC ? psum * rh_coef : 0.0);
                double bad = 0.0;
                const int rc = flux_merge<VISC>(kp.gas, tw, acc, F, Ft, bad);
                if (rc) {
                    if (owned) report_error(kp, err_key(kp.stage, 0, item, p, 2, rc), bad);
                    fail = 1;
                }
            }
            }
            if (!fail && !kp.report) {
                // face-local -> global (dg.hpp:336-345)
                const long fidx = (long)i + (long)nx * (j + (long)ny * k);
                double* out = face + (long)(p * 10) * kp.fs + fidx;
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
                if (!FTO) {
#pragma unroll
                    for (int v = 0; v < 5; ++v) out[v * kp.fs] = G[v];
                }
#pragma unroll
                for (int v = 0; v < 5; ++v) out[(5 + v) * kp.fs] = Gt[v];
                if (kp.count_fluxes && owned) atomicAdd(kp.flux_count, 1ull);
            }
        }
        }  // points of this warp
        race_shake(kp, 1, n);
        __syncthreads();  // this stage is free for the prefetch two tiles ahead
        if (HGKS_FACE_STAGES == 1) {
            if (has_next) prefetch(nxt, smem);
            cp_async_commit();
        }
        cur = nxt;
    }
    if (!tma) cp_async_wait<0>();
}

// -------------------------------------------------------------- cell kernel

// value + global derivatives at a volume point of class PS (canonical index)
// (eval_tabulated, dg.hpp:139-161); m0..m2: the point's sign masks
template <int P, int DIM, int TC, int PS>
__device__ __forceinline__ void vol_eval_canon(unsigned m0, unsigned m1, unsigned m2,
                                               const double* __restrict__ c, const double* i2h, double* e) {
    using SH = Shape<P, DIM>;
    constexpr int N = SH::N;
#pragma unroll
    for (int m = 0; m < 20; ++m) e[m] = 0.0;
#pragma unroll
    for (int n = 0; n < N; ++n) {
        const double b = ctab<P, DIM>.vB[PS][n];
        const double d0 = ctab<P, DIM>.vdB[PS][0][n];
        const double d1 = ctab<P, DIM>.vdB[PS][1][n];
        const double d2 = ctab<P, DIM>.vdB[PS][2][n];
        const unsigned mn = (ctab<P, DIM>.par[0][n] ? m0 : 0u) ^ (ctab<P, DIM>.par[1][n] ? m1 : 0u) ^
                            (ctab<P, DIM>.par[2][n] ? m2 : 0u);
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            const double cv = flip_sign(c[(n * 5 + v) * TC], mn);
            if (b != 0.0) e[v] += b * cv;
            if (d0 != 0.0) e[5 + v] += d0 * cv;
            if (d1 != 0.0) e[10 + v] += d1 * cv;
            if (d2 != 0.0) e[15 + v] += d2 * cv;
        }
    }
    const double s0 = flip_sign(i2h[0], m0), s1 = flip_sign(i2h[1], m1), s2 = flip_sign(i2h[2], m2);
#pragma unroll
    for (int v = 0; v < 5; ++v) {
        e[5 + v] *= s0;
        e[10 + v] *= s1;
        e[15 + v] *= s2;
    }
}

// volume point p = (i, j, k), k fastest -> its class' evaluator
template <int P, int DIM, int TC>
__device__ __forceinline__ void vol_eval_sym(int p, const double* __restrict__ c, const double* i2h,
                                             double* e) {
    static_assert(gauss_symmetric<P, DIM>(), "basis tables are not sign-symmetric");
    constexpr int NQ = Shape<P, DIM>::NQ, NQZ = DIM == 3 ? NQ : 1;
    const int i = p / (NQ * NQZ), j = (p / NQZ) % NQ, k = p % NQZ;
    const unsigned m0 = g_neg(NQ, i) ? kSignBit : 0u, m1 = g_neg(NQ, j) ? kSignBit : 0u,
                   m2 = g_neg(NQZ, k) ? kSignBit : 0u;
    constexpr auto PC = [](int zi, int zj, int zk) {
        return ((zi ? NQ / 2 : NQ - 1) * NQ + (zj ? NQ / 2 : NQ - 1)) * NQZ + (zk ? NQZ / 2 : NQZ - 1);
    };
    if constexpr (NQ == 2) {
        vol_eval_canon<P, DIM, TC, PC(0, 0, 0)>(m0, m1, m2, c, i2h, e);
    } else {
        const int cls = (g_zero(NQ, i) ? 4 : 0) | (g_zero(NQ, j) ? 2 : 0) | (g_zero(NQZ, k) ? 1 : 0);
        switch (cls) {
            case 0: vol_eval_canon<P, DIM, TC, PC(0, 0, 0)>(m0, m1, m2, c, i2h, e); break;
            case 1: vol_eval_canon<P, DIM, TC, PC(0, 0, 1)>(m0, m1, m2, c, i2h, e); break;
            case 2: vol_eval_canon<P, DIM, TC, PC(0, 1, 0)>(m0, m1, m2, c, i2h, e); break;
            case 3: vol_eval_canon<P, DIM, TC, PC(0, 1, 1)>(m0, m1, m2, c, i2h, e); break;
            case 4: vol_eval_canon<P, DIM, TC, PC(1, 0, 0)>(m0, m1, m2, c, i2h, e); break;
            case 5: vol_eval_canon<P, DIM, TC, PC(1, 0, 1)>(m0, m1, m2, c, i2h, e); break;
            case 6: vol_eval_canon<P, DIM, TC, PC(1, 1, 0)>(m0, m1, m2, c, i2h, e); break;
            default: vol_eval_canon<P, DIM, TC, PC(1, 1, 1)>(m0, m1, m2, c, i2h, e); break;
        }
    }
}

// Phase-B order of the volume points: sorted by class, so the points a warp
// evaluates together (32 / TC of them) share one evaluator where possible.
template <int P, int DIM>
struct VolOrder {
    int p[27];
};
template <int P, int DIM>
constexpr VolOrder<P, DIM> make_vol_order() {
    VolOrder<P, DIM> o{};
    constexpr int NQ = Shape<P, DIM>::NQ, NQZ = DIM == 3 ? NQ : 1, NVP = Shape<P, DIM>::NVP;
    int n = 0;
    for (int cls = 0; cls < 8; ++cls)
        for (int q = 0; q < NVP; ++q) {
            const int i = q / (NQ * NQZ), j = (q / NQZ) % NQ, k = q % NQZ;
            const int c = (g_zero(NQ, i) ? 4 : 0) | (g_zero(NQ, j) ? 2 : 0) | (g_zero(NQZ, k) ? 1 : 0);
            if (c == cls) o.p[n++] = q;
        }
    return o;
}
template <int P, int DIM>
__device__ constexpr VolOrder<P, DIM> kVolOrder = make_vol_order<P, DIM>();

enum : int { MODE_RESIDUAL = 0, MODE_STAGE1 = 1, MODE_STAGE2 = 2 };

// shared-memory plan of one cell-kernel CTA (doubles). Face and volume flux
// rows are (F|Ft) x var; the S2O4 second stage keeps only the Ft rows
// (RW = 5, RO = 5), so its tile is half as large. Every region starts
// 128-byte aligned (TMA destinations): sizes rounded to 16 doubles.
constexpr int pad16(int n) { return (n + 15) / 16 * 16; }
template <int V>
using IC = std::integral_constant<int, V>;
template <int P, int DIM, int MODE>
struct CellTile {
    using SH = Shape<P, DIM>;
    static constexpr int TC = SH::TC, NC = SH::NC, NVP = SH::NVP;
    static constexpr int NFX = SH::template nfp<0>(), NFY = SH::template nfp<1>(),
                         NFZ = SH::template nfp<2>();
    static constexpr int RW = MODE == MODE_STAGE2 ? 5 : 10, RO = 10 - RW;
    static constexpr int XS = TC + 2;                    // x faces i0..i0+TC (+1 pad: even box width)
    static constexpr int COEF = pad16(NC * TC);          // one coefficient tile [NC][TC]
    static constexpr int FX = pad16(NFX * RW * XS);      // x faces [pf][c][XS]
    static constexpr int FYH = pad16(NFY * RW * TC);     // y faces of one row [pf][c][TC]
    static constexpr int FZH = pad16(NFZ * RW * TC);
    static constexpr int FY = pad16(2 * FYH);            // rows j, j+1   [half][pf][c][TC]
    static constexpr int FZ = pad16(2 * FZH);            // layers k, k+1 [half][pf][c][TC]
    static constexpr int VFW = 3 * RW;                   // flux rows per volume point
    static constexpr int VF = pad16(NVP * VFW * TC);     // volume-point fluxes [p][VFW][TC]
    // stage 1 of 3-D P1/P2 as one thread per (cell, volume point) at 3 CTAs
    // per SM (HGKS_CELL_S1X): the F and Ft items of a (cell, var) sit in
    // adjacent lanes and swap L1 / Lt1 by a shuffle, so no L, Lt tile
    static constexpr bool S1X = HGKS_CELL_S1X && MODE == MODE_STAGE1 && P < 3 && DIM == 3;
    static constexpr int LB = MODE == MODE_STAGE1 && !S1X ? pad16(2 * NC * TC) : 0;  // L, Lt of the tile (stage-1 q*)
    static constexpr int GEO = 2 * TC + 4;               // widths of a tile: dx, 2/dx [TC]; dy, dz, 2/dy, 2/dz
    // stage 2: the tile's A = q + dt L1 + dt^2/6 Lt1 [NC][TC], prefetched with the faces
    static constexpr int AB = MODE == MODE_STAGE2 ? COEF : 0;
    // projection items (cell, var, F|Ft); stage 2 projects only Ft
    static constexpr int NITEMS = TC * 5 * (MODE == MODE_STAGE2 ? 1 : 2);
    static constexpr int SMEM = 2 * COEF + FX + FY + FZ + VF + LB + AB + pad16(2 * GEO);
    // bytes the face group of a tile lands (TMA transaction count)
    static constexpr unsigned FACE_TX =
        8u * (NFX * RW * XS + 2 * NFY * RW * TC + 2 * NFZ * RW * TC + (MODE == MODE_STAGE2 ? NC * TC : 0));
    // threads / resident CTAs: stage 2 (half the tile, ~150 registers) runs
    // one thread per (cell, volume point) at 3 CTAs per SM for 3-D P1/P2
    static constexpr bool S2X = MODE == MODE_STAGE2 && P < 3 && DIM == 3;
    static constexpr int NT = S2X ? TC * NVP : S1X ? (P == 2 ? HGKS_CELL_S1X_NT : TC * NVP) : (P == 3 && MODE == MODE_STAGE2) ? HGKS_CELL_P3_NT2 : SH::NT_CELL;
    static constexpr int MINB = S2X ? (P == 1 ? HGKS_CELL_S2_MINB_P1 : HGKS_CELL_S2_MINB) : S1X ? HGKS_CELL_S1_MINB : (P == 3 && MODE == MODE_STAGE2) ? HGKS_CELL_P3_MINB2 : SH::MINB_CELL;
    // P3: projection items split into two basis ranges (see HGKS_CELL_P3_SPLIT2)
    static constexpr bool SPLIT = P == 3 && (MODE == MODE_STAGE2 ? HGKS_CELL_P3_SPLIT2 : HGKS_CELL_P3_SPLIT1);
};

// TMA tensor maps of one cell-kernel launch: the input state and stage 2's A
// (box {TC, 1, NC} of the (x, row, comp) view), the three face buffers (box
// {XS | TC, 1, RW, nfp} of the (x, row, F|Ft x var, point) view)
struct CellMaps {
    CUtensorMap coef, A, fx, fy, fz;
};

// Persistent CTA over tiles of TC consecutive cells along x, software
// pipelined: while tile t is computed, the coefficients of tile t+grid and
// the face fluxes of tile t stream into shared memory — by TMA
// (KParams::cell_tma: one elected thread, mbarrier completion) or cp.async.
// Phase B: one (cell, volume point) item per thread -> smooth fluxes.
// Phase C: one (cell, var, F|Ft) item per thread -> face gather + volume
// projection + M^-1 (+ S2O4 combine); stage 1 then forms q* per coefficient
// from shared memory, stage 2 needs only Lt2.
template <int P, int DIM, bool VISC, int MODE>
__global__ void __launch_bounds__(CellTile<P, DIM, MODE>::NT, CellTile<P, DIM, MODE>::MINB)
    cell_kernel(KParams kp, const double* __restrict__ qin, const double* __restrict__ f0,
                const double* __restrict__ f1, const double* __restrict__ f2,
                const double* __restrict__ qn, const double* __restrict__ L1,
                const double* __restrict__ Lt1, double* __restrict__ out0,
                double* __restrict__ out1, double* __restrict__ out2, int tile_first,
                int tile_count, const __grid_constant__ CellMaps maps) {
    using SH = Shape<P, DIM>;
    using CT = CellTile<P, DIM, MODE>;
    constexpr int N = SH::N, NC = SH::NC, NVP = SH::NVP, TC = SH::TC, XS = CT::XS;
    constexpr int NT = CT::NT, NAX = SH::NAX;
    extern __shared__ __align__(128) double smem[];  // 128 B: TMA destinations
    double* coefb = smem;                 // [2][NC][TC]
    double* fx = coefb + 2 * CT::COEF;    // [pf][c][XS]
    double* fy = fx + CT::FX;             // [half][pf][c][TC]
    double* fz = fy + CT::FY;
    double* vf = fz + CT::FZ;             // [NVP][VFW][TC]
    double* lb = vf + CT::VF;             // [2][NC][TC]
    double* ab = lb + CT::LB;             // [NC][TC] stage 2: A of the tile
    double* geob = ab + CT::AB;           // [2][GEO], staged with the coefficients
    __shared__ uint64_t mb_c[2], mb_f;    // TMA: coefficient buffers, face group

    if (kp.scal[SC_ACTIVE] == 0.0) return;  // halted device loop: no-op step
    const double dt = kp.scal[SC_DT];
    const bool tma = kp.cell_tma != 0;
    constexpr int NITEMS = CT::NITEMS;
    const int tid = threadIdx.x;
    const int nx = kp.nx, ny = kp.ny;
    const int ntx = (nx + TC - 1) / TC;
    const int tile_end = tile_first + tile_count;
    const int step = kp.report ? tile_count : gridDim.x;

    using TI = TileWalk::TI;
    const TileWalk walk(ntx, ny, TC, step);
    // one [NC][TC] state tile (coefficients of TC cells) -> shared memory
    auto prefetch_state = [&](const double* __restrict__ base, const TI& ti, double* dst) {
        const long cbase = (long)(ti.k + 1) * kp.S + (long)ti.j * nx;
        if constexpr (NT % TC == 0) {
            // fixed column per thread, components strided by NT / TC
            constexpr int CST = NT / TC;
            const int l = tid % TC;
            const bool ok = ti.i0 + l < nx;
            const double* src = base + (long)(tid / TC) * kp.cs + cbase + (ok ? ti.i0 + l : 0);
            const long sst = CST * kp.cs;
#pragma unroll 4
            for (int comp = tid / TC; comp < NC; comp += CST, src += sst) cp_async8(dst + comp * TC + l, src, ok);
        } else {
            for (int e = tid; e < NC * TC; e += NT) {
                const int l = e % TC, comp = e / TC;
                const bool ok = ti.i0 + l < nx;
                cp_async8(dst + comp * TC + l, base + comp * kp.cs + cbase + (ok ? ti.i0 + l : 0), ok);
            }
        }
    };
    // the tile's widths (always cp.async, by TC + 4 threads)
    auto prefetch_geo = [&](const TI& ti, double* gdst) {
        if (tid < TC) {
            const bool ok = ti.i0 + tid < nx;
            const int i = ok ? ti.i0 + tid : 0;
            cp_async8(gdst + tid, kp.dx + i, ok);
            cp_async8(gdst + TC + tid, kp.i2dx + i, ok);
        } else if (tid < TC + 4) {
            const int r = tid - TC;
            const double* src = r == 0 ? kp.dy + ti.j : r == 1 ? kp.dz + ti.k + 1 : r == 2 ? kp.i2dy + ti.j
                                                                                          : kp.i2dz + ti.k + 1;
            cp_async8(gdst + 2 * TC + r, src, true);
        }
    };
    auto coef_tma = [&](const TI& ti, double* dst, uint64_t* bar) {
        mbar_expect_tx(bar, 8u * NC * TC);
        tma_load3(dst, &maps.coef, ti.i0, ti.j + ny * (ti.k + 1), 0, bar);
    };
    // stage 2 consumes only the Ft rows (the face pass stores only those)
    constexpr int RW = CT::RW, RO = CT::RO;
    auto face_rows = [&](const TI& ti, long& rowk, long& rowp, long& rowz, int& jp, int& kp1) {
        rowk = (long)nx * (ti.j + (long)ny * ti.k);
        jp = ti.j + 1 == ny ? 0 : ti.j + 1;
        rowp = (long)nx * (jp + (long)ny * ti.k);
        kp1 = (ti.k + 1 == kp.zface_layers && kp.z_wrap) ? 0 : ti.k + 1;
        rowz = (long)nx * (ti.j + (long)ny * kp1);
    };
    auto faces_tma = [&](const TI& ti) {
        long rowk, rowp, rowz;
        int jp, kp1;
        face_rows(ti, rowk, rowp, rowz, jp, kp1);
        mbar_expect_tx(&mb_f, CT::FACE_TX);
        const int r0 = ti.j + ny * ti.k;
        tma_load4(fx, &maps.fx, ti.i0, r0, RO, 0, &mb_f);
        tma_load4(fy, &maps.fy, ti.i0, r0, RO, 0, &mb_f);
        tma_load4(fy + CT::FYH, &maps.fy, ti.i0, jp + ny * ti.k, RO, 0, &mb_f);
        tma_load4(fz, &maps.fz, ti.i0, r0, RO, 0, &mb_f);
        tma_load4(fz + CT::FZH, &maps.fz, ti.i0, ti.j + ny * kp1, RO, 0, &mb_f);
        if (MODE == MODE_STAGE2) tma_load3(ab, &maps.A, ti.i0, ti.j + ny * (ti.k + 1), 0, &mb_f);
    };
    auto prefetch_faces = [&](const TI& ti) {
        if (MODE == MODE_STAGE2) prefetch_state(L1, ti, ab);
        const int i0 = ti.i0;
        long rowk, rowp, rowz;
        int jp, kp1;
        face_rows(ti, rowk, rowp, rowz, jp, kp1);
        if constexpr (2 * TC == 32) {
            // one face row per warp instruction: x rows hold TC+1 faces
            // (lanes 0..TC), y/z rows the TC faces of both neighbour rows
            constexpr int NW = NT / 32;
            const int lane = tid & 31, warp = tid >> 5;
            const int igx = i0 + lane;
            const bool okx = lane <= TC && igx <= nx;  // x is periodic: face nx is face 0
            const long ox = rowk + (okx ? (igx == nx ? 0 : igx) : 0);
            const int ig = i0 + (lane % TC);
            const bool ok = ig < nx;
            const int half = lane < TC ? 0 : 1;
            const long oy = (half ? rowp : rowk) + (ok ? ig : 0);
            const long oz = (half ? rowz : rowk) + (ok ? ig : 0);
            // a warp owns component rows c (F/Ft x var) and walks the face
            // points with constant strides: row pf*10 + RO + c
            const long pst = 10 * kp.fs;
            for (int c = warp; c < RW; c += NW) {
                const int r0 = RO + c;
                const double* sx = f0 + (long)r0 * kp.fs + ox;
                const double* sy = f1 + (long)r0 * kp.fs + oy;
                const double* sz = f2 + (long)r0 * kp.fs + oz;
#pragma unroll
                for (int pf = 0; pf < CT::NFX; ++pf)
                    if (lane <= TC) cp_async8(fx + (pf * RW + c) * XS + lane, sx + pf * pst, okx);
#pragma unroll
                for (int pf = 0; pf < CT::NFY; ++pf)
                    cp_async8(fy + half * CT::FYH + (pf * RW + c) * TC + lane % TC, sy + pf * pst, ok);
#pragma unroll
                for (int pf = 0; pf < CT::NFZ; ++pf)
                    cp_async8(fz + half * CT::FZH + (pf * RW + c) * TC + lane % TC, sz + pf * pst, ok);
            }
        } else {
            auto row_of = [](int rr) { return (rr / RW) * 10 + RO + rr % RW; };
            for (int e = tid; e < CT::NFX * RW * (TC + 1); e += NT) {  // x faces i0 .. i0+TC (periodic wrap at nx)
                const int l = e % (TC + 1), rr = e / (TC + 1);
                const int ig = i0 + l;
                const bool ok = ig <= nx;  // x is always periodic: face nx is face 0
                const int iw = ig == nx ? 0 : ig;
                cp_async8(fx + rr * XS + l, f0 + (long)row_of(rr) * kp.fs + rowk + (ok ? iw : 0), ok);
            }
            for (int e = tid; e < CT::NFY * RW * 2 * TC; e += NT) {  // y faces of rows j, j+1
                const int l = e % TC, rr = (e / TC) % (CT::NFY * RW), half = e / (TC * CT::NFY * RW);
                const int ig = i0 + l;
                const bool ok = ig < nx;
                cp_async8(fy + half * CT::FYH + rr * TC + l,
                          f1 + (long)row_of(rr) * kp.fs + (half ? rowp : rowk) + (ok ? ig : 0), ok);
            }
            for (int e = tid; e < CT::NFZ * RW * 2 * TC; e += NT) {  // z faces of layers k, k+1
                const int l = e % TC, rr = (e / TC) % (CT::NFZ * RW), half = e / (TC * CT::NFZ * RW);
                const int ig = i0 + l;
                const bool ok = ig < nx;
                cp_async8(fz + half * CT::FZH + rr * TC + l,
                          f2 + (long)row_of(rr) * kp.fs + (half ? rowz : rowk) + (ok ? ig : 0), ok);
            }
        }
    };
    const int t0 = tile_first + (kp.report ? 0 : blockIdx.x);
    TI cur = walk.of(t0);
    if (tma) {
        if (tid == 0) {
            mbar_init(&mb_c[0], 1);
            mbar_init(&mb_c[1], 1);
            mbar_init(&mb_f, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0 && t0 < tile_end) coef_tma(cur, coefb, &mb_c[0]);
    } else if (t0 < tile_end) {
        prefetch_state(qin, cur, coefb);
    }
    if (t0 < tile_end) prefetch_geo(cur, geob);
    cp_async_commit();
    int n = 0;
    for (int t = t0; t < tile_end; t += step, ++n) {
        double* sc = coefb + (n & 1) * CT::COEF;
        const bool has_next = t + step < tile_end;
        const TI nxt = walk.next(cur);
        const int i0 = cur.i0, j = cur.j, k = cur.k;
        const long cbase = (long)(k + 1) * kp.S + (long)j * nx;
        const double* gg = geob + (n & 1) * CT::GEO;
        const long cglob_row = (long)nx * (j + (long)ny * (k + kp.kglob0));
        race_shake(kp, 2, n);
        // this tile's coefficients and widths (issued a tile ahead)
        if (tma) mbar_wait(&mb_c[n & 1], (n >> 1) & 1);
        cp_async_wait<0>();
        __syncthreads();
        // every buffer the previous tile read is free: the tile's faces (+
        // stage 2's A), then the next tile's coefficients and widths
        if (tma) {
            if (tid == 0) {
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                if (!kp.report) faces_tma(cur);
                if (has_next) coef_tma(nxt, coefb + ((n + 1) & 1) * CT::COEF, &mb_c[(n + 1) & 1]);
            }
        } else {
            if (!kp.report) prefetch_faces(cur);
            cp_async_commit();
            if (has_next) prefetch_state(qin, nxt, coefb + ((n + 1) & 1) * CT::COEF);
        }
        if (has_next) prefetch_geo(nxt, geob + ((n + 1) & 1) * CT::GEO);
        cp_async_commit();
        const double hy = gg[2 * TC], hz = gg[2 * TC + 1];
        const double i2hy = gg[2 * TC + 2], i2hz = gg[2 * TC + 3];

        // periodic x: the face at x = nx is face 0 (TMA has no wrap; that
        // column arrived zero-filled), patched by threads [t0, t0 + nthr)
        auto patch_x = [&](int t0p, int nthr) {
            if (i0 + TC >= nx) {
                const long rowk = (long)nx * (j + (long)ny * k);
                for (int e = tid - t0p; e < CT::NFX * RW; e += nthr) {
                    const int r0 = (e / RW) * 10 + RO + e % RW;
                    fx[e * XS + (nx - i0)] = f0[(long)r0 * kp.fs + rowk];
                }
            }
        };
        // face part of projection item it (dg.hpp:404-425): + w jac B- F(minus
        // face) - w jac B+ F(plus face), Legendre parity B+(p,n) = (-1)^{n_a} B-(p,n)
        auto face_part = [&](int it, double* R, auto M0c, auto M1c) {
            constexpr int M0 = decltype(M0c)::value, M1 = decltype(M1c)::value;
            int l, v, ft;
            if (CT::S1X) {
                ft = it & 1;
                l = (it >> 1) % TC;
                v = (it >> 1) / TC;
            } else {
                l = it % TC;
                v = (it / TC) % 5;
                ft = (MODE == MODE_STAGE2 ? 1 : 0) + (it / TC) / 5;
            }
            const int row = 5 * ft + v;
            const double hx = gg[l];
            const double jac[3] = {hy * hz * 0.25, hz * hx * 0.25, hx * hy * 0.25};
#pragma unroll
            for (int m = M0; m < M1; ++m) R[m] = 0.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int nfp = a == 0 ? CT::NFX : a == 1 ? CT::NFY : CT::NFZ;
                double acc[N];
#pragma unroll
                for (int m = M0; m < M1; ++m) acc[m] = 0.0;
#pragma unroll
                for (int pf = 0; pf < nfp; ++pf) {
                    const int r = pf * RW + row - RO;
                    double Fm, Fp;
                    if (a == 0) {
                        Fm = fx[r * XS + l];
                        Fp = fx[r * XS + l + 1];
                    } else {
                        const double* fa = a == 1 ? fy : fz;
                        const int hh = a == 1 ? CT::FYH : CT::FZH;
                        Fm = fa[r * TC + l];
                        Fp = fa[hh + r * TC + l];
                    }
                    const double Dm = Fm - Fp, Sm = Fm + Fp;
#pragma unroll
                    for (int m = M0; m < M1; ++m) {
                        const double c = ctab<P, DIM>.fw[a][pf] * ctab<P, DIM>.fB[a][0][pf][m];
                        const bool odd = ctab<P, DIM>.par[a][m] != 0;
                        if (c != 0.0) acc[m] += c * (odd ? Sm : Dm);
                    }
                }
#pragma unroll
                for (int m = M0; m < M1; ++m) R[m] += jac[a] * acc[m];
            }
        };

        // ---- phase B: smooth fluxes at volume points
        for (int it = tid; it < TC * NVP; it += NT) {
            const int l = it % TC;
            const int p = SH::NQ == 2 ? it / TC : kVolOrder<P, DIM>.p[it / TC];
            const int i = i0 + l;
            if (i >= nx) continue;
            const double i2h[3] = {gg[TC + l], i2hy, i2hz};
            double e[20];
            vol_eval_sym<P, DIM, TC>(p, sc + l, i2h, e);
            double o[30];
            double bad = 0.0;
            const int rc = smooth_flux<VISC, NAX, MODE == MODE_STAGE2>(e, kp.gas, o, bad);
            if (rc) {
                report_error(kp, err_key(kp.stage, 1, cglob_row + i, p, 0, rc), bad);
#pragma unroll
                for (int m = 0; m < 30; ++m) o[m] = 0.0;
            }
#pragma unroll
            for (int m = 0; m < 10 * NAX; ++m)
                if (m % 10 >= RO) vf[(p * CT::VFW + (m / 10) * RW + m % 10 - RO) * TC + l] = o[m];
        }
        if (kp.report) return;
        race_shake(kp, 3, n);
        // this tile's face fluxes (+ stage 2's A tile)
        if (tma) {
            mbar_wait(&mb_f, n & 1);
            patch_x(0, NT);
        } else {
            cp_async_wait<1>();
        }
        __syncthreads();

        // ---- phase C: gather + projection + inverse mass (+ stage-2 combine)
        constexpr int FT0 = MODE == MODE_STAGE2 ? 1 : 0;
        // one projection item restricted to the basis functions [M0, M1)
        // (compile-time range: the table zeros stay folded)
        auto item_range = [&](int it, auto M0c, auto M1c) {
            constexpr int M0 = decltype(M0c)::value, M1 = decltype(M1c)::value;
            int l, v, ft;  // ft: 0 -> F (R), 1 -> Ft (Rt)
            if (CT::S1X) {  // F / Ft of a (cell, var) in adjacent lanes
                ft = it & 1;
                l = (it >> 1) % TC;
                v = (it >> 1) / TC;
            } else {
                l = it % TC;
                v = (it / TC) % 5;
                ft = FT0 + (it / TC) / 5;
            }
            const int i = i0 + l;
            if (!CT::S1X && i >= nx) return;  // (S1X: every lane joins the shuffle; stores are predicated)
            const double hx = gg[l];
            const double i2h[3] = {gg[TC + l], i2hy, i2hz};
            const int row = 5 * ft + v;
            double R[N];
            face_part(it, R, M0c, M1c);
            // volume (dg.hpp:427-448): + w (h0 h1 h2 / 8) (2/h_a) dB_a F_a
            const double vol = hx * hy * hz;
            const double vjac = vol * 0.125;
#pragma unroll
            for (int a = 0; a < NAX; ++a) {
                double acc[N];
#pragma unroll
                for (int m = M0; m < M1; ++m) acc[m] = 0.0;
#pragma unroll
                for (int p = 0; p < NVP; ++p) {
                    const double F = vf[(p * CT::VFW + a * RW + row - RO) * TC + l];
#pragma unroll
                    for (int m = M0; m < M1; ++m) {
                        const double c = ctab<P, DIM>.vw[p] * ctab<P, DIM>.vdB[p][a][m];
                        if (c != 0.0) acc[m] += c * F;
                    }
                }
                const double sa = vjac * i2h[a];
#pragma unroll
                for (int m = M0; m < M1; ++m) R[m] += sa * acc[m];
            }
            const long g0 = (long)v * kp.cs + cbase + i;
            if (MODE == MODE_RESIDUAL) {
                double* o = ft ? out1 : out0;
#pragma unroll
                for (int m = M0; m < M1; ++m) o[g0 + (long)(m * 5) * kp.cs] = R[m];
                return;
            }
            // mass_diag (dg.hpp:42-50): 1/M_n = (2nx+1)(2ny+1)(2nz+1)/vol (solver.hpp:49-51)
            const double ivol = 1.0 / vol;
            const double c6 = dt * dt / 6.0;
            if (CT::S1X) {
                // the partner lane holds the other of (L1, Lt1):
                //   q* = q + dt/2 L1 + dt^2/8 Lt1 (F lane -> out0)
                //   A  = q + (dt L1 + dt^2/6 Lt1)  (Ft lane -> out1)
                const bool valid = i < nx;
#pragma unroll
                for (int m = M0; m < M1; ++m) {
                    const double L = R[m] * (ctab<P, DIM>.massf[m] * ivol);
                    const double Lo = __shfl_xor_sync(0xffffffffu, L, 1);
                    const double q = sc[(m * 5 + v) * TC + l];
                    const long gi = g0 + (long)(m * 5) * kp.cs;
                    if (valid) {
                        if (ft) out1[gi] = q + (dt * Lo + c6 * L);
                        else out0[gi] = q + 0.5 * dt * L + 0.125 * dt * dt * Lo;
                    }
                }
                return;
            }
#pragma unroll
            for (int m = M0; m < M1; ++m) {
                const double L = R[m] * (ctab<P, DIM>.massf[m] * ivol);
                const long gi = g0 + (long)(m * 5) * kp.cs;
                if (MODE == MODE_STAGE1) {
                    lb[(ft * NC + m * 5 + v) * TC + l] = L;
                } else {
                    // q^{n+1} = q + dt L1 + dt^2/6 (Lt1 + 2 Lt2) (integrator.hpp:72-74)
                    // = A + dt^2/6 * 2 Lt2, A formed by stage 1
                    out0[gi] = ab[(m * 5 + v) * TC + l] + c6 * (2.0 * L);
                }
            }
        };
        // (S1X: 160 items on 128 threads, warp 0 takes the last 32; splitting
        // those 32 by basis range over the four warps measured slower:
        // stage 1 2.36 vs 2.22 ms)
        if constexpr (CT::SPLIT) {
            // P3 stage 2: 40 items would leave most of the 7 warps idle; each
            // item is split into two basis ranges [0, N/2) and [N/2, N), one
            // per warp of a pair, so a warp's lanes share one range
            const int w = tid >> 5, lane = tid & 31;
            for (int base = (w >> 1) * 32; base < NITEMS; base += (NT / 64) * 32) {
                const int it = base + lane;
                if (it >= NITEMS || w >= (NT / 64) * 2) continue;
                if (w & 1) item_range(it, IC<N / 2>{}, IC<N>{});
                else item_range(it, IC<0>{}, IC<N / 2>{});
            }
        } else {
            for (int it = tid; it < NITEMS; it += NT) item_range(it, IC<0>{}, IC<N>{});
        }
        if (MODE == MODE_STAGE1 && !CT::S1X) {
            // from shared memory, per coefficient (integrator.hpp:69-74):
            //   q* = q + dt/2 L1 + dt^2/8 Lt1           -> out0
            //   A  = q + (dt L1 + dt^2/6 Lt1)           -> out1 (stage 2 adds dt^2/6 * 2 Lt2)
            race_shake(kp, 4, n);
            __syncthreads();
            const double c6 = dt * dt / 6.0;
            // unrolled with predicated stores: all shared-memory loads of the
            // thread's elements issue before the first use
#pragma unroll
            for (int e = tid; e < NC * TC; e += NT) {
                const int l = e % TC, comp = e / TC;
                const double q = sc[comp * TC + l], L = lb[comp * TC + l], Lt = lb[(NC + comp) * TC + l];
                const long gi = comp * kp.cs + cbase + i0 + l;
                if (i0 + l < nx) {
                    out0[gi] = q + 0.5 * dt * L + 0.125 * dt * dt * Lt;
                    out1[gi] = q + (dt * L + c6 * Lt);
                }
            }
        }
        cur = nxt;
    }
    cp_async_wait<0>();
}

}  // namespace hgks_dev
