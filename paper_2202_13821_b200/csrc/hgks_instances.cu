// Explicit kernel instantiation unit: one translation unit per
// (degree, dim) family (HGKS_INST_P, HGKS_INST_DIM), compiled in parallel by
// build.py. Each exports pick_<P>_<DIM>() for the dispatcher in hgks_capi.cu.
#include <algorithm>

#include "hgks_launch.h"

#ifndef HGKS_INST_P
#define HGKS_INST_P 2
#define HGKS_INST_DIM 3
#endif

namespace hgks_dev {
namespace {

// kernel argument when no tensor map is needed (cp.async staging)
inline const CUtensorMap& map_or_null(const CUtensorMap* m) {
    static const CUtensorMap zero{};
    return m ? *m : zero;
}

inline const CellMaps& cmaps_or_null(const CellMaps* m) {
    static const CellMaps zero{};
    return m ? *m : zero;
}

// persistent grid size: resident CTAs on the GPU, optionally capped
// (KParams::grid_cap, a test hook that makes every CTA walk many tiles)
inline int capped(const KParams& kp, int g) {
    g = std::max(1, g);
    return kp.grid_cap > 0 ? std::min(g, kp.grid_cap) : g;
}

template <int P, int DIM, bool VISC>
struct Launch {
    using SH = Shape<P, DIM>;
    template <int AXIS = 2>
    static int face_smem() {
        // staged coefficients of both neighbours (double-buffered by default)
        // [+ the flux accumulators when they live in shared memory]
        return (HGKS_FACE_STAGES * FaceStage<SH::NC, AXIS>::STG +
                (HGKS_FACE_ACC_SMEM ? 35 * FaceCTA<P, DIM, AXIS>::NT : 0)) *
               (int)sizeof(double);
    }
    // persistent face kernels: resident CTAs on the whole GPU per axis
    static inline int face_grid[3] = {0, 0, 0};
    template <int MODE = MODE_STAGE1>
    static int cell_smem() { return CellTile<P, DIM, MODE>::SMEM * (int)sizeof(double); }
    // persistent cell kernel: resident CTAs on the whole GPU (set by configure)
    static inline int cell_grid[3] = {0, 0, 0};

    template <int AXIS>
    static void face_axis(const KParams& kp, const double* q, const CUtensorMap* qm, double* f, cudaStream_t st,
                          int report, const int* tile) {
        const int layers = AXIS == 2 ? kp.zface_layers : kp.nzl;
        int t[3] = {0, 0, 0};
        if (report) {
            t[0] = tile[0];
            t[1] = tile[1];
            t[2] = tile[2];
        }
        constexpr int NFP = SH::template nfp<AXIS>();
        const int ntx = (kp.nx + 31) / 32;
        const int ntiles = ntx * kp.ny * layers;
        int first = 0, count = ntiles;
        int grid = std::min(ntiles, capped(kp, face_grid[AXIS]));
        if (report) {  // the failing face's tile only
            first = t[0] + ntx * (t[1] + kp.ny * t[2]);
            count = 1;
            grid = 1;
        }
        (void)NFP;
        launch_face<AXIS>(kp, grid, q, qm, f, first, count, st);
    }
    // stage-2 passes (kp.ft_only) run the Ft-only instantiation
    template <int AXIS>
    static void launch_face(const KParams& kp, int grid, const double* q, const CUtensorMap* qm, double* f,
                            int first, int count, cudaStream_t st) {
        const CUtensorMap m = map_or_null(qm ? qm + (AXIS == 0 ? 1 : 0) : nullptr);
        if (kp.ft_only)
            face_kernel<P, DIM, VISC, AXIS, true><<<grid, FaceCTA<P, DIM, AXIS>::NT, face_smem<AXIS>(), st>>>(
                kp, q, f, first, count, m);
        else
            face_kernel<P, DIM, VISC, AXIS, false><<<grid, FaceCTA<P, DIM, AXIS>::NT, face_smem<AXIS>(), st>>>(
                kp, q, f, first, count, m);
    }
    template <int AXIS>
    static void face_axis_layers(const KParams& kp, const double* q, const CUtensorMap* qm, double* f,
                                 cudaStream_t st, int kb, int ke) {
        const int ntx = (kp.nx + 31) / 32;
        const int first = ntx * kp.ny * kb, count = ntx * kp.ny * (ke - kb);
        if (count <= 0) return;
        const int grid = std::min(count, capped(kp, face_grid[AXIS]));
        launch_face<AXIS>(kp, grid, q, qm, f, first, count, st);
    }
    static void face_axis_range(const KParams& kp, int axis, const double* q, const CUtensorMap* qm, double* f,
                                cudaStream_t st, int kb, int ke) {
        if (axis == 0) face_axis_layers<0>(kp, q, qm, f, st, kb, ke);
        else if (axis == 1) face_axis_layers<1>(kp, q, qm, f, st, kb, ke);
        else face_axis_layers<2>(kp, q, qm, f, st, kb, ke);
    }
    static void face_layers(const KParams& kp, const double* q, const CUtensorMap* qm, double* const f[3],
                            cudaStream_t st, int kb, int ke) {
        face_axis_layers<0>(kp, q, qm, f[0], st, kb, ke);
        face_axis_layers<1>(kp, q, qm, f[1], st, kb, ke);
        face_axis_layers<2>(kp, q, qm, f[2], st, kb, ke);
    }
    static void cell_layers(const KParams& kp, const CellMaps* cm, int mode, const double* qin, double* const f[3],
                            const double* qn, const double* L1, const double* Lt1, double* o0,
                            double* o1, double* o2, cudaStream_t st, int kb, int ke) {
        const int ntx = (kp.nx + SH::TC - 1) / SH::TC;
        const int first = ntx * kp.ny * kb, count = ntx * kp.ny * (ke - kb);
        if (count <= 0) return;
        const int grid = std::min(count, capped(kp, cell_grid[mode]));
        if (mode == MODE_STAGE1)
            cell_kernel<P, DIM, VISC, MODE_STAGE1><<<grid, CellTile<P, DIM, MODE_STAGE1>::NT,
                                                     cell_smem<MODE_STAGE1>(), st>>>(
                kp, qin, f[0], f[1], f[2], qn, L1, Lt1, o0, o1, o2, first, count, cmaps_or_null(cm));
        else
            cell_kernel<P, DIM, VISC, MODE_STAGE2><<<grid, CellTile<P, DIM, MODE_STAGE2>::NT,
                                                     cell_smem<MODE_STAGE2>(), st>>>(
                kp, qin, f[0], f[1], f[2], qn, L1, Lt1, o0, o1, o2, first, count, cmaps_or_null(cm));
    }
    static void face(const KParams& kp, const double* q, const CUtensorMap* qm, double* const f[3], cudaStream_t st,
                     int report, const int* tile) {
        // report mode re-runs only the failing axis' tile (tile[3] = axis)
        if (!report || tile[3] == 0) face_axis<0>(kp, q, qm, f[0], st, report, tile);
        if (!report || tile[3] == 1) face_axis<1>(kp, q, qm, f[1], st, report, tile);
        if (!report || tile[3] == 2) face_axis<2>(kp, q, qm, f[2], st, report, tile);
    }
    static void cell(const KParams& kp, const CellMaps* cm, int mode, const double* qin, double* const f[3],
                     const double* qn, const double* L1, const double* Lt1, double* o0, double* o1,
                     double* o2, cudaStream_t st, int report, const int* tile) {
        const int ntx = (kp.nx + SH::TC - 1) / SH::TC;
        const int ntiles = ntx * kp.ny * kp.nzl;
        int first = 0, count = ntiles;
        int grid = std::min(ntiles, capped(kp, cell_grid[mode]));
        if (report) {  // the failing cell's tile only
            first = tile[0] + ntx * (tile[1] + kp.ny * tile[2]);
            count = 1;
            grid = 1;
        }
        if (mode == MODE_RESIDUAL)
            cell_kernel<P, DIM, VISC, MODE_RESIDUAL><<<grid, CellTile<P, DIM, MODE_RESIDUAL>::NT,
                                                       cell_smem<MODE_RESIDUAL>(), st>>>(
                kp, qin, f[0], f[1], f[2], qn, L1, Lt1, o0, o1, o2, first, count, cmaps_or_null(cm));
        else if (mode == MODE_STAGE1)
            cell_kernel<P, DIM, VISC, MODE_STAGE1><<<grid, CellTile<P, DIM, MODE_STAGE1>::NT,
                                                     cell_smem<MODE_STAGE1>(), st>>>(
                kp, qin, f[0], f[1], f[2], qn, L1, Lt1, o0, o1, o2, first, count, cmaps_or_null(cm));
        else
            cell_kernel<P, DIM, VISC, MODE_STAGE2><<<grid, CellTile<P, DIM, MODE_STAGE2>::NT,
                                                     cell_smem<MODE_STAGE2>(), st>>>(
                kp, qin, f[0], f[1], f[2], qn, L1, Lt1, o0, o1, o2, first, count, cmaps_or_null(cm));
    }
    static cudaError_t configure() {
        cudaError_t e = cudaSuccess;
        auto set = [&](const void* fn, int bytes) {
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        };
        set((const void*)face_kernel<P, DIM, VISC, 0>, face_smem<0>());
        set((const void*)face_kernel<P, DIM, VISC, 1>, face_smem<1>());
        set((const void*)face_kernel<P, DIM, VISC, 2>, face_smem<2>());
        set((const void*)face_kernel<P, DIM, VISC, 0, true>, face_smem<0>());
        set((const void*)face_kernel<P, DIM, VISC, 1, true>, face_smem<1>());
        set((const void*)face_kernel<P, DIM, VISC, 2, true>, face_smem<2>());
        set((const void*)cell_kernel<P, DIM, VISC, MODE_RESIDUAL>, cell_smem<MODE_RESIDUAL>());
        set((const void*)cell_kernel<P, DIM, VISC, MODE_STAGE1>, cell_smem<MODE_STAGE1>());
        set((const void*)cell_kernel<P, DIM, VISC, MODE_STAGE2>, cell_smem<MODE_STAGE2>());
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0;
        e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const void* fns[3] = {(const void*)cell_kernel<P, DIM, VISC, MODE_RESIDUAL>,
                              (const void*)cell_kernel<P, DIM, VISC, MODE_STAGE1>,
                              (const void*)cell_kernel<P, DIM, VISC, MODE_STAGE2>};
        for (int m = 0; m < 3 && e == cudaSuccess; ++m) {
            int nb = 0;
            const int nts[3] = {CellTile<P, DIM, MODE_RESIDUAL>::NT, CellTile<P, DIM, MODE_STAGE1>::NT,
                                CellTile<P, DIM, MODE_STAGE2>::NT};
            const int shm[3] = {cell_smem<MODE_RESIDUAL>(), cell_smem<MODE_STAGE1>(), cell_smem<MODE_STAGE2>()};
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fns[m], nts[m], shm[m]);
            cell_grid[m] = std::max(1, nb) * sms;
        }
        const void* ffn[3] = {(const void*)face_kernel<P, DIM, VISC, 0>,
                              (const void*)face_kernel<P, DIM, VISC, 1>,
                              (const void*)face_kernel<P, DIM, VISC, 2>};
        const int fnt[3] = {FaceCTA<P, DIM, 0>::NT, FaceCTA<P, DIM, 1>::NT, FaceCTA<P, DIM, 2>::NT};
        const int fsm[3] = {face_smem<0>(), face_smem<1>(), face_smem<2>()};
        for (int a = 0; a < 3 && e == cudaSuccess; ++a) {
            int nb = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, ffn[a], fnt[a], fsm[a]);
            face_grid[a] = std::max(1, nb) * sms;
        }
        return e;
    }
    static KernelSet set() {
        KernelSet k;
        k.face = &face;
        k.cell = &cell;
        k.face_layers = &face_layers;
        k.face_axis = &face_axis_range;
        k.cell_layers = &cell_layers;
        k.face_smem[0] = face_smem<0>();
        k.face_smem[1] = face_smem<1>();
        k.face_smem[2] = face_smem<2>();
        k.cell_smem = cell_smem();
        k.cell_tc = SH::TC;
        k.face_tma = HGKS_FACE_STAGES == 2;  // the TMA path needs the double-buffered stage
        k.cell_xs = CellTile<P, DIM, MODE_STAGE1>::XS;
        k.nfp[0] = SH::template nfp<0>();
        k.nfp[1] = SH::template nfp<1>();
        k.nfp[2] = SH::template nfp<2>();
        return k;
    }
};

}  // namespace

#define HGKS_CAT(a, b, c) a##_##b##_##c
#define HGKS_PICKNAME(P, D) HGKS_CAT(pick, P, D)

bool HGKS_PICKNAME(HGKS_INST_P, HGKS_INST_DIM)(bool visc, KernelSet& ks, cudaError_t& err) {
    if (visc) {
        err = Launch<HGKS_INST_P, HGKS_INST_DIM, true>::configure();
        ks = Launch<HGKS_INST_P, HGKS_INST_DIM, true>::set();
    } else {
        err = Launch<HGKS_INST_P, HGKS_INST_DIM, false>::configure();
        ks = Launch<HGKS_INST_P, HGKS_INST_DIM, false>::set();
    }
    return true;
}

}  // namespace hgks_dev
