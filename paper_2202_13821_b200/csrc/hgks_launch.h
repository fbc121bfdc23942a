// Kernel-set dispatch shared by the C-ABI and the per-(degree, dim)
// instantiation units (hgks_instances.cu).
#pragma once

#include <cuda_runtime.h>

#include "hgks_kernels.cuh"

namespace hgks_dev {

struct KernelSet {
    // qmap: the two TMA tensor maps of q (x, row, comp) — box {32, 1, NC} for
    // the y / z faces, {34, 1, NC} for the x faces — or null (cp.async staging)
    void (*face)(const KParams&, const double* q, const CUtensorMap* qmap, double* const f[3], cudaStream_t,
                 int report, const int* tile);
    // cm: the launch's TMA tensor maps (KParams::cell_tma) or null
    void (*cell)(const KParams&, const CellMaps* cm, int mode, const double* qin, double* const f[3],
                 const double* qn, const double* L1, const double* Lt1, double* o0, double* o1, double* o2,
                 cudaStream_t, int report, const int* tile);
    // the same kernels restricted to owned z layers [kb, ke) (all three face
    // axes / the cell update of those layers), for the streamed host step
    void (*face_layers)(const KParams&, const double* q, const CUtensorMap* qmap, double* const f[3],
                        cudaStream_t, int kb, int ke);
    // one face axis over z layers [kb, ke) (z: up to zface_layers), for the
    // multi-slab step that overlaps the halo exchange with interior faces
    void (*face_axis)(const KParams&, int axis, const double* q, const CUtensorMap* qmap, double* f,
                      cudaStream_t, int kb, int ke);
    void (*cell_layers)(const KParams&, const CellMaps* cm, int mode, const double* qin, double* const f[3],
                        const double* qn, const double* L1, const double* Lt1, double* o0,
                        double* o1, double* o2, cudaStream_t, int kb, int ke);
    int face_tma;  // 1: the face kernels can stage by TMA (given qmap)
    int cell_xs;   // x-face box width of the cell kernel (TC + 2)
    int face_smem[3];
    int cell_smem;
    int cell_tc;
    int nfp[3];
};

// one per instantiated (degree, dim): configures shared memory and fills ks
bool pick_kernels(int degree, int dim, bool visc, KernelSet& ks, cudaError_t& err);

#define HGKS_DECLARE_PICK(P, D) \
    bool pick_##P##_##D(bool visc, KernelSet& ks, cudaError_t& err);
HGKS_DECLARE_PICK(1, 3)
HGKS_DECLARE_PICK(2, 3)
HGKS_DECLARE_PICK(3, 3)
HGKS_DECLARE_PICK(2, 2)
HGKS_DECLARE_PICK(3, 2)

}  // namespace hgks_dev
