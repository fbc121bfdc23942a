/* hgks_b200 — C ABI of the B200-native DG-HGKS time step.
 *
 * The drop-in boundary: plain pointers and sizes, no torch or CUDA types.
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/hgks/). The C++ host
 * header include/hgks_b200/hgks.hpp wraps these in the reference's own
 * hgks:: names and exception types; INTEGRATION.md shows the bindings.
 *
 * Host layouts are the reference's: coefficients AoS [(cell*N + n)*5 + var]
 * (dg.hpp:15-17, cell = i + nx*(j + ny*k), mesh.hpp:34); face buffers
 * [face*(npts*10) + p*10 + (F|Ft)] (dg.hpp:287). The device keeps SoA
 * [n*5+var][cell] with one ghost cell layer above and below in z.
 *
 * Return codes: HGKS_OK, or
 *   HGKS_ERR_STATE   invalid_state_error: non-positive density / pressure
 *                    (core.hpp:58-70), message "item <i>: non-positive ..."
 *                    exactly as worker_error shapes it (runtime.hpp:37-41)
 *   HGKS_ERR_CONFIG  std::invalid_argument-class configuration error
 *   HGKS_ERR_DT      non_positive_dt (integrator.hpp:17-19, :43)
 *   HGKS_ERR_CUDA    CUDA runtime failure (no CPU fallback exists)
 * hgks_last_error() returns the message of the most recent failure.
 */
#ifndef HGKS_B200_H
#define HGKS_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define HGKS_OK 0
#define HGKS_ERR_STATE 1
#define HGKS_ERR_CONFIG 2
#define HGKS_ERR_DT 3
#define HGKS_ERR_CUDA 4

#define HGKS_ABI_VERSION 2

typedef struct hgks_solver hgks_solver;

/* Mesh + Scheme (mesh.hpp:11-30, dg.hpp:269-281, core.hpp:35-42). */
typedef struct {
    int nx, ny, nz;                  /* global cells per axis */
    const double* xs;                /* nx+1 node coordinates, strictly increasing */
    const double* ys;                /* ny+1 */
    const double* zs;                /* nz+1 */
    int degree;                      /* 2 or 3 (reference); 1 = P1 extension */
    int dim;                         /* 3 (2 = degenerate 2D mode, nz must be 1) */
    double gamma;                    /* GasModel::make gamma */
    double mu;                       /* mu_ref = 1/Re; 0 selects the Euler (tau = 0) limit */
    int device;                      /* CUDA device ordinal */
    int z_begin, z_count;            /* owned z-slab [z_begin, z_begin+z_count); z_count<=0: all */
} hgks_config;

int hgks_abi_version(void);

/* Creates the solver on cfg->device. Scheme::make + ResidualWorkspace::resize
 * + TwoStageScratch in one object (dg.hpp:274, :294; integrator.hpp:50). */
int hgks_create(const hgks_config* cfg, hgks_solver** out);
void hgks_destroy(hgks_solver* s);
const char* hgks_last_error(const hgks_solver* s);
/* structured form of the last failure: code, phase (0 face, 1 cell, 2 dt),
 * reference item index, offending value */
void hgks_error_info(const hgks_solver* s, int* code, int* phase, long* item, double* value);

int hgks_num_basis(const hgks_solver* s);      /* BasisSet::N (basis.hpp:64-82) */
long hgks_num_coeffs(const hgks_solver* s);    /* owned cells * N * 5 */
int hgks_face_points(const hgks_solver* s, int axis); /* face_minus[axis].npts */

/* DGState coefficients (dg.hpp:18-38) of the owned cells, host AoS. */
int hgks_set_state(hgks_solver* s, const double* coeffs, double time);
int hgks_get_state(hgks_solver* s, double* coeffs, double* time);

/* residual(coeffs, mesh, scheme, dt, ws) (dg.hpp:354-450): R, Rt as ws.R /
 * ws.Rt; face0..2 (optional, may be NULL) as ws.face[a]. coeffs may be NULL
 * to use the current state. */
int hgks_residual(hgks_solver* s, const double* coeffs, double dt, double* R, double* Rt,
                  double* face0, double* face1, double* face2);

/* detail::apply_inverse_mass(R, L, mesh, basis, part) (solver.hpp:42-54) */
int hgks_apply_inverse_mass(hgks_solver* s, const double* R, double* L);

/* compute_dt(state, mesh, gas, ctrl, degree) (integrator.hpp:27-45) on the
 * current state, ctrl.cfl = cfl. */
int hgks_compute_dt(hgks_solver* s, double cfl, double* dt);
/* the same with the degree of the viscous bound given explicitly (the
 * reference's compute_dt takes it as an argument, independent of the state's
 * basis: integrator.hpp:27, :40) */
int hgks_compute_dt_k(hgks_solver* s, double cfl, int degree, double* dt);

/* two_stage_step(q, dt, eval, scratch) (integrator.hpp:64-75) with the eval
 * of solver.hpp:81-88 (residual + inverse mass, the same full dt in both
 * stages), applied to the device-resident state; state time += dt.
 * On failure the state is left unchanged. */
int hgks_step(hgks_solver* s, double dt);

/* The same step on a caller-owned host vector q (AoS, hgks_num_coeffs):
 * host->device, step, device->host. The literal drop-in for
 * two_stage_step(r.state.coeffs, dt, eval, scratch). */
int hgks_two_stage_step_host(hgks_solver* s, double* q, double dt);

/* The same step with the host<->device traffic streamed: the z range is cut
 * into `nchunks` slabs (<= 0: automatic, ~2.7 z layers each, at most 48)
 * whose uploads, face/cell kernels (a z-wavefront) and
 * downloads overlap on three streams. Results are bitwise identical to
 * hgks_two_stage_step_host; on a state error q is restored to q^n (the
 * reference's two_stage_step leaves q untouched). Single slab only;
 * otherwise it falls back to hgks_two_stage_step_host. */
int hgks_two_stage_step_host_streamed(hgks_solver* s, double* q, double dt, int nchunks);

/* advance() (solver.hpp:62-108), device-resident: steps from the current
 * time to t_end with dt = compute_dt(cfl) or dt_fixed (> 0), clipped to t_end
 * and, when record_interval > 0, to the next record time (the first one is
 * first_record; the reference starts at record_interval). dt, the clipping,
 * the t update and the failure checks run on the device (CUDA graph per
 * step, no host round trip between steps); max_steps > 0 stops after that
 * many steps. After every step that lands on a record time, on_record(user,
 * s, t) is called with the solver showing that step's state (get_state,
 * tgv_diagnostics, error_norms read it; the callback must not step s).
 * State errors get " at t=<t>" appended (the failing step's start time);
 * compute_dt failures are the bare error, as in the reference. On failure the
 * state is q^n of the failing step. Writes the number of steps taken. */
typedef int (*hgks_record_fn)(void* user, hgks_solver* s, double t);
int hgks_advance_records(hgks_solver* s, double t_end, double cfl, double dt_fixed,
                         double record_interval, double first_record, int max_steps,
                         hgks_record_fn on_record, void* user, int* steps);
/* the same without records: first_record = the next multiple of
 * record_interval after the current time */
int hgks_advance(hgks_solver* s, double t_end, double cfl, double dt_fixed,
                 double record_interval, int* steps);

/* ResidualWorkspace::count_fluxes debug tally (dg.hpp:291-292, :393): counts
 * owned face-point flux evaluations. */
void hgks_set_count_fluxes(hgks_solver* s, int on);
long hgks_flux_evaluations(const hgks_solver* s);

/* project(initial_field(cfg)) (dg.hpp:193-220, cases.hpp:127-137) on the
 * device: case_name adv2d | adv3d | vortex2d | tgv (gamma 1.4, Ma 0.1,
 * eps 5 as CaseConfig::named, cases.hpp:12-46); exact field at time t. */
int hgks_project_case(hgks_solver* s, const char* case_name, double t);

/* tgv_diagnostics (cases.hpp:165-204) of the current state: Ek, epsZeta
 * (fixed-order device reduction; sums over owned cells only). */
int hgks_tgv_diagnostics(hgks_solver* s, double* ek_vol, double* ens_vol, double* volume);

/* error_norms (dg.hpp:228-266) of the current state against the named case's
 * exact field at time t, as UNREDUCED sums over owned cells: out[0] = L1,
 * out[1] = L2^2, out[2] = cell-average error^2 (ErrorNorms = {out0,
 * sqrt(out1), sqrt(out2)} after summing over slabs). */
int hgks_error_norms(hgks_solver* s, const char* case_name, double t, double* out);

/* project(field, mesh, tab, part) (dg.hpp:193-220) for a caller-supplied
 * field: samples[(cell*npts + p)*5 + var] are the field's conserved values at
 * the projection points of the owned cells, x = center + h/2 * ref_p with the
 * (k+2)^dim Gauss points in the reference's order (dg.hpp:102-105); the
 * weighted sums run on the device. npts = hgks_projection_npts. */
int hgks_projection_npts(const hgks_solver* s);
int hgks_project_samples(hgks_solver* s, const double* samples, double t);
/* error_norms(state, mesh, tab, exact, part) (dg.hpp:228-266) for a
 * caller-supplied exact field: rho_exact[cell*npts + p] at the projection
 * points; out as hgks_error_norms (unreduced sums). */
int hgks_error_norms_samples(hgks_solver* s, const double* rho_exact, double* out);

/* ---- multi-GPU z-slabs. The halo is one layer of cell
 * coefficients below and above the owned slab, packed contiguously:
 * [comp][cell-in-layer], hgks_halo_bytes() per direction. */
long hgks_halo_bytes(const hgks_solver* s);
/* device pointers (as integers) of the solver-owned contiguous halo buffers:
 * send_lo/send_hi hold the packed bottom/top owned layers, recv_lo/recv_hi
 * receive the neighbours' layers. */
int hgks_halo_buffers(hgks_solver* s, unsigned long long* send_lo, unsigned long long* send_hi,
                      unsigned long long* recv_lo, unsigned long long* recv_hi);
/* which = 0: the state q^n, 1: the stage array q*. pack: owned boundary
 * layers -> send buffers; unpack: recv buffers -> ghost layers. Both are
 * kernels on the solver stream. */
int hgks_halo_pack(hgks_solver* s, int which);
int hgks_halo_unpack(hgks_solver* s, int which);
/* callback run at each exchange point (after pack, before unpack), on the
 * solver's stream; moves send_lo -> lower neighbour's recv_hi and send_hi ->
 * upper neighbour's recv_lo; returns 0 on success. Without one, a multi-slab
 * hgks_step fails; a single slab fills its ghosts by the periodic wrap. */
typedef int (*hgks_halo_fn)(void* user, hgks_solver* s, int which);
void hgks_set_halo_exchange(hgks_solver* s, hgks_halo_fn fn, void* user);
/* Overlapped exchange (takes precedence over the single callback when both
 * are set): start(user, s, which) runs right after the pack and must only
 * ENQUEUE the transfer behind the solver stream; the faces that need no ghost
 * layer (x and y faces of every owned layer, z faces of layers 1..nzl-1) are
 * then launched, and finish(user, s, which) must make the solver stream wait
 * for the transfer; unpack and the two boundary z-face layers follow. */
void hgks_set_halo_exchange_split(hgks_solver* s, hgks_halo_fn start, hgks_halo_fn finish, void* user);
/* Split-phase step for callers that drive the exchange themselves (several
 * slabs in one process): phase 0 = stage 1 (needs q^n ghosts), phase 1 =
 * stage 2 (needs q* ghosts), phase 2 = error check + commit. A single slab
 * fills its own ghosts; a multi-slab solver expects them unpacked already. */
int hgks_step_phase(hgks_solver* s, double dt, int phase);
/* Host reduction hook for host-driven transports (halo callbacks): every
 * rank calls it at the same points with op HGKS_REDUCE_MIN_U64 (error keys,
 * dt bits: positive doubles order like their bits) or HGKS_REDUCE_SUM_F64
 * (the offending value of a failure, diagnostics); the values are reduced in
 * place over the slabs. Ranks whose own cells failed still join, so a state
 * error raises the same, globally first, item on every rank. */
#define HGKS_REDUCE_MIN_U64 0
#define HGKS_REDUCE_SUM_F64 1
typedef int (*hgks_reduce_fn)(void* user, int op, void* values, int n);
void hgks_set_host_reduce(hgks_solver* s, hgks_reduce_fn fn, void* user);

/* ---- in-library data plane: the z-slab ring over NCCL (NVLink / NVSwitch).
 * Rank 0 creates an id (NCCL_UNIQUE_ID_BYTES = 128 bytes) and hands it to
 * every rank (MPI_Bcast, torch.distributed, a file); each rank attaches its
 * slab solver. The halo moves with ncclSend/ncclRecv on a comm stream while
 * the ghost-free faces compute; dt and the error keys are min-reduced on the
 * device (one 16-byte all-reduce per step for dt, 8 bytes for the key), so a
 * step needs no host round trip. world = 1 runs the same exchange with the
 * slab as its own neighbour. libnccl.so.2 is loaded at attach time
 * (HGKS_NCCL_LIB overrides the name). */
int hgks_nccl_unique_id(char* id_out, int nbytes);
int hgks_attach_nccl(hgks_solver* s, const char* unique_id, int rank, int world);
/* the same with a caller-owned communicator (an ncclComm_t) */
int hgks_attach_nccl_comm(hgks_solver* s, void* nccl_comm, int rank, int world);
/* in-place sum of n host doubles over the slabs (NCCL, or the host reduce
 * hook; a single slab leaves them unchanged): diagnostics partial sums */
int hgks_slab_reduce_sum(hgks_solver* s, double* values, int n);

/* ---- runtime plumbing */
int hgks_set_stream(hgks_solver* s, void* cuda_stream); /* NULL = solver-owned stream */
void* hgks_get_stream(hgks_solver* s);
int hgks_synchronize(hgks_solver* s);
/* kernel launches issued by this solver so far (for the bench's gpu_launches) */
long hgks_launch_count(const hgks_solver* s);
/* duration in ms of the last hgks_step's face and cell kernels (CUDA events on
 * the solver stream) when timing is enabled */
void hgks_set_kernel_timing(hgks_solver* s, int on);
int hgks_kernel_times(hgks_solver* s, double* face_ms, double* cell_ms, double* other_ms);
/* the same per S2O4 stage (0 or 1) of the last timed step */
int hgks_kernel_times_stage(hgks_solver* s, int stage, double* face_ms, double* cell_ms);
/* CUDA graphs for the device-resident advance loop (default on; kernel
 * timing disables them) */
void hgks_set_graphs(hgks_solver* s, int on);
/* test hook: cap the persistent face / cell grids at `ctas` CTAs (0 = the
 * resident count), so every CTA walks many tiles even on small meshes */
void hgks_set_grid_cap(hgks_solver* s, int ctas);
/* test hook: seed != 0 makes every warp of the persistent kernels sleep a
 * pseudo-random 0..4 us before each cp.async wait and barrier (a race
 * shaker: results must stay bitwise identical); 0 = off */
void hgks_set_race_shake(hgks_solver* s, unsigned seed);
/* face-kernel staging: 1 (default) = TMA boxes (cp.async.bulk.tensor +
 * mbarrier) when nx is even, 0 = per-lane cp.async (A/B and tests) */
void hgks_set_face_tma(hgks_solver* s, int on);
/* cell-kernel staging of the coefficient, face-flux and stage-2 A tiles: 1
 * (default) = TMA boxes when nx is even, 0 = per-lane cp.async */
void hgks_set_cell_tma(hgks_solver* s, int on);

/* Roofline denominator: sustained FP64 FMA throughput of `device`, measured
 * with a DFMA-chain kernel over ~`ms` milliseconds (CUDA events). Writes
 * TFLOP/s (2 flops per DFMA). */
int hgks_measure_fp64_peak(int device, double ms, double* tflops);

#ifdef __cplusplus
}
#endif
#endif
