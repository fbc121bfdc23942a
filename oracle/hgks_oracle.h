/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the DG-HGKS time step.
 *
 * A plain-C restatement of the reference algorithm (arXiv 2202.13821 as
 * implemented in /root/reference/proj/include/hgks). Each function cites the
 * reference file:line it restates. It is the checker for the CUDA path and is
 * loaded only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg; the product never links or calls it.
 *
 * Parity pin: validated against the reference headers compiled unmodified
 * (oracle/_ref/libhgks_ref.so, see oracle/ref_driver.cpp) and against the
 * golden vectors in tests/golden/ generated from that build
 * (tests/golden/make_golden.py).
 *
 * Layouts follow the reference: coefficients AoS [(cell*N + n)*5 + var]
 * (dg.hpp:15-17); face buffers [face*(npts*10) + p*10 + (F|Ft)] (dg.hpp:287).
 */
#ifndef HGKS_ORACLE_H
#define HGKS_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* error codes (mirror the reference exception types, core.hpp:58-70,
 * integrator.hpp:17-19) */
enum { ORC_OK = 0, ORC_NONPOS_DENSITY = 1, ORC_NONPOS_PRESSURE = 2, ORC_NONPOS_DT = 3, ORC_CONFIG = 4 };

typedef struct {
    int code;      /* ORC_* */
    int item;      /* face task (axis*ncells + f) or cell index; -1 if none */
    double value;  /* offending rho or p */
    char msg[256]; /* reference-shaped message */
} orc_error;

typedef struct orc_solver orc_solver;

/* setup_run (solver.hpp:29): case mesh, scheme and projected initial state.
 * case_name: adv2d | adv3d | vortex2d | tgv. Returns NULL on config error. */
orc_solver* orc_setup(const char* case_name, int n, int degree, int nonuniform, orc_error* err);
/* Mesh/scheme from explicit node arrays (mesh.hpp:22-37), zero state. */
orc_solver* orc_create(int nx, int ny, int nz, const double* xs, const double* ys,
                       const double* zs, int degree, int dim, double gamma, double mu,
                       orc_error* err);
void orc_free(orc_solver* s);

int orc_N(const orc_solver* s);
int orc_ncells(const orc_solver* s);
long orc_ncoeffs(const orc_solver* s);
double* orc_state(orc_solver* s); /* AoS coefficients, writable */
int orc_face_npts(const orc_solver* s, int axis);

/* residual (dg.hpp:354-450). R, Rt sized ncoeffs; faces (may be NULL) sized
 * ncells*npts*10 per axis. Returns ORC_OK or the first failing item's code. */
int orc_residual(orc_solver* s, const double* coeffs, double dt, double* R, double* Rt,
                 double* face0, double* face1, double* face2, long* flux_evals, orc_error* err);
/* detail::apply_inverse_mass (solver.hpp:42-54) */
void orc_apply_inverse_mass(const orc_solver* s, const double* R, double* L);
/* compute_dt (integrator.hpp:27-45) on the solver state */
int orc_compute_dt(const orc_solver* s, double cfl, double* dt, orc_error* err);
/* two_stage_step (integrator.hpp:64-75) with the eval of solver.hpp:81-88 */
int orc_step(orc_solver* s, double dt, orc_error* err);
/* tgv_diagnostics (cases.hpp:165-204): out = {Ek, epsZeta} */
void orc_tgv_diagnostics(const orc_solver* s, double* out);
/* error_norms (dg.hpp:228-266) against the named case's exact field at t */
int orc_error_norms(const orc_solver* s, double t, double* out3);

/* kinetics (flux.hpp:71-124, :128-177): traces are q[5], dq[3][5] */
int orc_interface_flux(const double* tl, const double* tr, double gamma, double tau, double dt,
                       double* full, double* half, orc_error* err);
int orc_smooth_flux(const double* t, double gamma, double tau, double dt, int axis, double* full,
                    double* half, orc_error* err);
/* moments.hpp:27-60: out = u[9], upos[9], uneg[9], v[9], w[9], xi2, xi4 */
void orc_maxwellian_moments(const double* prim, double gamma, double* out);

#ifdef __cplusplus
}
#endif
#endif
