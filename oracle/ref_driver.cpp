// TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// C-ABI driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/hgks/*.hpp, compiled in place with -I; no
// reference source is copied into this repository). Built by oracle/Makefile
// into oracle/_ref/libhgks_ref.so. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, as the checker and
// as the CPU baseline — never as the thing measured for the GPU arm.
//
// Every entry point calls the reference's own public API:
//   setup_run            proj/include/hgks/solver.hpp:29
//   residual             proj/include/hgks/dg.hpp:354
//   apply_inverse_mass   proj/include/hgks/solver.hpp:42
//   two_stage_step       proj/include/hgks/integrator.hpp:64
//   compute_dt           proj/include/hgks/integrator.hpp:27
//   run_case / advance   proj/include/hgks/solver.hpp:110 / :62
//   interface_flux_integrals / smooth_flux_integrals  proj/include/hgks/flux.hpp:71 / :148
//   tgv_diagnostics      proj/include/hgks/cases.hpp:165
//   error_norms          proj/include/hgks/dg.hpp:228
#include <cstring>
#include <memory>
#include <string>

#include "hgks/hgks.hpp"

using namespace hgks;

namespace {

struct RefRun {
    CaseConfig cfg;
    RunOptions opt;
    RunResult run;
    ResidualWorkspace ws;
    TwoStageScratch scratch;
    int ws_workers = -1;
};

void put_err(char* err, int errlen, const std::string& msg) {
    if (!err || errlen <= 0) return;
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
}

// 0 ok, 1 invalid state (numerical), 2 configuration, 3 non-positive dt, 4 other
template <class F>
int guarded(char* err, int errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const invalid_state_error& e) {
        put_err(err, errlen, e.what());
        return 1;
    } catch (const worker_error& e) {
        put_err(err, errlen, e.what());
        return 1;
    } catch (const non_positive_dt& e) {
        put_err(err, errlen, e.what());
        return 3;
    } catch (const std::invalid_argument& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 4;
    }
}

void ensure_ws(RefRun* r, int workers) {
    if (r->ws_workers != workers) {
        r->ws.resize(r->run.mesh, r->run.scheme, workers);
        r->ws_workers = workers;
    }
}

FaceTrace trace_from(const double* t) {
    FaceTrace f;
    f.q = Conserved::from({t[0], t[1], t[2], t[3], t[4]});
    for (int d = 0; d < 3; ++d)
        for (int v = 0; v < 5; ++v) f.dq[d][v] = t[5 + 5 * d + v];
    return f;
}

}  // namespace

extern "C" {

void* ref_setup(const char* case_name, int n, int degree, int nonuniform, int workers, char* err,
                int errlen) {
    auto r = std::make_unique<RefRun>();
    const int rc = guarded(err, errlen, [&] {
        r->cfg = CaseConfig::named(case_name, n);
        r->cfg.nonuniform = nonuniform != 0;
        r->opt.degree = degree;
        r->opt.workers = workers;
        r->run = setup_run(r->cfg, r->opt);
    });
    if (rc != 0) return nullptr;
    return r.release();
}

void ref_free(void* h) { delete static_cast<RefRun*>(h); }

void ref_info(void* h, int* dims /*nx,ny,nz,N,dim,degree*/, double* gas /*gamma,K,mu*/) {
    auto* r = static_cast<RefRun*>(h);
    dims[0] = r->run.mesh.nx;
    dims[1] = r->run.mesh.ny;
    dims[2] = r->run.mesh.nz;
    dims[3] = r->run.scheme.basis.N;
    dims[4] = r->run.scheme.basis.dim;
    dims[5] = r->run.scheme.basis.degree;
    gas[0] = r->run.scheme.gas.gamma;
    gas[1] = r->run.scheme.gas.K;
    gas[2] = r->run.scheme.gas.mu_ref;
}

void ref_nodes(void* h, double* xs, double* ys, double* zs) {
    auto* r = static_cast<RefRun*>(h);
    std::memcpy(xs, r->run.mesh.xs.data(), r->run.mesh.xs.size() * sizeof(double));
    std::memcpy(ys, r->run.mesh.ys.data(), r->run.mesh.ys.size() * sizeof(double));
    std::memcpy(zs, r->run.mesh.zs.data(), r->run.mesh.zs.size() * sizeof(double));
}

long ref_ncoeffs(void* h) { return static_cast<long>(static_cast<RefRun*>(h)->run.state.coeffs.size()); }

void ref_get_state(void* h, double* out, double* time) {
    auto* r = static_cast<RefRun*>(h);
    std::memcpy(out, r->run.state.coeffs.data(), r->run.state.coeffs.size() * sizeof(double));
    if (time) *time = r->run.state.time;
}

void ref_set_state(void* h, const double* in, double time) {
    auto* r = static_cast<RefRun*>(h);
    std::memcpy(r->run.state.coeffs.data(), in, r->run.state.coeffs.size() * sizeof(double));
    r->run.state.time = time;
}

/// Stage-level residual (dg.hpp:354). Any output pointer may be null.
int ref_residual(void* h, const double* coeffs, double dt, int workers, double* R, double* Rt,
                 double* f0, double* f1, double* f2, long* flux_evals, char* err, int errlen) {
    auto* r = static_cast<RefRun*>(h);
    ensure_ws(r, workers);
    r->ws.count_fluxes = flux_evals != nullptr;
    r->ws.flux_evaluations = 0;
    const int rc = guarded(err, errlen, [&] {
        residual(coeffs ? coeffs : r->run.state.coeffs.data(), r->run.mesh, r->run.scheme, dt, r->ws);
    });
    if (flux_evals) *flux_evals = r->ws.flux_evaluations.load();
    const size_t n = r->ws.R.size();
    if (R) std::memcpy(R, r->ws.R.data(), n * sizeof(double));
    if (Rt) std::memcpy(Rt, r->ws.Rt.data(), n * sizeof(double));
    double* fs[3] = {f0, f1, f2};
    for (int a = 0; a < 3; ++a)
        if (fs[a]) std::memcpy(fs[a], r->ws.face[a].data(), r->ws.face[a].size() * sizeof(double));
    return rc;
}

/// detail::apply_inverse_mass (solver.hpp:42) on a caller buffer.
void ref_apply_inverse_mass(void* h, const double* R, double* L, int workers) {
    auto* r = static_cast<RefRun*>(h);
    std::vector<double> in(R, R + r->run.state.coeffs.size()), out(in.size());
    detail::apply_inverse_mass(in, out, r->run.mesh, r->run.scheme.basis,
                               Partition::make(r->run.mesh.ncells(), workers));
    std::memcpy(L, out.data(), out.size() * sizeof(double));
}

/// compute_dt (integrator.hpp:27) on the run's current state.
int ref_compute_dt(void* h, double cfl, double* dt_out, char* err, int errlen) {
    auto* r = static_cast<RefRun*>(h);
    return guarded(err, errlen, [&] {
        StepControl ctrl;
        ctrl.cfl = cfl;
        *dt_out = compute_dt(r->run.state, r->run.mesh, r->run.scheme.gas, ctrl, r->opt.degree);
    });
}

/// One S2O4 step (integrator.hpp:64) with the eval of solver.hpp:81-88.
int ref_step(void* h, double dt, int workers, char* err, int errlen) {
    auto* r = static_cast<RefRun*>(h);
    ensure_ws(r, workers);
    r->ws.count_fluxes = false;
    const Partition cell_part = Partition::make(r->run.mesh.ncells(), workers);
    const auto eval = [&](const std::vector<double>& q, std::vector<double>& L,
                          std::vector<double>& Lt) {
        L.resize(q.size());
        Lt.resize(q.size());
        residual(q.data(), r->run.mesh, r->run.scheme, dt, r->ws);
        detail::apply_inverse_mass(r->ws.R, L, r->run.mesh, r->run.scheme.basis, cell_part);
        detail::apply_inverse_mass(r->ws.Rt, Lt, r->run.mesh, r->run.scheme.basis, cell_part);
    };
    return guarded(err, errlen, [&] {
        two_stage_step(r->run.state.coeffs, dt, eval, r->scratch);
        r->run.state.time += dt;
        ++r->run.steps;
    });
}

/// advance (solver.hpp:62) from the current state with run_case's TGV
/// recording (solver.hpp:110-126). dt_fixed <= 0 selects the CFL step.
int ref_advance(void* h, double t_end, double cfl, double dt_fixed, double record_interval,
                int workers, int* steps, double* rec /*[max_rec*4] t,Ek,epsEk,epsZeta*/,
                int max_rec, int* nrec, char* err, int errlen) {
    auto* r = static_cast<RefRun*>(h);
    RunOptions opt = r->opt;
    opt.cfl = cfl;
    opt.t_end = t_end;
    if (dt_fixed > 0) opt.dt_fixed = dt_fixed;
    opt.workers = workers;
    opt.record_interval = record_interval;
    r->run.records.clear();
    const int steps0 = r->run.steps;
    const Partition part = Partition::make(r->run.mesh.ncells(), workers);
    const int rc = guarded(err, errlen, [&] {
        advance(r->run, r->cfg, opt, [&](RunResult& rr) {
            if (r->cfg.name == "tgv")
                rr.records.push_back(
                    tgv_diagnostics(rr.state, rr.mesh, rr.scheme.tab, rr.scheme.gas, part));
        });
    });
    if (r->run.records.size() >= 3) {
        std::vector<double> ek(r->run.records.size());
        for (size_t i = 0; i < ek.size(); ++i) ek[i] = r->run.records[i].Ek;
        const auto eps = dissipation_from_series(ek, record_interval);
        for (size_t i = 0; i < ek.size(); ++i) r->run.records[i].epsEk = eps[i];
    }
    if (steps) *steps = r->run.steps - steps0;
    int k = 0;
    for (const auto& x : r->run.records) {
        if (k >= max_rec) break;
        rec[4 * k + 0] = x.t;
        rec[4 * k + 1] = x.Ek;
        rec[4 * k + 2] = x.epsEk;
        rec[4 * k + 3] = x.epsZeta;
        ++k;
    }
    if (nrec) *nrec = k;
    return rc;
}

/// tgv_diagnostics (cases.hpp:165) of the current state.
void ref_tgv_diagnostics(void* h, double* out /*t, Ek, epsZeta*/) {
    auto* r = static_cast<RefRun*>(h);
    const Partition part = Partition::make(r->run.mesh.ncells(), 1);
    const TgvRecord rec =
        tgv_diagnostics(r->run.state, r->run.mesh, r->run.scheme.tab, r->run.scheme.gas, part);
    out[0] = rec.t;
    out[1] = rec.Ek;
    out[2] = rec.epsZeta;
}

/// error_norms (dg.hpp:228) against the case's exact field at time t.
int ref_error_norms(void* h, double t, double* out /*l1,l2,cell_avg*/, char* err, int errlen) {
    auto* r = static_cast<RefRun*>(h);
    return guarded(err, errlen, [&] {
        const auto exact = exact_field(r->cfg, t);
        if (!exact) throw std::invalid_argument("case has no exact solution: " + r->cfg.name);
        const ErrorNorms e = error_norms(r->run.state, r->run.mesh, r->run.scheme.tab, exact,
                                         Partition::make(r->run.mesh.ncells(), 1));
        out[0] = e.l1;
        out[1] = e.l2;
        out[2] = e.cell_avg;
    });
}

/// interface_flux_integrals (flux.hpp:71): traces are 20 doubles
/// (q[5], dq_normal[5], dq_t1[5], dq_t2[5]) in the face-local frame.
int ref_interface_flux(const double* tl, const double* tr, double gamma, double tau, double dt,
                       double* full, double* half, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const GasModel gas = GasModel::make(gamma);
        const auto [If, Ih] = interface_flux_integrals(trace_from(tl), trace_from(tr), gas, tau, dt);
        for (int v = 0; v < 5; ++v) {
            full[v] = If[v];
            half[v] = Ih[v];
        }
    });
}

/// make_smooth_point + smooth_flux_integrals (flux.hpp:128-165).
int ref_smooth_flux(const double* t, double gamma, double tau, double dt, int axis, double* full,
                    double* half, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const GasModel gas = GasModel::make(gamma);
        const FaceTrace ft = trace_from(t);
        const SmoothPoint sp = make_smooth_point(ft.q, ft.dq, gas);
        const auto [If, Ih] = smooth_flux_integrals(sp, tau, dt, axis);
        for (int v = 0; v < 5; ++v) {
            full[v] = If[v];
            half[v] = Ih[v];
        }
    });
}

/// maxwellian_moments (moments.hpp:27): out = u[9], upos[9], uneg[9], v[9], w[9], xi2, xi4.
int ref_maxwellian_moments(const double* prim, double gamma, double* out) {
    const GasModel gas = GasModel::make(gamma);
    const MomentTable m = maxwellian_moments({prim[0], prim[1], prim[2], prim[3], prim[4]}, gas);
    for (int n = 0; n < 9; ++n) {
        out[n] = m.u[n];
        out[9 + n] = m.upos[n];
        out[18 + n] = m.uneg[n];
        out[27 + n] = m.v[n];
        out[36 + n] = m.w[n];
    }
    out[45] = m.xi2;
    out[46] = m.xi4;
    return 0;
}

/// Basis tables (dg.hpp:91-128) for cross-checking the device tables:
/// which = 0 vol, 1 proj, 2+a face_minus[a], 5+a face_plus[a]. Writes B[npts*N],
/// dB[npts*3*N], w[npts], ref[npts*3]; returns npts.
int ref_tables(int degree, int dim, int which, double* B, double* dB, double* w, double* ref) {
    const BasisSet b = build_basis(degree, dim);
    const DGTables t = DGTables::make(b);
    const detail::PointBasis* pb = which == 0   ? &t.vol
                                   : which == 1 ? &t.proj
                                   : which < 5  ? &t.face_minus[which - 2]
                                                : &t.face_plus[which - 5];
    if (B) std::memcpy(B, pb->B.data(), pb->B.size() * sizeof(double));
    if (dB) std::memcpy(dB, pb->dB.data(), pb->dB.size() * sizeof(double));
    if (w) std::memcpy(w, pb->wq.data(), pb->wq.size() * sizeof(double));
    if (ref)
        for (int p = 0; p < pb->npts; ++p)
            for (int a = 0; a < 3; ++a) ref[3 * p + a] = pb->ref[p][a];
    return pb->npts;
}

}  // extern "C"
