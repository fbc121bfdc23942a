// hgks_b200/hgks.hpp — C++ drop-in for the reference's solver interface,
// backed by the B200 kernels through the C ABI (include/hgks_b200.h).
//
// A reference user replaces the include path proj/include with
//     -I include/hgks_b200/compat -I include
// (compat/hgks/*.hpp forward the reference's header names here) and links
// libhgks_b200.so; or includes "hgks_b200/hgks.hpp" directly. Names,
// argument meanings, host layouts and exception types are the reference's:
//
//   core.hpp, moments.hpp, microslope.hpp types   -> hgks_b200/core.hpp
//   quadrature.hpp, basis.hpp, mesh.hpp, dg.hpp helpers -> hgks_b200/discretization.hpp
//   runtime.hpp                                    -> hgks_b200/runtime.hpp
//   Scheme::make                    dg.hpp:269-281
//   ResidualWorkspace, residual     dg.hpp:286-303, :354-455
//   project, error_norms            dg.hpp:193-266
//   detail::apply_inverse_mass      solver.hpp:42-54
//   StepControl, compute_dt, non_positive_dt, default_cfl   integrator.hpp:11-45
//   TwoStageScratch, two_stage_step integrator.hpp:47-75
//   CaseConfig, build_mesh, case fields, initial_field, exact_field,
//   TgvRecord, tgv_diagnostics, dissipation_from_series     cases.hpp:12-216
//   RunOptions, RunResult, setup_run, advance<OnRecord>, run_case,
//   run_error_norms, StudyOptions, StudyRow, convergence_study,
//   scaling_report                  solver.hpp:10-240
//
// Where the work goes: residual, inverse mass, compute_dt, projection, error
// norms, TGV diagnostics and the whole advance loop run on the GPU (the
// device-resident loop of hgks_advance_records: dt, clipping, commit and
// failure checks on the device, one CUDA graph per step; records download the
// state only for a caller's on_record). There is no host fallback: without a
// GPU every device call throws device_error. The host-side pieces are the
// reference's caller-facing utilities (Partition, field sampling for a
// caller's std::function, the generic two_stage_step for an arbitrary eval).
// One device solver per (mesh, scheme) is shared by every call on it.
#pragma once

#include <chrono>
#include <cmath>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../hgks_b200.h"
#include "core.hpp"
#include "discretization.hpp"
#include "runtime.hpp"

namespace hgks {

/// CUDA / device failure (no CPU path exists)
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct non_positive_dt : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// Everything the residual needs besides the state (dg.hpp:269-281).
struct Scheme {
    BasisSet basis;
    DGTables tab;
    GasModel gas;

    static Scheme make(int degree, int dim, const GasModel& gas) {
        Scheme s;
        s.basis = build_basis(degree, dim);
        s.tab = DGTables::make(s.basis);
        s.gas = gas;
        return s;
    }
    /// P1 extension (unpinned: the reference has no k = 1)
    static Scheme make_extended(int degree, int dim, const GasModel& gas) {
        Scheme s;
        s.basis = build_basis_extended(degree, dim);
        s.tab = DGTables::make(s.basis);
        s.gas = gas;
        return s;
    }
};

// ------------------------------------------------------- device handles
namespace detail {

inline void throw_from(hgks_solver* s, int rc) {
    const std::string msg = s ? hgks_last_error(s) : "hgks: no solver";
    if (rc == HGKS_ERR_STATE) {
        int code = 0, phase = -1;
        long item = -1;
        double value = 0;
        hgks_error_info(s, &code, &phase, &item, &value);
        if (phase == 0 || phase == 1) {
            // worker_error prefixes "item <i>: " itself (runtime.hpp:37-41)
            const std::string pre = "item " + std::to_string(item) + ": ";
            const std::string inner = msg.rfind(pre, 0) == 0 ? msg.substr(pre.size()) : msg;
            throw worker_error(static_cast<int>(item), inner);
        }
        if (msg.find("density") != std::string::npos) throw non_positive_density(value);
        throw non_positive_pressure(value);
    }
    if (rc == HGKS_ERR_DT) throw non_positive_dt(msg);
    if (rc == HGKS_ERR_CONFIG) throw std::invalid_argument(msg);
    throw device_error(msg);
}

/// One device solver (mesh + scheme + device-resident state).
struct Device {
    hgks_solver* s = nullptr;
    int nx, ny, nz, degree, dim, device;
    double gamma, mu;
    std::vector<double> xs, ys, zs;

    Device(const Mesh& m, int degree_, int dim_, const GasModel& gas, int device_)
        : nx(m.nx), ny(m.ny), nz(m.nz), degree(degree_), dim(dim_), device(device_), gamma(gas.gamma),
          mu(gas.mu_ref), xs(m.xs), ys(m.ys), zs(m.zs) {
        hgks_config cfg{};
        cfg.nx = nx;
        cfg.ny = ny;
        cfg.nz = nz;
        cfg.xs = xs.data();
        cfg.ys = ys.data();
        cfg.zs = zs.data();
        cfg.degree = degree;
        cfg.dim = dim;
        cfg.gamma = gamma;
        cfg.mu = mu;
        cfg.device = device;
        hgks_solver* h = nullptr;
        const int rc = hgks_create(&cfg, &h);
        if (rc != HGKS_OK) {
            const std::string msg = h ? hgks_last_error(h) : "hgks_create failed";
            if (h) hgks_destroy(h);
            if (rc == HGKS_ERR_CONFIG) throw std::invalid_argument(msg);
            throw device_error(msg);
        }
        s = h;
    }
    ~Device() {
        if (s) hgks_destroy(s);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    bool same_mesh(const Mesh& m) const {
        return m.nx == nx && m.ny == ny && m.nz == nz && m.xs == xs && m.ys == ys && m.zs == zs;
    }
    bool matches(const Mesh& m, int deg, int d, const GasModel& gas, int dev) const {
        return same_mesh(m) && deg == degree && d == dim && gas.gamma == gamma && gas.mu_ref == mu && dev == device;
    }
    void check(int rc) const {
        if (rc != HGKS_OK) throw_from(s, rc);
    }
    void upload(const DGState& st) const { check(hgks_set_state(s, st.coeffs.data(), st.time)); }
    void download(DGState& st) const {
        st.coeffs.resize(static_cast<size_t>(hgks_num_coeffs(s)));
        check(hgks_get_state(s, st.coeffs.data(), &st.time));
    }
};

/// Process-wide registry: one live solver per (mesh, degree, dim, gas,
/// device), shared by workspaces and the free functions; the two most
/// recently used stay alive between calls.
class Registry {
  public:
    static Registry& get() {
        static Registry r;
        return r;
    }
    std::shared_ptr<Device> acquire(const Mesh& m, int degree, int dim, const GasModel& gas, int device) {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = live_.begin(); it != live_.end();) {
            auto sp = it->lock();
            if (!sp) {
                it = live_.erase(it);
                continue;
            }
            if (sp->matches(m, degree, dim, gas, device)) {
                touch(sp);
                return sp;
            }
            ++it;
        }
        auto sp = std::make_shared<Device>(m, degree, dim, gas, device);
        live_.push_back(sp);
        touch(sp);
        return sp;
    }
    /// any live solver on this mesh and basis (the inverse mass matrix does
    /// not depend on the gas); else a new one with air
    std::shared_ptr<Device> acquire_basis(const Mesh& m, int degree, int dim, int device) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (auto& w : live_)
                if (auto sp = w.lock())
                    if (sp->same_mesh(m) && sp->degree == degree && sp->dim == dim && sp->device == device) {
                        touch(sp);
                        return sp;
                    }
        }
        return acquire(m, degree, dim, GasModel::make(1.4), device);
    }
    void release_all() {
        std::lock_guard<std::mutex> lk(mu_);
        recent_.clear();
    }

  private:
    void touch(const std::shared_ptr<Device>& sp) {
        for (auto it = recent_.begin(); it != recent_.end(); ++it)
            if (*it == sp) {
                recent_.erase(it);
                break;
            }
        recent_.insert(recent_.begin(), sp);
        if (recent_.size() > 2) recent_.resize(2);
    }
    std::mutex mu_;
    std::vector<std::weak_ptr<Device>> live_;
    std::vector<std::shared_ptr<Device>> recent_;
};

inline std::shared_ptr<Device> device_for(const Mesh& m, const Scheme& sch, int device = 0) {
    return Registry::get().acquire(m, sch.basis.degree, sch.basis.dim, sch.gas, device);
}

}  // namespace detail

/// Drop every cached device solver that no workspace or result still holds.
inline void release_device_memory() { detail::Registry::get().release_all(); }

// ------------------------------------------------------------ residual
/// Reused buffers for residual assembly (dg.hpp:286-303); the device solver
/// holding the face buffers lives behind `dev`.
struct ResidualWorkspace {
    std::array<std::vector<double>, 3> face;  // [face*(npts*10) + p*10 + (F|Ft)]
    std::vector<double> R, Rt;                // [(cell*N + n)*5 + var]
    Partition cells{1, {{0, 0}}};
    Partition faces{1, {{0, 0}}};
    bool count_fluxes = false;
    std::atomic<long> flux_evaluations{0};
    std::shared_ptr<detail::Device> dev;
    int device = 0;

    void resize(const Mesh& mesh, const Scheme& sch, int workers) {
        dev = detail::device_for(mesh, sch, device);
        const int nc = mesh.ncells();
        for (int a = 0; a < 3; ++a)
            face[a].assign(static_cast<size_t>(nc) * sch.tab.face_minus[a].npts * 10, 0.0);
        R.assign(static_cast<size_t>(nc) * sch.basis.N * 5, 0.0);
        Rt.assign(static_cast<size_t>(nc) * sch.basis.N * 5, 0.0);
        cells = Partition::make(nc, workers);
        faces = Partition::make(3 * nc, workers);
    }
};

/// residual (dg.hpp:354): R, Rt and the face buffers of `coeffs`, on the GPU.
inline void residual(const double* coeffs, const Mesh& mesh, const Scheme& sch, double dt, ResidualWorkspace& ws) {
    if (!ws.dev || !ws.dev->matches(mesh, sch.basis.degree, sch.basis.dim, sch.gas, ws.device) ||
        ws.R.size() != static_cast<size_t>(mesh.ncells()) * sch.basis.N * 5)
        ws.resize(mesh, sch, ws.cells.workers);
    hgks_set_count_fluxes(ws.dev->s, ws.count_fluxes ? 1 : 0);
    ws.dev->check(hgks_residual(ws.dev->s, coeffs, dt, ws.R.data(), ws.Rt.data(), ws.face[0].data(),
                                ws.face[1].data(), ws.face[2].data()));
    if (ws.count_fluxes) ws.flux_evaluations += hgks_flux_evaluations(ws.dev->s);
}

inline void residual(const DGState& s, const Mesh& mesh, const Scheme& sch, double dt, ResidualWorkspace& ws) {
    residual(s.coeffs.data(), mesh, sch, dt, ws);
}

namespace detail {
/// L = R * (1/M) per cell (solver.hpp:42-54), on the GPU.
inline void apply_inverse_mass(const std::vector<double>& R, std::vector<double>& L, const Mesh& mesh,
                               const BasisSet& basis, const Partition&) {
    auto d = Registry::get().acquire_basis(mesh, basis.degree, basis.dim, 0);
    L.resize(R.size());
    d->check(hgks_apply_inverse_mass(d->s, R.data(), L.data()));
}
}  // namespace detail

// ---------------------------------------------------------- integrator
struct StepControl {
    double cfl = 0.15;
    double t_end = 1.0;
    std::optional<double> dt_fixed;
};

inline double default_cfl(int degree) { return degree == 2 ? 0.15 : 0.09; }

/// compute_dt (integrator.hpp:27-45) from the cell means, on the GPU. Only
/// the means enter, and `degree` only through the viscous bound, so the means
/// of any state are evaluated on the mesh's P2 device solver.
inline double compute_dt(const DGState& s, const Mesh& mesh, const GasModel& gas, const StepControl& ctrl,
                         int degree) {
    if (ctrl.dt_fixed) return *ctrl.dt_fixed;
    const int dim = mesh.nz > 1 ? 3 : 2;
    const int N = dim == 3 ? 10 : 6;
    auto d = detail::Registry::get().acquire(mesh, 2, dim, gas, 0);
    if (s.N == N) {
        d->upload(s);
    } else {
        DGState m = DGState::zeros(mesh.ncells(), N);
        for (int c = 0; c < mesh.ncells(); ++c)
            for (int v = 0; v < 5; ++v) m.coeff(c, 0, v) = s.coeff(c, 0, v);
        m.time = s.time;
        d->upload(m);
    }
    double dt = 0.0;
    d->check(hgks_compute_dt_k(d->s, ctrl.cfl, degree, &dt));
    return dt;
}

struct TwoStageScratch {
    std::vector<double> qstar, L1, Lt1, L2, Lt2;
    void resize(size_t n) {
        qstar.resize(n);
        L1.resize(n);
        Lt1.resize(n);
        L2.resize(n);
        Lt2.resize(n);
    }
};

/// two_stage_step (integrator.hpp:64-75) for an arbitrary operator: eval(q,
/// L, Lt) exactly twice; the combine is the reference's (the operator itself
/// is the caller's, e.g. residual + apply_inverse_mass on the GPU).
template <class Eval>
void two_stage_step(std::vector<double>& q, double dt, Eval&& eval, TwoStageScratch& ws) {
    const size_t n = q.size();
    ws.resize(n);
    eval(q, ws.L1, ws.Lt1);
    for (size_t i = 0; i < n; ++i) ws.qstar[i] = q[i] + 0.5 * dt * ws.L1[i] + 0.125 * dt * dt * ws.Lt1[i];
    eval(ws.qstar, ws.L2, ws.Lt2);
    const double c = dt * dt / 6.0;
    for (size_t i = 0; i < n; ++i) q[i] += dt * ws.L1[i] + c * (ws.Lt1[i] + 2.0 * ws.Lt2[i]);
}

/// The solver.hpp:81-88 eval (residual + inverse mass, the same full dt in
/// both stages) named as a type: two_stage_step then runs the whole fused
/// step on the GPU (one upload, both stages + combine on the device, one
/// download).
struct DeviceEval {
    ResidualWorkspace* ws;
};

inline void two_stage_step(std::vector<double>& q, double dt, DeviceEval eval, TwoStageScratch&) {
    eval.ws->dev->check(hgks_two_stage_step_host_streamed(eval.ws->dev->s, q.data(), dt, 0));
}

// ---------------------------------------------------------- projection
namespace detail {
/// field values at the projection points of every cell, [(c*npts + p)*5 + v]
/// (x = center + h/2 * ref_p, dg.hpp:205-209), sampled over the partition
inline std::vector<double> sample_field(const std::function<Conserved(std::array<double, 3>)>& f,
                                        const Mesh& mesh, const DGTables& tab, const Partition& part,
                                        bool rho_only) {
    const int np = tab.proj.npts, per = rho_only ? 1 : 5;
    std::vector<double> out(static_cast<size_t>(mesh.ncells()) * np * per);
    parallel_map_cells(part, [&](int c) {
        const auto ctr = mesh.center(c);
        const auto h = mesh.widths(c);
        for (int p = 0; p < np; ++p) {
            const auto& r = tab.proj.ref[p];
            const Conserved q = f({ctr[0] + 0.5 * h[0] * r[0], ctr[1] + 0.5 * h[1] * r[1], ctr[2] + 0.5 * h[2] * r[2]});
            double* o = out.data() + (static_cast<size_t>(c) * np + p) * per;
            if (rho_only) {
                o[0] = q.rho;
            } else {
                const Vec5 v = q.vec();
                for (int k = 0; k < 5; ++k) o[k] = v[k];
            }
        }
    });
    return out;
}
}  // namespace detail

/// L2 projection of a field onto the basis (dg.hpp:193-220): the field is
/// sampled on the host (it is the caller's function), the quadrature sums
/// run on the GPU.
inline DGState project(const std::function<Conserved(std::array<double, 3>)>& field, const Mesh& mesh,
                       const DGTables& tab, const Partition& part) {
    auto d = detail::Registry::get().acquire_basis(mesh, tab.basis.degree, tab.basis.dim, 0);
    const std::vector<double> smp = detail::sample_field(field, mesh, tab, part, false);
    d->check(hgks_project_samples(d->s, smp.data(), 0.0));
    DGState s = DGState::zeros(mesh.ncells(), tab.basis.N);
    d->download(s);
    s.time = 0.0;
    return s;
}

/// Density error norms against an exact field (dg.hpp:228-266), on the GPU.
inline ErrorNorms error_norms(const DGState& s, const Mesh& mesh, const DGTables& tab,
                              const std::function<Conserved(std::array<double, 3>)>& exact,
                              const Partition& part) {
    auto d = detail::Registry::get().acquire_basis(mesh, tab.basis.degree, tab.basis.dim, 0);
    d->upload(s);
    const std::vector<double> rho = detail::sample_field(exact, mesh, tab, part, true);
    double out[3];
    d->check(hgks_error_norms_samples(d->s, rho.data(), out));
    return {out[0], std::sqrt(out[1]), std::sqrt(out[2])};
}

// --------------------------------------------------------------- cases
/// Built-in problems (cases.hpp:12-46).
struct CaseConfig {
    std::string name;
    int dim = 2;
    int n = 8;
    bool nonuniform = false;
    double gamma = 1.4;
    double mach0 = 0.1;
    double reynolds = 1600;
    double eps = 5.0;
    double t_end = 2.0;

    static CaseConfig named(const std::string& name, int n) {
        CaseConfig c;
        c.name = name;
        c.n = n;
        if (name == "adv2d" || name == "adv3d") {
            c.dim = name == "adv3d" ? 3 : 2;
            c.t_end = 2.0;
        } else if (name == "vortex2d" || name == "tgv") {
            c.dim = name == "tgv" ? 3 : 2;
            c.t_end = 10.0;
        } else {
            throw std::invalid_argument("unknown case: " + name);
        }
        return c;
    }
    double viscosity() const { return name == "tgv" ? 1.0 / reynolds : 0.0; }
};

/// x = xi + 0.05 sin(pi xi) on the uniform parameter nodes (cases.hpp:50-57)
inline std::vector<double> case_axis_nodes(double lo, double hi, int n, bool nonuniform) {
    std::vector<double> v(n + 1);
    for (int i = 0; i <= n; ++i) {
        const double xi = lo + (hi - lo) * i / n;
        v[i] = nonuniform ? xi + 0.05 * std::sin(M_PI * xi) : xi;
    }
    return v;
}

/// cases.hpp:59-73: 2-D cases on the degenerate box with one z cell
inline Mesh build_mesh(const CaseConfig& cfg) {
    if (cfg.n < 4) throw std::invalid_argument("build_mesh: need at least 4 cells per axis");
    const double lo = cfg.name == "tgv" ? -M_PI : 0.0;
    const double hi = cfg.name == "tgv" ? M_PI : cfg.name == "vortex2d" ? 10.0 : 2.0;
    auto ax = [&] { return case_axis_nodes(lo, hi, cfg.n, cfg.nonuniform); };
    if (cfg.dim == 2) return Mesh::make(ax(), ax(), {lo, hi});
    return Mesh::make(ax(), ax(), ax());
}

/// rho = 1 + 0.2 sin(pi (sum x - dim t)), unit pressure and velocities (cases.hpp:78-87)
inline Conserved density_wave(int dim, const std::array<double, 3>& x, double t, double gamma = 1.4) {
    const double s = dim == 3 ? x[0] + x[1] + x[2] - 3.0 * t : x[0] + x[1] - 2.0 * t;
    const double rho = 1.0 + 0.2 * std::sin(M_PI * s);
    const double W = dim == 3 ? 1.0 : 0.0;
    const double E = 1.0 / (gamma - 1.0) + 0.5 * rho * (1.0 + 1.0 + W * W);
    return {rho, rho, rho, rho * W, E};
}

/// isotropic vortex on [0,10]^2 moving with (1,1) (cases.hpp:91-112)
inline Conserved isotropic_vortex(const std::array<double, 3>& x, double t, double eps, double gamma) {
    auto wrap = [](double v) {
        v = std::fmod(v, 10.0);
        if (v < -5.0) v += 10.0;
        if (v >= 5.0) v -= 10.0;
        return v;
    };
    const double dx = wrap(x[0] - 5.0 - t), dy = wrap(x[1] - 5.0 - t);
    const double r2 = dx * dx + dy * dy;
    const double g = eps / (2.0 * M_PI) * std::exp(0.5 * (1.0 - r2));
    const double U = 1.0 - g * dy, V = 1.0 + g * dx;
    const double T = 1.0 - (gamma - 1.0) * eps * eps / (8.0 * gamma * M_PI * M_PI) * std::exp(1.0 - r2);
    const double rho = std::pow(T, 1.0 / (gamma - 1.0));
    const double p = rho * T;
    return {rho, rho * U, rho * V, 0.0, p / (gamma - 1.0) + 0.5 * rho * (U * U + V * V)};
}

/// Taylor-Green field on [-pi, pi]^3, p0 = 1/(gamma M0^2), rho = p/p0 (cases.hpp:115-124)
inline Conserved taylor_green_init(const std::array<double, 3>& x, const CaseConfig& cfg) {
    const double p0 = 1.0 / (cfg.gamma * cfg.mach0 * cfg.mach0);
    const double U = std::sin(x[0]) * std::cos(x[1]) * std::cos(x[2]);
    const double V = -std::cos(x[0]) * std::sin(x[1]) * std::cos(x[2]);
    const double p = p0 + (std::cos(2.0 * x[0]) + std::cos(2.0 * x[1])) * (std::cos(2.0 * x[2]) + 2.0) / 16.0;
    const double rho = p / p0;
    return {rho, rho * U, rho * V, 0.0, p / (cfg.gamma - 1.0) + 0.5 * rho * (U * U + V * V)};
}

inline std::function<Conserved(std::array<double, 3>)> initial_field(const CaseConfig& cfg) {
    if (cfg.name == "adv2d" || cfg.name == "adv3d")
        return [d = cfg.dim, g = cfg.gamma](std::array<double, 3> x) { return density_wave(d, x, 0.0, g); };
    if (cfg.name == "vortex2d")
        return [e = cfg.eps, g = cfg.gamma](std::array<double, 3> x) { return isotropic_vortex(x, 0.0, e, g); };
    return [cfg](std::array<double, 3> x) { return taylor_green_init(x, cfg); };
}

/// exact solution at t, or null for tgv (cases.hpp:140-153)
inline std::function<Conserved(std::array<double, 3>)> exact_field(const CaseConfig& cfg, double t) {
    if (cfg.name == "adv2d" || cfg.name == "adv3d")
        return [d = cfg.dim, g = cfg.gamma, t](std::array<double, 3> x) { return density_wave(d, x, t, g); };
    if (cfg.name == "vortex2d")
        return [e = cfg.eps, g = cfg.gamma, t](std::array<double, 3> x) { return isotropic_vortex(x, t, e, g); };
    return nullptr;
}

struct TgvRecord {
    double t;
    double Ek;
    double epsEk = 0.0;
    double epsZeta;
};

namespace detail {
inline TgvRecord tgv_record(hgks_solver* s, double mu_ref, double t) {
    double e = 0, z = 0, v = 0;
    const int rc = hgks_tgv_diagnostics(s, &e, &z, &v);
    if (rc != HGKS_OK) throw_from(s, rc);
    TgvRecord r;
    r.t = t;
    r.Ek = e / v;
    r.epsZeta = 2.0 * mu_ref * z / v;
    return r;
}
}  // namespace detail

/// Kinetic energy and enstrophy dissipation (cases.hpp:165-204), on the GPU.
inline TgvRecord tgv_diagnostics(const DGState& s, const Mesh& mesh, const DGTables& tab, const GasModel& gas,
                                 const Partition&) {
    auto d = detail::Registry::get().acquire_basis(mesh, tab.basis.degree, tab.basis.dim, 0);
    d->upload(s);
    return detail::tgv_record(d->s, gas.mu_ref, s.time);
}

/// -dEk/dt by second-order differences (cases.hpp:208-216)
inline std::vector<double> dissipation_from_series(const std::vector<double>& Ek, double dt) {
    const size_t n = Ek.size();
    if (n < 3) throw std::invalid_argument("dissipation_from_series: need at least 3 samples");
    std::vector<double> eps(n);
    eps[0] = -(-3.0 * Ek[0] + 4.0 * Ek[1] - Ek[2]) / (2.0 * dt);
    for (size_t i = 1; i + 1 < n; ++i) eps[i] = -(Ek[i + 1] - Ek[i - 1]) / (2.0 * dt);
    eps[n - 1] = -(3.0 * Ek[n - 1] - 4.0 * Ek[n - 2] + Ek[n - 3]) / (2.0 * dt);
    return eps;
}

// -------------------------------------------------------------- solver
struct RunOptions {
    int degree = 2;
    double cfl = 0.0;  // 0 selects the per-degree default
    std::optional<double> dt_fixed;
    std::optional<double> t_end;
    int workers = 1;  // signature parity; the device ignores it
    double record_interval = 0.05;
};

struct RunResult {
    Mesh mesh;
    Scheme scheme;
    DGState state;
    int steps = 0;
    std::vector<TgvRecord> records;
};

/// solver.hpp:29-37: mesh, scheme, projected initial state (projection of the
/// named case on the GPU).
inline RunResult setup_run(const CaseConfig& cfg, const RunOptions& opt) {
    RunResult r;
    r.mesh = build_mesh(cfg);
    r.scheme = Scheme::make(opt.degree, cfg.dim, GasModel::make(cfg.gamma, cfg.viscosity()));
    auto d = detail::device_for(r.mesh, r.scheme);
    d->check(hgks_project_case(d->s, cfg.name.c_str(), 0.0));
    r.state = DGState::zeros(r.mesh.ncells(), r.scheme.basis.N);
    d->download(r.state);
    r.state.time = 0.0;
    return r;
}

namespace detail {
struct RecordCtx {
    std::function<void(double)> fn;
    std::exception_ptr err;
};
inline int record_trampoline(void* user, hgks_solver*, double t) {
    auto* ctx = static_cast<RecordCtx*>(user);
    try {
        ctx->fn(t);
        return 0;
    } catch (...) {
        ctx->err = std::current_exception();
        return 1;
    }
}

/// the device-resident advance loop on r's device (solver.hpp:62-108);
/// on_step_record(t) runs at each record time with the device showing that
/// state
inline void advance_on_device(RunResult& r, const CaseConfig& cfg, const RunOptions& opt, Device& d,
                              const std::function<void(double)>& on_step_record) {
    const double cfl = opt.cfl > 0.0 ? opt.cfl : default_cfl(opt.degree);
    const double t_end = opt.t_end ? *opt.t_end : cfg.t_end;
    const bool record = cfg.name == "tgv";
    RecordCtx ctx{on_step_record, nullptr};
    int steps = 0;
    const int rc = hgks_advance_records(d.s, t_end, cfl, opt.dt_fixed ? *opt.dt_fixed : 0.0,
                                        record ? opt.record_interval : 0.0, opt.record_interval, 0,
                                        record ? &record_trampoline : nullptr, &ctx, &steps);
    r.steps += steps;
    if (ctx.err) std::rethrow_exception(ctx.err);
    if (rc == HGKS_ERR_STATE) {
        int code = 0, phase = -1;
        long item = -1;
        double value = 0;
        hgks_error_info(d.s, &code, &phase, &item, &value);
        // compute_dt failures propagate as they are; a failing step is
        // rewrapped with " at t=<t>" (solver.hpp:95-99)
        if (phase == 2) throw_from(d.s, rc);
        throw invalid_state_error(hgks_last_error(d.s));
    }
    d.check(rc);
}
}  // namespace detail

/// March a prepared run to t_end (solver.hpp:62-108): on_record(r) at t = 0
/// and at every record time of the tgv case, with r.state the state at that
/// time. The loop runs on the GPU; records download the state for the callback.
template <class OnRecord>
inline void advance(RunResult& r, const CaseConfig& cfg, const RunOptions& opt, OnRecord&& on_record) {
    auto d = detail::device_for(r.mesh, r.scheme);
    on_record(r);
    d->upload(r.state);
    detail::advance_on_device(r, cfg, opt, *d, [&](double t) {
        d->download(r.state);
        r.state.time = t;
        on_record(r);
    });
    d->download(r.state);
}

inline RunResult run_case(const CaseConfig& cfg, const RunOptions& opt) {
    RunResult r = setup_run(cfg, opt);
    auto d = detail::device_for(r.mesh, r.scheme);
    const bool tgv = cfg.name == "tgv";
    // records straight from the device state (no download per record)
    d->upload(r.state);
    if (tgv) r.records.push_back(detail::tgv_record(d->s, r.scheme.gas.mu_ref, r.state.time));
    detail::advance_on_device(r, cfg, opt, *d, [&](double t) {
        r.records.push_back(detail::tgv_record(d->s, r.scheme.gas.mu_ref, t));
    });
    d->download(r.state);
    if (!r.records.empty()) {
        std::vector<double> ek;
        for (const auto& x : r.records) ek.push_back(x.Ek);
        const auto eps = dissipation_from_series(ek, opt.record_interval);
        for (size_t i = 0; i < ek.size(); ++i) r.records[i].epsEk = eps[i];
    }
    return r;
}

/// error norms of a finished run against the case's exact solution
/// (solver.hpp:129-134), on the GPU.
inline ErrorNorms run_error_norms(const RunResult& r, const CaseConfig& cfg, int) {
    if (!exact_field(cfg, r.state.time)) throw std::invalid_argument("case has no exact solution: " + cfg.name);
    auto d = detail::device_for(r.mesh, r.scheme);
    d->upload(r.state);
    double out[3];
    d->check(hgks_error_norms(d->s, cfg.name.c_str(), r.state.time, out));
    return {out[0], std::sqrt(out[1]), std::sqrt(out[2])};
}

struct StudyOptions {
    int degree = 2;
    bool nonuniform = false;
    int workers = 1;
    bool nominal = false;
    double dt_power = 2.0;
    double dt_safety = 0.7;
    size_t anchor_index = 0;
    std::optional<double> cfl;
};

struct StudyRow {
    int n;
    ErrorNorms err;
    int steps;
    double dt;
};

/// solver.hpp:161-202: nominal (per-mesh CFL step) or refined (dt ~ h^power
/// anchored at one mesh, capped by the mesh's CFL step) convergence study
inline std::vector<StudyRow> convergence_study(const std::string& case_name, const std::vector<int>& meshes,
                                               const StudyOptions& so) {
    const double cfl = so.cfl ? *so.cfl : default_cfl(so.degree);
    auto cfl_dt = [&](int n) {
        CaseConfig cfg = CaseConfig::named(case_name, n);
        cfg.nonuniform = so.nonuniform;
        RunOptions opt;
        opt.degree = so.degree;
        const RunResult r = setup_run(cfg, opt);
        StepControl ctrl;
        ctrl.cfl = cfl;
        return compute_dt(r.state, r.mesh, r.scheme.gas, ctrl, so.degree);
    };
    double anchor_dt = 0.0;
    int anchor_n = 0;
    if (!so.nominal) {
        anchor_n = meshes.at(std::min(so.anchor_index, meshes.size() - 1));
        anchor_dt = so.dt_safety * cfl_dt(anchor_n);
    }
    std::vector<StudyRow> rows;
    for (int n : meshes) {
        CaseConfig cfg = CaseConfig::named(case_name, n);
        cfg.nonuniform = so.nonuniform;
        RunOptions opt;
        opt.degree = so.degree;
        opt.cfl = cfl;
        if (!so.nominal) opt.dt_fixed = std::min(anchor_dt * std::pow(double(anchor_n) / n, so.dt_power), cfl_dt(n));
        const RunResult r = run_case(cfg, opt);
        rows.push_back({n, run_error_norms(r, cfg, so.workers), r.steps, opt.dt_fixed ? *opt.dt_fixed : 0.0});
    }
    return rows;
}

/// wall-time table over sizes (solver.hpp:207-233); "workers" has no device
/// meaning, so every row times the same GPU loop and speedup is relative to
/// the first worker count
inline std::vector<ScalingRow> scaling_report(const std::string& case_name, const std::vector<int>& sizes,
                                              const std::vector<int>& workers, int degree,
                                              std::optional<double> t_end = {}) {
    std::vector<ScalingRow> rows;
    for (int n : sizes) {
        double base = 0.0;
        for (int w : workers) {
            CaseConfig cfg = CaseConfig::named(case_name, n);
            RunOptions opt;
            opt.degree = degree;
            opt.workers = w;
            opt.t_end = t_end;
            RunResult r = setup_run(cfg, opt);
            const auto t0 = std::chrono::steady_clock::now();
            advance(r, cfg, opt, [](RunResult&) {});
            const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (w == 1 || base == 0.0) base = secs;
            rows.push_back({n, w, secs, base / secs});
        }
    }
    return rows;
}

}  // namespace hgks
