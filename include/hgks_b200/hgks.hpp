// hgks_b200/hgks.hpp — C++ drop-in for the reference's hot path, backed by
// the B200 kernels through the C ABI (include/hgks_b200.h).
//
// A reference user replaces
//     #include "hgks/hgks.hpp"         (proj/include/hgks/hgks.hpp)
// with
//     #include "hgks_b200/hgks.hpp"
// and links libhgks_b200.so. The names, argument meanings, layouts and
// exception types of the hot path are the reference's:
//
//   GasModel::make            core.hpp:35-42
//   Mesh::make / cell_index   mesh.hpp:22-37
//   Scheme::make              dg.hpp:274-280
//   DGState                   dg.hpp:18-38   (AoS [(c*N+n)*5+v])
//   ResidualWorkspace         dg.hpp:286-303 (R, Rt, face[3], count_fluxes,
//                                             flux_evaluations, resize)
//   residual(...)             dg.hpp:354, :452
//   detail::apply_inverse_mass solver.hpp:42
//   StepControl, compute_dt   integrator.hpp:11-45
//   TwoStageScratch, two_stage_step integrator.hpp:47-75
//   invalid_state_error, non_positive_density, non_positive_pressure,
//   worker_error, non_positive_dt  core.hpp:58-70, runtime.hpp:37-41,
//                                  integrator.hpp:17-19
//
// The workspace owns the device solver (one per mesh/scheme), created by
// ResidualWorkspace::resize exactly where the reference sizes its buffers.
// Every computation runs on the GPU; there is no host fallback.
#pragma once

#include <array>
#include <atomic>
#include <cmath>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../hgks_b200.h"

namespace hgks {

// ------------------------------------------------------------ exceptions
struct invalid_state_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct non_positive_density : invalid_state_error {
    using invalid_state_error::invalid_state_error;
};
struct non_positive_pressure : invalid_state_error {
    using invalid_state_error::invalid_state_error;
};
struct worker_error : std::runtime_error {
    int item;
    worker_error(int item_, const std::string& what) : std::runtime_error(what), item(item_) {}
};
struct non_positive_dt : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------- gas, mesh
struct GasModel {
    double gamma;
    double K;
    double Pr = 1.0;
    double mu_ref = 0.0;
    static GasModel make(double gamma, double mu = 0.0) {
        GasModel g;
        g.gamma = gamma;
        g.K = (5.0 - 3.0 * gamma) / (gamma - 1.0);
        g.mu_ref = mu;
        if (g.K < 0.0) throw std::invalid_argument("GasModel: gamma gives negative internal dof");
        return g;
    }
};

struct Mesh {
    int nx = 0, ny = 0, nz = 0;
    std::vector<double> xs, ys, zs;
    static Mesh make(std::vector<double> x, std::vector<double> y, std::vector<double> z) {
        Mesh m;
        m.nx = static_cast<int>(x.size()) - 1;
        m.ny = static_cast<int>(y.size()) - 1;
        m.nz = static_cast<int>(z.size()) - 1;
        m.xs = std::move(x);
        m.ys = std::move(y);
        m.zs = std::move(z);
        for (const auto* v : {&m.xs, &m.ys, &m.zs})
            for (size_t i = 1; i < v->size(); ++i)
                if (!((*v)[i] > (*v)[i - 1]))
                    throw std::invalid_argument("Mesh: node coordinates must be strictly increasing");
        return m;
    }
    int ncells() const { return nx * ny * nz; }
    int cell_index(int i, int j, int k) const { return i + nx * (j + ny * k); }
    std::array<double, 3> widths(int c) const {
        const int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
        return {xs[i + 1] - xs[i], ys[j + 1] - ys[j], zs[k + 1] - zs[k]};
    }
    double volume(int c) const {
        const auto h = widths(c);
        return h[0] * h[1] * h[2];
    }
};

struct BasisSet {
    int degree = 2, dim = 3, N = 0;
};

struct Scheme {
    BasisSet basis;
    GasModel gas;
    static Scheme make(int degree, int dim, const GasModel& gas) {
        if (degree < 1 || degree > 3) throw std::invalid_argument("build_basis: degree must be 2 or 3");
        if (dim != 2 && dim != 3) throw std::invalid_argument("build_basis: dim must be 2 or 3");
        Scheme s;
        s.basis.degree = degree;
        s.basis.dim = dim;
        int n = 0;
        for (int a = 0; a <= degree; ++a)
            for (int b = 0; b <= degree; ++b)
                for (int c = 0; c <= (dim == 3 ? degree : 0); ++c)
                    if (a + b + c <= degree) ++n;
        s.basis.N = n;
        s.gas = gas;
        return s;
    }
};

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

// ------------------------------------------------------- device handle
namespace detail {

inline void throw_from(hgks_solver* s, int rc) {
    const std::string msg = hgks_last_error(s);
    if (rc == HGKS_ERR_STATE) {
        int code = 0, phase = -1;
        long item = -1;
        double value = 0;
        hgks_error_info(s, &code, &phase, &item, &value);
        if (phase == 0 || phase == 1) throw worker_error(static_cast<int>(item), msg);
        if (msg.find("density") != std::string::npos) throw non_positive_density(msg);
        throw non_positive_pressure(msg);
    }
    if (rc == HGKS_ERR_DT) throw non_positive_dt(msg);
    if (rc == HGKS_ERR_CONFIG) throw std::invalid_argument(msg);
    throw device_error(msg);
}

struct Device {
    hgks_solver* s = nullptr;
    int nx = -1, ny = -1, nz = -1, degree = -1, dim = -1;
    double gamma = 0, mu = -1;
    std::vector<double> xs, ys, zs;

    ~Device() {
        if (s) hgks_destroy(s);
    }
    bool matches(const Mesh& m, const Scheme& sch) const {
        return s && m.nx == nx && m.ny == ny && m.nz == nz && sch.basis.degree == degree &&
               sch.basis.dim == dim && sch.gas.gamma == gamma && sch.gas.mu_ref == mu &&
               m.xs == xs && m.ys == ys && m.zs == zs;
    }
    void open(const Mesh& m, const Scheme& sch, int device = 0) {
        if (matches(m, sch)) return;
        if (s) hgks_destroy(s);
        s = nullptr;
        hgks_config cfg{};
        cfg.nx = m.nx;
        cfg.ny = m.ny;
        cfg.nz = m.nz;
        cfg.xs = m.xs.data();
        cfg.ys = m.ys.data();
        cfg.zs = m.zs.data();
        cfg.degree = sch.basis.degree;
        cfg.dim = sch.basis.dim;
        cfg.gamma = sch.gas.gamma;
        cfg.mu = sch.gas.mu_ref;
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
        nx = m.nx;
        ny = m.ny;
        nz = m.nz;
        degree = sch.basis.degree;
        dim = sch.basis.dim;
        gamma = sch.gas.gamma;
        mu = sch.gas.mu_ref;
        xs = m.xs;
        ys = m.ys;
        zs = m.zs;
    }
    void check(int rc) const {
        if (rc != HGKS_OK) throw_from(s, rc);
    }
};

// process-wide device for the calls whose reference signature carries no
// workspace (apply_inverse_mass, compute_dt)
inline Device& shared_device() {
    static Device d;
    return d;
}

}  // namespace detail

// Partition is accepted for signature parity; the device ignores it.
struct Partition {
    int workers = 1;
    static Partition make(int, int w) {
        if (w < 1) throw std::invalid_argument("Partition: worker count must be >= 1");
        Partition p;
        p.workers = w;
        return p;
    }
};

struct ResidualWorkspace {
    std::array<std::vector<double>, 3> face;  // [face*(npts*10) + p*10 + (F|Ft)]
    std::vector<double> R, Rt;                // [(cell*N + n)*5 + var]
    Partition cells, faces;
    bool count_fluxes = false;
    std::atomic<long> flux_evaluations{0};
    std::shared_ptr<detail::Device> dev = std::make_shared<detail::Device>();
    int device = 0;

    void resize(const Mesh& mesh, const Scheme& sch, int workers) {
        dev->open(mesh, sch, device);
        const size_t n = static_cast<size_t>(mesh.ncells()) * sch.basis.N * 5;
        for (int a = 0; a < 3; ++a)
            face[a].assign(static_cast<size_t>(mesh.ncells()) * hgks_face_points(dev->s, a) * 10, 0.0);
        R.assign(n, 0.0);
        Rt.assign(n, 0.0);
        cells = Partition::make(mesh.ncells(), workers);
        faces = Partition::make(3 * mesh.ncells(), workers);
    }
};

/// residual (dg.hpp:354): fills ws.R, ws.Rt and ws.face on the GPU.
inline void residual(const double* coeffs, const Mesh& mesh, const Scheme& sch, double dt,
                     ResidualWorkspace& ws) {
    ws.dev->open(mesh, sch, ws.device);
    if (ws.R.size() != static_cast<size_t>(mesh.ncells()) * sch.basis.N * 5) ws.resize(mesh, sch, 1);
    hgks_set_count_fluxes(ws.dev->s, ws.count_fluxes ? 1 : 0);
    ws.dev->check(hgks_residual(ws.dev->s, coeffs, dt, ws.R.data(), ws.Rt.data(), ws.face[0].data(),
                                ws.face[1].data(), ws.face[2].data()));
    if (ws.count_fluxes) ws.flux_evaluations += hgks_flux_evaluations(ws.dev->s);
}

inline void residual(const DGState& s, const Mesh& mesh, const Scheme& sch, double dt,
                     ResidualWorkspace& ws) {
    residual(s.coeffs.data(), mesh, sch, dt, ws);
}

namespace detail {
/// apply_inverse_mass (solver.hpp:42-54) on the GPU.
inline void apply_inverse_mass(const std::vector<double>& R, std::vector<double>& L, const Mesh& mesh,
                               const BasisSet& basis, const Partition&) {
    Scheme sch;
    sch.basis = basis;
    sch.gas = GasModel::make(1.4);
    Device& d = shared_device();
    d.open(mesh, sch);
    L.resize(R.size());
    d.check(hgks_apply_inverse_mass(d.s, R.data(), L.data()));
}
}  // namespace detail

// ---------------------------------------------------------- integrator
struct StepControl {
    double cfl = 0.15;
    double t_end = 1.0;
    std::optional<double> dt_fixed;
};

inline double default_cfl(int degree) { return degree == 2 ? 0.15 : 0.09; }

/// compute_dt (integrator.hpp:27-45) on the GPU.
inline double compute_dt(const DGState& s, const Mesh& mesh, const GasModel& gas,
                         const StepControl& ctrl, int degree) {
    if (ctrl.dt_fixed) return *ctrl.dt_fixed;
    // the state's basis size tells the dimension (3-D: 4 / 10 / 20 for P1 / P2 / P3)
    const int n3 = degree == 1 ? 4 : degree == 2 ? 10 : 20;
    const Scheme sch = Scheme::make(degree, s.N == n3 ? 3 : 2, gas);
    detail::Device& d = detail::shared_device();
    d.open(mesh, sch);
    d.check(hgks_set_state(d.s, s.coeffs.data(), s.time));
    double dt = 0.0;
    d.check(hgks_compute_dt(d.s, ctrl.cfl, &dt));
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

/// The solver.hpp:81-88 eval (residual + inverse mass, same full dt in both
/// stages) as a device object; two_stage_step below runs the whole S2O4
/// step on the GPU for it.
struct DeviceEval {
    ResidualWorkspace* ws;
};

/// two_stage_step (integrator.hpp:64-75) with the device eval: one fused
/// device step on the caller's host vector (host->device, step, device->host).
inline void two_stage_step(std::vector<double>& q, double dt, DeviceEval eval, TwoStageScratch&) {
    eval.ws->dev->check(hgks_two_stage_step_host(eval.ws->dev->s, q.data(), dt));
}

/// Generic two_stage_step for an arbitrary eval callback (integrator.hpp:64-75).
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

/// advance's inner loop (solver.hpp:90-107) device-resident: steps `state` to
/// t_end with CFL (or fixed) dt clipped to t_end and the record cadence;
/// state errors get " at t=<t>" appended as the reference does.
inline int advance_device(DGState& state, const Mesh& mesh, const Scheme& sch, const StepControl& ctrl,
                          double record_interval, ResidualWorkspace& ws) {
    ws.dev->open(mesh, sch, ws.device);
    ws.dev->check(hgks_set_state(ws.dev->s, state.coeffs.data(), state.time));
    int steps = 0;
    const int rc = hgks_advance(ws.dev->s, ctrl.t_end, ctrl.cfl, ctrl.dt_fixed ? *ctrl.dt_fixed : 0.0,
                                record_interval, &steps);
    if (rc == HGKS_ERR_STATE) throw invalid_state_error(hgks_last_error(ws.dev->s));
    ws.dev->check(rc);
    ws.dev->check(hgks_get_state(ws.dev->s, state.coeffs.data(), &state.time));
    return steps;
}

}  // namespace hgks
