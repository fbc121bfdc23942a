// The C++ drop-in (include/hgks_b200/hgks.hpp) exercised the way the
// reference's own suites exercise hgks:: (proj/tests/test_runtime.cpp,
// test_solver.cpp, test_integrator.cpp), plus parity against the oracle
// (oracle/hgks_oracle.c, test infrastructure). Built and run by
// tests/test_gpu_dropin.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hgks_b200/hgks.hpp"

extern "C" {
#include "../../oracle/hgks_oracle.h"
}

using namespace hgks;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
        }                                                                        \
    } while (0)
#define TEST_CASE(name) static void name()

namespace {

std::vector<double> nodes(double lo, double hi, int n, bool nonuniform) {  // cases.hpp:50-57
    std::vector<double> v(n + 1);
    for (int i = 0; i <= n; ++i) {
        const double xi = lo + (hi - lo) * i / n;
        v[i] = nonuniform ? xi + 0.05 * std::sin(M_PI * xi) : xi;
    }
    return v;
}

struct Setup {
    Mesh mesh;
    Scheme sch;
    DGState state;
    orc_solver* orc = nullptr;
    ~Setup() { orc_free(orc); }
};

// the oracle projects the case (setup_run); the drop-in starts from that state
void setup(Setup& S, const char* name, int n, int degree, bool nonuni) {
    orc_error e{};
    S.orc = orc_setup(name, n, degree, nonuni ? 1 : 0, &e);
    const bool tgv = std::strcmp(name, "tgv") == 0;
    const bool two_d = name[3] == '2' || std::strcmp(name, "vortex2d") == 0;
    const double lo = tgv ? -M_PI : 0.0, hi = tgv ? M_PI : (std::strcmp(name, "vortex2d") == 0 ? 10.0 : 2.0);
    S.mesh = Mesh::make(nodes(lo, hi, n, nonuni), nodes(lo, hi, n, nonuni),
                        two_d ? std::vector<double>{lo, hi} : nodes(lo, hi, n, nonuni));
    S.sch = Scheme::make(degree, two_d ? 2 : 3, GasModel::make(1.4, tgv ? 1.0 / 1600 : 0.0));
    S.state = DGState::zeros(S.mesh.ncells(), S.sch.basis.N);
    std::memcpy(S.state.coeffs.data(), orc_state(S.orc), S.state.coeffs.size() * sizeof(double));
}

double rel(const std::vector<double>& a, const double* b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num = std::fmax(num, std::fabs(a[i] - b[i]));
        den = std::fmax(den, std::fabs(b[i]));
    }
    return den > 0 ? num / den : num;
}

}  // namespace

TEST_CASE(residual_matches_oracle) {
    for (auto [name, n, deg, nu] : {std::tuple{"adv3d", 4, 2, true}, std::tuple{"tgv", 6, 2, false},
                                    std::tuple{"tgv", 4, 3, false}}) {
        Setup S;
        setup(S, name, n, deg, nu);
        ResidualWorkspace ws;
        ws.resize(S.mesh, S.sch, 4);
        double dt = 0;
        orc_error e{};
        orc_compute_dt(S.orc, deg == 2 ? 0.15 : 0.09, &dt, &e);
        residual(S.state, S.mesh, S.sch, dt, ws);
        std::vector<double> R(ws.R.size()), Rt(ws.R.size());
        orc_residual(S.orc, nullptr, dt, R.data(), Rt.data(), nullptr, nullptr, nullptr, nullptr, &e);
        CHECK(rel(ws.R, R.data()) <= 1e-12);
        CHECK(rel(ws.Rt, Rt.data()) <= 1e-10);
    }
}

// test_runtime.cpp:63-78
TEST_CASE(each_face_flux_once) {
    Setup S;
    setup(S, "adv3d", 6, 2, false);
    ResidualWorkspace ws;
    ws.resize(S.mesh, S.sch, 4);
    ws.count_fluxes = true;
    residual(S.state, S.mesh, S.sch, 1e-3, ws);
    const long expected = 3L * S.mesh.ncells() * 4;
    CHECK(ws.flux_evaluations.load() == expected);
    residual(S.state, S.mesh, S.sch, 1e-3, ws);
    CHECK(ws.flux_evaluations.load() == 2 * expected);
}

// test_runtime.cpp:80-101: bitwise identical across worker counts
TEST_CASE(bitwise_across_workers) {
    Setup S;
    setup(S, "adv3d", 8, 2, false);
    std::vector<double> ref;
    for (int w : {1, 2, 4, 8}) {
        ResidualWorkspace ws;
        ws.resize(S.mesh, S.sch, w);
        residual(S.state, S.mesh, S.sch, 1e-3, ws);
        if (w == 1) ref = ws.R;
        else CHECK(std::memcmp(ref.data(), ws.R.data(), ref.size() * sizeof(double)) == 0);
    }
}

// test_solver.cpp:22-53, with the reference's own eval lambda (solver.hpp:81-88)
TEST_CASE(conservation_over_steps) {
    Setup S;
    setup(S, "adv2d", 8, 2, false);
    auto totals = [&] {
        std::array<double, 5> t{};
        for (int c = 0; c < S.mesh.ncells(); ++c)
            for (int v = 0; v < 5; ++v) t[v] += S.mesh.volume(c) * S.state.coeff(c, 0, v);
        return t;
    };
    const auto before = totals();
    StepControl ctrl;
    ctrl.cfl = 0.15;
    const Partition cp = Partition::make(S.mesh.ncells(), 2);
    ResidualWorkspace ws;
    ws.resize(S.mesh, S.sch, 2);
    TwoStageScratch scratch;
    double step_dt = 0;
    auto eval = [&](const std::vector<double>& q, std::vector<double>& L, std::vector<double>& Lt) {
        L.resize(q.size());
        Lt.resize(q.size());
        residual(q.data(), S.mesh, S.sch, step_dt, ws);
        detail::apply_inverse_mass(ws.R, L, S.mesh, S.sch.basis, cp);
        detail::apply_inverse_mass(ws.Rt, Lt, S.mesh, S.sch.basis, cp);
    };
    for (int s = 0; s < 20; ++s) {
        step_dt = compute_dt(S.state, S.mesh, S.sch.gas, ctrl, 2);
        two_stage_step(S.state.coeffs, step_dt, eval, scratch);
        const auto now = totals();
        for (int v = 0; v < 5; ++v)
            CHECK(std::fabs(now[v] - before[v]) <= 1e-12 * std::fmax(1.0, std::fabs(before[v])) * (s + 1));
    }
}

// the fused device step equals the generic eval path and the oracle
TEST_CASE(device_step_matches_eval_path_and_oracle) {
    Setup S;
    setup(S, "tgv", 6, 2, false);
    ResidualWorkspace ws;
    ws.resize(S.mesh, S.sch, 1);
    TwoStageScratch scratch;
    StepControl ctrl;
    std::vector<double> q = S.state.coeffs;
    for (int s = 0; s < 5; ++s) {
        DGState st = S.state;
        st.coeffs = q;
        const double dt = compute_dt(st, S.mesh, S.sch.gas, ctrl, 2);
        two_stage_step(q, dt, DeviceEval{&ws}, scratch);
        orc_error e{};
        orc_step(S.orc, dt, &e);
    }
    CHECK(rel(q, orc_state(S.orc)) <= 1e-10);
}

// test_integrator.cpp:13-24
TEST_CASE(compute_dt_rest_gas) {
    const Mesh mesh = Mesh::make({0.0, 0.1, 0.2}, {0.0, 0.1, 0.2}, {0.0, 0.1, 0.2});
    DGState s = DGState::zeros(mesh.ncells(), 10);
    for (int c = 0; c < mesh.ncells(); ++c) {
        s.coeff(c, 0, 0) = 1.0;
        s.coeff(c, 0, 4) = 1.0 / 0.4;
    }
    StepControl ctrl;
    ctrl.cfl = 0.15;
    const double dt = compute_dt(s, mesh, GasModel::make(1.4), ctrl, 2);
    CHECK(std::fabs(dt - 0.15 * 0.1 / std::sqrt(1.4)) <= 1e-12 * dt);
    ctrl.dt_fixed = 0.123;
    CHECK(compute_dt(s, mesh, GasModel::make(1.4), ctrl, 2) == 0.123);
}

// test_solver.cpp:122-140
TEST_CASE(blowup_is_diagnosable) {
    Setup S;
    setup(S, "adv3d", 6, 2, false);
    S.state.coeff(2, 0, 0) = 1.0;
    S.state.coeff(2, 0, 1) = 10.0;
    S.state.coeff(2, 0, 4) = 1.0;
    ResidualWorkspace ws;
    ws.resize(S.mesh, S.sch, 2);
    bool threw = false;
    try {
        residual(S.state, S.mesh, S.sch, 1e-3, ws);
    } catch (const worker_error& e) {
        threw = true;
        CHECK(std::string(e.what()).find("pressure") != std::string::npos);
        CHECK(std::string(e.what()).rfind("item ", 0) == 0);
    }
    CHECK(threw);
    bool threw_dt = false;
    try {
        StepControl ctrl;
        compute_dt(S.state, S.mesh, S.sch.gas, ctrl, 2);
    } catch (const invalid_state_error&) {
        threw_dt = true;
    } catch (const non_positive_dt&) {
        threw_dt = true;
    }
    CHECK(threw_dt);
}

int main() {
    residual_matches_oracle();
    each_face_flux_once();
    bitwise_across_workers();
    conservation_over_steps();
    device_step_matches_eval_path_and_oracle();
    compute_dt_rest_gas();
    blowup_is_diagnosable();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
