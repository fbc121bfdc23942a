// TEST INFRASTRUCTURE: compiles the product's __host__ __device__ kinetics
// (paper_2202_13821_b200/csrc/hgks_kinetics.cuh) for the CPU so the
// restructured moment algebra is checked against the reference here, without
// a GPU. Built by tests/conftest.py into tests/native/_build/.
#include "hgks_kinetics.cuh"

using namespace hgks_dev;

static GasC gas_of(double gamma, double mu) {
    GasC g;
    g.gamma = gamma;
    g.gm1 = gamma - 1.0;
    g.K = (5.0 - 3.0 * gamma) / (gamma - 1.0);
    g.D = g.K + 3.0;
    g.mu = mu;
    g.four_D = 4.0 / g.D;
    return g;
}

extern "C" {

// linearised interface flux: F[5], Ft[5]; returns ERR_* and stage
int hk_interface_flux(const double* tl, const double* tr, double gamma, double tau, double dt,
                      double* F, double* Ft, int* stage, double* bad) {
    const GasC g = gas_of(gamma, 0.0);
    const TimeW tw = time_weights(tau, dt);
    int st = -1;
    double b = 0;
    const int rc = tau > 0.0 ? interface_flux<true>(tl, tr, g, tw, F, Ft, st, b)
                             : interface_flux<false>(tl, tr, g, tw, F, Ft, st, b);
    if (stage) *stage = st;
    if (bad) *bad = b;
    return rc;
}

// linearised smooth flux along 3 axes: out[30] = (F_a[5], Ft_a[5]) per axis
int hk_smooth_flux(const double* t, double gamma, double mu, double* out, double* bad) {
    const GasC g = gas_of(gamma, mu);
    double b = 0;
    const int rc = mu > 0.0 ? smooth_flux<true, 3>(t, g, out, b) : smooth_flux<false, 3>(t, g, out, b);
    if (bad) *bad = b;
    return rc;
}

void hk_time_weights(double tau, double dt, double* w12) {
    const TimeW w = time_weights(tau, dt);
    const double v[12] = {w.g0F, w.g0Ft, w.abF, w.abFt, w.AbF, w.AbFt,
                          w.f0F, w.f0Ft, w.anF, w.anFt, w.AnF, w.AnFt};
    for (int i = 0; i < 12; ++i) w12[i] = v[i];
}
}
