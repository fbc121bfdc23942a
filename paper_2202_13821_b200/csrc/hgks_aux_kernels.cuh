// Auxiliary device kernels: AoS<->SoA transforms at the ABI, inverse mass
// matrix, L2 projection of the case fields (dg.hpp:193-220, cases.hpp:78-137)
// and the Taylor-Green diagnostics (cases.hpp:165-204).
#pragma once

#include "hgks_kernels.cuh"

namespace hgks_dev {

// host AoS [(c*NC) + comp] (owned cells) <-> device SoA comp*cs + S + c.
// 32 cells per block, staged through shared memory so both sides coalesce.
// cells [cbeg, cend) of the owned range (cend < 0: all)
__global__ void aos_to_soa_kernel(KParams kp, const double* __restrict__ aos,
                                  double* __restrict__ soa, int NC, long cbeg = 0, long cend = -1) {
    __shared__ double st[100 * 33];
    const long ncell = cend < 0 ? (long)kp.S * kp.nzl : cend;
    for (long c0 = cbeg + (long)blockIdx.x * 32; c0 < ncell; c0 += (long)gridDim.x * 32) {
        const int nc = (int)min(32L, ncell - c0);
        for (int e = threadIdx.x; e < nc * NC; e += blockDim.x) {
            const int l = e / NC, comp = e - l * NC;
            st[comp * 33 + l] = aos[c0 * NC + e];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 32 * NC; e += blockDim.x) {
            const int l = e & 31, comp = e >> 5;
            if (l < nc) soa[comp * kp.cs + kp.S + c0 + l] = st[comp * 33 + l];
        }
        __syncthreads();
    }
}

__global__ void soa_to_aos_kernel(KParams kp, const double* __restrict__ soa,
                                  double* __restrict__ aos, int NC, long cbeg = 0, long cend = -1) {
    __shared__ double st[100 * 33];
    const long ncell = cend < 0 ? (long)kp.S * kp.nzl : cend;
    for (long c0 = cbeg + (long)blockIdx.x * 32; c0 < ncell; c0 += (long)gridDim.x * 32) {
        const int nc = (int)min(32L, ncell - c0);
        for (int e = threadIdx.x; e < 32 * NC; e += blockDim.x) {
            const int l = e & 31, comp = e >> 5;
            if (l < nc) st[comp * 33 + l] = soa[comp * kp.cs + kp.S + c0 + l];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nc * NC; e += blockDim.x) {
            const int l = e / NC, comp = e - l * NC;
            aos[c0 * NC + e] = st[comp * 33 + l];
        }
        __syncthreads();
    }
}

// L = R * (1/M_nn) in place (solver.hpp:42-54, mass_diag dg.hpp:42-50)
__global__ void inverse_mass_kernel(KParams kp, double* q, int NC) {
    const long ncell = (long)kp.S * kp.nzl;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < ncell * NC;
         e += (long)gridDim.x * blockDim.x) {
        const long c = e % ncell;
        const int comp = (int)(e / ncell);
        const int n = comp / 5;
        const int i = (int)(c % kp.nx), j = (int)((c / kp.nx) % kp.ny), k = (int)(c / kp.S);
        const double m = kp.dx[i] * kp.dy[j] * kp.dz[k + 1] / kp.tab[kp.off_massf + n];
        const double inv = 1.0 / m;
        double* p = q + comp * kp.cs + kp.S + c;
        *p = *p * inv;
    }
}

// ---------------------------------------------------------------- dt kernel
// compute_dt (integrator.hpp:27-45): min over owned cells of cfl h / (|U|+|V|+
// |W|+c) and the viscous bound. Positive doubles order like their bit
// patterns, so the min is an integer atomicMin (order independent, exact).
__global__ void dt_kernel(KParams kp, const double* __restrict__ q, double cfl, int degree,
                          unsigned long long* dt_bits) {
    const long n_owned = (long)kp.S * kp.nzl;
    double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < n_owned;
         c += (long)gridDim.x * blockDim.x) {
        const int i = (int)(c % kp.nx);
        const int j = (int)((c / kp.nx) % kp.ny);
        const int k = (int)(c / kp.S);
        const long g = c + kp.S;  // skip the ghost layer
        double avg[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) avg[v] = __ldg(q + v * kp.cs + g);
        Prim w;
        double bad = 0.0;
        const int rc = prim_from_q(avg, kp.gas, w, bad);
        if (rc) {
            const long item = (long)i + (long)kp.nx * (j + (long)kp.ny * (k + kp.kglob0));
            report_error(kp, err_key(0, 0, item, 0, 0, rc), bad);
            continue;
        }
        const double h = fmin(fmin(__ldg(kp.dx + i), __ldg(kp.dy + j)), __ldg(kp.dz + k + 1));
        const double p = 0.5 * w.rho / w.lam;
        const double cs = sqrt(kp.gas.gamma * p / w.rho);
        const double speed = fabs(w.U) + fabs(w.V) + fabs(w.W) + cs;
        const double cand = cfl * h / speed;
        if (cand < best) best = cand;
        if (kp.gas.mu > 0.0) {
            const double vis = cfl * h * h * w.rho / (2.0 * kp.gas.mu * (2.0 * degree + 1.0));
            if (vis < best) best = vis;
        }
    }
    // warp min then one atomic per warp (NaN never wins: comparisons are false)
    unsigned long long bits = (unsigned long long)__double_as_longlong(best);
    if (!(best >= 0.0)) bits = 0x7ff0000000000000ULL;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
        bits = other < bits ? other : bits;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(dt_bits, bits);
}

// ------------------------------------------------ step control on the device
// Key block (unsigned 64-bit words, solver-owned): the two dt words are
// min-reduced together across slabs (one 16-byte allreduce), the step key
// after stage 2.
enum : int { K_DTERR = 0, K_DT = 1, K_STEP = 2, K_FLUX = 3, K_SCRATCH = 4, K_WORDS = 8 };
constexpr unsigned long long kNoKey = ~0ull;
constexpr unsigned long long kInfBits = 0x7ff0000000000000ULL;

// step scalars for a host-given dt (hgks_step, residual, streamed step)
__global__ void set_scalars_kernel(double* scal, double dt, double mu) {
    scal[SC_DT] = dt;
    scal[SC_INV_DT] = dt != 0.0 ? 1.0 / dt : 0.0;
    scal[SC_RH] = mu > 0.0 ? dt / (4.0 * mu) : 0.0;
    scal[SC_ACTIVE] = 1.0;
}

// Control block of the device-resident advance loop (solver.hpp:90-107).
struct StepCtl {
    double t, t_end, next_record, record_interval, dt_fixed, mu;
    unsigned long long fail_key;  // the key that halted the loop (step or dt)
    int halted;                   // HALT_* below
    int record;                   // clip dt to the record cadence
    int steps;                    // committed steps
    int rec_hit;                  // the last committed step landed on a record time
};
enum : int { HALT_NONE = 0, HALT_DONE = 1, HALT_STEP = 2, HALT_DT_STATE = 3, HALT_DT = 4 };
// what the host reads back per step (pinned ring)
struct StepStatus {
    double t, dt;
    unsigned long long fail_key;
    int halted, steps, rec_hit, active;
};

// dt of the next step from the (reduced) dt words, clipped to t_end and the
// next record time exactly as advance does (solver.hpp:90-93); a halted or
// finished loop makes the step a no-op (SC_ACTIVE = 0).
__global__ void dt_finalize_kernel(StepCtl* c, const unsigned long long* keys, double* scal) {
    scal[SC_ACTIVE] = 0.0;
    if (c->halted) return;
    if (!(c->t < c->t_end - 1e-14 * c->t_end)) {
        c->halted = HALT_DONE;
        return;
    }
    double dt;
    if (c->dt_fixed > 0.0) {
        dt = c->dt_fixed;  // compute_dt's dt_fixed override (integrator.hpp:28)
    } else {
        if (keys[K_DTERR] != kNoKey) {
            c->halted = HALT_DT_STATE;
            c->fail_key = keys[K_DTERR];
            return;
        }
        dt = __longlong_as_double((long long)keys[K_DT]);
        if (!(dt > 0.0) || !isfinite(dt)) {  // integrator.hpp:43
            c->halted = HALT_DT;
            return;
        }
    }
    const double rem = c->t_end - c->t;
    dt = rem < dt ? rem : dt;  // std::min(dt, t_end - t)
    if (c->record) {
        const double rr = c->next_record - c->t;
        dt = rr < dt ? rr : dt;
    }
    scal[SC_DT] = dt;
    scal[SC_INV_DT] = 1.0 / dt;
    scal[SC_RH] = c->mu > 0.0 ? dt / (4.0 * c->mu) : 0.0;
    scal[SC_ACTIVE] = 1.0;
}

// After stage 2 (and the cross-slab key reduction): commit or halt, then
// re-arm the dt words for the next step and publish the status.
__global__ void commit_kernel(StepCtl* c, unsigned long long* keys, const double* scal, StepStatus* st) {
    const bool active = scal[SC_ACTIVE] != 0.0;
    if (active && !c->halted) {
        if (keys[K_STEP] != kNoKey) {
            c->halted = HALT_STEP;
            c->fail_key = keys[K_STEP];
        } else {
            c->t += scal[SC_DT];  // t += dt (solver.hpp:101)
            ++c->steps;
            c->rec_hit = 0;
            if (c->record && c->t >= c->next_record - 1e-12) {  // solver.hpp:104
                c->rec_hit = 1;
                c->next_record += c->record_interval;
            }
        }
    }
    keys[K_DT] = kInfBits;
    keys[K_DTERR] = kNoKey;
    st->t = c->t;
    st->dt = active ? scal[SC_DT] : 0.0;
    st->fail_key = c->fail_key;
    st->halted = c->halted;
    st->steps = c->steps;
    st->rec_hit = active && !c->halted ? c->rec_hit : 0;
    st->active = active ? 1 : 0;
}

// periodic single slab: ghost layer -1 <- layer nzl-1, ghost nzl <- layer 0
__global__ void ghost_wrap_kernel(KParams kp, double* q, int ncomp) {
    const long per = (long)kp.S;
    const long total = per * ncomp * 2;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long c = e % per;
        const long r = e / per;
        const int comp = (int)(r >> 1);
        const int top = (int)(r & 1);
        double* base = q + comp * kp.cs;
        if (top)
            base[(long)(kp.nzl + 1) * per + c] = base[per + c];
        else
            base[c] = base[(long)kp.nzl * per + c];
    }
}

// halo layers <-> contiguous buffers [send_lo|send_hi|recv_lo|recv_hi][comp][S]
__global__ void halo_pack_kernel(KParams kp, const double* __restrict__ a, double* __restrict__ buf, int NC) {
    const long L = (long)kp.S * NC;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < L; e += (long)gridDim.x * blockDim.x) {
        const long comp = e / kp.S, c = e - comp * kp.S;
        buf[e] = a[comp * kp.cs + kp.S + c];                      // owned layer 0
        buf[L + e] = a[comp * kp.cs + (long)kp.nzl * kp.S + c];  // owned layer nzl-1
    }
}

__global__ void halo_unpack_kernel(KParams kp, double* __restrict__ a, const double* __restrict__ buf, int NC) {
    const long L = (long)kp.S * NC;
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < L; e += (long)gridDim.x * blockDim.x) {
        const long comp = e / kp.S, c = e - comp * kp.S;
        a[comp * kp.cs + c] = buf[2 * L + e];                                // ghost below
        a[comp * kp.cs + (long)(kp.nzl + 1) * kp.S + c] = buf[3 * L + e];   // ghost above
    }
}

// FP64 pipe peak: DFMA_CHAINS independent dependency chains per thread
#define DFMA_CHAINS 8
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters) {
    double a[DFMA_CHAINS];
#pragma unroll
    for (int k = 0; k < DFMA_CHAINS; ++k) a[k] = threadIdx.x * 1e-3 + k;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < DFMA_CHAINS; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < DFMA_CHAINS; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

enum : int { CASE_ADV2D = 0, CASE_ADV3D = 1, CASE_VORTEX2D = 2, CASE_TGV = 3 };

struct CaseParams {
    int cid, dim;
    double gamma, mach0, eps, t;
    int npts;
};

// initial / exact fields (cases.hpp:78-124)
__device__ __forceinline__ void case_field(const CaseParams& c, const double* x, double* q) {
    const double pi = 3.14159265358979323846;
    if (c.cid == CASE_ADV2D || c.cid == CASE_ADV3D) {
        double s = x[0] + x[1] - 2.0 * c.t;
        if (c.cid == CASE_ADV3D) s = x[0] + x[1] + x[2] - 3.0 * c.t;
        const double rho = 1.0 + 0.2 * sin(pi * s);
        const double W = c.cid == CASE_ADV3D ? 1.0 : 0.0;
        const double E = 1.0 / (c.gamma - 1.0) + 0.5 * rho * (1.0 + 1.0 + W * W);
        q[0] = rho;
        q[1] = rho;
        q[2] = rho;
        q[3] = rho * W;
        q[4] = E;
    } else if (c.cid == CASE_VORTEX2D) {
        auto wrap = [](double v) {
            v = fmod(v, 10.0);
            if (v < -5.0) v += 10.0;
            if (v >= 5.0) v -= 10.0;
            return v;
        };
        const double dx = wrap(x[0] - 5.0 - c.t), dy = wrap(x[1] - 5.0 - c.t);
        const double r2 = dx * dx + dy * dy;
        const double g = c.eps / (2.0 * pi) * exp(0.5 * (1.0 - r2));
        const double U = 1.0 - g * dy, V = 1.0 + g * dx;
        const double T = 1.0 - (c.gamma - 1.0) * c.eps * c.eps / (8.0 * c.gamma * pi * pi) * exp(1.0 - r2);
        const double rho = pow(T, 1.0 / (c.gamma - 1.0));
        const double p = rho * T;
        q[0] = rho;
        q[1] = rho * U;
        q[2] = rho * V;
        q[3] = 0.0;
        q[4] = p / (c.gamma - 1.0) + 0.5 * rho * (U * U + V * V);
    } else {
        const double p0 = 1.0 / (c.gamma * c.mach0 * c.mach0);
        const double U = sin(x[0]) * cos(x[1]) * cos(x[2]);
        const double V = -cos(x[0]) * sin(x[1]) * cos(x[2]);
        const double p = p0 + (cos(2.0 * x[0]) + cos(2.0 * x[1])) * (cos(2.0 * x[2]) + 2.0) / 16.0;
        const double rho = p / p0;
        q[0] = rho;
        q[1] = rho * U;
        q[2] = rho * V;
        q[3] = 0.0;
        q[4] = p / (c.gamma - 1.0) + 0.5 * rho * (U * U + V * V);
    }
}

// project (dg.hpp:193-220): one thread per owned cell, (k+2)^3 points
template <int NC>
__global__ void __launch_bounds__(128) project_kernel(KParams kp, CaseParams cp,
                                                      const double* __restrict__ ctr,
                                                      double* __restrict__ q, long ncell,
                                                      const double* __restrict__ samples, long c0) {
    // samples (optional): the field at the projection points of cells
    // [c0, c0 + ncell), [(cell - c0) * npts + p][5], evaluated by the caller
    // (a host-side field function, dg.hpp:193); else the named case's field
    constexpr int N = NC / 5;
    const long c = c0 + blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (c >= c0 + ncell) return;
    const int i = (int)(c % kp.nx), j = (int)((c / kp.nx) % kp.ny), k = (int)(c / kp.S);
    const double h[3] = {kp.dx[i], kp.dy[j], kp.dz[k + 1]};
    const double x0[3] = {ctr[i], ctr[kp.nx + j], ctr[kp.nx + kp.ny + k]};
    double acc[NC];
#pragma unroll
    for (int m = 0; m < NC; ++m) acc[m] = 0.0;
    for (int p = 0; p < cp.npts; ++p) {
        const double* r = kp.tab + kp.off_pref + 3 * p;
        const double x[3] = {x0[0] + 0.5 * h[0] * r[0], x0[1] + 0.5 * h[1] * r[1], x0[2] + 0.5 * h[2] * r[2]};
        double f[5];
        if (samples) {
#pragma unroll
            for (int v = 0; v < 5; ++v) f[v] = samples[((c - c0) * cp.npts + p) * 5 + v];
        } else {
            case_field(cp, x, f);
        }
        const double wq = kp.tab[kp.off_pw + p];
        const double* B = kp.tab + kp.off_pB + p * N;
#pragma unroll
        for (int n = 0; n < N; ++n) {
            const double wb = wq * B[n];
#pragma unroll
            for (int v = 0; v < 5; ++v) acc[n * 5 + v] += wb * f[v];
        }
    }
#pragma unroll
    for (int n = 0; n < N; ++n) {
        const double bn = kp.tab[kp.off_massf + n] / 8.0;
#pragma unroll
        for (int v = 0; v < 5; ++v) q[(n * 5 + v) * kp.cs + kp.S + c] = acc[n * 5 + v] * bn;
    }
}

// tgv_diagnostics partial sums (cases.hpp:165-204): per block
// {sum vjac*ek, sum vjac*ens, sum vol}, fixed-order tree inside the block
template <int NC>
__global__ void __launch_bounds__(256) tgv_kernel(KParams kp, int npts,
                                                  const double* __restrict__ q, long ncell,
                                                  double* __restrict__ part) {
    constexpr int N = NC / 5;
    __shared__ double red[3][256];
    double se = 0, sz = 0, sv = 0;
    for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < ncell;
         c += (long)gridDim.x * blockDim.x) {
        const int i = (int)(c % kp.nx), j = (int)((c / kp.nx) % kp.ny), k = (int)(c / kp.S);
        const double h[3] = {kp.dx[i], kp.dy[j], kp.dz[k + 1]};
        const double vjac = h[0] * h[1] * h[2] / 8.0;
        double co[NC];
#pragma unroll
        for (int m = 0; m < NC; ++m) co[m] = q[m * kp.cs + kp.S + c];
        double ek = 0, ens = 0;
        for (int p = 0; p < npts; ++p) {
            const double* B = kp.tab + kp.off_pB + p * N;
            const double* dB = kp.tab + kp.off_pdB + p * 3 * N;
            double e[20];
#pragma unroll
            for (int m = 0; m < 20; ++m) e[m] = 0.0;
#pragma unroll
            for (int n = 0; n < N; ++n) {
#pragma unroll
                for (int v = 0; v < 5; ++v) {
                    const double cv = co[n * 5 + v];
                    e[v] += B[n] * cv;
                    e[5 + v] += dB[n] * cv;
                    e[10 + v] += dB[N + n] * cv;
                    e[15 + v] += dB[2 * N + n] * cv;
                }
            }
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                e[5 + v] *= 2.0 / h[0];
                e[10 + v] *= 2.0 / h[1];
                e[15 + v] *= 2.0 / h[2];
            }
            const double inv = 1.0 / e[0];
            const double U = e[1] * inv, V = e[2] * inv, W = e[3] * inv;
            const double wq = kp.tab[kp.off_pw + p];
            ek += wq * 0.5 * (e[1] * U + e[2] * V + e[3] * W);
            const double vel[4] = {0.0, U, V, W};
#define DVEL(comp, ax) ((e[5 + 5 * (ax) + (comp)] - vel[comp] * e[5 + 5 * (ax)]) * inv)
            const double wx = DVEL(3, 1) - DVEL(2, 2);
            const double wy = DVEL(1, 2) - DVEL(3, 0);
            const double wz = DVEL(2, 0) - DVEL(1, 1);
#undef DVEL
            ens += wq * 0.5 * e[0] * (wx * wx + wy * wy + wz * wz);
        }
        se += vjac * ek;
        sz += vjac * ens;
        sv += h[0] * h[1] * h[2];
    }
    red[0][threadIdx.x] = se;
    red[1][threadIdx.x] = sz;
    red[2][threadIdx.x] = sv;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int r = 0; r < 3; ++r) red[r][threadIdx.x] += red[r][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int r = 0; r < 3; ++r) part[3 * blockIdx.x + r] = red[r][0];
}

inline void launch_project(int degree, int dim, const KParams& kp, const CaseParams& cp,
                           const double* ctr, double* q, long ncell, cudaStream_t st,
                           const double* samples = nullptr, long c0 = 0) {
    const int blocks = (int)((ncell + 127) / 128);
    const int NC = 5 * (dim == 3 ? (degree == 1 ? 4 : degree == 2 ? 10 : 20) : (degree == 2 ? 6 : 10));
    if (NC == 20) project_kernel<20><<<blocks, 128, 0, st>>>(kp, cp, ctr, q, ncell, samples, c0);
    else if (NC == 30) project_kernel<30><<<blocks, 128, 0, st>>>(kp, cp, ctr, q, ncell, samples, c0);
    else if (NC == 50) project_kernel<50><<<blocks, 128, 0, st>>>(kp, cp, ctr, q, ncell, samples, c0);
    else project_kernel<100><<<blocks, 128, 0, st>>>(kp, cp, ctr, q, ncell, samples, c0);
}

inline void launch_tgv(int degree, int dim, const KParams& kp, int npts, const double* q, long ncell,
                       double* part, int blocks, cudaStream_t st) {
    const int NC = 5 * (dim == 3 ? (degree == 1 ? 4 : degree == 2 ? 10 : 20) : (degree == 2 ? 6 : 10));
    if (NC == 20) tgv_kernel<20><<<blocks, 256, 0, st>>>(kp, npts, q, ncell, part);
    else if (NC == 30) tgv_kernel<30><<<blocks, 256, 0, st>>>(kp, npts, q, ncell, part);
    else if (NC == 50) tgv_kernel<50><<<blocks, 256, 0, st>>>(kp, npts, q, ncell, part);
    else tgv_kernel<100><<<blocks, 256, 0, st>>>(kp, npts, q, ncell, part);
}

// error_norms (dg.hpp:228-266) partial sums per block: {sum vol/8 l1_c,
// sum vol/8 l2_c, sum vol davg^2} with the (k+2)^3 projection rule; fixed-
// order tree inside the block (deterministic)
template <int N>
__global__ void __launch_bounds__(256) error_kernel(KParams kp, CaseParams cp, const double* __restrict__ ctr,
                                                    const double* __restrict__ q, long ncell,
                                                    double* __restrict__ part,
                                                    const double* __restrict__ rho_samples) {
    // rho_samples (optional): the exact density at the projection points,
    // [cell * npts + p], evaluated by the caller (dg.hpp:228 takes a function)
    __shared__ double red[3][256];
    double s1 = 0, s2 = 0, sc = 0;
    for (long c = blockIdx.x * (long)blockDim.x + threadIdx.x; c < ncell; c += (long)gridDim.x * blockDim.x) {
        const int i = (int)(c % kp.nx), j = (int)((c / kp.nx) % kp.ny), k = (int)(c / kp.S);
        const double h[3] = {kp.dx[i], kp.dy[j], kp.dz[k + 1]};
        const double x0[3] = {ctr[i], ctr[kp.nx + j], ctr[kp.nx + kp.ny + k]};
        const double vol = h[0] * h[1] * h[2];
        double rho_c[N];
#pragma unroll
        for (int n = 0; n < N; ++n) rho_c[n] = q[(n * 5) * kp.cs + kp.S + c];
        double l1 = 0, l2 = 0, avg = 0;
        for (int p = 0; p < cp.npts; ++p) {
            const double* r = kp.tab + kp.off_pref + 3 * p;
            const double x[3] = {x0[0] + 0.5 * h[0] * r[0], x0[1] + 0.5 * h[1] * r[1], x0[2] + 0.5 * h[2] * r[2]};
            double f[5];
            if (rho_samples) f[0] = rho_samples[c * cp.npts + p];
            else case_field(cp, x, f);
            const double* B = kp.tab + kp.off_pB + p * N;
            double rh = 0;
#pragma unroll
            for (int n = 0; n < N; ++n) rh += B[n] * rho_c[n];
            const double d = fabs(f[0] - rh);
            const double w = kp.tab[kp.off_pw + p];
            l1 += w * d;
            l2 += w * d * d;
            avg += w * f[0];
        }
        avg /= 8.0;
        const double davg = avg - rho_c[0];
        s1 += vol / 8.0 * l1;
        s2 += vol / 8.0 * l2;
        sc += vol * davg * davg;
    }
    red[0][threadIdx.x] = s1;
    red[1][threadIdx.x] = s2;
    red[2][threadIdx.x] = sc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int r = 0; r < 3; ++r) red[r][threadIdx.x] += red[r][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int r = 0; r < 3; ++r) part[3 * blockIdx.x + r] = red[r][0];
}

inline void launch_error(int degree, int dim, const KParams& kp, const CaseParams& cp, const double* ctr,
                         const double* q, long ncell, double* part, int blocks, cudaStream_t st,
                         const double* rho_samples = nullptr) {
    const int N = dim == 3 ? (degree == 1 ? 4 : degree == 2 ? 10 : 20) : (degree == 2 ? 6 : 10);
    if (N == 4) error_kernel<4><<<blocks, 256, 0, st>>>(kp, cp, ctr, q, ncell, part, rho_samples);
    else if (N == 6) error_kernel<6><<<blocks, 256, 0, st>>>(kp, cp, ctr, q, ncell, part, rho_samples);
    else if (N == 10) error_kernel<10><<<blocks, 256, 0, st>>>(kp, cp, ctr, q, ncell, part, rho_samples);
    else error_kernel<20><<<blocks, 256, 0, st>>>(kp, cp, ctr, q, ncell, part, rho_samples);
}

}  // namespace hgks_dev
