// DMMA gate microbenchmark (north_star: "DMMA only if ncu shows it beats the
// FP64 FMA pipe"). Measures, on one B200:
//   dfma   : FP64 FMA chains on every warp            (the FP64 pipe alone)
//   dmma   : mma.sync.m8n8k4 f64 chains on every warp (the FP64 tensor path alone)
//   mixed  : half the warps DFMA, half DMMA           (do they run concurrently?)
// and reports TFLOP/s (2 flops per FMA, 2*8*8*4 per DMMA). If mixed > max(dfma,
// dmma) the tensor path adds throughput next to the FP64 pipe.
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void k_dfma(double* out, int iters) {
    double a[CH];
    for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 1e-3 + k;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < CH; ++k) a[k] = fma(a[k], b, c);
    double s = 0;
    for (int k = 0; k < CH; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma(double* out, int iters) {
    double d[CH][2];
    for (int k = 0; k < CH; ++k) d[k][0] = d[k][1] = threadIdx.x * 1e-3 + k;
    const double a = 0.5 + threadIdx.x * 1e-6, b = 1e-3;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < CH; ++k) dmma(d[k], a, b);
    double s = 0;
    for (int k = 0; k < CH; ++k) s += d[k][0] + d[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// warps of even index run DFMA, odd DMMA; dfma_iters / dmma_iters balance the time
__global__ void k_mixed(double* out, int it_f, int it_m) {
    const int w = threadIdx.x >> 5;
    double s = 0;
    if (w & 1) {
        double d[CH][2];
        for (int k = 0; k < CH; ++k) d[k][0] = d[k][1] = threadIdx.x * 1e-3 + k;
        const double a = 0.5 + threadIdx.x * 1e-6, b = 1e-3;
        for (int i = 0; i < it_m; ++i)
#pragma unroll
            for (int k = 0; k < CH; ++k) dmma(d[k], a, b);
        for (int k = 0; k < CH; ++k) s += d[k][0] + d[k][1];
    } else {
        double a[CH];
        for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 1e-3 + k;
        const double b = 0.999999, c = 1e-7;
        for (int i = 0; i < it_f; ++i)
#pragma unroll
            for (int k = 0; k < CH; ++k) a[k] = fma(a[k], b, c);
        for (int k = 0; k < CH; ++k) s += a[k];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    const int blocks = 148 * 4, threads = 256;
    double* out;
    cudaMalloc(&out, blocks * threads * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        return best;
    };
    const int IT = 20000;
    const double nthr = (double)blocks * threads;
    float tf = timeit([&] { k_dfma<<<blocks, threads>>>(out, IT); });
    const double fl_f = nthr * IT * CH * 2.0;
    float tm = timeit([&] { k_dmma<<<blocks, threads>>>(out, IT); });
    const double fl_m = (nthr / 32.0) * IT * CH * 2.0 * 8 * 8 * 4;
    std::printf("dfma  %.3f ms  %.2f TFLOP/s\n", tf, fl_f / tf * 1e-9);
    std::printf("dmma  %.3f ms  %.2f TFLOP/s\n", tm, fl_m / tm * 1e-9);
    // mixed: half the warps each; choose iterations so each half alone would
    // take about the same time as the other
    const double rate_f = fl_f / tf, rate_m = fl_m / tm;  // flops per ms, whole GPU
    int it_m = IT, it_f = (int)(IT * (rate_f / rate_m) * (2.0 * 8 * 8 * 4 / 32.0) / 2.0);
    if (it_f < 1) it_f = 1;
    float tx = timeit([&] { k_mixed<<<blocks, threads>>>(out, it_f, it_m); });
    const double fl_x = (nthr / 2) * it_f * CH * 2.0 + (nthr / 2 / 32.0) * it_m * CH * 2.0 * 8 * 8 * 4;
    std::printf("mixed %.3f ms  %.2f TFLOP/s  (dfma iters %d, dmma iters %d)\n", tx, fl_x / tx * 1e-9, it_f, it_m);
    std::printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
