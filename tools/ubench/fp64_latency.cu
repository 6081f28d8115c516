// Microbenchmark: dependent-chain latency and per-SM throughput of DADD/DMUL/
// FFMA on this GPU (informs the ordered-chain kernel's outputs-per-thread).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dadd(double *out, double a, int n, long long *cyc) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_ffma(float *out, float a, int n, long long *cyc) {
    float x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __fmaf_rn(x, a, a);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
// throughput: K independent chains per thread, many warps
template <int K>
__global__ void tput_dadd(double *out, double a, int n) {
    double x[K];
    for (int k = 0; k < K; ++k) x[k] = a + threadIdx.x + k;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = __dadd_rn(x[k], a);
    double s = 0;
    for (int k = 0; k < K; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double *d; float *f; long long *c;
    cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 20); cudaMalloc(&c, 8);
    const int n = 1 << 16;
    long long cyc;
    chain_dadd<<<1, 32>>>(d, 1e-300, n, c); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f clk\n", (double)cyc / n);
    chain_ffma<<<1, 32>>>(f, 1e-30f, n, c); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent latency: %.2f clk\n", (double)cyc / n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps = 4; warps <= 32; warps *= 2) {
        const int iters = 4096;
        tput_dadd<8><<<sms, warps * 32>>>(d, 1e-300, iters);
        cudaEventRecord(e0);
        tput_dadd<8><<<sms, warps * 32>>>(d, 1e-300, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)sms * warps * 32 * iters * 8;
        printf("DADD throughput, %2d warps/SM x 8 chains: %.1f Gop/s = %.1f lane-ops/clk/SM (clock %d MHz)\n",
               warps, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    return 0;
}
