// Floor of cfg1's structure: 49,023 independent float64 chains of 1,024
// steps (acc = acc + x*h, separately rounded), operands in registers --
// no memory traffic.  R chains per thread, 32-thread CTAs.
#include <cstdio>
#include <cuda_runtime.h>

template <int R>
__global__ void chains(double *out, int n_chains, int steps, double x0, double h0) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc[R], h[R], xv[8];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0, h[r] = h0 - r;
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = x0 + t + u;
    for (int s = 0; s < steps; s += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = __dadd_rn(acc[r], __dmul_rn(xv[u], h[r]));
#pragma unroll
        for (int r = 0; r < R; ++r) h[r] = __dadd_rn(h[r], 1e-9);  // one op per 8 steps keeps the loop honest
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += acc[r];
    if (t * R < n_chains) out[t] = s;
}

template <int R>
void run(double *d) {
    const int n = 49023, threads = (n + R - 1) / R;
    const int grid = (threads + 31) / 32;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains<R><<<grid, 32>>>(d, n, 1024, 1.0, 0.5);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) chains<R><<<grid, 32>>>(d, n, 1024, 1.0, 0.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("R=%d: %.2f us per launch (1024 steps x 49,023 chains, DMUL + DADD per step, operands in registers)\n", R, ms * 100);
}

int main() {
    double *d;
    cudaMalloc(&d, 1 << 20);
    run<1>(d);
    run<2>(d);
    run<4>(d);
    return 0;
}
