// Microbenchmark: per-SM throughput of DMUL / DFMA / DADD on this GPU, and
// the cfg1 chain floor (49,023 chains x 1,024 separately rounded steps) with
// the product taken by DMUL or by DFMA(x, h, +0) (the same rounded product).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int K>
__global__ void tput(double *out, double a, int n) {
    double x[K];
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = a + threadIdx.x + k;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (OP == 0) x[k] = __dadd_rn(x[k], a);
            if (OP == 1) x[k] = __dmul_rn(x[k], a);
            if (OP == 2) x[k] = __fma_rn(x[k], a, a);
        }
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int R, bool FMA>
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
            for (int r = 0; r < R; ++r)
                acc[r] = __dadd_rn(acc[r], FMA ? __fma_rn(xv[u], h[r], 0.0) : __dmul_rn(xv[u], h[r]));
#pragma unroll
        for (int r = 0; r < R; ++r) h[r] = __dadd_rn(h[r], 1e-9);
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += acc[r];
    if (t * R < n_chains) out[t] = s;
}

static float time_ms(void (*f)(double *, int), double *d, int arg) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f(d, arg);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) f(d, arg);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 10;
}

template <int OP>
void run_tput(double *d, int sms) {
    const char *nm[] = {"DADD", "DMUL", "DFMA"};
    for (int warps = 4; warps <= 32; warps *= 2) {
        const int iters = 4096;
        auto f = [](double *dd, int w) {
            int s;
            cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, 0);
            tput<OP, 8><<<s, w * 32>>>(dd, 1.0000001, 4096);
        };
        const float ms = time_ms(f, d, warps);
        const double ops = (double)sms * warps * 32 * iters * 8;
        printf("%s throughput, %2d warps/SM x 8 chains: %.1f lane-ops/clk/SM at 1965 MHz\n", nm[OP], warps,
               ops / (ms * 1e-3) / sms / 1965e6);
    }
}

template <int R, bool FMA, int TBK>
void run_chain(double *d) {
    for (int steps = 1024; steps <= 2048; steps *= 2) {
        static int st;
        st = steps;
        auto f = [](double *dd, int s) {
            const int n = 49023, threads = (n + R - 1) / R;
            chains<R, FMA><<<(threads + TBK - 1) / TBK, TBK>>>(dd, n, s, 1.0, 0.5);
        };
        const float ms = time_ms(f, d, steps);
        printf("chain R=%d %s CTA=%3d steps=%d: %.2f us per launch (%.1f clk/step at 1965 MHz)\n", R,
               FMA ? "DFMA(x,h,0)" : "DMUL       ", TBK, steps, ms * 1e3, ms * 1e-3 * 1965e6 / steps);
    }
}


// products of u-block k+1 are taken in loop iteration k (the loop is not
// unrolled, so ptxas cannot sink them next to their DADDs)
template <int R>
__global__ void chains_sp(double *out, int n_chains, int steps, double x0, double h0) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc[R], h[R], xv[8], p[8][R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0, h[r] = h0 - r;
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = x0 + t + u;
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) p[u][r] = __dmul_rn(xv[u], h[r]);
#pragma unroll 1
    for (int s = 0; s < steps; s += 8) {
#pragma unroll
        for (int r = 0; r < R; ++r) h[r] = __dadd_rn(h[r], 1e-9);
        double q[8][R];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) q[u][r] = __dmul_rn(xv[u], h[r]);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = __dadd_rn(acc[r], p[u][r]);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) p[u][r] = q[u][r];
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += acc[r];
    if (t * R < n_chains) out[t] = s;
}

template <int R, int TBK>
void run_chain_sp(double *d) {
    for (int steps = 8; steps <= 2048; steps *= (steps == 8 ? 128 : 2)) {
        auto f = [](double *dd, int s) {
            const int n = 49023, threads = (n + R - 1) / R;
            chains_sp<R><<<(threads + TBK - 1) / TBK, TBK>>>(dd, n, s, 1.0, 0.5);
        };
        const float ms = time_ms(f, d, steps);
        printf("chain_sp R=%d CTA=%3d steps=%d: %.2f us per launch (%.1f clk/step at 1965 MHz)\n", R, TBK, steps,
               ms * 1e3, ms * 1e-3 * 1965e6 / steps);
    }
}

int main() {
    double *d;
    cudaMalloc(&d, 1 << 26);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run_chain_sp<1, 32>(d);
    run_chain_sp<1, 128>(d);
    run_chain_sp<2, 32>(d);
    run_chain_sp<4, 32>(d);
    run_chain<1, false, 32>(d);
    run_chain<1, true, 32>(d);
    run_chain<1, true, 64>(d);
    run_chain<1, true, 128>(d);
    run_chain<2, false, 32>(d);
    run_chain<2, true, 32>(d);
    run_chain<4, true, 32>(d);
    return 0;
}
