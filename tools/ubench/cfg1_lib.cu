// cfg1 through the library's C ABI (sc_fir_full, float64, ordered): per-launch
// device time (a) back to back, (b) one launch between events after an L2
// flush (bench.py's method).  SC_CHAIN_SMALL=0 selects the windowed chain.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "scatterconv_b200.h"

int main(int argc, char **argv) {
    const int64_t ne = argc > 1 ? atoll(argv[1]) : 48000, nh = argc > 2 ? atoll(argv[2]) : 1024, no = ne + nh - 1;
    printf("ne=%lld nh=%lld ", (long long)ne, (long long)nh);
    std::vector<double> x(ne), h(nh);
    srand(1);
    for (auto &v : x) v = 2.0 * rand() / RAND_MAX - 1.0;
    for (auto &v : h) v = 2.0 * rand() / RAND_MAX - 1.0;
    double *dx, *dh, *dy;
    char *flush;
    cudaMalloc(&dx, ne * 8);
    cudaMalloc(&dh, nh * 8);
    cudaMalloc(&dy, no * 8);
    cudaMalloc(&flush, 256 << 20);
    cudaMemcpy(dx, x.data(), ne * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dh, h.data(), nh * 8, cudaMemcpyHostToDevice);
    cudaStream_t s;
    cudaStreamCreate(&s);
    auto call = [&] {
        if (sc_fir_full(SC_F64, SC_MODE_ORDERED, dx, ne, dh, nh, dy, SC_SKIP_NONE, 0.0, s) != 0) {
            printf("error %s\n", sc_last_error());
            exit(1);
        }
    };
    for (int i = 0; i < 5; ++i) call();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 50; ++i) call();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("back to back: %.2f us per launch\n", ms * 1e3 / 50);
    float tot = 0;
    for (int i = 0; i < 50; ++i) {
        cudaMemsetAsync(flush, i, 256 << 20, s);
        cudaEventRecord(e0, s);
        call();
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
    }
    printf("single launch after L2 flush: %.2f us\n", tot * 1e3 / 50);
    tot = 0;
    for (int i = 0; i < 50; ++i) {
        cudaEventRecord(e0, s);
        call();
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
    }
    printf("single launch, warm L2: %.2f us\n", tot * 1e3 / 50);
    return 0;
}
