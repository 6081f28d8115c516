// Kernel-boundary cost on this GPU: a chain of N dependent tiny kernels,
// (a) plain stream launches, (b) PDL launches (programmatic stream
// serialisation, griddepcontrol in the kernel), (c)/(d) the same captured
// into a CUDA graph and replayed.  Per-kernel time = total / N.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(float *p, int pdl) {
    if (pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (threadIdx.x == 0) p[blockIdx.x] += 1.0f;
}

static void launch(cudaStream_t s, float *p, int grid, bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? at : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_tiny, p, (int)pdl);
}

int main() {
    float *p;
    cudaMalloc(&p, 1 << 20);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int N = 20;
    for (int grid : {148, 600}) {
        for (int pdl = 0; pdl < 2; ++pdl) {
            for (int i = 0; i < N; ++i) launch(s, p, grid, pdl);
            cudaStreamSynchronize(s);
            float best = 1e9, ms;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0, s);
                for (int i = 0; i < N; ++i) launch(s, p, grid, pdl);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("grid %4d stream %s: %.2f us per kernel\n", grid, pdl ? "PDL  " : "plain", best * 1e3 / N);
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < N; ++i) launch(s, p, grid, pdl);
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
            best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0, s);
                cudaGraphLaunch(ge, s);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("grid %4d graph  %s: %.2f us per kernel\n", grid, pdl ? "PDL  " : "plain", best * 1e3 / N);
        }
    }
    // one kernel between two events: plain launch vs a one-node graph
    for (int grid : {148, 511}) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        launch(s, p, grid, false);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        float tp = 0, tg = 0, ms;
        for (int r = 0; r < 50; ++r) {
            cudaStreamSynchronize(s);
            cudaEventRecord(e0, s);
            launch(s, p, grid, false);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            tp += ms;
            cudaEventRecord(e0, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            tg += ms;
        }
        printf("grid %4d single kernel between events: plain %.2f us, one-node graph %.2f us\n", grid, tp * 1e3 / 50,
               tg * 1e3 / 50);
    }
    return 0;
}
