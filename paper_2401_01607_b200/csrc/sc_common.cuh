// sc_common.cuh -- shared helpers for the scatterconv B200 library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/scatterconv_b200.h"

namespace sc {

// ------------------------------------------------------------------ errors

void set_error(const char *fmt, ...);

#define SC_CHECK_CUDA(expr)                                                            \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess) {                                                       \
            ::sc::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),   \
                            __FILE__, __LINE__);                                       \
            return SC_ERR_CUDA;                                                        \
        }                                                                              \
    } while (0)

void note_launch();  // bumps the sc_launch_count() counter
// records one k_tc_fir launch for sc_tc_stats (drain period, tile width, and
// the padded MACs of its MMAs: tiles x 128*tile_n outputs x 128 taps x shifts)
// and which kernel issued them (SC_TC_KERNEL_IMAGE / SC_TC_KERNEL_FUSED_SPLIT)
void note_tc_launch(int ssh, int tile_n, int64_t padded_macs, int kernel);
// counters around a CUDA-graph capture, re-applied on every replay
void note_launches(int64_t k);
int64_t launches_so_far();
void tc_stats_now(int64_t *launches, int64_t *padded, int *ssh, int *tile_n);
void note_tc_replay(int64_t launches, int64_t padded, int ssh, int tile_n);

#define SC_CHECK_LAUNCH()                                                              \
    do {                                                                               \
        ::sc::note_launch();                                                           \
        cudaError_t _e = cudaGetLastError();                                           \
        if (_e != cudaSuccess) {                                                       \
            ::sc::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), \
                            __FILE__, __LINE__);                                       \
            return SC_ERR_CUDA;                                                        \
        }                                                                              \
    } while (0)

#define SC_REQUIRE(cond, ...)                                                          \
    do {                                                                               \
        if (!(cond)) {                                                                 \
            ::sc::set_error(__VA_ARGS__);                                              \
            return SC_ERR_ARG;                                                         \
        }                                                                              \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();  // of the current device (cached per device)

// Grow-only per-device scratch buffer (workspace for split-K partials and
// padded taps).  Stream-ordered: a buffer is only reallocated after a
// cudaStreamSynchronize of the requesting stream.
void *scratch(size_t bytes, int slot, cudaStream_t stream, int *err);
// bumped whenever a scratch buffer is (re)allocated: cached CUDA graphs that
// captured scratch addresses are keyed by it
int64_t scratch_generation();
// while on: scratch(.., from) resolves to stream `to`'s buffers and never grows
void scratch_capture_alias(cudaStream_t from, cudaStream_t to, bool on);

// Small pinned host blocks from a process-wide pool (nullptr on failure).
void *pinned_small(size_t bytes);
void pinned_small_free(void *p);

// ------------------------------------------------------------------ exact arithmetic

// Separately rounded multiply then add: the reference's strict order
// (_kernels.py:1-8).  These never contract into FMA.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// One step of an ordered chain, acc + x*h.  float64: product and sum rounded
// separately -- the reference's exact arithmetic, hence bit-identical results.
// float32 (no bit-exact reference exists; the reference computes in float64):
// one fused multiply-add, i.e. a single rounding per step -- every float32
// ordered kernel uses this same step, so stream == batch and block-size
// invariance stay bit-exact in float32 too.
__device__ __forceinline__ double mac_rn(double acc, double x, double h) { return __dadd_rn(acc, __dmul_rn(x, h)); }
__device__ __forceinline__ float mac_rn(float acc, float x, float h) { return __fmaf_rn(x, h, acc); }
// FUSED = true: one rounding per step (fma) for double too -- the float64
// FAST mode (chain order kept, product rounding dropped; within 1e-12).
template <bool FUSED>
__device__ __forceinline__ double mac_step(double acc, double x, double h) {
    return FUSED ? __fma_rn(x, h, acc) : mac_rn(acc, x, h);
}
template <bool FUSED>
__device__ __forceinline__ float mac_step(float acc, float x, float h) { return mac_rn(acc, x, h); }

// Zero-skip predicates, compared in float64 like the reference (a float32
// sample widens exactly; the threshold is never rounded to float32).
template <int SKIP, typename T>
__device__ __forceinline__ bool skipped(T x, double thr) {
    if (SKIP == SC_SKIP_LE) return fabs((double)x) <= thr;       // core.py:164 (NaN not skipped)
    if (SKIP == SC_SKIP_NOT_GT) return !(fabs((double)x) > thr); // _kernels.py:33 (NaN skipped)
    return false;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels on a dependent chain (the FAST fused stream, the tensor-core FIR's
// prep -> MMA -> reduce) are launched with programmatic stream
// serialisation: the next kernel's launch and prologue overlap this one's
// tail.  Every such kernel calls pdl_begin() first: it lets its own
// successor launch and waits for its predecessors' memory (a no-op when the
// kernel was launched without the attribute).
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

#define SC_LAUNCH_PDL(...)                                                                  \
    do {                                                                                    \
        cudaError_t _e = ::sc::launch_pdl(__VA_ARGS__);                                     \
        if (_e != cudaSuccess) {                                                            \
            ::sc::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e),     \
                            __FILE__, __LINE__);                                            \
            return SC_ERR_CUDA;                                                             \
        }                                                                                   \
        ::sc::note_launch();                                                                \
    } while (0)

}  // namespace sc

// ------------------------------------------------------------------ internal launchers
// (implemented in the .cu files, used by capi.cu / engine.cu)

namespace sc {

struct ChainSeg {
    const void *h;    // taps of the IR active for drive samples [m_lo, m_hi)
    int64_t nh;
    int64_t m_lo, m_hi;
};
constexpr int kMaxSegs = 32;

// Ordered chain: outputs t in [t0, t0+n_out):
//   acc = init (init[t-t0] if t-t0 < init_len (host value, or *init_len_dev
//         when non-null), else +0)
//   for each seg, for m ascending in seg ∩ [t-nh+1, t]: unless skipped,
//         acc = acc + x[m - x_off] * h[t-m]   (separately rounded)
//   t-t0 < n_a -> out_a[t-t0], else out_b[t-t0-n_a]
int launch_chain(int dtype, int skip_mode, double threshold, const void *x, int64_t x_off,
                 const ChainSeg *segs, int nseg, const void *init, int64_t init_len,
                 const int64_t *init_len_dev, int64_t t0, int64_t n_out, void *out_a,
                 int64_t n_a, void *out_b, cudaStream_t stream, const unsigned *run_if = nullptr,
                 const struct ChainBatch *batch = nullptr, bool fused = false);

// Optional channel batching for launch_chain (grid.y = channel): channel c
// reads x + c*ldx, every segment's taps + c*ldh, its residue init + c*ld_init
// with length *(init_len_dev + c*ld_st), and writes out_a + c*ldo and
// out_b + c*ld_outb.
struct ChainBatch {
    int64_t channels, ldx, ldh, ldo;
    int64_t ld_init = 0, ld_outb = 0, ld_st = 0;
};

// Fast FP32 FIR over an output range (see k_fast_f32.cu).  With run_if set,
// every kernel of the launch exits immediately unless *run_if != 0.
int launch_fir_f32_fast(const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi,
                        const float *h, int64_t ldh, int64_t nh, float *y, int64_t ldy,
                        int64_t n_begin, int64_t n_end, int64_t channels, cudaStream_t stream,
                        const unsigned *run_if = nullptr);

// Per-channel max |x| / max |h| (float bit patterns at amax[2c], amax[2c+1])
// and the non-finite flag of a tensor-core FIR launch, computed by the caller
// in a pass it makes anyway (the engine's mask pass): the launch then skips
// its own max pass.
struct TcPre {
    const unsigned *amax;
    unsigned *flag;
};

// Tensor-core (tcgen05, FP16 hi/lo split, 3 MMAs) FP32-accurate FIR (k_tc_fir.cu).
// *nonfinite_out receives a device flag that is nonzero when an input sample
// is NaN/Inf; the tensor-core kernel then writes nothing and the caller's
// FFMA launch (gated on the same flag) produces the reference's NaN pattern.
bool tc_fir_supported(int64_t nh);
int launch_fir_f32_tc(const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi,
                      const float *h, int64_t ldh, int64_t nh, float *y, int64_t ldy, int64_t n_begin,
                      int64_t n_end, int64_t channels, cudaStream_t stream,
                      const unsigned **nonfinite_out, const TcPre *pre = nullptr,
                      bool *fallback_folded = nullptr);

// FAST-mode dispatch: tensor cores for long filters, FFMA2 kernel otherwise.
int launch_fir_f32(int mode, const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi,
                   const float *h, int64_t ldh, int64_t nh, float *y, int64_t ldy, int64_t n_begin,
                   int64_t n_end, int64_t channels, cudaStream_t stream, const TcPre *pre = nullptr);

int launch_direct_form(const double *e, int64_t ne, const double *h, int64_t nh, double *y,
                       unsigned *status, cudaStream_t stream);

}  // namespace sc
