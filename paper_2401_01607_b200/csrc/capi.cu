// capi.cu -- C ABI entry points for the whole-signal paths + shared runtime.
//
// Each sc_* function validates its arguments, picks the kernel for the
// requested dtype/mode and launches on the caller's stream.  See
// include/scatterconv_b200.h for the contract and the reference interface
// each entry point replaces.

#include <atomic>
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "sc_common.cuh"

namespace sc {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// tensor-core launch bookkeeping (sc_tc_stats): the work k_tc_fir issues
static std::atomic<int64_t> g_tc_launches{0}, g_tc_padded{0};
static std::atomic<int> g_tc_last_ssh{0}, g_tc_last_tn{0}, g_tc_last_kernel{SC_TC_KERNEL_NONE};
void note_launches(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
int64_t launches_so_far() { return g_launches.load(std::memory_order_relaxed); }

void note_tc_launch(int ssh, int tile_n, int64_t padded_macs, int kernel) {
    g_tc_last_kernel.store(kernel, std::memory_order_relaxed);
    g_tc_launches.fetch_add(1, std::memory_order_relaxed);
    g_tc_padded.fetch_add(padded_macs, std::memory_order_relaxed);
    g_tc_last_ssh.store(ssh, std::memory_order_relaxed);
    g_tc_last_tn.store(tile_n, std::memory_order_relaxed);
}

void tc_stats_now(int64_t *launches, int64_t *padded, int *ssh, int *tile_n) {
    *launches = g_tc_launches.load(std::memory_order_relaxed);
    *padded = g_tc_padded.load(std::memory_order_relaxed);
    *ssh = g_tc_last_ssh.load(std::memory_order_relaxed);
    *tile_n = g_tc_last_tn.load(std::memory_order_relaxed);
}

void note_tc_replay(int64_t launches, int64_t padded, int ssh, int tile_n) {
    if (launches <= 0) return;
    g_tc_launches.fetch_add(launches, std::memory_order_relaxed);
    g_tc_padded.fetch_add(padded, std::memory_order_relaxed);
    g_tc_last_ssh.store(ssh, std::memory_order_relaxed);
    g_tc_last_tn.store(tile_n, std::memory_order_relaxed);
}

// FAST mode routes long filters to the tensor-core kernel (validated on B200
// against the oracle, tests/test_tc_gpu.py).
static bool g_fast_uses_tc = true;

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int sm_count() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
    cache[dev] = n;
    return n;
}

// Small pinned host blocks (state read-backs; portable and mapped, so any
// device's kernels may store into them) carved from 256 KB arenas:
// cudaHostAlloc costs ~1 ms per call, far too much for a per-engine buffer.
namespace {
struct PinnedPool {
    static constexpr size_t kArena = 256 * 1024;
    std::mutex mu;
    std::map<size_t, std::vector<void *>> free_lists;  // size class -> blocks
    std::map<void *, size_t> owner;                     // block -> size class
    char *arena = nullptr;
    size_t arena_left = 0;
};
PinnedPool &pinned_pool() {
    static PinnedPool *p = new PinnedPool();  // never destroyed: blocks may outlive static teardown
    return *p;
}
}  // namespace

void *pinned_small(size_t bytes) {
    if (bytes == 0) return nullptr;
    PinnedPool &pp = pinned_pool();
    size_t cls = 64;
    while (cls < bytes) cls <<= 1;
    std::lock_guard<std::mutex> lk(pp.mu);
    auto &fl = pp.free_lists[cls];
    if (!fl.empty()) {
        void *p = fl.back();
        fl.pop_back();
        return p;
    }
    void *p = nullptr;
    if (cls > PinnedPool::kArena / 4) {
        if (cudaHostAlloc(&p, cls, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    } else {
        if (pp.arena_left < cls) {
            void *a = nullptr;
            if (cudaHostAlloc(&a, PinnedPool::kArena, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
            pp.arena = static_cast<char *>(a);
            pp.arena_left = PinnedPool::kArena;
        }
        p = pp.arena;
        pp.arena += cls;
        pp.arena_left -= cls;
    }
    pp.owner[p] = cls;
    return p;
}

void pinned_small_free(void *p) {
    if (!p) return;
    PinnedPool &pp = pinned_pool();
    std::lock_guard<std::mutex> lk(pp.mu);
    auto it = pp.owner.find(p);
    if (it != pp.owner.end()) pp.free_lists[it->second].push_back(p);  // reused by the next request
}

static std::atomic<int64_t> g_scratch_gen{0};
int64_t scratch_generation() { return g_scratch_gen.load(std::memory_order_relaxed); }

// Graph capture on a private stream stands in for a caller stream: scratch
// lookups from the capture stream resolve to the caller stream's buffers
// (the graph is launched there), and nothing may grow while capturing.
static thread_local cudaStream_t t_alias_from = nullptr, t_alias_to = nullptr;
static thread_local bool t_capturing = false;
void scratch_capture_alias(cudaStream_t from, cudaStream_t to, bool on) {
    t_alias_from = from;
    t_alias_to = to;
    t_capturing = on;
}

void *scratch(size_t bytes, int slot, cudaStream_t stream, int *err) {
    if (t_capturing && stream == t_alias_from) stream = t_alias_to;
    // Grow-only buffers keyed by (device, stream, slot): concurrent streams
    // (or host threads driving different devices) never share a buffer.
    struct Buf {
        void *p = nullptr;
        size_t n = 0;
    };
    static std::mutex mu;
    static std::map<std::tuple<int, uintptr_t, int>, Buf> bufs;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    Buf &b = bufs[std::make_tuple(dev, reinterpret_cast<uintptr_t>(stream), slot)];
    if (b.n < bytes && t_capturing) {
        set_error("scratch: would grow during graph capture");
        *err = SC_ERR_STATE;
        return nullptr;
    }
    if (b.n < bytes) {
        if (b.p) {
            // kernels queued on this stream may still read the old buffer
            cudaStreamSynchronize(stream);
            cudaFree(b.p);
            b.p = nullptr;
            b.n = 0;
        }
        size_t want = bytes + bytes / 4 + 256;
        if (cudaMalloc(&b.p, want) != cudaSuccess) {
            cudaGetLastError();
            set_error("scratch: cudaMalloc(%zu) failed", want);
            *err = SC_ERR_ALLOC;
            return nullptr;
        }
        b.n = want;
        g_scratch_gen.fetch_add(1, std::memory_order_relaxed);
    }
    *err = 0;
    return b.p;
}

constexpr int64_t kTcShortMinTaps = 26;  // see launch_fir_f32

int launch_fir_f32(int mode, const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi,
                   const float *h, int64_t ldh, int64_t nh, float *y, int64_t ldy, int64_t n_begin,
                   int64_t n_end, int64_t channels, cudaStream_t stream, const TcPre *pre) {
    bool tc = false, guard = false;
    if (mode == SC_MODE_TC) {
        tc = guard = true;
    } else if (mode == SC_MODE_FAST) {
        // tensor cores from 256 taps; from 26 taps too when the launch is big
        // enough to amortise their set-up: the fused-split kernel
        // (k_tc_fir_fs, no split image in HBM) takes a flat ~0.12 ms for
        // 2^26 outputs at any tap count up to 255 (HBM-bound), while the
        // CUDA-core short-filter kernels grow ~2.5 us per tap from 0.095 ms
        // at 16 taps (32 taps: 0.135 vs 0.120 ms on tensor cores)
        const double macs = (double)(n_end - n_begin) * (double)nh * (double)channels;
        tc = g_fast_uses_tc && (tc_fir_supported(nh) || (nh >= kTcShortMinTaps && macs >= 1073741824.0));
        guard = tc;
    } else if (mode != SC_MODE_FFMA) {
        set_error("fir: bad mode %d", mode);
        return SC_ERR_ARG;
    }
    if (!tc)
        return launch_fir_f32_fast(x, ldx, x_base, x_lo, x_hi, h, ldh, nh, y, ldy, n_begin, n_end,
                                   channels, stream);
    const unsigned *nonfinite = nullptr;
    bool folded = false;  // a split reduce already computes the flagged case
    int rc = launch_fir_f32_tc(x, ldx, x_base, x_lo, x_hi, h, ldh, nh, y, ldy, n_begin, n_end, channels,
                               stream, &nonfinite, pre, &folded);
    if (rc || !guard || !nonfinite || folded) return rc;
    // NaN/Inf inputs, and magnitudes whose power-of-two scales leave float
    // range (k_tc_fir.cu channel_scales), are routed (on the device, no host sync) to
    // the ORDERED kernel, which visits exactly the reference's (m, k) pairs
    // and so reproduces its NaN/Inf pattern (0*Inf included).  Each launch
    // exits immediately when the flag is clear.
    ChainSeg seg{h, nh, x_lo, x_hi};
    ChainBatch batch{channels, ldx, ldh, ldy};
    return launch_chain(SC_F32, SC_SKIP_NONE, 0.0, x, x_base, &seg, 1, nullptr, 0, nullptr, n_begin,
                        n_end - n_begin, y, n_end - n_begin, nullptr, stream, nonfinite, &batch);
}

static size_t dtype_size(int dtype) { return dtype == SC_F64 ? 8 : (dtype == SC_F32 ? 4 : 0); }

}  // namespace sc

using namespace sc;

extern "C" {

int sc_abi_version(void) { return SC_ABI_VERSION; }

int64_t sc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char *sc_last_error(void) { return g_err; }

int sc_tc_stats(int64_t *launches, int64_t *padded_macs, int *last_ssh, int *last_tile_n) {
    if (launches) *launches = g_tc_launches.load(std::memory_order_relaxed);
    if (padded_macs) *padded_macs = g_tc_padded.load(std::memory_order_relaxed);
    if (last_ssh) *last_ssh = g_tc_last_ssh.load(std::memory_order_relaxed);
    if (last_tile_n) *last_tile_n = g_tc_last_tn.load(std::memory_order_relaxed);
    return SC_OK;
}

int sc_tc_last_kernel(void) { return g_tc_last_kernel.load(std::memory_order_relaxed); }

void sc_tc_stats_reset(void) {
    g_tc_launches.store(0, std::memory_order_relaxed);
    g_tc_padded.store(0, std::memory_order_relaxed);
}

int sc_fir_full(int dtype, int mode, const void *x, int64_t ne, const void *h, int64_t nh,
                void *y, int skip_mode, double threshold, void *stream) {
    SC_REQUIRE(dtype_size(dtype) != 0, "sc_fir_full: bad dtype %d", dtype);
    SC_REQUIRE(ne >= 1, "sc_fir_full: input signal is empty");
    SC_REQUIRE(nh >= 1, "sc_fir_full: impulse response is empty");
    SC_REQUIRE(x && h && y, "sc_fir_full: null pointer");
    SC_REQUIRE(skip_mode >= SC_SKIP_NONE && skip_mode <= SC_SKIP_NOT_GT, "sc_fir_full: bad skip_mode");
    SC_REQUIRE(threshold >= 0.0, "sc_fir_full: threshold must be non-negative, got %g", threshold);
    const int64_t nout = ne + nh - 1;
    cudaStream_t st = as_stream(stream);
    if (mode != SC_MODE_ORDERED && dtype == SC_F32 && skip_mode == SC_SKIP_NONE) {
        return launch_fir_f32(mode, static_cast<const float *>(x), 0, 0, 0, ne,
                              static_cast<const float *>(h), 0, nh, static_cast<float *>(y), 0, 0, nout,
                              1, st);
    }
    // float64 outside ORDERED mode: the same chain with fused multiply-adds
    ChainSeg seg{h, nh, 0, ne};
    return launch_chain(dtype, skip_mode, threshold, x, 0, &seg, 1, nullptr, 0, nullptr, 0, nout,
                        y, nout, nullptr, st, nullptr, nullptr, dtype == SC_F64 && mode != SC_MODE_ORDERED);
}

int sc_fir_range(int dtype, int mode, const void *x, int64_t x_begin, int64_t x_end, const void *h,
                 int64_t nh, void *y, int64_t n_begin, int64_t n_end, void *stream) {
    SC_REQUIRE(dtype == SC_F32, "sc_fir_range: only float32 (fast mode) is supported");
    SC_REQUIRE(mode != SC_MODE_ORDERED, "sc_fir_range: ordered mode is not supported");
    SC_REQUIRE(nh >= 1, "sc_fir_range: impulse response is empty");
    SC_REQUIRE(x_end >= x_begin && n_end >= n_begin, "sc_fir_range: bad range");
    SC_REQUIRE(h && y && (x || x_end == x_begin), "sc_fir_range: null pointer");
    return launch_fir_f32(mode, static_cast<const float *>(x), 0, x_begin, x_begin, x_end,
                          static_cast<const float *>(h), 0, nh, static_cast<float *>(y), 0, n_begin,
                          n_end, 1, as_stream(stream));
}

int sc_fir_batched(int dtype, int mode, const void *x, int64_t ldx, const void *h, int64_t ldh,
                   void *y, int64_t ldy, int64_t channels, int64_t ne, int64_t nh, void *stream) {
    SC_REQUIRE(dtype == SC_F32, "sc_fir_batched: only float32 (fast mode) is supported");
    SC_REQUIRE(mode != SC_MODE_ORDERED, "sc_fir_batched: ordered mode is not supported");
    SC_REQUIRE(ne >= 1, "sc_fir_batched: input signal is empty");
    SC_REQUIRE(nh >= 1, "sc_fir_batched: impulse response is empty");
    SC_REQUIRE(channels >= 1, "sc_fir_batched: channels must be >= 1");
    SC_REQUIRE(ldx >= ne && ldh >= nh && ldy >= ne + nh - 1, "sc_fir_batched: bad leading dims");
    SC_REQUIRE(x && h && y, "sc_fir_batched: null pointer");
    return launch_fir_f32(mode, static_cast<const float *>(x), ldx, 0, 0, ne,
                          static_cast<const float *>(h), ldh, nh, static_cast<float *>(y), ldy, 0,
                          ne + nh - 1, channels, as_stream(stream));
}

int sc_direct_form(const double *e, int64_t ne, const double *h, int64_t nh, double *y, unsigned *status,
                   void *stream) {
    SC_REQUIRE(ne >= 1, "sc_direct_form: input signal is empty");
    SC_REQUIRE(nh >= 1, "sc_direct_form: impulse response is empty");
    SC_REQUIRE(e && h && y, "sc_direct_form: null pointer");
    return launch_direct_form(e, ne, h, nh, y, status, as_stream(stream));
}

}  // extern "C"
