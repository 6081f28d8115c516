// k_ordered.cu -- ordered ("strict") scatter-convolution kernels.
//
// Every output is computed as ONE chain over input index m ascending,
// starting from +0.0 (or from a carried residue), acc = acc + x[m]*h[t-m]
// (float64: product and sum rounded separately; float32: fused, see
// mac_rn in sc_common.cuh).  That is exactly the
// order in which the reference's scatter loops touch each slot:
//   core._scatter_full        pkg/src/scatterconv/core.py:80-92
//   _kernels.scatter_block    pkg/src/scatterconv/_kernels.py:31-51
// so float64 results are bit-identical to the reference, and streamed
// results equal batch results for every block partition (the residue carry
// continues the same chain).
//
// Gather form on the device: output-stationary, one thread per output slot,
// drive samples and taps staged through shared memory per 256-sample chunk.
// The drive chunk is a shared-memory broadcast; taps are read at consecutive
// addresses by consecutive threads (conflict-free).  Zero-skip predicates are
// warp-uniform (all threads of a chunk visit the same m).

#include <algorithm>

#include "sc_common.cuh"

namespace sc {
namespace {

constexpr int TB = 256;  // outputs per CTA
constexpr int MC = 256;  // drive samples per shared-memory chunk

template <typename T>
struct ChainArgs {
    const T *x;
    int64_t x_off;
    ChainSeg seg[kMaxSegs];
    int nseg;
    const T *init;
    int64_t init_len;
    const int64_t *init_len_dev;
    int64_t t0, n_out;
    T *out_a;
    int64_t n_a;
    T *out_b;
    double thr;
    const unsigned *run_if;  // optional device gate: run only if *run_if != 0
    int64_t ldx, ldh, ldo;   // channel strides (grid.y = channel); 0 = one channel
    int64_t ld_init, ld_outb, ld_st;
};

template <typename T, int SKIP>
__global__ void __launch_bounds__(TB) k_chain(ChainArgs<T> a) {
    __shared__ T xs[MC];
    __shared__ T hs[MC + TB - 1];
    if (a.run_if && *a.run_if == 0) return;  // block-uniform
    // batched channel (grid.y): channel-local base pointers (the param struct
    // itself is never written, so it stays in the constant bank)
    const T *xb = a.x + blockIdx.y * a.ldx;
    T *outa = a.out_a + blockIdx.y * a.ldo;
    const int64_t hoff = blockIdx.y * a.ldh;
    const T *initc = a.init ? a.init + blockIdx.y * a.ld_init : nullptr;
    T *outb = a.out_b ? a.out_b + blockIdx.y * a.ld_outb : nullptr;
    const int64_t n_tiles = (a.n_out + TB - 1) / TB;
    const int64_t init_len = a.init_len_dev ? a.init_len_dev[blockIdx.y * a.ld_st] : a.init_len;
    for (int64_t tb = blockIdx.x; tb < n_tiles; tb += gridDim.x) {
    __syncthreads();  // smem reuse across tiles of this CTA
    const int64_t tile0 = a.t0 + tb * TB;
    const int64_t t_end = a.t0 + a.n_out;
    const int64_t tile_last = (tile0 + TB < t_end ? tile0 + TB : t_end) - 1;
    const int64_t t = tile0 + threadIdx.x;
    const bool active = t < t_end;

    T acc = T(0);
    if (active && initc != nullptr && (t - a.t0) < init_len) acc = initc[t - a.t0];

    for (int s = 0; s < a.nseg; ++s) {
        const T *__restrict__ h = static_cast<const T *>(a.seg[s].h) + hoff;
        const int64_t nh = a.seg[s].nh;
        const int64_t m_lo = a.seg[s].m_lo, m_hi = a.seg[s].m_hi;
        const int64_t blo = tile0 - nh + 1 > m_lo ? tile0 - nh + 1 : m_lo;
        const int64_t bhi = tile_last + 1 < m_hi ? tile_last + 1 : m_hi;  // exclusive
        const int64_t my_lo = t - nh + 1 > m_lo ? t - nh + 1 : m_lo;
        const int64_t my_hi = t < m_hi - 1 ? t : m_hi - 1;  // inclusive
        for (int64_t mc = blo; mc < bhi; mc += MC) {
            __syncthreads();
            for (int i = threadIdx.x; i < MC; i += TB) {
                const int64_t m = mc + i;
                xs[i] = m < bhi ? xb[m - a.x_off] : T(0);
            }
            const int64_t kbase = tile0 - mc - MC + 1;
            for (int i = threadIdx.x; i < MC + TB - 1; i += TB) {
                const int64_t k = kbase + i;
                hs[i] = (k >= 0 && k < nh) ? h[k] : T(0);
            }
            __syncthreads();
            if (active) {
                const int64_t lo64 = my_lo > mc ? my_lo : mc;
                const int64_t hi64 = my_hi < mc + MC - 1 ? my_hi : mc + MC - 1;
                if (lo64 <= hi64) {
                    const int lo = (int)(lo64 - mc), hi = (int)(hi64 - mc);
                    const T *hp = hs + threadIdx.x + MC - 1;
#pragma unroll 4
                    for (int im = lo; im <= hi; ++im) {
                        const T xv = xs[im];
                        if (skipped<SKIP>(xv, a.thr)) continue;
                        acc = mac_rn(acc, xv, hp[-im]);
                    }
                }
            }
        }
    }
    if (active) {
        const int64_t i = t - a.t0;
        if (i < a.n_a)
            outa[i] = acc;
        else if (outb != nullptr)
            outb[i - a.n_a] = acc;
    }
    }  // tiles
}

// ---------------------------------------------------------------- register-tiled chain
// Same arithmetic and order as k_chain (each output: one ascending-m chain of
// separately rounded mul/add), but each thread carries RT_R consecutive
// outputs: per drive sample m the tap window slides by one, so with a
// rotating register window of RT_R + RT_U - 1 taps one shared-memory load
// feeds RT_R/ (RT_R+RT_U-1) * RT_U MACs instead of one.  Used for large
// ordered launches (whole signals in float64, fused streaming).  The tap
// stage is padded (one slot every 32 floats / 16 doubles) so the stride-RT_R
// accesses of a warp hit distinct banks.
constexpr int RT_TB = 128;
constexpr int RT_R = 8;
constexpr int RT_TILE = RT_TB * RT_R;  // 1024 outputs per CTA
constexpr int RT_MC = 128;            // drive samples per smem chunk
constexpr int RT_U = 8;               // m-steps per register window
static_assert(RT_MC == RT_TB, "one staged drive sample per thread (the scatter-mask ballot)");
static_assert(32 % RT_U == 0, "a u-block's scatter bits sit in one mask word");

template <typename T>
__device__ __forceinline__ int rt_pos(int i) {
    return sizeof(T) == 8 ? i + (i >> 4) : i + (i >> 5);
}

template <typename T, int SKIP>
__global__ void __launch_bounds__(RT_TB) k_chain_rt(ChainArgs<T> a) {
    constexpr int HS = RT_TILE + RT_MC - 1;
    __shared__ T xs[RT_MC];
    __shared__ unsigned xmask[RT_MC / 32];
    __shared__ T hs[HS + HS / 16 + 2];
    if (a.run_if && *a.run_if == 0) return;
    // batched channel (grid.y): channel-local base pointers (the param struct
    // itself is never written, so it stays in the constant bank)
    const T *xb = a.x + blockIdx.y * a.ldx;
    T *outa = a.out_a + blockIdx.y * a.ldo;
    const int64_t hoff = blockIdx.y * a.ldh;
    const T *initc = a.init ? a.init + blockIdx.y * a.ld_init : nullptr;
    T *outb = a.out_b ? a.out_b + blockIdx.y * a.ld_outb : nullptr;
    const int64_t n_tiles = (a.n_out + RT_TILE - 1) / RT_TILE;
    const int64_t t_end = a.t0 + a.n_out;
    const int64_t init_len = a.init_len_dev ? a.init_len_dev[blockIdx.y * a.ld_st] : a.init_len;
    for (int64_t tb = blockIdx.x; tb < n_tiles; tb += gridDim.x) {
        __syncthreads();
        const int64_t tile0 = a.t0 + tb * RT_TILE;
        const int64_t tile_last = (tile0 + RT_TILE < t_end ? tile0 + RT_TILE : t_end) - 1;
        const int64_t tj = tile0 + (int64_t)threadIdx.x * RT_R;  // this thread's first output
        T acc[RT_R];
#pragma unroll
        for (int r = 0; r < RT_R; ++r) {
            const int64_t t = tj + r;
            acc[r] = (initc != nullptr && t < t_end && (t - a.t0) < init_len) ? initc[t - a.t0] : T(0);
        }
        for (int s = 0; s < a.nseg; ++s) {
            const T *__restrict__ h = static_cast<const T *>(a.seg[s].h) + hoff;
            const int64_t nh = a.seg[s].nh;
            const int64_t m_lo = a.seg[s].m_lo, m_hi = a.seg[s].m_hi;
            const int64_t blo = tile0 - nh + 1 > m_lo ? tile0 - nh + 1 : m_lo;
            const int64_t bhi = tile_last + 1 < m_hi ? tile_last + 1 : m_hi;
            for (int64_t mc = blo; mc < bhi; mc += RT_MC) {
                __syncthreads();
                // stage the drive chunk and, by warp ballot, a bit per sample
                // that scatters (the zero-skip test runs once per sample, not
                // once per thread and sample)
                for (int i = threadIdx.x; i < RT_MC; i += RT_TB) {
                    const int64_t m = mc + i;
                    const T v = m < bhi ? xb[m - a.x_off] : T(0);
                    xs[i] = v;
                    const unsigned live_bits = __ballot_sync(0xffffffffu, m < bhi && !skipped<SKIP>(v, a.thr));
                    if ((i & 31) == 0) xmask[i >> 5] = live_bits;
                }
                const int64_t kbase = tile0 - mc - RT_MC + 1;
                for (int i = threadIdx.x; i < HS; i += RT_TB) {
                    const int64_t k = kbase + i;
                    hs[rt_pos<T>(i)] = (k >= 0 && k < nh) ? h[k] : T(0);
                }
                __syncthreads();
                const int mcount = (int)(bhi - mc < RT_MC ? bhi - mc : RT_MC);
                // every (output of the tile, m of the chunk) pair is a valid tap
                const bool full = (mc >= tile_last - nh + 1) && (mc + mcount - 1 <= tile0);
                // edge chunks: output r takes sample im iff lo_r <= im <= hi_r
                // (int32, relative to the chunk): m <= t and m > t - nh
                const int rel = (int)(tj - mc);  // t - m = rel + r - im
                const int hb = threadIdx.x * RT_R + RT_MC - 1;  // hs index of tap for (r=0, im=0)
                for (int im0 = 0; im0 < mcount; im0 += RT_U) {
                    T w[RT_R + RT_U - 1];  // w[q] = hs[hb - im0 - (RT_U-1) + q]
#pragma unroll
                    for (int q = 0; q < RT_R + RT_U - 1; ++q) w[q] = hs[rt_pos<T>(hb - im0 - (RT_U - 1) + q)];
                    // scatter bits of samples im0..im0+7 (RT_U = 8 divides 32)
                    const unsigned bits = (xmask[im0 >> 5] >> (im0 & 31)) & 0xFFu;
                    if (full && bits == 0xFFu) {
                        // common case (dense signal, interior chunk): no tests at all
#pragma unroll
                        for (int u = 0; u < RT_U; ++u) {
                            const T xv = xs[im0 + u];
#pragma unroll
                            for (int r = 0; r < RT_R; ++r) acc[r] = mac_rn(acc[r], xv, w[r - u + RT_U - 1]);
                        }
                    } else if (full) {
#pragma unroll
                        for (int u = 0; u < RT_U; ++u) {
                            if (!(bits & (1u << u))) continue;
                            const T xv = xs[im0 + u];
#pragma unroll
                            for (int r = 0; r < RT_R; ++r) acc[r] = mac_rn(acc[r], xv, w[r - u + RT_U - 1]);
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < RT_U; ++u) {
                            if (!(bits & (1u << u))) continue;
                            const T xv = xs[im0 + u];
#pragma unroll
                            for (int r = 0; r < RT_R; ++r) {
                                const int d = rel + r - (im0 + u);  // = t - m
                                if (d >= 0 && d < nh) acc[r] = mac_rn(acc[r], xv, w[r - u + RT_U - 1]);
                            }
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RT_R; ++r) {
            const int64_t t = tj + r;
            if (t < t_end) {
                const int64_t i = t - a.t0;
                if (i < a.n_a)
                    outa[i] = acc[r];
                else if (outb != nullptr)
                    outb[i - a.n_a] = acc[r];
            }
        }
    }
}

template <typename T>
int launch_chain_t(int skip_mode, double threshold, const void *x, int64_t x_off,
                   const ChainSeg *segs, int nseg, const void *init, int64_t init_len,
                   const int64_t *init_len_dev, int64_t t0, int64_t n_out, void *out_a,
                   int64_t n_a, void *out_b, cudaStream_t stream, const unsigned *run_if,
                   const ChainBatch *batch) {
    if (n_out <= 0) return SC_OK;
    SC_REQUIRE(nseg >= 0 && nseg <= kMaxSegs, "chain: bad segment count %d", nseg);
    ChainArgs<T> a{};
    a.x = static_cast<const T *>(x);
    a.x_off = x_off;
    for (int i = 0; i < nseg; ++i) a.seg[i] = segs[i];
    a.nseg = nseg;
    a.init = static_cast<const T *>(init);
    a.init_len = init_len;
    a.init_len_dev = init_len_dev;
    a.t0 = t0;
    a.n_out = n_out;
    a.out_a = static_cast<T *>(out_a);
    a.n_a = n_a;
    a.out_b = static_cast<T *>(out_b);
    a.thr = threshold;
    a.run_if = run_if;
    int64_t channels = 1;
    if (batch) {
        channels = batch->channels;
        a.ldx = batch->ldx;
        a.ldh = batch->ldh;
        a.ldo = batch->ldo;
        a.ld_init = batch->ld_init;
        a.ld_outb = batch->ld_outb;
        a.ld_st = batch->ld_st;
        SC_REQUIRE(channels >= 1 && channels < 65536, "chain: bad batch");
    }
    // Grid-stride over 256-output tiles.  A device-gated launch (run_if) is
    // usually a no-op, so it gets a small grid that exits in microseconds.
    const int64_t cap = run_if ? std::max<int64_t>(1, 4 * (int64_t)sm_count() / channels)
                               : (int64_t)INT32_MAX - 1;
    // Large launches: register-tiled variant (8 outputs/thread).  Small ones
    // (one streaming block) keep one output per thread for parallelism.
    static const int64_t rt_min = [] {
        const char *v = getenv("SC_CHAIN_RT_MIN");  // experiment knob (outputs)
        return v ? (int64_t)atoll(v) : (int64_t)2 * 148 * RT_TILE;
    }();
    if (n_out >= rt_min) {
        const dim3 grid((unsigned)std::min<int64_t>(cdiv(n_out, RT_TILE), cap), (unsigned)channels);
        switch (skip_mode) {
            case SC_SKIP_NONE: k_chain_rt<T, SC_SKIP_NONE><<<grid, RT_TB, 0, stream>>>(a); break;
            case SC_SKIP_LE: k_chain_rt<T, SC_SKIP_LE><<<grid, RT_TB, 0, stream>>>(a); break;
            case SC_SKIP_NOT_GT: k_chain_rt<T, SC_SKIP_NOT_GT><<<grid, RT_TB, 0, stream>>>(a); break;
            default: SC_REQUIRE(false, "chain: bad skip_mode %d", skip_mode);
        }
        SC_CHECK_LAUNCH();
        return SC_OK;
    }
    const dim3 grid((unsigned)std::min<int64_t>(cdiv(n_out, TB), cap), (unsigned)channels);
    switch (skip_mode) {
        case SC_SKIP_NONE: k_chain<T, SC_SKIP_NONE><<<grid, TB, 0, stream>>>(a); break;
        case SC_SKIP_LE: k_chain<T, SC_SKIP_LE><<<grid, TB, 0, stream>>>(a); break;
        case SC_SKIP_NOT_GT: k_chain<T, SC_SKIP_NOT_GT><<<grid, TB, 0, stream>>>(a); break;
        default: SC_REQUIRE(false, "chain: bad skip_mode %d", skip_mode);
    }
    SC_CHECK_LAUNCH();
    return SC_OK;
}

// ---------------------------------------------------------------- direct form
// Gather form of direct_form (core.py:102-119).  The reference sums the
// individually rounded products e[m]*h[n-m] with math.fsum (exact rounding).
// Here: products rounded the same way, summed with the compensated
// "Sum2" scheme (TwoSum error-free transformation, error terms accumulated
// and folded in once) -- as accurate as a double-double accumulator, which
// is exactly rounded except under extreme cancellation.

__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

__global__ void __launch_bounds__(TB) k_direct_dd(const double *__restrict__ e, int64_t ne,
                                                  const double *__restrict__ h, int64_t nh,
                                                  double *__restrict__ y) {
    const int64_t n = (int64_t)blockIdx.x * TB + threadIdx.x;
    if (n >= ne + nh - 1) return;
    const int64_t lo = n - nh + 1 > 0 ? n - nh + 1 : 0;
    const int64_t hi = n < ne - 1 ? n : ne - 1;
    double s = 0.0, c = 0.0;
    for (int64_t m = lo; m <= hi; ++m) {
        const double p = __dmul_rn(e[m], h[n - m]);
        double q;
        two_sum(s, p, s, q);
        c = __dadd_rn(c, q);
    }
    y[n] = __dadd_rn(s, c);
}

}  // namespace

int launch_chain(int dtype, int skip_mode, double threshold, const void *x, int64_t x_off,
                 const ChainSeg *segs, int nseg, const void *init, int64_t init_len,
                 const int64_t *init_len_dev, int64_t t0, int64_t n_out, void *out_a,
                 int64_t n_a, void *out_b, cudaStream_t stream, const unsigned *run_if,
                 const ChainBatch *batch) {
    if (dtype == SC_F64)
        return launch_chain_t<double>(skip_mode, threshold, x, x_off, segs, nseg, init, init_len,
                                      init_len_dev, t0, n_out, out_a, n_a, out_b, stream, run_if, batch);
    if (dtype == SC_F32)
        return launch_chain_t<float>(skip_mode, threshold, x, x_off, segs, nseg, init, init_len,
                                     init_len_dev, t0, n_out, out_a, n_a, out_b, stream, run_if, batch);
    set_error("chain: bad dtype %d", dtype);
    return SC_ERR_ARG;
}

int launch_direct_form_dd(const double *e, int64_t ne, const double *h, int64_t nh, double *y,
                          cudaStream_t stream) {
    const int64_t nout = ne + nh - 1;
    if (nout <= 0) return SC_OK;
    k_direct_dd<<<(unsigned)cdiv(nout, TB), TB, 0, stream>>>(e, ne, h, nh, y);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

}  // namespace sc
