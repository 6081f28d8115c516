// k_fast_f32.cu -- output-stationary, register-tiled FP32 FIR for sm_100a.
//
// Computes y[n] = sum_k h[k] * X(n-k) over an output range, the gather
// restatement of the reference's scatter loop y[k+n] += x[k]*h[n]
// (core.py:80-92, _kernels.py:31-42).  Same result within FP32 rounding
// (fixed, deterministic summation order; not the reference's chain order --
// SC_MODE_ORDERED provides that).
//
// Tiling (one CTA = 256 threads = 8192 consecutive outputs):
//  * the tile is two halves A = [n0, n0+4096) and B = [n0+4096, n0+8192);
//    thread j owns the 16 output PAIRS (y[n0+16j+p], y[n0+4096+16j+p]),
//    p = 0..15, as 16 float2 accumulators.  Pairing outputs 4096 apart keeps
//    the pair alignment fixed while the tap index slides, so every MAC is
//    one lane of an FFMA2 (fma.rn.f32x2) with the tap broadcast:
//        acc[p] += (X(n0+16j+p-k), X(n0+4096+16j+p-k)) * h[k]
//  * taps are walked in chunks of 16; a thread's 31-pair sliding window for
//    a chunk is two 16-pair groups read with LDS.128 from a shared-memory
//    RING of input pairs.  Full unrolling turns the window shift into
//    register renaming: 256 FFMA2 (512 MAC) per 16 LDS.128 + 4 LDG.128 (taps).
//  * the ring holds 272 groups of 16 pairs, each group padded by 2 pairs
//    (16 B) so lanes j and j+1 (groups 144 B apart) hit disjoint banks.  As
//    the tap index advances by 64 (one pipeline stage = 4 chunks) the window
//    slides by 64 pairs: 4 new groups (128 floats) are fetched into
//    registers during the stage and stored after it -- the ring is sized so
//    the new groups never alias groups still being read, so ONE
//    __syncthreads per 64 taps suffices and global traffic per CTA is just
//    the input halo plus taps (~12 bytes per 64 taps per thread).
//  * long filters with few tiles are split over taps (grid.y); partials go
//    to a workspace and a second kernel sums them in fixed split order
//    (deterministic, no atomics).  grid.z = channel (batched multichannel).

#include "sc_common.cuh"

namespace sc {
namespace {

constexpr int FT_THREADS = 256;
constexpr int FT_PAIRS = 16;                    // output pairs per thread
constexpr int FT_HALF = FT_THREADS * FT_PAIRS;  // 4096
constexpr int FT_TILE = 2 * FT_HALF;            // 8192 outputs per CTA
constexpr int FT_KC = 16;                       // taps per register chunk
constexpr int FT_CPS = 4;                       // chunks per pipeline stage
constexpr int FT_STAGE_TAPS = FT_KC * FT_CPS;   // 64
constexpr int FT_GSTRIDE = 18;                  // float2 per group incl. skew
constexpr int FT_NG = 272;                      // ring groups (>= 256 + 2*FT_CPS + 1)
constexpr int FT_FILL_GROUPS = FT_THREADS + FT_CPS;  // groups live in stage 0: [-CPS+1 .. 256]

struct FastArgs {
    const float *x;
    int64_t ldx;      // channel stride of x
    int64_t x_base;   // absolute index of x[0]
    int64_t x_lo, x_hi;  // valid absolute input range
    const float *hp;  // padded taps, channel stride ldhp, zero beyond nh
    int64_t ldhp;
    int64_t nh;       // true tap count
    int64_t nh_pad;   // multiple of FT_STAGE_TAPS
    int64_t taps_per_split;  // multiple of FT_STAGE_TAPS
    float *y;         // if nsplit == 1: final output (channel stride ldy)
    int64_t ldy;
    float *ws;        // partials [nsplit][channels][n_len] when nsplit > 1
    int64_t n_begin, n_len;
    int nsplit, channels;
    const unsigned *run_if;  // optional device gate (FAST-mode fallback)
};

__device__ __forceinline__ float load_x(const FastArgs &a, const float *xc, int64_t m) {
    return (m >= a.x_lo && m < a.x_hi) ? __ldg(xc + (m - a.x_base)) : 0.0f;
}

// Ring slot of relative group g (can be negative).
__device__ __forceinline__ int ring_slot(int64_t g) {
    int r = (int)(g % FT_NG);
    return r < 0 ? r + FT_NG : r;
}

__global__ void __launch_bounds__(FT_THREADS, 2) k_fir_f32_fast(FastArgs a) {
    __shared__ __align__(16) float2 ring[FT_NG * FT_GSTRIDE];
    if (a.run_if && *a.run_if == 0) return;  // gated fallback not needed (block-uniform)

    const int j = threadIdx.x;
    const int ch = blockIdx.z;
    const int split = blockIdx.y;
    const int64_t n0 = a.n_begin + (int64_t)blockIdx.x * FT_TILE;
    const int64_t ks = (int64_t)split * a.taps_per_split;
    int64_t ke = ks + a.taps_per_split;
    if (ke > a.nh_pad) ke = a.nh_pad;
    const float *xc = a.x + (int64_t)ch * a.ldx;
    const float *hc = a.hp + (int64_t)ch * a.ldhp;

    // Relative group g covers pair indices q in [qb + 16g, qb + 16g + 16),
    // qb = -ks - 16; pair q = (X(n0+q), X(n0+4096+q)).  At chunk c thread j
    // reads groups j-c and j-c+1.
    const int64_t qb = -ks - FT_KC;

    // ---- initial fill: groups [-(CPS-1), 256] (stage 0 = chunks 0..CPS-1)
    for (int i = j; i < FT_FILL_GROUPS * 16; i += FT_THREADS) {
        const int64_t g = (int64_t)(i >> 4) - (FT_CPS - 1);
        const int64_t q = qb + 16 * g + (i & 15);
        float2 v;
        v.x = load_x(a, xc, n0 + q);
        v.y = load_x(a, xc, n0 + FT_HALF + q);
        ring[ring_slot(g) * FT_GSTRIDE + (i & 15)] = v;
    }

    float2 acc[FT_PAIRS];
#pragma unroll
    for (int p = 0; p < FT_PAIRS; ++p) acc[p] = make_float2(0.0f, 0.0f);

    const int64_t n_chunks = (ke - ks) / FT_KC;  // multiple of CPS
    // taps of the first chunk
    float4 hv[4];
    {
        const float4 *h4 = reinterpret_cast<const float4 *>(hc + ks);
#pragma unroll
        for (int i = 0; i < 4; ++i) hv[i] = __ldg(h4 + i);
    }
    __syncthreads();

    for (int64_t c0 = 0; c0 < n_chunks; c0 += FT_CPS) {
        // Prefetch the 4 groups the next stage adds: g in [-c0-2CPS+1, -c0-CPS].
        float pre = 0.0f;
        int pre_slot = -1;
        const bool has_next = c0 + FT_CPS < n_chunks;
        if (has_next && j < FT_CPS * 32) {
            const int gi = j >> 5;            // 0..CPS-1
            const int w = j & 31;             // 0..15 half A, 16..31 half B
            const int64_t g = -c0 - 2 * FT_CPS + 1 + gi;
            const int64_t q = qb + 16 * g + (w & 15);
            pre = load_x(a, xc, n0 + q + (w >= 16 ? FT_HALF : 0));
            pre_slot = ring_slot(g) * FT_GSTRIDE + (w & 15);
        }

#pragma unroll 1
        for (int cc = 0; cc < FT_CPS; ++cc) {
            const int64_t c = c0 + cc;
            // next chunk's taps (padded array: always in bounds up to nh_pad)
            float4 hn[4];
            {
                const int64_t kn = ks + (c + 1) * FT_KC;
                const float4 *h4 = reinterpret_cast<const float4 *>(hc + (kn < a.nh_pad ? kn : ks));
#pragma unroll
                for (int i = 0; i < 4; ++i) hn[i] = __ldg(h4 + i);
            }
            const float4 *gA = reinterpret_cast<const float4 *>(ring + ring_slot(j - c) * FT_GSTRIDE);
            const float4 *gB = reinterpret_cast<const float4 *>(ring + ring_slot(j - c + 1) * FT_GSTRIDE);
            float2 W[2 * FT_PAIRS];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float4 va = gA[i];
                const float4 vb = gB[i];
                W[2 * i] = make_float2(va.x, va.y);
                W[2 * i + 1] = make_float2(va.z, va.w);
                W[16 + 2 * i] = make_float2(vb.x, vb.y);
                W[16 + 2 * i + 1] = make_float2(vb.z, vb.w);
            }
            const float *hs = reinterpret_cast<const float *>(hv);
            // Taps past nh (zero padding) are never multiplied: 0*NaN / 0*Inf
            // inputs must not reach outputs the reference leaves finite.
            const int64_t kc = ks + c * FT_KC;
            if (kc + FT_KC <= a.nh) {
#pragma unroll
                for (int t = 0; t < FT_KC; ++t) {
                    const float2 h2 = make_float2(hs[t], hs[t]);
#pragma unroll
                    for (int p = 0; p < FT_PAIRS; ++p) acc[p] = __ffma2_rn(W[p - t + 16], h2, acc[p]);
                }
            } else if (kc < a.nh) {
                const int tv = (int)(a.nh - kc);
#pragma unroll
                for (int t = 0; t < FT_KC; ++t) {
                    if (t < tv) {
                        const float2 h2 = make_float2(hs[t], hs[t]);
#pragma unroll
                        for (int p = 0; p < FT_PAIRS; ++p) acc[p] = __ffma2_rn(W[p - t + 16], h2, acc[p]);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) hv[i] = hn[i];
        }
        if (pre_slot >= 0) reinterpret_cast<float *>(ring)[2 * pre_slot + ((j & 31) >= 16 ? 1 : 0)] = pre;
        __syncthreads();
    }

    // ---- epilogue
    float *dst;
    int64_t dst_off;
    if (a.nsplit == 1) {
        dst = a.y + (int64_t)ch * a.ldy;
        dst_off = -a.n_begin;
    } else {
        dst = a.ws + ((int64_t)split * a.channels + ch) * a.n_len;
        dst_off = -a.n_begin;
    }
    const int64_t n_end = a.n_begin + a.n_len;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int64_t nb = n0 + half * FT_HALF + 16 * j;
        float *d = dst + (nb + dst_off);
        const bool full = nb + FT_PAIRS <= n_end;
        if (full && ((reinterpret_cast<uintptr_t>(d) & 15) == 0)) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float4 v;
                v.x = half ? acc[4 * i].y : acc[4 * i].x;
                v.y = half ? acc[4 * i + 1].y : acc[4 * i + 1].x;
                v.z = half ? acc[4 * i + 2].y : acc[4 * i + 2].x;
                v.w = half ? acc[4 * i + 3].y : acc[4 * i + 3].x;
                reinterpret_cast<float4 *>(d)[i] = v;
            }
        } else {
#pragma unroll
            for (int p = 0; p < FT_PAIRS; ++p)
                if (nb + p < n_end) d[p] = half ? acc[p].y : acc[p].x;
        }
    }
}

// Sum split partials in fixed (ascending) split order.
__global__ void k_split_reduce(const float *__restrict__ ws, int nsplit, int channels,
                               int64_t n_len, float *__restrict__ y, int64_t ldy, const unsigned *run_if) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int ch = blockIdx.y;
    if (i >= n_len || (run_if && *run_if == 0)) return;
    float s = ws[(int64_t)ch * n_len + i];
    for (int k = 1; k < nsplit; ++k) s += ws[((int64_t)k * channels + ch) * n_len + i];
    y[(int64_t)ch * ldy + i] = s;
}

// Copy taps into a zero-padded, 16-byte aligned workspace.
__global__ void k_pad_taps(const float *__restrict__ h, int64_t ldh, int64_t nh,
                           float *__restrict__ hp, int64_t ldhp, const unsigned *run_if) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int ch = blockIdx.y;
    if (i >= ldhp || (run_if && *run_if == 0)) return;
    hp[(int64_t)ch * ldhp + i] = i < nh ? h[(int64_t)ch * ldh + i] : 0.0f;
}

int choose_splits(int64_t tiles, int64_t stages, int slots) {
    // Pick the split count (over tap stages) that best fills whole waves of
    // `slots` resident CTAs; each split keeps >= 16 stages (1024 taps) so
    // the ring fill stays amortised.  Prefer fewer splits on ties.
    int best = 1;
    double best_eff = 0.0;
    const int max_split = (int)(stages / 16 > 1 ? (stages / 16 < 64 ? stages / 16 : 64) : 1);
    for (int s = 1; s <= max_split; ++s) {
        const int64_t units = tiles * s;
        const int64_t waves = (units + slots - 1) / slots;
        const double eff = (double)units / (double)(waves * slots);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = s;
        }
        if (best_eff > 0.97) break;
    }
    return best;
}

}  // namespace

int launch_fir_f32_fast(const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi,
                        const float *h, int64_t ldh, int64_t nh, float *y, int64_t ldy,
                        int64_t n_begin, int64_t n_end, int64_t channels, cudaStream_t stream,
                        const unsigned *run_if) {
    const int64_t n_len = n_end - n_begin;
    if (n_len <= 0 || channels <= 0) return SC_OK;
    SC_REQUIRE(nh >= 1, "fir: empty impulse response");
    SC_REQUIRE(channels < 65536, "fir: too many channels");
    const int64_t nh_pad = cdiv(nh, FT_STAGE_TAPS) * FT_STAGE_TAPS;
    const int64_t tiles = cdiv(n_len, FT_TILE);
    SC_REQUIRE(tiles < (int64_t)INT32_MAX, "fir: output range too large");
    const int64_t stages = nh_pad / FT_STAGE_TAPS;

    static int slots_per_sm = -1;
    if (slots_per_sm < 0) {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fir_f32_fast, FT_THREADS, 0) !=
                cudaSuccess || nb < 1)
            nb = 1;
        slots_per_sm = nb;
    }
    const int slots = sm_count() * slots_per_sm;
    const int nsplit = choose_splits(tiles * channels, stages, slots);
    const int64_t stages_per_split = cdiv(stages, nsplit);
    const int64_t taps_per_split = stages_per_split * FT_STAGE_TAPS;
    const int nsplit_eff = (int)cdiv(stages, stages_per_split);

    int err = 0;
    const int64_t ldhp = nh_pad + FT_STAGE_TAPS;  // + one stage of zeros for the h prefetch
    float *hp = static_cast<float *>(scratch(sizeof(float) * ldhp * channels, 0, stream, &err));
    if (err) return err;
    {
        dim3 g((unsigned)cdiv(ldhp, 256), (unsigned)channels);
        k_pad_taps<<<g, 256, 0, stream>>>(h, ldh, nh, hp, ldhp, run_if);
        SC_CHECK_LAUNCH();
    }
    float *ws = nullptr;
    if (nsplit_eff > 1) {
        ws = static_cast<float *>(
            scratch(sizeof(float) * (size_t)n_len * channels * nsplit_eff, 1, stream, &err));
        if (err) return err;
    }
    FastArgs a;
    a.x = x;
    a.ldx = ldx;
    a.x_base = x_base;
    a.x_lo = x_lo;
    a.x_hi = x_hi;
    a.hp = hp;
    a.ldhp = ldhp;
    a.nh = nh;
    a.nh_pad = nh_pad;
    a.taps_per_split = taps_per_split;
    a.y = y;
    a.ldy = ldy;
    a.ws = ws;
    a.n_begin = n_begin;
    a.n_len = n_len;
    a.nsplit = nsplit_eff;
    a.channels = (int)channels;
    a.run_if = run_if;
    dim3 grid((unsigned)tiles, (unsigned)nsplit_eff, (unsigned)channels);
    k_fir_f32_fast<<<grid, FT_THREADS, 0, stream>>>(a);
    SC_CHECK_LAUNCH();
    if (nsplit_eff > 1) {
        dim3 g((unsigned)cdiv(n_len, 256), (unsigned)channels);
        k_split_reduce<<<g, 256, 0, stream>>>(ws, nsplit_eff, (int)channels, n_len, y, ldy, run_if);
        SC_CHECK_LAUNCH();
    }
    return SC_OK;
}

}  // namespace sc
