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

#include <cstdlib>

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

        // ring slots of groups j - c and j - c + 1, stepped down per chunk
        // (no 64-bit modulo in the inner loop)
        int sA = ring_slot(j - c0), sB = ring_slot(j - c0 + 1);
#pragma unroll 2  // (full unrolling spills at the 128-register cap)
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
            const float4 *gA = reinterpret_cast<const float4 *>(ring + sA * FT_GSTRIDE);
            const float4 *gB = reinterpret_cast<const float4 *>(ring + sB * FT_GSTRIDE);
            sB = sA;
            sA = sA == 0 ? FT_NG - 1 : sA - 1;
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

// ---------------------------------------------------------------- short filters, HBM-bound (Nh <= 32)
// Nh <= 32 (HBM-bound up to ~40 taps; longer filters use k_fir_short_smem
// below, whose smem window feeds more FMAs per L1 wavefront): no staging of x at
// all.  Each thread owns 8 consecutive outputs t0..t0+7 and slides a
// 12-float register window over x in float4 steps: for the 4 taps
// 4kb..4kb+3 it needs x[t0-4kb-3 .. t0-4kb+7], and moving to the next 4 taps
// drops the top float4 and loads one new float4 below (renaming only: the
// tap-block loop is unrolled at compile time, NKB = ceil(Nh/4) blocks).  So
// a thread issues NKB+2 LDG.128 (L1 hits for all but ~1/3: neighbouring
// threads share windows), one broadcast LDS.128 of taps and 32 FFMA per 4
// taps, and two float4 stores.  Each output accumulates taps in ascending
// order (fmaf), identical in interior and edge tiles.  Taps past Nh (zero
// padding of the last block) are never multiplied, so NaN/Inf inputs next to
// them cannot leak.  Tiles whose window leaves the valid input range [x_lo,
// x_hi) (the first and last few) take a guarded scalar path that multiplies
// only taps whose input exists -- the reference's edge semantics.
// (16 outputs per thread measured slower at every length: lanes 64 B apart
// double the L1 wavefronts per LDG.128 along with the FFMAs it feeds.)
constexpr int SH_THREADS = 256;
constexpr int SH_R = 8;
constexpr int SH_MAXNH = 256;

template <int NKB, int SH_R>
__global__ void __launch_bounds__(SH_THREADS) k_fir_short(const float *__restrict__ x, int64_t ldx, int64_t x_base,
                                                          int64_t x_lo, int64_t x_hi, const float *__restrict__ h,
                                                          int64_t ldh, int nh, float *__restrict__ y, int64_t ldy,
                                                          int64_t n_begin, int64_t n_end, const unsigned *run_if) {
    constexpr int SH_TILE = SH_THREADS * SH_R;  // outputs per CTA
    constexpr int NW = SH_R / 4 + 1;            // float4s in the register window
    __shared__ __align__(16) float hsm[4 * NKB];
    if (run_if && *run_if == 0) return;
    const int ch = blockIdx.y;
    const float *xc = x + (int64_t)ch * ldx;
    const float *hc = h + (int64_t)ch * ldh;
    float *yc = y + (int64_t)ch * ldy;
    for (int k = threadIdx.x; k < 4 * NKB; k += SH_THREADS) hsm[k] = k < nh ? hc[k] : 0.0f;
    __syncthreads();
    const int64_t n0 = n_begin + (int64_t)blockIdx.x * SH_TILE;
    const int64_t t0 = n0 + (int64_t)threadIdx.x * SH_R;
    const int nkb = (nh + 3) >> 2;
    const int nfull = nh >> 2;  // blocks whose 4 taps all exist
    float acc[SH_R];
#pragma unroll
    for (int r = 0; r < SH_R; ++r) acc[r] = 0.0f;
    // CTA-uniform: every float4 the window reads lies in [x_lo, x_hi), is
    // aligned, and the tile is whole
    const float *xt = xc + (n0 - x_base);
    const bool interior = n0 - 4 * nkb >= x_lo && n0 + SH_TILE <= x_hi && n0 + SH_TILE <= n_end &&
                          ((reinterpret_cast<uintptr_t>(xt) | reinterpret_cast<uintptr_t>(yc + (n0 - n_begin)) |
                            (uintptr_t)(ldx * 4) | (uintptr_t)(ldy * 4)) & 15) == 0;
    if (interior && nkb == NKB && nfull == NKB) {
        // Nh == 4*NKB: the tap-block loop is entirely compile-time (no
        // per-block tests, the window shift is pure register renaming)
        // g[c] = x[t0 - 4 + 4c .. t0 + 4c - 1]: window of taps 4kb..4kb+3
        const float4 *xp = reinterpret_cast<const float4 *>(xc + (t0 - x_base));
        float4 g[NW];
#pragma unroll
        for (int c = 0; c < NW; ++c) g[c] = __ldg(xp + c - 1);
        const float4 *h4 = reinterpret_cast<const float4 *>(hsm);
#pragma unroll
        for (int kb = 0; kb < NKB; ++kb) {
            float w[4 * NW];
#pragma unroll
            for (int c = 0; c < NW; ++c) {
                w[4 * c] = g[c].x;
                w[4 * c + 1] = g[c].y;
                w[4 * c + 2] = g[c].z;
                w[4 * c + 3] = g[c].w;
            }
            const float4 hq = h4[kb];
            const float hk[4] = {hq.x, hq.y, hq.z, hq.w};
            float4 gn = g[0];
            if (kb + 1 < NKB) gn = __ldg(xp - (kb + 2));  // next window in flight during the FMAs
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int r = 0; r < SH_R; ++r) acc[r] = fmaf(w[r - u + 4], hk[u], acc[r]);
#pragma unroll
            for (int c = NW - 1; c > 0; --c) g[c] = g[c - 1];
            g[0] = gn;
        }
        float4 *d = reinterpret_cast<float4 *>(yc + (t0 - n_begin));
#pragma unroll
        for (int c = 0; c < SH_R / 4; ++c)
            d[c] = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
        return;
    }
    if (interior) {
        const float4 *xp = reinterpret_cast<const float4 *>(xc + (t0 - x_base));  // x[t0 .. t0+3]
        float4 g[NW];                                                             // x[t0-4 .. t0+SH_R-1]
#pragma unroll
        for (int c = 0; c < NW; ++c) g[c] = __ldg(xp + c - 1);
        const float4 *h4 = reinterpret_cast<const float4 *>(hsm);
#pragma unroll
        for (int kb = 0; kb < NKB; ++kb) {
            if (kb < nkb) {
                float w[4 * NW];
#pragma unroll
                for (int c = 0; c < NW; ++c) {
                    w[4 * c] = g[c].x;
                    w[4 * c + 1] = g[c].y;
                    w[4 * c + 2] = g[c].z;
                    w[4 * c + 3] = g[c].w;
                }
                const float4 hq = h4[kb];
                const float hk[4] = {hq.x, hq.y, hq.z, hq.w};
                // next window (x[t0-4kb-8 .. t0-4kb-5]) in flight during the FMAs
                const float4 gn = kb + 1 < nkb ? __ldg(xp - (kb + 2)) : g[0];
                if (kb < nfull) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int r = 0; r < SH_R; ++r) acc[r] = fmaf(w[r - u + 4], hk[u], acc[r]);
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * kb + u < nh)
#pragma unroll
                            for (int r = 0; r < SH_R; ++r) acc[r] = fmaf(w[r - u + 4], hk[u], acc[r]);
                }
#pragma unroll
                for (int c = NW - 1; c > 0; --c) g[c] = g[c - 1];
                g[0] = gn;
            }
        }
        float4 *d = reinterpret_cast<float4 *>(yc + (t0 - n_begin));
#pragma unroll
        for (int c = 0; c < SH_R / 4; ++c)
            d[c] = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
        return;
    }
    // edge tiles: scalar, only taps whose input exists, k ascending
    for (int k = 0; k < nh; ++k) {
        const float hk = hsm[k];
#pragma unroll
        for (int r = 0; r < SH_R; ++r) {
            const int64_t m = t0 + r - k;
            if (m >= x_lo && m < x_hi) acc[r] = fmaf(__ldg(xc + (m - x_base)), hk, acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < SH_R; ++r)
        if (t0 + r < n_end) yc[t0 + r - n_begin] = acc[r];
}

// ---------------------------------------------------------------- short filters, taps in registers (Nh <= 64)
// Tap-stationary form: every thread holds the whole filter in registers and
// walks C chunks of 4 consecutive outputs, keeping the last 4*NH4+4 inputs in
// a register ring of NH4+1 float4 slots (the chunk loop is unrolled by NH4+1,
// so advancing the window is register renaming).  Per chunk a thread reads
// ONE float4 of x and writes one float4 of y, both in shared memory, for
// 4*Nh FFMA: at 32 taps 128 FFMA per LDS.128 + STS.128 (the register-window
// kernel above needs one L1 wavefront per 4 FFMA there).  The CTA stages its
// x tile (+ the 4*NH4-sample halo) with coalesced 16-byte loads and copies
// the y tile out the same way.  Lane stride in smem is C float4s, C odd, so
// LDS/STS.128 are conflict-free.
// Each output is one fmaf chain over taps k = 0..Nh-1 ascending from +0 --
// bit-identical to k_fir_short.  Edge tiles (inputs outside [x_lo, x_hi) or
// a partial tile) multiply only taps whose input exists.
constexpr int TR_THREADS = 128;

template <int NH4>
struct TapReg {
    // ring of S >= NH4+1 float4 slots, S odd; C = chunks per thread, a
    // multiple of S (so a whole number of ring cycles) and odd (so the lane
    // stride in smem is conflict-free for LDS/STS.128)
    static constexpr int S = (NH4 % 2 == 0) ? NH4 + 1 : NH4 + 2;
    static constexpr int C = S < 5 ? 3 * S : S;
    static constexpr int TILE = TR_THREADS * 4 * C;    // outputs per CTA
    static constexpr int NX4 = TR_THREADS * C + NH4;   // staged x float4s (halo first)
    static constexpr int SMEM = 16 * (NX4 + TR_THREADS * C);
};

template <int NH4>
__device__ __forceinline__ void tapreg_walk(const float4 *xs, float4 *ys, const float (&hr)[4 * NH4], int nh) {
    using T = TapReg<NH4>;
    constexpr int S = T::S;
    const int f0 = threadIdx.x * T::C;  // x float4 of this thread's first window; y float4 of its first chunk
    float4 W[S];
#pragma unroll
    for (int q = 0; q < NH4; ++q) W[q] = xs[f0 + q];
#pragma unroll 1
    for (int g = 0; g < T::C / S; ++g) {
#pragma unroll
        for (int jj = 0; jj < S; ++jj) {
            const int j = g * S + jj;
            // float4 f0+j+q of the window lives in W[(jj+q) % S]; the newest
            // one (q = NH4) is loaded here
            W[(jj + NH4) % S] = xs[f0 + j + NH4];
            float xw[4 * NH4 + 4];
#pragma unroll
            for (int q = 0; q <= NH4; ++q) {
                const float4 v = W[(jj + q) % S];
                xw[4 * q] = v.x;
                xw[4 * q + 1] = v.y;
                xw[4 * q + 2] = v.z;
                xw[4 * q + 3] = v.w;
            }
            // output i of the chunk (n = n_first + 4j + i) times tap k reads
            // x[n-k] = xw[4*NH4 + i - k]
            float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int k = 0; k < 4 * NH4; ++k) {
                if (k >= 4 * (NH4 - 1) && k >= nh) break;  // taps past Nh are never multiplied
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[i] = fmaf(xw[4 * NH4 + i - k], hr[k], acc[i]);
            }
            ys[f0 + j] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        }
    }
}

// One tile per CTA (blockIdx.x = tile, blockIdx.y = channel); several CTAs
// per SM overlap one tile's staging with another's FMAs (a persistent
// double-buffered loop measured slower: it doubled the registers).
// Edge tiles: plain runtime loops over the same stage (structurally unlike the
// unrolled walk, so the compiler cannot merge the two into one predicated
// body), multiplying only taps whose input exists.
template <int NH4>
__device__ __forceinline__ void tapreg_walk_edge(const float4 *xs, float4 *ys, const float *hc, int nh,
                                                 int64_t n_first, int64_t x_lo, int64_t x_hi) {
    using T = TapReg<NH4>;
    const float *xsf = reinterpret_cast<const float *>(xs);
    const int f0 = threadIdx.x * T::C;
#pragma unroll 1
    for (int j = 0; j < T::C; ++j) {
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 1
        for (int k = 0; k < nh; ++k) {
            const float hk = __ldg(hc + k);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t m = n_first + 4 * j + i - k;
                if (m >= x_lo && m < x_hi) acc[i] = fmaf(xsf[4 * (f0 + j) + 4 * NH4 + i - k], hk, acc[i]);
            }
        }
        ys[f0 + j] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    }
}

template <int NH4>
__global__ void __launch_bounds__(TR_THREADS) k_fir_tapreg(const float *__restrict__ x, int64_t ldx, int64_t x_base,
                                                           int64_t x_lo, int64_t x_hi, const float *__restrict__ h,
                                                           int64_t ldh, int nh, float *__restrict__ y, int64_t ldy,
                                                           int64_t n_begin, int64_t n_end, const unsigned *run_if) {
    using T = TapReg<NH4>;
    extern __shared__ float4 tr_smem[];  // T::SMEM bytes: the x stage, then the y stage
    float4 *xs = tr_smem;
    float4 *ys = tr_smem + T::NX4;
    if (run_if && *run_if == 0) return;
    const int ch = blockIdx.y;
    const float *xc = x + (int64_t)ch * ldx;
    const float *hc = h + (int64_t)ch * ldh;
    float *yc = y + (int64_t)ch * ldy;
    float hr[4 * NH4];  // warp-uniform: the compiler keeps them in uniform registers where they fit
#pragma unroll
    for (int k = 0; k < 4 * NH4; ++k) hr[k] = k < nh ? __ldg(hc + k) : 0.0f;
    const int64_t n0 = n_begin + (int64_t)blockIdx.x * T::TILE;
    const int64_t m0 = n0 - 4 * NH4;  // input index of staged float4 0
    const float *src = xc + (m0 - x_base);
    const bool edge = m0 < x_lo || n0 + T::TILE > x_hi || n0 + T::TILE > n_end;
    if (!edge && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        // 16-byte async copies: the whole stage in flight without registers
        const uint32_t xs_s = (uint32_t)__cvta_generic_to_shared(xs);
        for (int f = threadIdx.x; f < T::NX4; f += TR_THREADS)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(xs_s + 16 * f), "l"(src + 4 * f)
                         : "memory");
        asm volatile("cp.async.wait_all;\n" ::: "memory");
    } else {
        float *xsf = reinterpret_cast<float *>(xs);
        for (int i = threadIdx.x; i < 4 * T::NX4; i += TR_THREADS) {
            const int64_t m = m0 + i;
            xsf[i] = (m >= x_lo && m < x_hi) ? __ldg(xc + (m - x_base)) : 0.0f;
        }
    }
    __syncthreads();
    const int64_t n_first = n0 + (int64_t)threadIdx.x * 4 * T::C;
    if (!edge)
        tapreg_walk<NH4>(xs, ys, hr, nh);
    else
        tapreg_walk_edge<NH4>(xs, ys, hc, nh, n_first, x_lo, x_hi);
    __syncthreads();
    float *dst = yc + (n0 - n_begin);
    if (!edge && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        float4 *d4 = reinterpret_cast<float4 *>(dst);
        for (int f = threadIdx.x; f < TR_THREADS * T::C; f += TR_THREADS) d4[f] = ys[f];
    } else {
        const float *ysf = reinterpret_cast<const float *>(ys);
        const int64_t lim = n_end - n0 < T::TILE ? n_end - n0 : T::TILE;
        for (int i = threadIdx.x; i < lim; i += TR_THREADS) dst[i] = ysf[i];
    }
}

constexpr int TR_MAXNH4 = 8;

template <int NH4>
int launch_tapreg(const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi, const float *h,
                  int64_t ldh, int64_t nh, float *y, int64_t ldy, int64_t n_begin, int64_t n_end,
                  int64_t channels, cudaStream_t stream, const unsigned *run_if) {
    using T = TapReg<NH4>;
    static const cudaError_t attr =
        cudaFuncSetAttribute(k_fir_tapreg<NH4>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
    SC_REQUIRE(attr == cudaSuccess, "fir: tap-register kernel smem attribute: %s", cudaGetErrorString(attr));
    const int64_t tiles = cdiv(n_end - n_begin, (int64_t)T::TILE);
    SC_REQUIRE(tiles < (int64_t)INT32_MAX, "fir: output range too large");
    dim3 g((unsigned)tiles, (unsigned)channels);
    k_fir_tapreg<NH4><<<g, TR_THREADS, T::SMEM, stream>>>(x, ldx, x_base, x_lo, x_hi, h, ldh, (int)nh, y, ldy,
                                                          n_begin, n_end, run_if);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

// ---------------------------------------------------------------- short filters, FMA-bound (32 < Nh <= 256)
// 32 < Nh <= 256 (FMA-bound): the ring/split machinery above is overhead.  Each CTA stages one
// contiguous x tile (4096 outputs + Nh-1 halo, float4 loads) and the taps in
// smem; each thread computes 16 consecutive outputs.  Per 4 taps a thread
// reads its 20-float input window with 5 LDS.128 plus the 4 taps with one
// broadcast LDS.128 and issues 64 FFMA; the stage starts Nh rounded up to 4
// before the tile so every window is float4-aligned and the window shift is
// pure register renaming.
// The x stage is padded by 4 floats every 16 (row pitch 80 B) so the 64 B
// stride between lanes is bank-conflict-free.  HBM-bound for short filters
// (8 B per output), FMA-bound beyond ~40 taps.  Edge tiles (touching the ends
// of the valid input range) only multiply taps whose input exists, so
// non-finite taps propagate exactly as in the reference.
constexpr int SM_THREADS = 256;
constexpr int SM_R = 16;
constexpr int SM_TILE = SM_THREADS * SM_R;  // 4096

__device__ __forceinline__ int sh_pos(int i) { return i + ((i >> 4) << 2); }

__global__ void __launch_bounds__(SM_THREADS) k_fir_short_smem(const float *__restrict__ x, int64_t ldx, int64_t x_base,
                                                          int64_t x_lo, int64_t x_hi, const float *__restrict__ h,
                                                          int64_t ldh, int nh, float *__restrict__ y, int64_t ldy,
                                                          int64_t n_begin, int64_t n_end, const unsigned *run_if) {
    // xs[i] = X(n0 - nh_pad + 1 + i) with nh_pad = nh rounded up to 4 (so the
    // tile start is float4-aligned whenever n0 is), i in [0, 4096 + nh_pad + 4)
    constexpr int XS = SM_TILE + SH_MAXNH + 8;
    __shared__ __align__(16) float xs[XS + XS / 4];
    __shared__ __align__(16) float hsm[SH_MAXNH + 4];
    if (run_if && *run_if == 0) return;
    const int ch = blockIdx.y;
    const float *xc = x + (int64_t)ch * ldx;
    const float *hc = h + (int64_t)ch * ldh;
    float *yc = y + (int64_t)ch * ldy;
    const int nhp = (nh + 3) & ~3;
    const int64_t n0 = n_begin + (int64_t)blockIdx.x * SM_TILE;
    const int64_t m0 = n0 - nhp;  // input index of xs[0] (float4-aligned with n0)
    const int nx = SM_TILE + nhp;
    for (int k = threadIdx.x; k < SH_MAXNH + 4; k += SM_THREADS) hsm[k] = k < nh ? hc[k] : 0.0f;
    const bool edge = m0 < x_lo || n0 + SM_TILE > x_hi;
    const float *src = xc + (m0 - x_base);
    if (!edge && m0 + nx <= x_hi && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        for (int i4 = threadIdx.x; i4 < nx / 4; i4 += SM_THREADS)
            *reinterpret_cast<float4 *>(&xs[sh_pos(4 * i4)]) = __ldg(reinterpret_cast<const float4 *>(src) + i4);
    } else {
        for (int i = threadIdx.x; i < nx; i += SM_THREADS) {
            const int64_t m = m0 + i;
            xs[sh_pos(i)] = (m >= x_lo && m < x_hi) ? __ldg(xc + (m - x_base)) : 0.0f;
        }
    }
    __syncthreads();
    float acc[SM_R];
#pragma unroll
    for (int r = 0; r < SM_R; ++r) acc[r] = 0.0f;
    const int j16 = threadIdx.x * SM_R;
    const int64_t t0 = n0 + j16;  // this thread's first output
    // output t0+r, tap k reads X(t0 + r - k) = xs[j16 + r - k + nhp]
    int k_done = 0;
    if (!edge) {
        // Interior tiles: the 20-sample window slides by 4 samples per 4
        // taps, so each step loads ONE new float4 (into the slot of the
        // dropped one) plus the broadcast taps: 2 LDS.128 per 64 FFMA
        // instead of 6.  Five slots in a cycle, unrolled by 5, so the slot
        // rotation is pure register renaming; whole groups of 20 taps here,
        // the remainder in the reload loop below (a static tail of slide
        // steps measured slower: 76 registers).
        const int b0 = j16 + nhp - 4;
        const int ngrp = nh / 20;
        if (ngrp > 0) {
            float4 S[5];
#pragma unroll
            for (int c = 0; c < 5; ++c) S[c] = *reinterpret_cast<const float4 *>(&xs[sh_pos(b0 + 4 * c)]);
            for (int g = 0; g < ngrp; ++g) {
                const int k0 = 20 * g;
#pragma unroll
                for (int st = 0; st < 5; ++st) {
                    const int kk = k0 + 4 * st;
                    float w[20];
#pragma unroll
                    for (int c = 0; c < 5; ++c) {
                        const float4 q = S[(5 - st + c) % 5];
                        w[4 * c] = q.x;
                        w[4 * c + 1] = q.y;
                        w[4 * c + 2] = q.z;
                        w[4 * c + 3] = q.w;
                    }
                    // next lowest float4 (the stage holds nhp+4 samples below
                    // b0+4, so this stays inside it; unused after the last step)
                    const float4 nxt = *reinterpret_cast<const float4 *>(&xs[sh_pos(b0 - kk - 4 + (kk + 4 >= nhp ? 4 : 0))]);
                    const float4 hq = *reinterpret_cast<const float4 *>(&hsm[kk]);
                    const float hk[4] = {hq.x, hq.y, hq.z, hq.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int r = 0; r < SM_R; ++r) acc[r] = fmaf(w[r - u + 4], hk[u], acc[r]);
                    S[(9 - st) % 5] = nxt;  // the dropped (highest) slot becomes the new lowest
                }
            }
            k_done = 20 * ngrp;
        }
    }
    // remaining taps (all of them on edge tiles): reload the window per 4 taps
    for (int k0 = k_done; k0 < nh; k0 += 4) {
        // window: xs[b .. b+20) with b = j16 + nhp - 4 - k0 (a multiple of 4,
        // so both the staging and the window loads are float4-aligned);
        // tap k0+u, output r -> w[r - u + 4]
        const int b = j16 + nhp - 4 - k0;
        float w[20];
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            const float4 q = *reinterpret_cast<const float4 *>(&xs[sh_pos(b + 4 * c)]);
            w[4 * c] = q.x;
            w[4 * c + 1] = q.y;
            w[4 * c + 2] = q.z;
            w[4 * c + 3] = q.w;
        }
        const float4 hq = *reinterpret_cast<const float4 *>(&hsm[k0]);
        const float hk[4] = {hq.x, hq.y, hq.z, hq.w};
        if (!edge) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (k0 + u < nh) {
#pragma unroll
                    for (int r = 0; r < SM_R; ++r) acc[r] = fmaf(w[r - u + 4], hk[u], acc[r]);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = k0 + u;
                if (k < nh) {
#pragma unroll
                    for (int r = 0; r < SM_R; ++r) {
                        const int64_t m = t0 + r - k;
                        if (m >= x_lo && m < x_hi) acc[r] = fmaf(w[r - u + 4], hk[u], acc[r]);
                    }
                }
            }
        }
    }
    float *d = yc + (t0 - n_begin);
    if (t0 + SM_R <= n_end && (reinterpret_cast<uintptr_t>(d) & 15) == 0) {
#pragma unroll
        for (int c = 0; c < SM_R / 4; ++c)
            reinterpret_cast<float4 *>(d)[c] = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
    } else {
#pragma unroll
        for (int r = 0; r < SM_R; ++r)
            if (t0 + r < n_end) d[r] = acc[r];
    }
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
    // 9..32 taps: the tap-stationary kernel (16 taps 0.096 vs 0.103 ms, 32 taps
    // 0.135 vs 0.146 on 2^26 outputs); <= 8 taps the register-window kernel
    // (HBM-bound, 0.93 of the copy bandwidth; tap-stationary 0.091 ms); 33..256
    // the smem kernel (tap-stationary with 64 taps in registers: par, and
    // an FFMA2 pairing of the tap-stationary walk measured slower everywhere)
    static const int knob_kind = [] {  // experiment knob: 1 = default choice, 0 = never tap-stationary
        const char *v = getenv("SC_SHORT_KIND");
        return v ? atoi(v) : 1;
    }();
    if (knob_kind == 1 && nh > 8 && nh <= 4 * TR_MAXNH4) {
        const int nh4 = (int)((nh + 3) / 4);
        int rc = SC_OK;
#define SC_TAPREG(N)                                                                                        \
    case N: rc = launch_tapreg<N>(x, ldx, x_base, x_lo, x_hi, h, ldh, nh, y, ldy, n_begin, n_end, channels, \
                                  stream, run_if);                                                          \
        break
        switch (nh4) {
            SC_TAPREG(3); SC_TAPREG(4); SC_TAPREG(5); SC_TAPREG(6); SC_TAPREG(7); SC_TAPREG(8);
            default: SC_REQUIRE(false, "fir: tap-register kernel, bad tap count");
        }
#undef SC_TAPREG
        return rc;
    }
    if (nh > 32 && nh <= SH_MAXNH) {
        const int64_t tiles = cdiv(n_len, SM_TILE);
        SC_REQUIRE(tiles < (int64_t)INT32_MAX, "fir: output range too large");
        dim3 g((unsigned)tiles, (unsigned)channels);
        k_fir_short_smem<<<g, SM_THREADS, 0, stream>>>(x, ldx, x_base, x_lo, x_hi, h, ldh, (int)nh, y, ldy, n_begin,
                                                       n_end, run_if);
        SC_CHECK_LAUNCH();
        return SC_OK;
    }
    if (nh <= SH_MAXNH) {
        const int64_t tiles = cdiv(n_len, (int64_t)SH_THREADS * SH_R);
        SC_REQUIRE(tiles < (int64_t)INT32_MAX, "fir: output range too large");
        dim3 g((unsigned)tiles, (unsigned)channels);
#define SC_SHORT(NKB)                                                                                          \
    case NKB:                                                                                                  \
        k_fir_short<NKB, SH_R><<<g, SH_THREADS, 0, stream>>>(x, ldx, x_base, x_lo, x_hi, h, ldh, (int)nh, y, ldy, \
                                                             n_begin, n_end, run_if);                              \
        break
        // NKB = ceil(Nh/4) exactly (the compile-time path for multiples of 4)
        switch ((int)((nh + 3) / 4)) {
            SC_SHORT(1); SC_SHORT(2); SC_SHORT(3); SC_SHORT(4);
            SC_SHORT(5); SC_SHORT(6); SC_SHORT(7); SC_SHORT(8);
            default: SC_REQUIRE(false, "fir: short kernel, bad tap count");
        }
#undef SC_SHORT
        SC_CHECK_LAUNCH();
        return SC_OK;
    }
    const int64_t nh_pad = cdiv(nh, FT_STAGE_TAPS) * FT_STAGE_TAPS;
    const int64_t tiles = cdiv(n_len, FT_TILE);
    SC_REQUIRE(tiles < (int64_t)INT32_MAX, "fir: output range too large");
    const int64_t stages = nh_pad / FT_STAGE_TAPS;

    // queried per launch (cheap, host-only): thread-safe and per-device
    int slots_per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&slots_per_sm, k_fir_f32_fast, FT_THREADS, 0) !=
            cudaSuccess || slots_per_sm < 1)
        slots_per_sm = 1;
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
