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
// Gather form on the device: output-stationary, each thread owns R
// consecutive output slots (k_chain_w below); drive samples and taps are
// staged through shared memory per 128-sample chunk, the drive as a
// broadcast, the taps through a per-thread register window.  Zero-skip tests
// run once per staged sample (a warp-ballot scatter mask).  The direct-form
// oracle restatement (k_direct_dd) closes the file.

#include <algorithm>

#include "sc_common.cuh"

namespace sc {
namespace {

constexpr int TB = 256;  // direct-form CTA size

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

// ---------------------------------------------------------------- windowed chain
// One kernel for every ordered launch.  A CTA of TB threads (32 or 128) owns
// a tile of TB*R consecutive outputs, thread j the R consecutive outputs
// tj..tj+R-1 (R = 8, 4, 2 or 1, picked per launch so the grid keeps every SM
// sub-partition busy).  Drive samples go through shared memory in chunks of
// 128, the taps of the chunk x tile in a padded stage (TapStage: conflict-
// free 16-byte tap loads).  Per 8-sample "u-block" a thread keeps a register
// window of R+7 taps; sliding to the next u-block reuses R-1 of them, so a
// u-block costs 8 taps (two float / four double 16-byte loads for R >= 4)
// and two (float) / four (double) broadcast vector loads of the drive for
// 8R MACs.  Interior chunks of a dense drive
// (every (output, sample) pair valid, nothing skipped) run a fully unrolled
// path with no tests; edge u-blocks test validity per thread and only the
// u-blocks that straddle an edge pay per-MAC predicates.  The next chunk's
// drive and taps are loaded into registers while the current chunk is
// computed (double-buffered stage, one barrier per chunk).
constexpr int CW_MC = 128;  // drive samples per chunk
constexpr int CW_U = 8;     // samples per u-block
constexpr int CW_WIDE = CW_MC < 128 ? CW_MC : 128;  // the wide-CTA variant (SC_CHAIN_TB=128)
static_assert(32 % CW_U == 0, "a u-block's scatter bits sit in one mask word");

// Tap stage layout: the taps sit in groups of R (the stride between two
// threads' bases) padded to S elements.  Lane l's base is group l, so every
// tap address is a per-thread base S*l plus the compile-time (or 8-aligned)
// offset pos(c): [reg + imm] loads.  For R = 8 and 4 the strides (float 12 /
// 4, double 10 / 6 elements) are multiples of 16 bytes and put the 8 lanes of
// each 16-byte-load phase on distinct banks, so a thread reads its 8 new taps
// per u-block with two (float) or four (double) conflict-free LDS.128.  R = 2
// and 1 keep scalar loads with odd strides (3 and 1).
template <typename T, int R>
struct TapStage {
    static constexpr int S = R == 8 ? (sizeof(T) == 4 ? 12 : 10) : R == 4 ? (sizeof(T) == 4 ? 4 : 6) : R == 2 ? 3 : 1;
    static constexpr bool VEC = R >= 4;
    static constexpr int XV = 16 / (int)sizeof(T);  // elements per 16-byte load
    __host__ __device__ static constexpr int pos(int i) { return (i / R) * S + i % R; }
    // w[0..7] = taps c..c+7 of this thread, p = stage + S*l + pos(c), c % 8 == 0
    __device__ static __forceinline__ void load8(const T *p, T *w) {
        if constexpr (VEC) {
#pragma unroll
            for (int g = 0; g < 8 / R; ++g)
#pragma unroll
                for (int v = 0; v < R; v += XV) {
                    if constexpr (sizeof(T) == 4) {
                        const float4 f = *reinterpret_cast<const float4 *>(p + g * S + v);
                        w[g * R + v] = f.x, w[g * R + v + 1] = f.y, w[g * R + v + 2] = f.z, w[g * R + v + 3] = f.w;
                    } else {
                        const double2 d = *reinterpret_cast<const double2 *>(p + g * S + v);
                        w[g * R + v] = d.x, w[g * R + v + 1] = d.y;
                    }
                }
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) w[q] = p[pos(q)];
        }
    }
};
static_assert(TapStage<float, 8>::S * 4 % 16 == 0 && TapStage<double, 8>::S * 8 % 16 == 0 &&
                  TapStage<float, 4>::S * 4 % 16 == 0 && TapStage<double, 4>::S * 8 % 16 == 0,
              "16-byte aligned tap groups");

// The per-chunk barrier: a warp barrier for one-warp CTAs (it orders the
// warp's shared-memory accesses like __syncthreads).
template <int TB>
__device__ __forceinline__ void chunk_sync() {
    if constexpr (TB == 32)
        __syncwarp();
    else
        __syncthreads();
}

template <typename T, int SKIP, int R, bool FUSED, int CW_TB>
__global__ void __launch_bounds__(CW_TB, (sizeof(T) == 4 ? 6 : 4) * (128 / CW_TB)) k_chain_w(ChainArgs<T> a) {
    constexpr int TILE = CW_TB * R;
    constexpr int HS = TILE + CW_MC - 1;  // taps per stage
    using ST = TapStage<T, R>;
    // + one spare group: the window's initial load reads 8 taps past the
    // thread's base at chunk offset CW_MC (only R-1 of them are used)
    constexpr int HSP = (ST::pos(HS + 8) + 4) / 4 * 4;
    constexpr int HPT = (HS + CW_TB - 1) / CW_TB;  // tap loads per thread per chunk
    constexpr int XPT = CW_MC / CW_TB;             // drive samples staged per thread per chunk
    static_assert(CW_MC % CW_TB == 0 && CW_TB % 32 == 0, "chunk staging");
    constexpr int W = R + CW_U - 1;
    constexpr int XV = 16 / (int)sizeof(T);  // drive samples per vector load
    __shared__ __align__(16) T xs[2][CW_MC];
    __shared__ unsigned xmask[2][CW_MC / 32];
    // per chunk and warp: every staged drive sample and tap finite
    __shared__ unsigned xfin[2][CW_TB / 32];
    __shared__ __align__(16) T hs[2][HSP];
    // A gated launch (run_if: the tensor-core path's non-finite fallback) is
    // launched with programmatic stream serialisation: its CTAs become
    // resident while the tensor-core kernel runs and wait here for it (a
    // no-op for launches without the attribute), which hides this launch's
    // ~3 us of set-up behind that kernel.
    if (a.run_if) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.run_if && *a.run_if == 0) return;  // block-uniform
    // channel-local base pointers (the param struct stays in the constant bank)
    const T *xb = a.x + blockIdx.y * a.ldx;
    T *outa = a.out_a + blockIdx.y * a.ldo;
    const int64_t hoff = blockIdx.y * a.ldh;
    const T *initc = a.init ? a.init + blockIdx.y * a.ld_init : nullptr;
    T *outb = a.out_b ? a.out_b + blockIdx.y * a.ld_outb : nullptr;
    const int64_t n_tiles = (a.n_out + TILE - 1) / TILE;
    const int64_t t_end = a.t0 + a.n_out;
    const int64_t init_len = a.init_len_dev ? a.init_len_dev[blockIdx.y * a.ld_st] : a.init_len;
    const int tid = threadIdx.x;
    // the tap for (r, im) sits at stage index tid*R + (CW_MC - 1) + r - im
    const int hth = ST::S * tid;  // padded base of this thread

    for (int64_t tb = blockIdx.x; tb < n_tiles; tb += gridDim.x) {
        const int64_t tile0 = a.t0 + tb * TILE;
        const int64_t tile_last = (tile0 + TILE < t_end ? tile0 + TILE : t_end) - 1;
        const int64_t tj = tile0 + (int64_t)tid * R;
        T acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t t = tj + r;
            acc[r] = (initc != nullptr && t < t_end && (t - a.t0) < init_len) ? initc[t - a.t0] : T(0);
        }
        // chunk range of segment s for this tile: [blo, bhi)
        // The chunk walk: segment s, chunk start mc, and the segment's
        // fields cached in registers (hi = end of its drive range for this
        // tile), so stepping inside a segment is one add and one compare.
        struct Chunk {
            int s;
            int64_t mc, hi, nh;
            const T *h;
        };
        auto first_from = [&](int s) {  // first chunk of the first non-empty segment >= s
            Chunk c{s, 0, 0, 0, nullptr};
            for (; c.s < a.nseg; ++c.s) {
                c.nh = a.seg[c.s].nh;
                const int64_t lo = tile0 - c.nh + 1 > a.seg[c.s].m_lo ? tile0 - c.nh + 1 : a.seg[c.s].m_lo;
                c.hi = tile_last + 1 < a.seg[c.s].m_hi ? tile_last + 1 : a.seg[c.s].m_hi;
                if (lo < c.hi) {
                    c.mc = lo;
                    c.h = static_cast<const T *>(a.seg[c.s].h) + hoff;
                    break;
                }
            }
            return c;
        };
        auto next_of = [&](const Chunk &c) {
            if (c.mc + CW_MC < c.hi) {
                Chunk n = c;
                n.mc += CW_MC;
                return n;
            }
            return first_from(c.s + 1);
        };
        Chunk cur = first_from(0);
        // register prefetch of one chunk
        T px[XPT];
        bool pbit[XPT];
        T ph[HPT];
        auto fetch = [&](const Chunk &c) {
            const int64_t mc = c.mc;
            // Interior chunks (the whole chunk inside the segment, the whole
            // tap range inside the IR: block-uniform tests) load without
            // per-element 64-bit bounds checks, at [reg + imm] addresses.
            const int64_t bhi = c.hi;
            const T *xp = xb + (mc - a.x_off) + tid;
            if (mc + CW_MC <= bhi) {
#pragma unroll
                for (int k = 0; k < XPT; ++k) {
                    px[k] = xp[k * CW_TB];
                    pbit[k] = !skipped<SKIP>(px[k], a.thr);
                }
            } else {
                const int rem = (int)(bhi - mc);  // < CW_MC here
#pragma unroll
                for (int k = 0; k < XPT; ++k) {
                    const bool in = tid + k * CW_TB < rem;
                    px[k] = in ? xp[k * CW_TB] : T(0);
                    pbit[k] = in && !skipped<SKIP>(px[k], a.thr);
                }
            }
            const int64_t nh = c.nh;
            const int64_t kbase = tile0 - mc - CW_MC + 1;
            const T *__restrict__ hp = c.h + kbase + tid;
            if (kbase >= 0 && kbase + HS <= nh) {
#pragma unroll
                for (int j = 0; j < HPT; ++j)
                    ph[j] = (j * CW_TB + CW_TB <= HS || tid + j * CW_TB < HS) ? hp[j * CW_TB] : T(0);
            } else {
                // k = kbase + i in [0, nh): i in [-kbase, nh - kbase)
                const int ilo = kbase < 0 ? (int)(-kbase < HS ? -kbase : HS) : 0;
                const int64_t hi64 = nh - kbase;
                const int ihi = hi64 < 0 ? 0 : hi64 < HS ? (int)hi64 : HS;
#pragma unroll
                for (int j = 0; j < HPT; ++j) {
                    const int i = tid + j * CW_TB;
                    ph[j] = (i >= ilo && i < ihi) ? hp[j * CW_TB] : T(0);
                }
            }
        };
        auto stash = [&](int buf) {
            // Skipped samples are stored as zero: when every staged sample
            // and tap of the chunk is finite, adding x*h for a zeroed sample
            // or a zero (out-of-range) tap adds +-0, which leaves a chain
            // value unchanged (chains start at +0 or a residue and are never
            // -0), so the unpredicated path can run the whole chunk.
            bool fin = true;
#pragma unroll
            for (int k = 0; k < XPT; ++k) {
                xs[buf][tid + k * CW_TB] = pbit[k] ? px[k] : T(0);
                fin = fin && (!pbit[k] || isfinite((double)px[k]));
                const unsigned bits = __ballot_sync(0xffffffffu, pbit[k]);
                if ((tid & 31) == 0) xmask[buf][(tid + k * CW_TB) >> 5] = bits;
            }
#pragma unroll
            for (int j = 0; j < HPT; ++j) fin = fin && isfinite((double)ph[j]);
            const bool wfin = __all_sync(0xffffffffu, fin);
            if ((tid & 31) == 0) xfin[buf][tid >> 5] = wfin ? 1u : 0u;
#pragma unroll
            for (int j = 0; j < HPT; ++j) {
                const int i = tid + j * CW_TB;
                // pos(tid + j*TB) = pos(tid) + j*(TB/R)*S since TB % R == 0
                if (i < HS) hs[buf][ST::pos(tid) + j * (CW_TB / R) * ST::S] = ph[j];
            }
        };
        if (cur.s < a.nseg) {
            fetch(cur);
            stash(0);
        }
        chunk_sync<CW_TB>();
        int buf = 0;
        while (cur.s < a.nseg) {
            const Chunk nxt = next_of(cur);
            if (nxt.s < a.nseg) fetch(nxt);  // global loads in flight during the compute below

            const int64_t cmc = cur.mc;
            const int64_t nh = cur.nh;
            const int64_t bhi = cur.hi;
            const int mcount = (int)(bhi - cmc < CW_MC ? bhi - cmc : CW_MC);
            const T *xsb = xs[buf];
            const T *hsb = hs[buf];
            const bool full = (cmc >= tile_last - nh + 1) && (cmc + mcount - 1 <= tile0);
            bool dense = mcount == CW_MC;
            bool finite = true;
#pragma unroll
            for (int w = 0; w < CW_TB / 32; ++w) finite = finite && xfin[buf][w] != 0;
#pragma unroll
            for (int q = 0; q < CW_MC / 32; ++q) dense = dense && xmask[buf][q] == ~0u;
            if ((full && dense) || finite) {
                // interior: every (output, sample) pair valid, nothing skipped
                T w[W];
                {
                    T nx[8];
                    ST::load8(hsb + hth + ST::pos(CW_MC - CW_U), w);
                    ST::load8(hsb + hth + ST::pos(CW_MC), nx);
#pragma unroll
                    for (int q = 8; q < W; ++q) w[q] = nx[q - 8];
                }
#pragma unroll
                for (int ub = 0; ub < CW_MC / CW_U; ++ub) {
                    if (ub > 0) {
#pragma unroll
                        for (int p = R - 2; p >= 0; --p) w[CW_U + p] = w[p];
                        ST::load8(hsb + hth + ST::pos(CW_MC - CW_U - ub * CW_U), w);
                    }
                    T xv[CW_U];
#pragma unroll
                    for (int v = 0; v < CW_U; v += XV) {
                        if (sizeof(T) == 4) {
                            const float4 f = *reinterpret_cast<const float4 *>(&xsb[ub * CW_U + v]);
                            xv[v] = (T)f.x, xv[v + 1] = (T)f.y, xv[v + 2] = (T)f.z, xv[v + 3] = (T)f.w;
                        } else {
                            const double2 d = *reinterpret_cast<const double2 *>(&xsb[ub * CW_U + v]);
                            xv[v] = (T)d.x, xv[v + 1] = (T)d.y;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < CW_U; ++u)
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r] = mac_step<FUSED>(acc[r], xv[u], w[r - u + CW_U - 1]);
                }
            } else {
                // t - m = rel + r - im.  Only u-blocks with at least one valid
                // (output, sample) pair are visited: im0 in (rel - nh - 7 + R... ]
                // i.e. rel + R - 1 - im0 >= 0 and rel - im0 - 7 < nh.
                const int64_t rel = tj - cmc;
                int64_t ilo = rel - nh - (CW_U - 1) + 1;  // smallest im0 with rel - im0 - 7 < nh
                int64_t ihi = rel + R - 1;                // largest im0 with rel + R - 1 - im0 >= 0
                ilo = ilo < 0 ? 0 : (ilo + CW_U - 1) / CW_U * CW_U;
                ihi = ihi > mcount - 1 ? mcount - 1 : ihi;
                const int nh32 = (int)(nh < INT32_MAX ? nh : INT32_MAX);
                for (int im0 = (int)ilo; im0 <= (int)ihi; im0 += CW_U) {
                    T w[W];
                    // c0 = CW_MC - CW_U - im0 is a multiple of 8, so pos(c0 + q) = pos(c0) + pos(q)
                    const T *hp = hsb + hth + ST::pos(CW_MC - CW_U - im0);
                    {
                        T nx[8];
                        ST::load8(hp, w);
                        ST::load8(hp + ST::pos(8), nx);
#pragma unroll
                        for (int q = 8; q < W; ++q) w[q] = nx[q - 8];
                    }
                    // samples im0..im0+7 (bits past mcount are 0: m >= bhi)
                    const unsigned bits = (xmask[buf][im0 >> 5] >> (im0 & 31)) & 0xFFu;
                    const int e = (int)(rel - im0);  // |e| < nh + 8 here
                    const bool inside = (e - (CW_U - 1) >= 0) && (e + R - 1 < nh32);
                    if (bits == 0xFFu && inside) {
#pragma unroll
                        for (int u = 0; u < CW_U; ++u) {
                            const T xv = xsb[im0 + u];
#pragma unroll
                            for (int r = 0; r < R; ++r) acc[r] = mac_step<FUSED>(acc[r], xv, w[r - u + CW_U - 1]);
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < CW_U; ++u) {
                            if (!(bits & (1u << u))) continue;
                            const T xv = xsb[im0 + u];
#pragma unroll
                            for (int r = 0; r < R; ++r)  // 0 <= t - m < nh
                                if ((unsigned)(e + r - u) < (unsigned)nh32)
                                    acc[r] = mac_step<FUSED>(acc[r], xv, w[r - u + CW_U - 1]);
                        }
                    }
                }
            }
            if (nxt.s < a.nseg) stash(buf ^ 1);
            chunk_sync<CW_TB>();
            buf ^= 1;
            cur = nxt;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
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

template <typename T, int SKIP, bool FUSED, int TB>
int launch_chain_rf(int R, dim3 grid, cudaStream_t stream, const ChainArgs<T> &a) {
    auto go = [&](auto kern) -> cudaError_t {
        if (!a.run_if) {
            kern<<<grid, TB, 0, stream>>>(a);
            return cudaGetLastError();
        }
        return launch_pdl(kern, grid, dim3(TB), 0, stream, a);  // gated: see k_chain_w
    };
    cudaError_t e;
    switch (R) {
        case 8: e = go(k_chain_w<T, SKIP, 8, FUSED, TB>); break;
        case 4: e = go(k_chain_w<T, SKIP, 4, FUSED, TB>); break;
        case 2: e = go(k_chain_w<T, SKIP, 2, FUSED, TB>); break;
        default: e = go(k_chain_w<T, SKIP, 1, FUSED, TB>); break;
    }
    SC_REQUIRE(e == cudaSuccess, "chain: kernel launch failed: %s", cudaGetErrorString(e));
    return SC_OK;
}

// CTA width.  One-warp CTAs make the per-chunk barrier a warp barrier:
// 4-10 % faster for float chains and for small float64 launches.  Large
// float64 launches (at least 4 waves of 128-thread tiles) are FP64-pipe
// bound and run ~1 % faster on 128-thread CTAs.  SC_CHAIN_TB=32|128 forces.
int chain_tb(size_t es, int64_t n_out, int64_t channels, int R) {
    static const int forced = [] {
        const char *v = getenv("SC_CHAIN_TB");
        return v ? atoi(v) : 0;
    }();
    if (forced == 32 || forced == CW_WIDE) return forced;
    if (es == 8 && channels * cdiv(n_out, (int64_t)CW_WIDE * R) >= 4 * (int64_t)sm_count()) return CW_WIDE;
    return 32;
}

// float chains are always fused (one instantiation); double picks per call
template <typename T, int SKIP>
int launch_chain_r(int R, int tb, dim3 grid, cudaStream_t stream, const ChainArgs<T> &a, bool fused) {
    const bool narrow = tb == 32;
    if constexpr (sizeof(T) == 8) {
        if (fused)
            return narrow ? launch_chain_rf<T, SKIP, true, 32>(R, grid, stream, a)
                          : launch_chain_rf<T, SKIP, true, CW_WIDE>(R, grid, stream, a);
    }
    return narrow ? launch_chain_rf<T, SKIP, false, 32>(R, grid, stream, a)
                  : launch_chain_rf<T, SKIP, false, CW_WIDE>(R, grid, stream, a);
}

// Outputs per thread: the largest R that still gives every SM about 16 warps
// (two per sub-partition, each carrying R independent chains).
int pick_r(int64_t n_out, int64_t channels, size_t es) {
    static const int forced = [] {
        const char *v = getenv("SC_CHAIN_R");  // experiment knob
        return v ? atoi(v) : 0;
    }();
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8) return forced;
    // float64 chains run out of FP64-pipe and LDS throughput long before
    // they run out of warps: more independent chains per thread (larger R)
    // beat more warps (10 s through 17.6 M taps: R=8 0.946 s, R=4 0.989;
    // cfg1: R=2 26.5 us, R=1 29.2).  float32 wants ~16 warps per SM.
    const int64_t warps_per_sm = es == 8 ? 4 : 16;
    const int64_t want_threads = (int64_t)sm_count() * warps_per_sm * 32;
    for (int R = 8; R > 1; R >>= 1)
        if (channels * cdiv(n_out, R) >= want_threads) return R;
    return 1;
}

// ---------------------------------------------------------------- small strict float64
// k_chain_small: the latency kernel for small single-IR float64 strict
// launches (cfg1: 48,000 x 1,024 taps, 49,023 chains of 1,024 dependent
// DMUL+DADD steps).  Such launches cannot fill the FP64 pipe: there are only
// ~83 chains per SM sub-partition, so the time per step is set by how many
// chains share a sub-partition's 16-lane FP64 pipe and by how well one warp
// hides its own latencies.  Measured (tools/ubench/chain_small.cu): 3
// consecutive outputs per thread (96 chains per warp) beat 2 (two warps on
// some sub-partitions) and 4 (idle sub-partitions); 4-warp CTAs (one warp
// per sub-partition of the SM that holds the CTA; cfg1: 128 CTAs) beat 1-
// and 3-warp CTAs (cfg1 per bench step: 15.5 vs 16.6 and 22.4 us; large
// launches 1-3 % faster too); k_chain_w's chunked, windowed form took
// 22.6 us at cfg1.
//
// Every output t runs one chain over a fixed step count nhp = nh rounded up
// to 8: step j takes drive sample m = t - nhp + 1 + j and tap hs[nhp-1-j]
// (taps ascending in shared memory, zero beyond nh), the drive zero outside
// [m_lo, m_hi).  The steps the reference does not take add x*0 or 0*h = +-0,
// which leaves the chain unchanged when the operands are finite (chains start
// at +0 and never become -0), so the result is bit-identical to k_chain_w's
// and the reference's.  A CTA whose padded steps would meet a non-finite
// operand runs the bounded per-output loop instead (same products, same
// order, no padded terms).
//
// Staging: the CTA's drive window (TILE + nhp - 1 samples) and the taps
// arrive by cp.async.bulk on one mbarrier, issued by one thread while the
// warp writes the zero padding.  (Splitting the staging into per-128-step
// chunks so the chain could start earlier measured slower: the first chunk
// landed later than the whole window does in one transfer.)
constexpr int CS_R = 3;
constexpr int CS_TB = 128;
constexpr int CS_MAX_NH = 2048;                  // <= 34 KB of shared memory

__device__ __forceinline__ void cs_bulk(void *dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// Skip modes (scatter_convolve_skip_zeros, core.py:150-167): samples the
// reference skips are zeroed in the staged window, so a skipped sample adds
// x*0... = +-0 like a padded step -- exact when every tap is finite (checked
// by every CTA in skip mode); otherwise the bounded loop reads the drive from
// memory and skips those samples itself.
template <int R, int TB, int SKIP>
__global__ void __launch_bounds__(TB) k_chain_small(const double *__restrict__ x, int64_t x_off, int64_t m_lo,
                                                    int64_t m_hi, const double *__restrict__ h, int nh, int64_t t0,
                                                    int64_t n_out, double *__restrict__ y, double thr) {
    extern __shared__ __align__(16) unsigned char cs_smem[];
    constexpr int TILE = TB * R;
    const int nhp = (nh + 7) & ~7;
    const int P = nhp - nh;
    const int nxs = TILE + nhp - 1;
    const int64_t tile0 = t0 + (int64_t)blockIdx.x * TILE;
    const int64_t g0 = tile0 - nhp + 1;  // drive index m of xs[0]
    // 16-byte aligned drive samples m share one parity; shift xs by one
    // element when needed so they land 16-byte aligned in shared memory
    const uintptr_t xa = reinterpret_cast<uintptr_t>(x) - (uintptr_t)(x_off * 8);  // address of m = 0
    const int apar = (int)((xa >> 3) & 1);
    const int sx = (int)((apar - g0) & 1);
    uint64_t *bar = reinterpret_cast<uint64_t *>(cs_smem);
    double *hs = reinterpret_cast<double *>(cs_smem + 16);  // nhp taps ascending
    double *xs = hs + nhp + sx;                               // nxs drive samples
    const bool h_bulk = (reinterpret_cast<uintptr_t>(h) & 15) == 0;
    const int tid = threadIdx.x;
    const uint32_t bb = (uint32_t)__cvta_generic_to_shared(bar);
    // drive indices inside the signal: [a, b); bulk part [a16, a16 + n16)
    const int64_t a = max(g0, m_lo), b = min(g0 + nxs, m_hi);
    const int64_t a16 = a + ((int)(a & 1) != apar);
    const int64_t n16 = b > a16 ? (b - a16) & ~(int64_t)1 : 0;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bb), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        const uint32_t xbytes = (uint32_t)(n16 * 8), hbytes = h_bulk ? (uint32_t)(nh & ~1) * 8 : 0;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(xbytes + hbytes)
                     : "memory");
        if (xbytes) cs_bulk(xs + (a16 - g0), x + (a16 - x_off), xbytes, bb);
        if (hbytes) cs_bulk(hs, h, hbytes, bb);
    }
    // plain stores: zero drive outside [m_lo, m_hi) (edge CTAs), the (at
    // most two) unaligned ends of the bulk range, zero taps past nh, and
    // every tap when h is not 16-byte aligned
    const bool edge = g0 < m_lo || g0 + nxs > m_hi;
    if (edge)
        for (int i = tid; i < nxs; i += TB) {
            const int64_t m = g0 + i;
            if (m < m_lo || m >= m_hi) xs[i] = 0.0;
        }
    if (tid == 0 && a < b) {
        if (a16 > a) xs[a - g0] = x[a - x_off];
        for (int64_t m = a16 + n16; m < b; ++m) xs[m - g0] = x[m - x_off];
    }
    for (int k = nh + tid; k < nhp; k += TB) hs[k] = 0.0;
    if (!h_bulk)
        for (int k = tid; k < nh; k += TB) hs[k] = h[k];
    else if ((nh & 1) && tid == 0)
        hs[nh - 1] = h[nh - 1];
    __syncthreads();  // plain stores visible; the mbarrier init too
    {
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                " selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(bb)
                : "memory");
    }
    // Padded steps are exact only with finite operands: x meets a zero tap in
    // the P front steps (drive xs[0, TILE+P-1)), and a real tap meets zero
    // drive only in edge CTAs -- or, in skip mode, at any skipped sample --
    // which check the taps.
    bool fin = true;
    if (P > 0)
        for (int i = tid; i < TILE + P - 1; i += TB) fin &= isfinite(xs[i]);
    if (edge || SKIP != SC_SKIP_NONE)
        for (int k = tid; k < nh; k += TB) fin &= isfinite(hs[k]);
    if constexpr (SKIP != SC_SKIP_NONE) {
        __syncthreads();  // the front check read xs before it is masked
        for (int i = tid; i < nxs; i += TB)
            if (skipped<SKIP>(xs[i], thr)) xs[i] = 0.0;
    }
    fin = TB == 32 ? __all_sync(0xffffffffu, fin) : __syncthreads_and(fin);
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    const double *xb = xs + tid * R;  // xs index of (output r, step j) = tid*R + r + j
    if (fin) {
        double wx[R + 7];
#pragma unroll
        for (int k = 0; k < R - 1; ++k) wx[k] = xb[k];
        // unrolled 16 u-blocks deep: ptxas then interleaves the DMULs of
        // later steps into the DADD chains of earlier ones (cfg1 15.4 ->
        // 14.6 us against 4 deep; 32 deep measured 16.4)
#pragma unroll 16
        for (int jq = 0; jq < nhp; jq += 8) {  // steps jq..jq+7
            double hv[8];
#pragma unroll
            for (int k = 0; k < 8; k += 2) {  // their taps, descending in memory
                const double2 d = *reinterpret_cast<const double2 *>(hs + nhp - 8 - jq + k);
                hv[7 - k] = d.x, hv[6 - k] = d.y;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) wx[R - 1 + k] = xb[jq + R - 1 + k];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = __dadd_rn(acc[r], __dmul_rn(wx[u + r], hv[u]));
#pragma unroll
            for (int k = 0; k < R - 1; ++k) wx[k] = wx[8 + k];
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t t = tile0 + tid * R + r;
            // tap t-m in [0, nh) <=> j >= P; drive m in [m_lo, m_hi)
            const int64_t lo = max((int64_t)P, m_lo - t + nhp - 1);
            const int64_t hi = min((int64_t)nhp, m_hi - t + nhp - 1);
            if constexpr (SKIP == SC_SKIP_NONE) {
                for (int64_t j = lo; j < hi; ++j)
                    acc[r] = __dadd_rn(acc[r], __dmul_rn(xb[r + j], hs[nhp - 1 - j]));
            } else {
                // the staged window is masked: read the drive itself
                for (int64_t j = lo; j < hi; ++j) {
                    const double xv = x[t - nhp + 1 + j - x_off];
                    if (!skipped<SKIP>(xv, thr)) acc[r] = __dadd_rn(acc[r], __dmul_rn(xv, hs[nhp - 1 - j]));
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = (int64_t)blockIdx.x * TILE + tid * R + r;
        if (i < n_out) y[i] = acc[r];
    }
}

size_t chain_small_smem(int nh) {
    const int nhp = (nh + 7) & ~7;
    return 16 + sizeof(double) * (size_t)(2 * nhp + CS_TB * CS_R);
}

// Strict float64 launches of one IR of at most 2,048 taps (sc_fir_full,
// shards) take k_chain_small at every size: it also beats k_chain_w on
// large launches
// (tools/ubench/cfg1_lib.cu, one launch after an L2 flush: 8 M x 1,024 taps
// 1.01 ms vs 1.96 ms; 2 M x 2,048 0.57 vs 0.77; 4 M x 64 45 us vs 562).
// SC_CHAIN_SMALL=0 turns it off (A/B and tests).
bool chain_small_ok(int64_t n_out, int64_t nh) {
    static const int forced = [] {
        const char *v = getenv("SC_CHAIN_SMALL");
        return v ? atoi(v) : -1;
    }();
    (void)n_out;
    return forced != 0 && nh >= 1 && nh <= CS_MAX_NH;
}

template <typename T>
int launch_chain_t(int skip_mode, double threshold, const void *x, int64_t x_off,
                   const ChainSeg *segs, int nseg, const void *init, int64_t init_len,
                   const int64_t *init_len_dev, int64_t t0, int64_t n_out, void *out_a,
                   int64_t n_a, void *out_b, cudaStream_t stream, const unsigned *run_if,
                   const ChainBatch *batch, bool fused) {
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
    if constexpr (sizeof(T) == 8) {
        if (!fused && nseg == 1 && !init && !init_len_dev && !out_b && !run_if && !batch && n_a >= n_out &&
            chain_small_ok(n_out, segs[0].nh)) {
            const int nh = (int)segs[0].nh;
            const dim3 grid((unsigned)cdiv(n_out, (int64_t)CS_TB * CS_R));
            const size_t sm = chain_small_smem(nh);
            const double *xd = static_cast<const double *>(x), *hd = static_cast<const double *>(segs[0].h);
            double *yd = static_cast<double *>(out_a);
            const int64_t lo = segs[0].m_lo, hi = segs[0].m_hi;
            switch (skip_mode) {
                case SC_SKIP_NONE:
                    k_chain_small<CS_R, CS_TB, SC_SKIP_NONE><<<grid, CS_TB, sm, stream>>>(xd, x_off, lo, hi, hd, nh,
                                                                                           t0, n_out, yd, threshold);
                    break;
                case SC_SKIP_LE:
                    k_chain_small<CS_R, CS_TB, SC_SKIP_LE><<<grid, CS_TB, sm, stream>>>(xd, x_off, lo, hi, hd, nh,
                                                                                         t0, n_out, yd, threshold);
                    break;
                case SC_SKIP_NOT_GT:
                    k_chain_small<CS_R, CS_TB, SC_SKIP_NOT_GT><<<grid, CS_TB, sm, stream>>>(
                        xd, x_off, lo, hi, hd, nh, t0, n_out, yd, threshold);
                    break;
                default: SC_REQUIRE(false, "chain: bad skip_mode %d", skip_mode);
            }
            SC_CHECK_LAUNCH();
            return SC_OK;
        }
    }
    const int R = pick_r(n_out, channels, sizeof(T));
    // Grid-stride over tiles.  A device-gated launch (run_if) is usually a
    // no-op, so it gets a small grid that exits in microseconds.
    const int tb = chain_tb(sizeof(T), n_out, channels, R);
    const int64_t cap = run_if ? std::max<int64_t>(1, 4 * (128 / tb) * (int64_t)sm_count() / channels)
                               : (int64_t)INT32_MAX - 1;
    const dim3 grid((unsigned)std::min<int64_t>(cdiv(n_out, (int64_t)tb * R), cap), (unsigned)channels);
    switch (skip_mode) {
        case SC_SKIP_NONE: launch_chain_r<T, SC_SKIP_NONE>(R, tb, grid, stream, a, fused); break;
        case SC_SKIP_LE: launch_chain_r<T, SC_SKIP_LE>(R, tb, grid, stream, a, fused); break;
        case SC_SKIP_NOT_GT: launch_chain_r<T, SC_SKIP_NOT_GT>(R, tb, grid, stream, a, fused); break;
        default: SC_REQUIRE(false, "chain: bad skip_mode %d", skip_mode);
    }
    SC_CHECK_LAUNCH();
    return SC_OK;
}

// ---------------------------------------------------------------- direct form
// direct_form (core.py:102-119): each output is math.fsum of its individually
// rounded products e[m]*h[n-m], i.e. their EXACT sum rounded once.  One
// thread per output runs CPython's fsum: Shewchuk's non-overlapping
// "partials" (each new product is two-summed through them, so their exact
// sum is always the exact running sum), then the partials are added from the
// top with the round-half-even fix-up across partials -- the same published
// algorithm, so the results are bit-identical to math.fsum.  Non-overlapping
// doubles number at most ~40 (2098 exponent bits / 53), kept in local
// memory; the usual count is 1-3.  Non-finite summands follow fsum: a NaN
// or an Inf product short-circuits to their IEEE sum; -inf + inf and an
// intermediate overflow of finite products, which fsum raises on, set
// status bits 2 and 1 (the host raises ValueError / OverflowError).
constexpr int FSUM_MAXP = 48;

__global__ void __launch_bounds__(TB) k_direct_fsum(const double *__restrict__ e, int64_t ne,
                                                    const double *__restrict__ h, int64_t nh,
                                                    double *__restrict__ y, unsigned *status) {
    const int64_t n = (int64_t)blockIdx.x * TB + threadIdx.x;
    if (n >= ne + nh - 1) return;
    const int64_t lo = n - nh + 1 > 0 ? n - nh + 1 : 0;
    const int64_t hi = n < ne - 1 ? n : ne - 1;
    double p[FSUM_MAXP];
    int np = 0;
    double special = 0.0, inf_sum = 0.0;
    unsigned bad = 0;
    for (int64_t m = lo; m <= hi; ++m) {
        double x = __dmul_rn(e[m], h[n - m]);
        const double xsave = x;
        int i = 0;
        for (int j = 0; j < np; ++j) {
            double yv = p[j];
            if (fabs(x) < fabs(yv)) {
                const double t = x;
                x = yv;
                yv = t;
            }
            const double hs = __dadd_rn(x, yv);
            const double yr = __dsub_rn(hs, x);
            const double ls = __dsub_rn(yv, yr);
            if (ls != 0.0) p[i++] = ls;
            x = hs;
        }
        np = i;
        if (x != 0.0) {
            if (!isfinite(x)) {
                if (isfinite(xsave)) bad |= 1u;  // intermediate overflow
                if (isinf(xsave)) inf_sum = __dadd_rn(inf_sum, xsave);
                special = __dadd_rn(special, xsave);
                np = 0;
            } else if (np < FSUM_MAXP) {
                p[np++] = x;
            }
        }
    }
    double r = 0.0;
    if (special != 0.0 || isnan(special)) {
        if (isnan(inf_sum)) bad |= 2u;  // -inf + inf
        r = special;
    } else if (np > 0) {
        double hs = p[--np], ls = 0.0;
        while (np > 0) {
            const double x = hs;
            const double yv = p[--np];
            hs = __dadd_rn(x, yv);
            const double yr = __dsub_rn(hs, x);
            ls = __dsub_rn(yv, yr);
            if (ls != 0.0) break;
        }
        // round half to even across the partials below: if the rounding of
        // hs + ls was a tie and the next partial pushes past it, round away
        if (np > 0 && ((ls < 0.0 && p[np - 1] < 0.0) || (ls > 0.0 && p[np - 1] > 0.0))) {
            const double yv = ls * 2.0;
            const double x = __dadd_rn(hs, yv);
            const double yr = __dsub_rn(x, hs);
            if (yv == yr) hs = x;
        }
        r = hs;
    }
    y[n] = r;
    if (bad && status) atomicOr(status, bad);
}

}  // namespace

int launch_chain(int dtype, int skip_mode, double threshold, const void *x, int64_t x_off,
                 const ChainSeg *segs, int nseg, const void *init, int64_t init_len,
                 const int64_t *init_len_dev, int64_t t0, int64_t n_out, void *out_a,
                 int64_t n_a, void *out_b, cudaStream_t stream, const unsigned *run_if,
                 const ChainBatch *batch, bool fused) {
    if (dtype == SC_F64)
        return launch_chain_t<double>(skip_mode, threshold, x, x_off, segs, nseg, init, init_len,
                                      init_len_dev, t0, n_out, out_a, n_a, out_b, stream, run_if, batch, fused);
    if (dtype == SC_F32)
        return launch_chain_t<float>(skip_mode, threshold, x, x_off, segs, nseg, init, init_len,
                                     init_len_dev, t0, n_out, out_a, n_a, out_b, stream, run_if, batch, fused);
    set_error("chain: bad dtype %d", dtype);
    return SC_ERR_ARG;
}

int launch_direct_form(const double *e, int64_t ne, const double *h, int64_t nh, double *y,
                       unsigned *status, cudaStream_t stream) {
    const int64_t nout = ne + nh - 1;
    if (nout <= 0) return SC_OK;
    k_direct_fsum<<<(unsigned)cdiv(nout, TB), TB, 0, stream>>>(e, ne, h, nh, y, status);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

}  // namespace sc
