// k_tc_fir.cu -- FP32-accurate FIR on the 5th-gen tensor cores (tcgen05).
//
// Same output as the reference's scatter loop (core.py:80-92) within the
// north_star tolerance, computed as a block-Toeplitz GEMM:
//
//   y[n0 + 128*i + r] = sum_s sum_v X[i-s, v] * h[128*s + r - v]
//       X[rho, v] = x[n0 + 128*rho + v]   (the signal cut into 128-sample rows)
//
// For each "shift" s this is D[r', i] += T_s[r', v] * X[i-s, v] with
// r' = 127 - r (phases reversed, M = 128), i = output row (N = 128) and
// v = K (128 taps per shift).  Both operands come straight from compact
// shared-memory images through UMMA descriptors (SWIZZLE_NONE, K-major):
//
//  * T_s (A operand) is Toeplitz.  With H8[g][b][e] = h[C - 8g - b - e]
//    ("8 phase copies" of the reversed taps, 128 B per group g), core matrix
//    (row-group a, K-group j) of T_s is H8[g_s + a + j]: leading- and
//    stride-byte-offsets are both 128 B, so an 8 KB descriptor window covers a
//    dense 128x128 Toeplitz block.  Consecutive shifts slide by 16 groups.
//  * X (B operand) is stored K-group-major ([j][row][8]) so rows are 16 B
//    apart: moving to the next shift (one row down) is just start address
//    - 16 B.  One window of N + WP rows serves WP consecutive shifts.
//
// FP32 accuracy from FP16 tensor cores: x = x_hi + x_lo, h = h_hi + h_lo
// (each fp16, after exact power-of-two scaling of x and h into fp16 range),
// D += x_hi*h_hi + x_hi*h_lo + x_lo*h_hi (3 MMAs per K-step; fp16 products
// are exact in the FP32 accumulator).  Per-product relative error <= ~3*2^-22,
// i.e. worst case ~7% of the 1e-5*max|x|*||h||_1 tolerance.
//
// Pipeline (one persistent CTA per SM): warp 0 lane 0 is the producer
// (cp.async.bulk of X windows and H8 stages into smem, mbarrier
// complete_tx); warp 1 lane 0 issues tcgen05.mma kind::f16 (M128 x N x K16,
// FP32 accumulators in TMEM: two N-column buffers) and tcgen05.commit
// releases smem slots / publishes a drained stage; the epilogue warps (4 at
// N = 128, 8 at N = 256) tcgen05.ld, accumulate in FP32, unscale and store
// while the MMA warp works on the next stage.  N = 256-row tiles with
// 4-shift drains and 112-shift X windows for launches that fill the SMs;
// N = 128 with 8-shift drains (or 2 for <= 2-shift filters) otherwise.
//
// k_tc_fir_fs (end of file) is the fused-split variant for short and medium
// filters (up to 72 padded shifts, ~9,000 taps, on launches of >= 2 tiles per
// SM or one wave of 512-1,024-tap work): converter warps read x as FP32 and
// build each unit's hi/lo window in shared memory, so no split image goes
// through HBM; multi-stage units ring through four TMEM accumulators.

#include <cuda_fp16.h>

#include <algorithm>

#include <map>
#include <mutex>

#include "sc_common.cuh"

namespace sc {
namespace {

constexpr int TR = 128;              // phases per row (M) = taps per shift (K)
constexpr int KG = TR / 8;           // 16 K-groups of 8 fp16 (16 B)
#ifndef SC_TC_WP
#define SC_TC_WP 128
#endif
constexpr int NHSLOT = 2;            // H8 stage slots

// Tile geometry, by N = output rows per tile (the UMMA N): 128 (4 epilogue
// warps, 2 x 128 TMEM columns) or 256 (8 epilogue warps, all 512 TMEM
// columns).
template <int TNV>
struct TcGeo {
    static constexpr int TN = TNV;
    static constexpr int TTILE = TR * TNV;                 // outputs per tile
    static constexpr int NEPI = TNV / 32;                  // epilogue warps
    static constexpr int THREADS = 64 + 32 * NEPI;         // + producer and MMA warps
    static constexpr uint32_t TMEM_COLS = 2 * TNV;         // 2 accumulators x N fp32 columns
    // idesc: F32 accumulate (bit 4), A/B F16, K-major, N (>>3 at bit 17), M = 128 (>>4 at bit 24)
    static constexpr uint32_t IDESC = (1u << 4) | ((TNV >> 3) << 17) | ((TR >> 4) << 24);
};
constexpr uint32_t SM_XWIN = 0;
constexpr uint32_t SMEM_MAX = 232448;  // dynamic smem per CTA on sm_100

// Per (SSH, N): SSH = shifts per H8 stage = shifts per TMEM accumulator
// (drain period; 8 for long filters at N = 128, 4 at N = 256, 2 for filters
// of at most two 128-tap shifts), and the X window: the most shifts WP (<=
// 128, a multiple of 8) whose window of N + WP rows fits beside two H8
// stages.
template <int SSH, int TNV>
struct TcStage {
    static constexpr int SGROUPS = 2 * KG - 1 + KG * (SSH - 1);  // 143 groups per stage at SSH = 8
    static constexpr uint32_t HST_PART = SGROUPS * 128;            // one H8 stage, one part (18304 B)
    static constexpr int WP_FIT = (int)((SMEM_MAX - 128 - NHSLOT * 2 * HST_PART) / (2 * KG * 16)) - TNV;
    static constexpr int WP = (WP_FIT < SC_TC_WP ? WP_FIT : SC_TC_WP) / 8 * 8;  // shifts per X window
    static constexpr int WROWS = TNV + WP;                         // rows per window (WROWS-1 used)
    static constexpr uint32_t XWIN_PART = WROWS * KG * 16;         // one X window, one part
    static constexpr uint32_t SM_HST = 2 * XWIN_PART;
    static constexpr uint32_t SM_BAR = SM_HST + NHSLOT * 2 * HST_PART;  // 204288 B at N=128, SSH=8
    static constexpr uint32_t SM_TOTAL = SM_BAR + 128;
    static_assert(WP >= 8 && WP % SSH == 0, "X window too small");
    static_assert(SM_TOTAL <= SMEM_MAX, "smem");
};

struct TcArgs {
    const __half *xt[2];   // X in [ch][j][row][8] layout, hi / lo
    const __half *h8[2];   // H8 groups [ch][g][8][8], hi / lo
    int64_t xt_ch;         // elements per channel in xt
    int64_t h8_ch;         // elements per channel in h8
    int64_t nrows;         // rows in the X layout (per channel)
    int64_t row_min;       // row index of layout row 0
    int64_t s8;            // shifts (multiple of SSH)
    int64_t tiles_per_ch;
    int64_t n_tiles;       // tiles_per_ch * channels
    int64_t n_begin, n_end;  // output range; y[i] = out(n_begin + i)
    float *y;
    int64_t ldy;           // channel stride of y
    const float *scales;   // per channel: [3*ch+2] = 2^-(ex+eh)
    const unsigned *nonfinite;  // set by k_amax: inputs not representable -> skip
    int64_t nsplit;        // shift-range splits per tile
    int64_t sps;           // shifts per split (multiple of SSH)
    int64_t n_units;       // n_tiles * nsplit
    int64_t channels;
    float *ws;             // partials [nsplit][channels][n_end-n_begin] when nsplit > 1
};

// ---------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SWIZZLE_NONE K-major canonical layout; version 1 (bit 46).
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// One elected lane of a converged warp (the lowest active: lane 0 here).
// Issuing tcgen05.mma under elect.sync from a warp-wide loop lets ptxas keep
// the descriptors in uniform registers; a lane-0-only loop made it wrap
// every MMA in an elect / R2UR waterfall.
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- main kernel

template <int SSH, int TNV>
__global__ void __launch_bounds__(TcGeo<TNV>::THREADS, 1) k_tc_fir(TcArgs a) {
    using G = TcGeo<TNV>;
    using S = TcStage<SSH, TNV>;
    constexpr int TN = G::TN, WP = S::WP, WROWS = S::WROWS, NEPI = G::NEPI;
    constexpr uint32_t XWIN_PART = S::XWIN_PART, SM_HST = S::SM_HST, TMEM_COLS = G::TMEM_COLS, IDESC = G::IDESC;
    constexpr int64_t TTILE = G::TTILE;
    constexpr uint32_t HST_PART = S::HST_PART;
    constexpr uint32_t SM_BAR = S::SM_BAR;
    extern __shared__ __align__(1024) uint8_t smem[];
    pdl_begin();
    if (*a.nonfinite) return;  // block-uniform: the FFMA kernel handles this input
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform, provably
    const int lane = threadIdx.x & 31;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_xfull = sbase + SM_BAR + 0;
    const uint32_t bar_xempty = sbase + SM_BAR + 8;
    const uint32_t bar_hfull = sbase + SM_BAR + 16;   // + 8*slot
    const uint32_t bar_hempty = sbase + SM_BAR + 32;  // + 8*slot
    const uint32_t bar_tfull = sbase + SM_BAR + 48;   // + 8*acc
    const uint32_t bar_tempty = sbase + SM_BAR + 64;  // + 8*acc
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + SM_BAR + 96);

    if (threadIdx.x == 0) {
        mbar_init(bar_xfull, 1);
        mbar_init(bar_xempty, 1);
        for (int i = 0; i < NHSLOT; ++i) {
            mbar_init(bar_hfull + 8 * i, 1);
            mbar_init(bar_hempty + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar_tfull + 8 * i, 1);
            mbar_init(bar_tempty + 8 * i, NEPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform for the MMA operands

    // Work unit u = (tile, split): the split's shift range [sb, se) of that
    // tile (splits > 1 only when tiles alone leave SMs idle, e.g. cfg3).
    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ producer
            uint32_t xw = 0, hsc = 0;
            for (int64_t u = blockIdx.x; u < a.n_units; u += gridDim.x) {
                const int64_t tile = u / a.nsplit;
                const int64_t sb = (u - tile * a.nsplit) * a.sps;
                const int64_t se = sb + a.sps < a.s8 ? sb + a.sps : a.s8;
                const int64_t ch = tile / a.tiles_per_ch;
                const int64_t i0 = (tile - ch * a.tiles_per_ch) * TN;
                const __half *xt0 = a.xt[0] + ch * a.xt_ch, *xt1 = a.xt[1] + ch * a.xt_ch;
                const __half *h80 = a.h8[0] + ch * a.h8_ch, *h81 = a.h8[1] + ch * a.h8_ch;
                for (int64_t s0 = sb; s0 < se; s0 += WP) {
                    const int64_t s1 = s0 + WP < se ? s0 + WP : se;
                    if (xw > 0) mbar_wait(bar_xempty, (xw - 1) & 1);
                    // only the rows the window's shifts read: [WP - n_sh + 1, WROWS),
                    // rounded down to 8 rows (128 B) so the copies stay aligned
                    const int n_sh = (int)(s1 - s0);
                    const int r_first = ((WP - n_sh + 1) / 8) * 8;
                    const uint32_t rbytes = (uint32_t)(WROWS - r_first) * 16;
                    mbar_expect_tx(bar_xfull, 2 * KG * rbytes);
                    const int64_t row_lo = i0 - s0 - WP - a.row_min + r_first;  // layout row of window row r_first
                    for (int p = 0; p < 2; ++p)
                        for (int j = 0; j < KG; ++j)
                            bulk_g2s(sbase + SM_XWIN + p * XWIN_PART + j * (WROWS * 16) + r_first * 16,
                                     (p ? xt1 : xt0) + ((int64_t)j * a.nrows + row_lo) * 8, rbytes, bar_xfull);
                    ++xw;
                    for (int64_t sg = s0; sg < s1; sg += SSH) {
                        const uint32_t slot = hsc % NHSLOT;
                        if (hsc >= NHSLOT) mbar_wait(bar_hempty + 8 * slot, ((hsc / NHSLOT) - 1) & 1);
                        mbar_expect_tx(bar_hfull + 8 * slot, 2 * HST_PART);
                        // lowest group of the stage: g_s of its last shift
                        const int64_t glo = (a.s8 - 1 - (sg + SSH - 1)) * KG;
                        for (int p = 0; p < 2; ++p)
                            bulk_g2s(sbase + SM_HST + (slot * 2 + p) * HST_PART, (p ? h81 : h80) + glo * 64, HST_PART,
                                     bar_hfull + 8 * slot);
                        ++hsc;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        // Every H8 stage (SSH shifts) accumulates into a fresh TMEM buffer
        // (alternating), which the epilogue drains into FP32 registers.
        // The tensor core's FP32 accumulation truncates; bounding each
        // accumulator's chain to a stage of shifts x 8 K-steps x 3 MMAs keeps
        // the truncation drift ~1e-6 relative (it reached ~1.5e-3 over a full
        // 262k-tap chain).  The whole warp walks the schedule in 32-bit
        // arithmetic and elect.sync issues (see elect_one): the descriptors
        // stay in uniform registers, no per-MMA R2UR waterfall.
        {
            const int nsplit = (int)a.nsplit, sps = (int)a.sps, s8 = (int)a.s8, n_units = (int)a.n_units;
            uint32_t xw = 0, hsc = 0, dc = 0;
            for (int u = (int)blockIdx.x; u < n_units; u += (int)gridDim.x) {
                const int tile = u / nsplit;
                const int sb = (u - tile * nsplit) * sps;
                const int se = sb + sps < s8 ? sb + sps : s8;
                for (int s0 = sb; s0 < se; s0 += WP) {
                    const int s1 = s0 + WP < se ? s0 + WP : se;
                    mbar_wait(bar_xfull, xw & 1);
                    ++xw;
                    for (int sg = s0; sg < s1; sg += SSH) {
                        const uint32_t slot = hsc % NHSLOT;
                        mbar_wait(bar_hfull + 8 * slot, (hsc / NHSLOT) & 1);
                        ++hsc;
                        const uint32_t acc = dc & 1;
                        if (dc >= 2) mbar_wait(bar_tempty + 8 * acc, ((dc >> 1) - 1) & 1);
                        tc_fence_after();
                        const uint32_t d_tmem = tmem + acc * TN;
                        uint32_t accumulate = 0;
#pragma unroll 1
                        for (int ss = 0; ss < SSH; ++ss) {
                            const int s = sg + ss;
                            // A: T_s starts at group offset (SSH-1-ss)*KG inside the stage
                            const uint32_t a_hi = sbase + SM_HST + (slot * 2 + 0) * HST_PART + (SSH - 1 - ss) * KG * 128;
                            const uint32_t a_lo = a_hi + HST_PART;
                            // B: rows of shift s start WP + s0 - s rows into the window
                            const uint32_t b_hi = sbase + SM_XWIN + (uint32_t)(WP + s0 - s) * 16;
                            const uint32_t b_lo = b_hi + XWIN_PART;
                            const uint64_t ah0 = sdesc(a_hi, 128, 128), al0 = sdesc(a_lo, 128, 128);
                            const uint64_t bh0 = sdesc(b_hi, WROWS * 16, 128), bl0 = sdesc(b_lo, WROWS * 16, 128);
#pragma unroll
                            for (int kk = 0; kk < KG / 2; ++kk) {
                                // descriptor start addresses are in 16-byte units (low bits)
                                const uint64_t da = (uint64_t)((kk * 256) >> 4);
                                const uint64_t db = (uint64_t)((kk * 2 * (WROWS * 16)) >> 4);
                                if (elect_one()) {
                                    umma_f16(d_tmem, ah0 + da, bh0 + db, IDESC, accumulate);
                                    umma_f16(d_tmem, al0 + da, bh0 + db, IDESC, 1);
                                    umma_f16(d_tmem, ah0 + da, bl0 + db, IDESC, 1);
                                }
                                __syncwarp();
                                accumulate = 1;
                            }
                        }
                        if (elect_one()) {
                            umma_commit(bar_hempty + 8 * slot);
                            umma_commit(bar_tfull + 8 * acc);
                        }
                        __syncwarp();
                        ++dc;
                    }
                    if (elect_one()) umma_commit(bar_xempty);
                    __syncwarp();
                }
            }
        }
    } else {
        // ---------------------------------------------------------------- epilogue
        const int q = warp & 3;                // TMEM lane quarter of this warp
        const int half = (warp - 2) >> 2;      // which 128-column half of the N columns
        const int rp = q * 32 + lane;          // phase index r' = 127 - r
        uint32_t dc = 0;
        for (int64_t u = blockIdx.x; u < a.n_units; u += gridDim.x) {
            const int64_t tile = u / a.nsplit;
            const int64_t sp = u - tile * a.nsplit;
            const int64_t sb = sp * a.sps;
            const int64_t se = sb + a.sps < a.s8 ? sb + a.sps : a.s8;
            const int64_t n_stages = (se - sb) / SSH;
            const int64_t ch = tile / a.tiles_per_ch;
            const float inv = a.scales[3 * ch + 2];
            // with splits, each writes its (rescaled) partial to ws[sp][ch][.];
            // k_tc_split_reduce sums them in fixed split order (deterministic)
            float *yc = a.nsplit == 1 ? a.y + ch * a.ldy
                                      : a.ws + (sp * a.channels + ch) * (a.n_end - a.n_begin);
            // this thread's 128 outputs (one phase r', rows 128*half ..
            // 128*half+127), summed over the stage partials in FP32
            // round-to-nearest
            float sum[128];
#pragma unroll
            for (int i = 0; i < 128; ++i) sum[i] = 0.0f;
#pragma unroll 1
            for (int64_t st = 0; st < n_stages; ++st, ++dc) {
                const uint32_t acc = dc & 1;
                mbar_wait(bar_tfull + 8 * acc, (dc >> 1) & 1);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + acc * TN + half * 128;
#pragma unroll
                for (int c = 0; c < 128; c += 32) {
                    float v[32];
                    tmem_ld32(taddr + c, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i) sum[c + i] += v[i];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_tempty + 8 * acc);
            }
            const int64_t nb = a.n_begin + (tile - ch * a.tiles_per_ch) * TTILE + (int64_t)half * 128 * TR + (TR - 1 - rp);
#pragma unroll
            for (int i = 0; i < 128; ++i) {
                const int64_t n = nb + (int64_t)i * TR;
                if (n < a.n_end) yc[n - a.n_begin] = sum[i] * inv;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------- preprocessing

__device__ __forceinline__ void atomic_max_nonneg(unsigned *addr, float v) {
    // IEEE order of non-negative floats == order of their bit patterns
    atomicMax(addr, __float_as_uint(v));
}

// max|v| over one channel's n samples into *out, and a global flag if any
// sample is NaN/Inf (the tensor-core split cannot represent those; FAST mode
// then reroutes to the ordered kernel on the device, no host round-trip).
__device__ __forceinline__ void amax_body(const float *__restrict__ xc, int64_t n, int64_t tid, int64_t stride,
                                          unsigned *out, unsigned *nonfinite) {
    float m = 0.0f;
    bool bad = false;
    // scalar head up to 16-byte alignment, float4 body, scalar tail
    const int64_t mis = (int64_t)((16 - (reinterpret_cast<uintptr_t>(xc) & 15)) & 15) / 4;
    const int64_t head = mis < n ? mis : n;
    const int64_t n4 = (n - head) / 4;
    const float4 *x4 = reinterpret_cast<const float4 *>(xc + head);
    for (int64_t i = tid; i < n4; i += stride) {
        const float4 q = x4[i];
        const float a = fmaxf(fmaxf(fabsf(q.x), fabsf(q.y)), fmaxf(fabsf(q.z), fabsf(q.w)));
        bad |= !(fabsf(q.x) <= 3.4028235e38f) || !(fabsf(q.y) <= 3.4028235e38f) ||
               !(fabsf(q.z) <= 3.4028235e38f) || !(fabsf(q.w) <= 3.4028235e38f);
        m = a > m ? a : m;
    }
    for (int64_t i = tid; i < head + (n - head - 4 * n4); i += stride) {
        const int64_t k = i < head ? i : head + 4 * n4 + (i - head);
        const float v = fabsf(xc[k]);
        bad |= !(v <= 3.4028235e38f);
        m = v > m ? v : m;
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
}

// One launch for both operands: blocks [0, gx) reduce x (amax[2c]), blocks
// [gx, gridDim.x) reduce h (amax[2c+1]); grid.y = channel.
__global__ void k_amax2(const float *__restrict__ x, int64_t ldx, int64_t nx, int gx, const float *__restrict__ h,
                        int64_t ldh, int64_t nh, unsigned *amax, unsigned *nonfinite) {
    const int c = blockIdx.y;
    if ((int)blockIdx.x < gx)
        amax_body(x + (int64_t)c * ldx, nx, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                  (int64_t)gx * blockDim.x, amax + 2 * c, nonfinite);
    else
        amax_body(h + (int64_t)c * ldh, nh, (int64_t)(blockIdx.x - gx) * blockDim.x + threadIdx.x,
                  (int64_t)(gridDim.x - gx) * blockDim.x, amax + 2 * c + 1, nonfinite);
}

// per channel c: exact powers of two that put max|x|, max|h| in [2^14, 2^15):
// 2^ex, 2^eh, and the epilogue's unscale 2^-(ex+eh).  From amax[2c], [2c+1].
// Magnitudes whose scales would leave float range (max below 2^-100: 2^ex
// overflows from 2^-113 on; or |ex+eh| > 126: the unscale over/underflows)
// raise the fallback flag instead, so the ordered kernel computes the launch
// (flag-gated, like non-finite inputs) rather than returning Inf/NaN/0.
__device__ __forceinline__ float3 channel_scales(const unsigned *amax, int c, unsigned *fallback) {
    int e[2];
    bool out_of_range = false;
    for (int i = 0; i < 2; ++i) {
        const float m = __uint_as_float(amax[2 * c + i]);
        e[i] = (m > 0.0f && isfinite(m)) ? 14 - ilogbf(m) : 0;
        out_of_range |= e[i] > 114;
    }
    out_of_range |= e[0] + e[1] > 126 || e[0] + e[1] < -126;
    if (out_of_range) {
        if (threadIdx.x == 0) atomicOr(fallback, 1u);
        e[0] = e[1] = 0;
    }
    return make_float3(ldexpf(1.0f, e[0]), ldexpf(1.0f, e[1]), ldexpf(1.0f, -(e[0] + e[1])));
}

__device__ __forceinline__ void split16(float v, __half &hi, __half &lo) {
    hi = __float2half_rn(v);
    lo = __float2half_rn(v - __half2float(hi));
}

// XT[c][j][row][e] = split(scale_c * X_c(n_begin + (row + row_min)*128 + 8j + e))
__device__ __forceinline__ void split_x_tile(const float *__restrict__ x, int64_t ldx, int64_t x_base, int64_t x_lo,
                                             int64_t x_hi, int64_t n_begin, int64_t row_min, int64_t nrows,
                                             float sc, __half *__restrict__ xt_hi, __half *__restrict__ xt_lo,
                                             int64_t xt_ch, int64_t tile, float (*s)[132]) {
    // One CTA = 32 consecutive rows = 4096 contiguous samples: coalesced
    // float4 loads into a padded smem tile (row pitch 132 floats), then each
    // K-group j writes its 32 rows x 16 B = 512 B contiguous (fp16 hi and lo).
    const int c = blockIdx.y;
    const int64_t row0 = tile * 32;
    const float *xc = x + (int64_t)c * ldx;
    const int64_t m0 = n_begin + (row0 + row_min) * TR;  // first sample of the tile
    const bool inside = m0 >= x_lo && m0 + 4096 <= x_hi &&
                        ((reinterpret_cast<uintptr_t>(xc + (m0 - x_base)) & 15) == 0);
    if (inside) {
        const float4 *src = reinterpret_cast<const float4 *>(xc + (m0 - x_base));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int f = threadIdx.x + 256 * k;  // float4 index in the tile
            const float4 q = src[f];
            float *d = &s[f >> 5][(f & 31) * 4];
            d[0] = q.x * sc;
            d[1] = q.y * sc;
            d[2] = q.z * sc;
            d[3] = q.w * sc;
        }
    } else {
        for (int f = threadIdx.x; f < 4096; f += 256) {
            const int64_t m = m0 + f;
            s[f >> 7][f & 127] = (m >= x_lo && m < x_hi) ? xc[m - x_base] * sc : 0.0f;
        }
    }
    __syncthreads();
    const int r = threadIdx.x & 31;
    if (row0 + r >= nrows) return;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
        const int j = (threadIdx.x >> 5) + 8 * pass;
        __align__(16) __half hv[8], lv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) split16(s[r][8 * j + e], hv[e], lv[e]);
        const int64_t o = (int64_t)c * xt_ch + ((int64_t)j * nrows + row0 + r) * 8;
        *reinterpret_cast<uint4 *>(xt_hi + o) = *reinterpret_cast<const uint4 *>(hv);
        *reinterpret_cast<uint4 *>(xt_lo + o) = *reinterpret_cast<const uint4 *>(lv);
    }
}

// H8[c][g][b][e] = split(scale_c * h_c[C - 8g - b - e]), C = 128*s8 - 1
// y = sum of the split partials in ascending split order (deterministic).
// The launch's inputs, for the flagged (NaN/Inf or out-of-range scale) case:
// the reduce kernel then computes every output as the ordered FP32 chain
// itself -- the reference's (m, k) pairs in ascending m, one fused
// multiply-add per step, exactly what the gated k_chain_w launch would do --
// so a launch with shift splits needs no separate fallback kernel.
struct TcFallback {
    const float *x;
    int64_t ldx, x_base, x_lo, x_hi;
    const float *h;
    int64_t ldh, nh, n_begin;
};

__global__ void k_tc_split_reduce(const float *__restrict__ ws, int nsplit, int channels, int64_t n_len,
                                  float *__restrict__ y, int64_t ldy, const unsigned *nonfinite, TcFallback fb) {
    pdl_begin();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int ch = blockIdx.y;
    if (i >= n_len) return;
    if (*nonfinite) {
        const int64_t n = fb.n_begin + i;
        const int64_t m_lo = n - fb.nh + 1 > fb.x_lo ? n - fb.nh + 1 : fb.x_lo;
        const int64_t m_hi = n + 1 < fb.x_hi ? n + 1 : fb.x_hi;
        const float *xc = fb.x + ch * fb.ldx - fb.x_base;
        const float *hc = fb.h + ch * fb.ldh;
        float acc = 0.0f;
        for (int64_t m = m_lo; m < m_hi; ++m) acc = __fmaf_rn(xc[m], hc[n - m], acc);
        y[(int64_t)ch * ldy + i] = acc;
        return;
    }
    float s = ws[(int64_t)ch * n_len + i];
    for (int k = 1; k < nsplit; ++k) s += ws[((int64_t)k * channels + ch) * n_len + i];
    y[(int64_t)ch * ldy + i] = s;
}

__device__ __forceinline__ void build_h8_part(const float *__restrict__ h, int64_t ldh, int64_t nh, int64_t s8,
                                              int64_t ngroups, float sc, __half *__restrict__ h8_hi,
                                              __half *__restrict__ h8_lo, int64_t h8_ch, int64_t part) {
    const int64_t idx = part * blockDim.x + threadIdx.x;  // (g, b)
    if (idx >= ngroups * 8) return;
    const int c = blockIdx.y;
    const int64_t g = idx >> 3;
    const int b = (int)(idx & 7);
    const float *hc = h + (int64_t)c * ldh;
    const int64_t cc = (int64_t)TR * s8 - 1;
    __align__(16) __half hv[8], lv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int64_t k = cc - 8 * g - b - e;
        const float v = (k >= 0 && k < nh) ? hc[k] * sc : 0.0f;
        split16(v, hv[e], lv[e]);
    }
    const int64_t o = (int64_t)c * h8_ch + idx * 8;
    *reinterpret_cast<uint4 *>(h8_hi + o) = *reinterpret_cast<const uint4 *>(hv);
    *reinterpret_cast<uint4 *>(h8_lo + o) = *reinterpret_cast<const uint4 *>(lv);
}

// One launch for the operand images: blocks [0, gsplit) split x tiles,
// the rest build H8; each derives its channel's power-of-two scales from
// amax (block (0, c) also stores them for the tensor-core epilogue).
__global__ void __launch_bounds__(256) k_tc_prep(const float *__restrict__ x, int64_t ldx, int64_t x_base,
                                                 int64_t x_lo, int64_t x_hi, int64_t n_begin, int64_t row_min,
                                                 int64_t nrows, int gsplit, const float *__restrict__ h, int64_t ldh,
                                                 int64_t nh, int64_t s8, int64_t ngroups, const unsigned *amax,
                                                 float *scales, __half *__restrict__ xt_hi,
                                                 __half *__restrict__ xt_lo, int64_t xt_ch,
                                                 __half *__restrict__ h8_hi, __half *__restrict__ h8_lo,
                                                 int64_t h8_ch, unsigned *fallback) {
    pdl_begin();
    __shared__ __align__(16) float s[32][132];
    const int c = blockIdx.y;
    const float3 sc = channel_scales(amax, c, fallback);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        scales[3 * c] = sc.x;
        scales[3 * c + 1] = sc.y;
        scales[3 * c + 2] = sc.z;
    }
    if ((int)blockIdx.x < gsplit)
        split_x_tile(x, ldx, x_base, x_lo, x_hi, n_begin, row_min, nrows, sc.x, xt_hi, xt_lo, xt_ch, blockIdx.x, s);
    else
        build_h8_part(h, ldh, nh, s8, ngroups, sc.y, h8_hi, h8_lo, h8_ch, (int64_t)blockIdx.x - gsplit);
}

// ---------------------------------------------------------------- fused split
// Short and medium filters (at most FsGeo::WPF shifts): the tensor-core FIR
// reads x as FP32 straight from the signal -- no split image in HBM.  Every
// work unit (tile, shift range) needs one window of TN + shifts - 1 rows;
// four converter warps load it (coalesced float4), take its max |x|, pick
// the unit's own power-of-two scale, split it into the fp16 hi/lo K-group-
// major layout the UMMA descriptors read, and hand it to the MMA warp.  Two
// window slots: the next unit's conversion overlaps this unit's MMAs.  The
// epilogue unscales by 2^-(ex_unit + eh_channel).  HBM traffic: 4 B per input
// sample (plus the halo rows) and 4 B per output, against 16 B + 4 B for the
// image path (max pass, image write, image read).
// ONE: every unit is one drain stage (filters of at most SSH shifts, no
// shift splits) -- the epilogue streams each accumulator straight out (no
// per-thread sum over stages), which frees the registers for 8 converter
// warps instead of 4.
// converter warps of the one-stage kernel (env knob for A/B at build time)
#ifndef FS_NCONV1
#define FS_NCONV1 16
#endif
template <int SSH, bool ONE = false>
struct FsGeo {
    static constexpr int TN = 128;                                  // output rows per tile (UMMA N)
    // multi-stage units: FS_NEPI_MULTI epilogue warps (8 = two per TMEM lane
    // quarter, half the accumulator's columns each) and FS_NCONV_MULTI
    // converter warps (8 = two groups of four on alternating units)
#ifndef FS_NEPI_MULTI
#define FS_NEPI_MULTI 4
#endif
#ifndef FS_NCONV_MULTI
#define FS_NCONV_MULTI 4
#endif
    static constexpr int NEPI = ONE ? 4 : FS_NEPI_MULTI, NCONV = ONE ? FS_NCONV1 : FS_NCONV_MULTI;
    static constexpr int THREADS = 64 + 32 * (NEPI + NCONV);
    static constexpr int SGROUPS = 2 * KG - 1 + KG * (SSH - 1);
    static constexpr uint32_t HST_PART = SGROUPS * 128;
    // ONE: the unit's FP32 window (TN + SSH - 1 rows, contiguous in x) is
    // staged row-major by one bulk copy into RAW, then converted into the slot
    static constexpr uint32_t RAW = ONE ? (uint32_t)(TN + SSH - 1) * TR * 4 : 0;
    static constexpr int RAW_ROWS_A = 64;  // rows of RAW's first half (see the converters)
    // H8 stage slots: one-stage units keep their single stage resident (one
    // slot; a multi-channel launch reloads it when the channel changes)
    static constexpr int NHS = ONE ? 1 : NHSLOT;
    // TMEM accumulators: multi-stage units run four deep (all 512 columns), so
    // the MMA warp keeps issuing through a unit's output store
#ifndef FS_NACC_MULTI
#define FS_NACC_MULTI 4
#endif
    static constexpr int NACC = ONE ? 2 : FS_NACC_MULTI;
    static constexpr uint32_t BAR_BYTES = 320;
    static constexpr int WROWS_FIT = (int)((SMEM_MAX - BAR_BYTES - RAW - NHS * 2 * HST_PART) / (2 * 2 * KG * 16));
    static constexpr int WPF = ONE ? SSH : ((WROWS_FIT - 1 - TN) / 8) * 8;  // most shifts per unit
    // rows per window slot; WROWS = 1 (mod 8) puts the K-group stride at 16
    // (mod 128) bytes, so the converters' 16-byte accesses -- consecutive
    // threads on consecutive K-groups of one row -- are bank-conflict free
    static constexpr int WROWS = ((TN + WPF - 1 + 6) / 8) * 8 + 1;
    static constexpr uint32_t XPART = WROWS * KG * 16;              // one slot, one part (hi or lo)
    static constexpr uint32_t SM_RAW = 4 * XPART;                   // slot s, part p at (2s + p) * XPART
    static constexpr uint32_t SM_HST = SM_RAW + RAW;
    static constexpr uint32_t SM_BAR = SM_HST + NHS * 2 * HST_PART;
    static constexpr uint32_t SM_TOTAL = SM_BAR + BAR_BYTES;
    static constexpr uint32_t IDESC = TcGeo<TN>::IDESC;
    static_assert(WPF >= SSH && WPF % SSH == 0, "window");
    static_assert(SM_TOTAL <= SMEM_MAX, "smem");
};

struct FsArgs {
    const float *x;
    int64_t ldx, x_base, x_lo, x_hi;  // channel c's sample m at x[c*ldx + m - x_base], zero outside [x_lo, x_hi)
    const __half *h8[2];
    int64_t h8_ch;
    const int *eh;                    // per channel: h scale exponent
    int64_t s8, tiles_per_ch, n_tiles, n_begin, n_end, nsplit, sps, n_units, channels;
    float *y;
    int64_t ldy;
    float *ws;
    unsigned *flag;
    unsigned long long *trace;  // debug (SC_FS_TRACE): per CTA 0 unit timestamps
    // fold (one-stage, one channel): the kernel builds its H8 stage from the
    // taps itself and runs the non-finite fallback after a grid barrier
    int fold;
    const float *h;
    int64_t nh;
    unsigned long long *gbar;  // grid barrier word (generation << 32 | arrivals)
};

// Sense-reversing grid barrier for a cooperative (co-resident) grid: the
// last arrival clears the count and bumps the generation the others wait on.
__device__ __forceinline__ void fs_grid_barrier(unsigned long long *w) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long old = atomicAdd(w, 1ull);
        const unsigned gen = (unsigned)(old >> 32);
        if ((unsigned)(old & 0xffffffffull) + 1u == gridDim.x) {
            atomicExch(w, (unsigned long long)(gen + 1u) << 32);
        } else {
            while ((unsigned)(atomicAdd(w, 0ull) >> 32) == gen) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define FS_TRACE(field)                                                                  \
    do {                                                                                 \
        if (a.trace && blockIdx.x == 0 && uc < 32) a.trace[uc * 8 + (field)] = gtime(); \
    } while (0)

template <int NT>
__device__ __forceinline__ void conv_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NT) : "memory"); }

template <int SSH, bool ONE>
__global__ void __launch_bounds__(FsGeo<SSH, ONE>::THREADS, 1) k_tc_fir_fs(FsArgs a) {
    using G = FsGeo<SSH, ONE>;
    // converter groups of 4 warps; with two groups each takes every other
    // unit (its own window slot), so two windows' loads are in flight
    constexpr int TN = G::TN, WROWS = G::WROWS, NEPI = G::NEPI, NCONV = 4, NGRP = ONE ? 1 : G::NCONV / 4, NCT = 128;
    constexpr uint32_t XPART = G::XPART, SM_HST = G::SM_HST, HST_PART = G::HST_PART, SM_BAR = G::SM_BAR;
    constexpr int64_t TTILE = (int64_t)TR * TN;
    extern __shared__ __align__(1024) uint8_t smem[];
    pdl_begin();
    // non-finite taps (found by the H8 build): the gated fallback computes the launch
    if (!(ONE && a.fold) && *a.flag) return;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform, provably
    const int lane = threadIdx.x & 31;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_xfull = sbase + SM_BAR + 0;    // + 8*slot
    const uint32_t bar_xempty = sbase + SM_BAR + 16;  // + 8*slot
    const uint32_t bar_hfull = sbase + SM_BAR + 32;   // + 8*slot
    const uint32_t bar_hempty = sbase + SM_BAR + 48;  // + 8*slot
    constexpr int NACC = G::NACC;                       // TMEM accumulators in the ring
    const uint32_t bar_tfull = sbase + SM_BAR + 256;  // + 8*acc
    const uint32_t bar_tempty = sbase + SM_BAR + 288; // + 8*acc
    const uint32_t bar_exfull = sbase + SM_BAR + 96;  // + 8*k, k = unit % 4
    // RAW is filled and drained in two halves (rows [0, RAW_ROWS_A) and the
    // rest), so the next window's first half is in flight while this one's
    // second half is read
    const uint32_t bar_rawfull = sbase + SM_BAR + 128;
    const uint32_t bar_rawempty = sbase + SM_BAR + 136;
    const uint32_t bar_rawfull2 = sbase + SM_BAR + 232;
    const uint32_t bar_rawempty2 = sbase + SM_BAR + 240;
    int *ex_ring = reinterpret_cast<int *>(smem + SM_BAR + 144);   // [4]
    float *cmax = reinterpret_cast<float *>(smem + SM_BAR + 160);  // [NCONV <= 16]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + SM_BAR + 224);
    static_assert(G::NCONV <= 16, "cmax slots");

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar_xfull + 8 * i, 1);
            mbar_init(bar_xempty + 8 * i, 1);
            mbar_init(bar_hfull + 8 * i, 1);
            mbar_init(bar_hempty + 8 * i, 1);
        }
        for (int i = 0; i < NACC; ++i) {
            mbar_init(bar_tfull + 8 * i, 1);
            mbar_init(bar_tempty + 8 * i, NEPI);
        }
        for (int k = 0; k < 4; ++k) mbar_init(bar_exfull + 8 * k, 1);
        mbar_init(bar_rawfull, 1);
        mbar_init(bar_rawempty, 1);
        mbar_init(bar_rawfull2, 1);
        mbar_init(bar_rawempty2, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"((uint32_t)(NACC * TN)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

    // fold: every warp takes max |h| over the (<= 255) taps itself, the CTA
    // builds H8 stage 0 in slot 0 (what k_h8_fs + the producer's bulk copy
    // would have put there), and taps that are non-finite or too small skip
    // straight to the fallback
    bool fold_skip = false;
    int fold_eh = 0;
    if constexpr (ONE) {
        if (a.fold) {
            float mx = 0.0f;
            bool bad = false;
            for (int64_t k = lane; k < a.nh; k += 32) {
                const float v = a.h[k];
                mx = fmaxf(mx, fabsf(v));
                bad |= !isfinite(v);
            }
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            bad = __any_sync(0xffffffffu, bad);
            int e = (mx > 0.0f && isfinite(mx)) ? 14 - ilogbf(mx) : 0;
            const bool small = e > 114;
            if (small) e = 0;
            fold_eh = e;
            fold_skip = bad || small;
            if (fold_skip) {
                if (threadIdx.x == 0) atomicOr(a.flag, 1u);
            } else {
                const float sc = __int_as_float((127 + e) << 23);
                const int64_t cc = (int64_t)TR * a.s8 - 1;
                for (int idx = threadIdx.x; idx < G::SGROUPS * 8; idx += blockDim.x) {
                    const int g = idx >> 3, b = idx & 7;
                    __align__(16) __half hv[8], lv[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int64_t k = cc - 8 * g - b - q;
                        const float v = (k >= 0 && k < a.nh) ? a.h[k] * sc : 0.0f;
                        split16(v, hv[q], lv[q]);
                    }
                    *reinterpret_cast<uint4 *>(smem + SM_HST + idx * 16) = *reinterpret_cast<const uint4 *>(hv);
                    *reinterpret_cast<uint4 *>(smem + SM_HST + HST_PART + idx * 16) =
                        *reinterpret_cast<const uint4 *>(lv);
                }
                // generic-proxy stores -> visible to the tensor core's async proxy
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            }
            __syncthreads();
            if (threadIdx.x == 0 && !fold_skip) mbar_arrive(bar_hfull);  // slot 0 holds stage 0
        }
    }
    const int64_t NU = fold_skip ? 0 : a.n_units;
    auto EH = [&](int64_t ch) { return (ONE && a.fold) ? fold_eh : a.eh[ch]; };

    auto unit_of = [&](int64_t u, int64_t &tile, int64_t &sb, int64_t &se, int64_t &ch, int64_t &i0) {
        tile = u / a.nsplit;
        sb = (u - tile * a.nsplit) * a.sps;
        se = sb + a.sps < a.s8 ? sb + a.sps : a.s8;
        ch = tile / a.tiles_per_ch;
        i0 = (tile - ch * a.tiles_per_ch) * TN;
    };
    // a unit's window: samples [m0, m0 + 128*nrows) of channel ch; interior =
    // all of them inside [x_lo, x_hi) and 16-byte aligned (one bulk copy)
    auto window_of = [&](int64_t sb, int64_t se, int64_t ch, int64_t i0, int64_t &m0, int &nrows, bool &interior) {
        nrows = TN + (int)(se - sb) - 1;
        m0 = a.n_begin + (i0 - (se - 1)) * TR;
        const float *xc = a.x + ch * a.ldx - a.x_base;
        interior = m0 >= a.x_lo && m0 + (int64_t)nrows * TR <= a.x_hi &&
                   ((reinterpret_cast<uintptr_t>(xc + m0) & 15) == 0);
    };
    // Rows [r_lo, r_hi) of a window lie wholly inside [x_lo, x_hi): the one-
    // stage path bulk-copies them even in an edge window (16-byte aligned
    // rows only) and the converters fill just the rest.
    auto bulk_rows = [&](int64_t ch, int64_t m0, int nrows, int &r_lo, int &r_hi) {
        const float *xc = a.x + ch * a.ldx - a.x_base;
        if ((reinterpret_cast<uintptr_t>(xc + m0) & 15) != 0) {
            r_lo = r_hi = 0;
            return;
        }
        const int64_t lo = a.x_lo - m0 > 0 ? (a.x_lo - m0 + TR - 1) / TR : 0;
        const int64_t hi = a.x_hi - m0 >= 0 ? (a.x_hi - m0) / TR : 0;
        r_lo = (int)(lo < nrows ? lo : nrows);
        r_hi = (int)(hi < nrows ? hi : nrows);
        if (r_hi < r_lo) r_hi = r_lo;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ producer: H8 stages
            // A stage already in the previous slot (same channel and shift
            // range: every unit of a one-stage, one-channel launch) is not
            // loaded again -- the MMA warp keeps using it.
            uint32_t hsc = 0, rc = 0;
            int64_t last_key = -1;
            for (int64_t u = blockIdx.x; u < NU; u += gridDim.x, ++rc) {
                int64_t tile, sb, se, ch, i0;
                unit_of(u, tile, sb, se, ch, i0);
                if constexpr (ONE) {
                    // the unit's FP32 window, one bulk copy (edge windows: the
                    // converters fill RAW themselves after this arrive)
                    int64_t m0;
                    int nrows;
                    bool interior;
                    window_of(sb, se, ch, i0, m0, nrows, interior);
                    const float *src = a.x + ch * a.ldx - a.x_base + m0;
                    const int rows_a = nrows < G::RAW_ROWS_A ? nrows : G::RAW_ROWS_A;
                    int r_lo = 0, r_hi = nrows;  // bulk-copied rows
                    if (!interior) bulk_rows(ch, m0, nrows, r_lo, r_hi);
                    // half A: rows [0, rows_a), half B: [rows_a, nrows)
                    const int a0 = r_lo, a1 = r_hi < rows_a ? r_hi : rows_a;
                    const int b0 = r_lo > rows_a ? r_lo : rows_a, b1 = r_hi;
                    if (rc > 0) mbar_wait(bar_rawempty, (rc - 1) & 1);
                    const uint32_t bytes_a = a1 > a0 ? (uint32_t)(a1 - a0) * TR * 4 : 0;
                    mbar_expect_tx(bar_rawfull, bytes_a);
                    if (bytes_a)
                        bulk_g2s(sbase + G::SM_RAW + (uint32_t)a0 * TR * 4, src + (int64_t)a0 * TR, bytes_a,
                                 bar_rawfull);
                    if (rc > 0) mbar_wait(bar_rawempty2, (rc - 1) & 1);
                    const uint32_t bytes_b = b1 > b0 ? (uint32_t)(b1 - b0) * TR * 4 : 0;
                    mbar_expect_tx(bar_rawfull2, bytes_b);
                    if (bytes_b)
                        bulk_g2s(sbase + G::SM_RAW + (uint32_t)b0 * TR * 4, src + (int64_t)b0 * TR, bytes_b,
                                 bar_rawfull2);
                }
                if (ONE && a.fold) continue;  // stage 0 was built in slot 0 by the CTA
                const __half *h80 = a.h8[0] + ch * a.h8_ch, *h81 = a.h8[1] + ch * a.h8_ch;
                for (int64_t sg = sb; sg < se; sg += SSH) {
                    const int64_t key = ch * a.s8 + sg;
                    if (key == last_key) continue;
                    last_key = key;
                    const uint32_t slot = hsc % G::NHS;
                    if (hsc >= (uint32_t)G::NHS) mbar_wait(bar_hempty + 8 * slot, ((hsc / G::NHS) - 1) & 1);
                    mbar_expect_tx(bar_hfull + 8 * slot, 2 * HST_PART);
                    const int64_t glo = (a.s8 - 1 - (sg + SSH - 1)) * KG;
                    for (int p = 0; p < 2; ++p)
                        bulk_g2s(sbase + SM_HST + (slot * 2 + p) * HST_PART, (p ? h81 : h80) + glo * 64, HST_PART,
                                 bar_hfull + 8 * slot);
                    ++hsc;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        // The whole warp walks the schedule (so the descriptors are
        // warp-uniform values the compiler keeps in uniform registers) and
        // lane 0 issues: a single-thread loop made ptxas wrap every
        // tcgen05.mma in an elect / R2UR waterfall, ~110 clk per MMA against
        // the 64-clk floor of an M128 x N128 x K16 MMA.
        {
            // 32-bit unit arithmetic (n_units < 2^31, checked at launch): a
            // 64-bit division is a call whose results ptxas cannot treat as
            // warp-uniform
            const int nsplit = (int)a.nsplit, sps = (int)a.sps, s8 = (int)a.s8;
            const int n_units = (int)NU;
            uint32_t uc = 0, hsc = 0, dc = 0;
            int last_key = -1;
            uint32_t slot = 0;
            for (int u = (int)blockIdx.x; u < n_units; u += (int)gridDim.x, ++uc) {
                const int tile = u / nsplit;
                const int sb = (u - tile * nsplit) * sps;
                const int se = sb + sps < s8 ? sb + sps : s8;
                const int ch = tile / (int)a.tiles_per_ch;
                const uint32_t xs = uc & 1;
                mbar_wait(bar_xfull + 8 * xs, (uc >> 1) & 1);
                if (lane == 0) FS_TRACE(3);
                for (int sg = sb; sg < se; sg += SSH) {
                    const int key = ch * s8 + sg;
                    if (key != last_key) {
                        // leaving the previous stage: its slot is free once
                        // the MMAs issued so far complete
                        if (hsc > 0 && elect_one()) umma_commit(bar_hempty + 8 * slot);
                        last_key = key;
                        slot = hsc % G::NHS;
                        mbar_wait(bar_hfull + 8 * slot, (hsc / G::NHS) & 1);
                        ++hsc;
                    }
                    const uint32_t acc = dc % NACC;
                    if (dc >= NACC) mbar_wait(bar_tempty + 8 * acc, ((dc / NACC) - 1) & 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem + acc * TN;
                    uint32_t accumulate = 0;
#pragma unroll 1
                    for (int ss = 0; ss < SSH; ++ss) {
                        const int s = sg + ss;
                        const uint32_t a_hi = sbase + SM_HST + (slot * 2 + 0) * HST_PART + (SSH - 1 - ss) * KG * 128;
                        const uint32_t a_lo = a_hi + HST_PART;
                        // output row i of shift s reads window row i + (se - 1 - s)
                        const uint32_t b_hi = sbase + (2 * xs) * XPART + (uint32_t)(se - 1 - s) * 16;
                        const uint32_t b_lo = b_hi + XPART;
                        const uint64_t ah0 = sdesc(a_hi, 128, 128), al0 = sdesc(a_lo, 128, 128);
                        const uint64_t bh0 = sdesc(b_hi, WROWS * 16, 128), bl0 = sdesc(b_lo, WROWS * 16, 128);
#pragma unroll
                        for (int kk = 0; kk < KG / 2; ++kk) {
                            // descriptor start addresses are in 16-byte units (low bits)
                            const uint64_t da = (uint64_t)((kk * 256) >> 4);
                            const uint64_t db = (uint64_t)((kk * 2 * (WROWS * 16)) >> 4);
                            if (elect_one()) {
                                umma_f16(d_tmem, ah0 + da, bh0 + db, G::IDESC, accumulate);
                                umma_f16(d_tmem, al0 + da, bh0 + db, G::IDESC, 1);
                                umma_f16(d_tmem, ah0 + da, bl0 + db, G::IDESC, 1);
                            }
                            __syncwarp();
                            accumulate = 1;
                        }
                    }
                    if (elect_one()) umma_commit(bar_tfull + 8 * acc);
                    __syncwarp();
                    ++dc;
                }
                if (elect_one()) umma_commit(bar_xempty + 8 * xs);
                __syncwarp();
                if (lane == 0) FS_TRACE(4);
            }
        }
    } else if (warp < 2 + NEPI) {
        // ---------------------------------------------------------------- epilogue
        const int q = warp & 3;          // TMEM lane quarter
        const int rp = q * 32 + lane;    // phase r' = 127 - r
        uint32_t dc = 0, uc = 0;
        for (int64_t u = blockIdx.x; u < NU; u += gridDim.x, ++uc) {
            int64_t tile, sb, se, ch, i0;
            unit_of(u, tile, sb, se, ch, i0);
            const int64_t sp = u - tile * a.nsplit;
            const int64_t n_stages = (se - sb) / SSH;
            float *yc = a.nsplit == 1 ? a.y + ch * a.ldy : a.ws + (sp * a.channels + ch) * (a.n_end - a.n_begin);
            const int64_t nb = a.n_begin + i0 * TR + (TR - 1 - rp);
            if constexpr (ONE) {
                // one stage: the unit's x scale first, then stream the accumulator out
                mbar_wait(bar_exfull + 8 * (uc & 3), (uc >> 2) & 1);
                const int e = ex_ring[uc & 3] + EH(ch);
                const float inv = __int_as_float((127 - e) << 23);
                const uint32_t acc = dc % NACC;
                mbar_wait(bar_tfull + 8 * acc, (dc / NACC) & 1);
                if (threadIdx.x == 64) FS_TRACE(5);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + acc * TN;
#pragma unroll
                for (int c = 0; c < TN; c += 32) {
                    float v[32];
                    tmem_ld32(taddr + c, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int64_t n = nb + (int64_t)(c + i) * TR;
                        if (n < a.n_end) yc[n - a.n_begin] = v[i] * inv;
                    }
                }
                if (threadIdx.x == 64) FS_TRACE(6);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_tempty + 8 * acc);
                ++dc;
                continue;
            }
            // NEPI = 8: warps 2..5 take columns [0, TN/2), warps 6..9 the rest
            constexpr int CPW = TN / (NEPI / 4);
            const int c0 = ((warp - 2) >> 2) * CPW;
            float sum[CPW];
#pragma unroll
            for (int i = 0; i < CPW; ++i) sum[i] = 0.0f;
#pragma unroll 1
            for (int64_t st = 0; st < n_stages; ++st, ++dc) {
                const uint32_t acc = dc % NACC;
                mbar_wait(bar_tfull + 8 * acc, (dc / NACC) & 1);
                if (st == 0 && threadIdx.x == 64) FS_TRACE(5);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + acc * TN + c0;
#pragma unroll
                for (int c = 0; c < CPW; c += 32) {
                    float v[32];
                    tmem_ld32(taddr + c, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i) sum[c + i] += v[i];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_tempty + 8 * acc);
            }
            // the unit's x scale (written by the converters before this arrive)
            mbar_wait(bar_exfull + 8 * (uc & 3), (uc >> 2) & 1);
            const int e = ex_ring[uc & 3] + EH(ch);
            const float inv = __int_as_float((127 - e) << 23);  // 2^-e, |e| <= 126 (checked)
            if (threadIdx.x == 64) FS_TRACE(7);
            if (nb + (int64_t)(TN - 1) * TR < a.n_end) {
                // whole tile in range: immediate-offset stores, no per-element bound
                float *yp = yc + (nb - a.n_begin) + (int64_t)c0 * TR;
#pragma unroll
                for (int i = 0; i < CPW; ++i) yp[i * TR] = sum[i] * inv;
            } else {
#pragma unroll
                for (int i = 0; i < CPW; ++i) {
                    const int64_t n = nb + (int64_t)(c0 + i) * TR;
                    if (n < a.n_end) yc[n - a.n_begin] = sum[i] * inv;
                }
            }
            if (threadIdx.x == 64) FS_TRACE(6);
        }
    } else {
        // ---------------------------------------------------------------- converters
        if constexpr (ONE) {
            // The window arrived row-major in RAW by one bulk copy (or, at the
            // signal's edges, is filled here).  Pass 1: max |x| (float4 per
            // thread, contiguous); pass 2: each thread turns 4 samples into
            // 8 bytes of hi and 8 of lo in the slot's K-group-major layout.
            // RAW is released as soon as pass 2 has read it, so the next
            // window's copy overlaps this unit's MMAs.
            constexpr int NT1 = 32 * G::NCONV;  // converter threads
            const int ct = threadIdx.x - 32 * (2 + NEPI);  // 0..NT1-1
            const int cw = ct >> 5;
            const float4 *raw4 = reinterpret_cast<const float4 *>(smem + G::SM_RAW);
            uint32_t uc = 0;
            for (int64_t u = blockIdx.x; u < NU; u += gridDim.x, ++uc) {
                int64_t tile, sb, se, ch, i0, m0;
                int nrows;
                bool interior;
                unit_of(u, tile, sb, se, ch, i0);
                window_of(sb, se, ch, i0, m0, nrows, interior);
                const uint32_t xs = uc & 1;
                mbar_wait(bar_rawfull, uc & 1);
                if (ct == 0) FS_TRACE(0);
                const int n4 = nrows * (TR / 4);
                constexpr int Q = (((TN + SSH - 1) * (TR / 4)) + NT1 - 1) / NT1;
                constexpr int QA = G::RAW_ROWS_A * (TR / 4) / NT1;  // float4 rounds in half A
                static_assert(QA * NT1 == G::RAW_ROWS_A * (TR / 4) && QA < Q, "RAW halves");
                if (!interior) {
                    mbar_wait(bar_rawfull2, uc & 1);  // the previous window's half B is released too
                    int r_lo, r_hi;                   // rows the producer bulk-copied (see bulk_rows)
                    bulk_rows(ch, m0, nrows, r_lo, r_hi);
                    const int q_lo = r_lo * (TR / 4), q_hi = r_hi * (TR / 4);
                    // edge (or unaligned) window: every thread's loads in
                    // flight at once (unrolled, non-coherent), then the
                    // stores -- a loop of dependent load/store rounds took
                    // ~14 us per window, on the critical path of the CTA
                    // that owns the signal's first window
                    const float *xc = a.x + ch * a.ldx - a.x_base;
                    float4 *w4 = reinterpret_cast<float4 *>(smem + G::SM_RAW);
                    constexpr int QB = 8;  // float4 per batch: 32 loads in flight per thread
#pragma unroll
                    for (int k0 = 0; k0 < Q; k0 += QB) {
                        float v[QB][4];
#pragma unroll
                        for (int k = 0; k < QB; ++k) {
                            const int q = ct + NT1 * (k0 + k);
                            const int64_t m = m0 + 4 * (int64_t)q;
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                v[k][e] = (k0 + k < Q && q < n4 && (q < q_lo || q >= q_hi) && m + e >= a.x_lo &&
                                       m + e < a.x_hi)
                                              ? __ldg(xc + m + e) : 0.0f;
                        }
#pragma unroll
                        for (int k = 0; k < QB; ++k) {
                            const int q = ct + NT1 * (k0 + k);
                            if (k0 + k < Q && q < n4 && (q < q_lo || q >= q_hi))
                                w4[q] = make_float4(v[k][0], v[k][1], v[k][2], v[k][3]);
                        }
                    }
                    conv_bar<NT1>(1);
                }
                // RAW -> registers (<= 33 float4 per thread), then RAW is free
                // for the next window's copy while this unit converts
                float4 r[Q];
                float mx = 0.0f;
                bool bad = false;
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    if (k == QA) {
                        // half A read by every converter: release it, then half B
                        conv_bar<NT1>(1);
                        if (ct == 0) mbar_arrive(bar_rawempty);
                        mbar_wait(bar_rawfull2, uc & 1);
                    }
                    const int q = ct + NT1 * k;
                    r[k] = q < n4 ? raw4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
                    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(r[k].x), fabsf(r[k].y)), fmaxf(fabsf(r[k].z), fabsf(r[k].w))));
                    bad |= !(isfinite(r[k].x) && isfinite(r[k].y) && isfinite(r[k].z) && isfinite(r[k].w));
                }
                if (ct == 0) FS_TRACE(1);
                for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 1u);
                if (lane == 0) cmax[cw] = mx;
                conv_bar<NT1>(1);   // also: every thread has read RAW half B
                if (ct == 0) mbar_arrive(bar_rawempty2);
#pragma unroll
                for (int w = 0; w < G::NCONV; ++w) mx = fmaxf(mx, cmax[w]);
                int ex = (mx > 0.0f && isfinite(mx)) ? 14 - ilogbf(mx) : 0;
                const int e_tot = ex + EH(ch);
                if (ex > 114 || e_tot > 126 || e_tot < -126) {
                    if (ct == 0) atomicOr(a.flag, 1u);
                    ex = 0;
                }
                const float sc = __int_as_float((127 + ex) << 23);  // 2^ex
                if (uc >= 2) mbar_wait(bar_xempty + 8 * xs, ((uc >> 1) - 1) & 1);
                uint8_t *xhi = smem + (2 * xs) * XPART, *xlo = xhi + XPART;
#pragma unroll
                for (int k = 0; k < Q; ++k) {
                    const int q = ct + NT1 * k;
                    if (q < n4) {
                        const int w = q >> 5, j = (q >> 1) & 15, half = q & 1;
                        // packed: two samples per conversion instruction
                        const float2 a01 = make_float2(r[k].x * sc, r[k].y * sc);
                        const float2 a23 = make_float2(r[k].z * sc, r[k].w * sc);
                        const __half2 h01 = __float22half2_rn(a01), h23 = __float22half2_rn(a23);
                        const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
                        const __half2 l01 = __float22half2_rn(make_float2(a01.x - f01.x, a01.y - f01.y));
                        const __half2 l23 = __float22half2_rn(make_float2(a23.x - f23.x, a23.y - f23.y));
                        const uint32_t off = ((uint32_t)j * WROWS + (uint32_t)w) * 16 + half * 8;
                        *reinterpret_cast<uint2 *>(xhi + off) =
                            make_uint2(*reinterpret_cast<const uint32_t *>(&h01), *reinterpret_cast<const uint32_t *>(&h23));
                        *reinterpret_cast<uint2 *>(xlo + off) =
                            make_uint2(*reinterpret_cast<const uint32_t *>(&l01), *reinterpret_cast<const uint32_t *>(&l23));
                    }
                }
                // generic-proxy stores -> visible to the tensor core's async proxy
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                conv_bar<NT1>(1);
                if (ct == 0) {
                    ex_ring[uc & 3] = ex;
                    mbar_arrive(bar_exfull + 8 * (uc & 3));
                    mbar_arrive(bar_xfull + 8 * xs);
                    FS_TRACE(2);
                }
            }
        } else {
        // Work item = (window row w, K-group j): 8 consecutive samples.  The
        // raw FP32 samples land IN PLACE in the item's two 16-byte slots (hi
        // part, lo part) by cp.async -- every load of the window in flight at
        // once, no registers held -- then each thread takes the max over its
        // own items and, once the unit's scale is known, overwrites them with
        // the fp16 hi / lo split.
        const int cg = (threadIdx.x - 32 * (2 + NEPI)) / NCT;  // converter group
        const int ct = (threadIdx.x - 32 * (2 + NEPI)) % NCT;  // 0..127 within the group
        const int cw = ct >> 5;
        float *gmax = cmax + 4 * cg;
        uint32_t uc = 0;
        for (int64_t u = blockIdx.x; u < NU; u += gridDim.x, ++uc) {
            if ((int)(uc % NGRP) != cg) continue;
            int64_t tile, sb, se, ch, i0;
            unit_of(u, tile, sb, se, ch, i0);
            const uint32_t xs = uc & 1;
            if (uc >= 2) mbar_wait(bar_xempty + 8 * xs, ((uc >> 1) - 1) & 1);
            if (ct == 0) FS_TRACE(0);
            // window row w <-> global row i0 - (se - 1) + w; samples m0 + 128 w + v
            const int nrows = TN + (int)(se - sb) - 1;
            const int items = nrows * KG;
            const int64_t m0 = a.n_begin + (i0 - (se - 1)) * TR;
            const float *xc = a.x + ch * a.ldx - a.x_base;
            const int64_t lo = a.x_lo, hi = a.x_hi;
            // interior window: every sample inside [lo, hi) and 16-byte aligned
            const bool interior = m0 >= lo && m0 + (int64_t)nrows * TR <= hi &&
                                  ((reinterpret_cast<uintptr_t>(xc + m0) & 15) == 0);
            uint8_t *xhi = smem + (2 * xs) * XPART, *xlo = xhi + XPART;
            if (interior) {
                // unrolled: every copy's addresses in their own registers, so
                // the copies issue back to back (no waits on reused sources)
                const uint32_t shi = smem_u32(xhi), slo = smem_u32(xlo);
                for (int it0 = ct; it0 < items; it0 += 8 * NCT) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int it = it0 + k * NCT;
                        if (it < items) {
                            const float *src = xc + m0 + (int64_t)(it >> 4) * TR + (it & 15) * 8;
                            const uint32_t off = ((uint32_t)(it & 15) * WROWS + (uint32_t)(it >> 4)) * 16;
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(shi + off), "l"(src));
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(slo + off), "l"(src + 4));
                        }
                    }
                }
            } else {
                // edge (or unaligned) window: 4 items' loads in flight per
                // round (non-coherent), then their stores
                for (int it0 = ct; it0 < items; it0 += 4 * NCT) {
                    float v[4][8];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int it = it0 + k * NCT;
                        const int64_t m = m0 + (int64_t)(it >> 4) * TR + (it & 15) * 8;
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            v[k][e] = (it < items && m + e >= lo && m + e < hi) ? __ldg(xc + m + e) : 0.0f;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int it = it0 + k * NCT;
                        if (it < items) {
                            const uint32_t off = ((uint32_t)(it & 15) * WROWS + (uint32_t)(it >> 4)) * 16;
                            *reinterpret_cast<float4 *>(xhi + off) = make_float4(v[k][0], v[k][1], v[k][2], v[k][3]);
                            *reinterpret_cast<float4 *>(xlo + off) = make_float4(v[k][4], v[k][5], v[k][6], v[k][7]);
                        }
                    }
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            if (ct == 0) FS_TRACE(1);
            // max |x| over this thread's own items (it wrote them itself)
            float mx = 0.0f;
            bool bad = false;
            for (int it = ct; it < items; it += NCT) {
                const uint32_t off = ((uint32_t)(it & 15) * WROWS + (uint32_t)(it >> 4)) * 16;
                const float4 p0 = *reinterpret_cast<const float4 *>(xhi + off);
                const float4 p1 = *reinterpret_cast<const float4 *>(xlo + off);
                mx = fmaxf(mx, fmaxf(fmaxf(fabsf(p0.x), fabsf(p0.y)), fmaxf(fabsf(p0.z), fabsf(p0.w))));
                mx = fmaxf(mx, fmaxf(fmaxf(fabsf(p1.x), fabsf(p1.y)), fmaxf(fabsf(p1.z), fabsf(p1.w))));
                bad |= !(isfinite(p0.x) && isfinite(p0.y) && isfinite(p0.z) && isfinite(p0.w) && isfinite(p1.x) &&
                         isfinite(p1.y) && isfinite(p1.z) && isfinite(p1.w));
            }
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 1u);
            if (lane == 0) gmax[cw] = mx;
            conv_bar<NCT>(1 + cg);
#pragma unroll
            for (int w = 0; w < NCONV; ++w) mx = fmaxf(mx, gmax[w]);
            // the unit's exact power-of-two scale: max |x| into [2^14, 2^15);
            // scales (or the unscale with the taps' exponent) leaving float
            // range raise the fallback flag (the gated ordered launch)
            int ex = (mx > 0.0f && isfinite(mx)) ? 14 - ilogbf(mx) : 0;
            const int e_tot = ex + EH(ch);
            if (ex > 114 || e_tot > 126 || e_tot < -126) {
                if (ct == 0) atomicOr(a.flag, 1u);
                ex = 0;
            }
            const float sc = __int_as_float((127 + ex) << 23);  // 2^ex
            for (int it = ct; it < items; it += NCT) {
                const uint32_t off = ((uint32_t)(it & 15) * WROWS + (uint32_t)(it >> 4)) * 16;
                const float4 p0 = *reinterpret_cast<const float4 *>(xhi + off);
                const float4 p1 = *reinterpret_cast<const float4 *>(xlo + off);
                const float v[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
                __align__(16) __half hv[8], lv[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) split16(v[e] * sc, hv[e], lv[e]);
                *reinterpret_cast<uint4 *>(xhi + off) = *reinterpret_cast<const uint4 *>(hv);
                *reinterpret_cast<uint4 *>(xlo + off) = *reinterpret_cast<const uint4 *>(lv);
            }
            // generic-proxy stores -> visible to the tensor core's async proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            conv_bar<NCT>(1 + cg);
            if (ct == 0) {
                ex_ring[uc & 3] = ex;
                mbar_arrive(bar_exfull + 8 * (uc & 3));
                mbar_arrive(bar_xfull + 8 * xs);
                FS_TRACE(2);
            }
        }
    }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(NACC * TN)));
    }
    if constexpr (ONE) {
        if (a.fold) {
            // Every unit is written (and every non-finite sample has raised
            // the flag) once the whole grid is here.  Flagged launches then
            // recompute every output as the ordered FP32 chain -- the
            // reference's (m, k) pairs in ascending m, one fused multiply-add
            // each, exactly the gated k_chain_w launch this replaces -- and
            // clear the flag for the next launch.
            fs_grid_barrier(a.gbar);
            if (*reinterpret_cast<volatile unsigned *>(a.flag)) {
                const float *xc = a.x - a.x_base;
                for (int64_t n = a.n_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < a.n_end;
                     n += (int64_t)gridDim.x * blockDim.x) {
                    const int64_t m_lo = n - a.nh + 1 > a.x_lo ? n - a.nh + 1 : a.x_lo;
                    const int64_t m_hi = n + 1 < a.x_hi ? n + 1 : a.x_hi;
                    float acc = 0.0f;
                    for (int64_t m = m_lo; m < m_hi; ++m) acc = __fmaf_rn(xc[m], a.h[n - m], acc);
                    a.y[n - a.n_begin] = acc;
                }
                fs_grid_barrier(a.gbar);
                if (blockIdx.x == 0 && threadIdx.x == 0) *a.flag = 0u;
            }
        }
    }
}

// H8 images for the fused-split kernel with each channel's own h scale:
// every CTA takes max |h_c| over the whole (short) IR itself, so no separate
// max pass runs; CTA (0, c) publishes the exponent, non-finite taps raise
// the fallback flag.
// set_flag (one channel, no caller-owned flag): every CTA has seen all the
// taps, so each STORES the same flag value (no memset launch before this
// one); otherwise the flag is only raised (atomicOr).
__global__ void __launch_bounds__(256) k_h8_fs(const float *__restrict__ h, int64_t ldh, int64_t nh, int64_t s8,
                                               int64_t ngroups, __half *__restrict__ h8_hi,
                                               __half *__restrict__ h8_lo, int64_t h8_ch, int *eh, unsigned *flag,
                                               bool set_flag) {
    pdl_begin();
    const int c = blockIdx.y;
    const float *hc = h + (int64_t)c * ldh;
    float mx = 0.0f;
    bool bad = false;
    for (int64_t i = threadIdx.x; i < nh; i += blockDim.x) {
        const float v = hc[i];
        mx = fmaxf(mx, fabsf(v));
        bad |= !isfinite(v);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ float wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    bad = __syncthreads_or(bad);
    mx = wm[0];
    for (int w = 1; w < 8; ++w) mx = fmaxf(mx, wm[w]);
    int e = (mx > 0.0f && isfinite(mx)) ? 14 - ilogbf(mx) : 0;
    const bool small = e > 114;  // taps this small leave the split's range: ordered fallback
    if (small) e = 0;
    if (set_flag) {
        if (threadIdx.x == 0) *flag = (bad || small) ? 1u : 0u;
    } else {
        if (small && threadIdx.x == 0) atomicOr(flag, 1u);
        if (bad && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flag, 1u);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) eh[c] = e;
    build_h8_part(h, ldh, nh, s8, ngroups, __int_as_float((127 + e) << 23), h8_hi, h8_lo, h8_ch, blockIdx.x);
}

}  // namespace

// Fold control words (non-finite flag, grid-barrier word) of one (device,
// stream): zeroed once at creation; every folded launch leaves them clear.
struct FsCtl {
    unsigned flag, pad;
    unsigned long long gbar;
};

FsCtl *fs_ctl(cudaStream_t stream, int *err) {
    static std::mutex mu;
    static std::map<std::pair<int, uintptr_t>, FsCtl *> ctls;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    FsCtl *&c = ctls[std::make_pair(dev, reinterpret_cast<uintptr_t>(stream))];
    if (!c) {
        void *p = nullptr;
        if (cudaMalloc(&p, sizeof(FsCtl)) != cudaSuccess || cudaMemsetAsync(p, 0, sizeof(FsCtl), stream) != cudaSuccess) {
            cudaGetLastError();
            set_error("fir: fold control block allocation failed");
            *err = SC_ERR_ALLOC;
            return nullptr;
        }
        c = static_cast<FsCtl *>(p);
    }
    *err = 0;
    return c;
}

// Fused-split launch (see k_tc_fir_fs); returns SC_ERR_STATE when the filter
// has more shifts than one window holds (the image path then runs).
template <int SSH>
int launch_fs_impl(const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi, const float *h,
                   int64_t ldh, int64_t nh, float *y, int64_t ldy, int64_t n_begin, int64_t n_end, int64_t channels,
                   cudaStream_t stream, const unsigned **nonfinite_out, const TcPre *pre, bool *fallback_folded) {
    using G = FsGeo<SSH>;
    const int64_t n_len = n_end - n_begin;
    const int64_t s_needed = (nh + TR - 2) / TR + 1;
    const int64_t s8 = cdiv(s_needed, SSH) * SSH;
    // Short filters on launches with several tiles per SM (the converters of
    // the next tile then overlap this one's MMAs): measured 0.21 vs 0.28 ms
    // (128 taps, 2^26 outputs).  Longer filters and small launches keep the
    // image path (cfg2: 0.094 vs 0.108 ms).
    static const int64_t fs_max_s8 = [] {
        // Most (padded) shifts on this path: everything one window holds
        // (WPF = 72 at 2-shift drains: filters up to ~9,000 taps).  Measured on
        // 2^26 samples against the image path (profiles/r02_fs_max.txt):
        // 1,024 taps 0.481 -> 0.375 ms, 2,048 0.694 -> 0.607, 4,096 1.119 ->
        // 1.073, 8,192 2.007 -> 2.004 (the x image's extra HBM passes stop
        // mattering there).  SC_FS_MAX_S8=8 restores the round-2 bound (A/B).
        const char *v = getenv("SC_FS_MAX_S8");
        const int k = v ? atoi(v) : 0;
        return (int64_t)(k >= 2 && k <= G::WPF ? k : G::WPF);
    }();
    static const int64_t fs_min_tiles_x2 = [] {
        const char *v = getenv("SC_FS_MIN_TILES_X2");  // A/B knob: least tiles per SM, in halves (default 4 = 2 per SM)
        return (int64_t)(v ? atoi(v) : 4);
    }();
    // One-wave launches (a quarter to all of the SMs busy with one tile each)
    // of 512-1,024-tap filters also run here: measured against the image path
    // (profiles/r02_fs_small_launch.txt) 2^20 samples x 512 / 1,024 taps
    // 0.036 -> 0.032 / 0.038 -> 0.034 ms, 2^21 samples 0.038 -> 0.032 / 0.046
    // -> 0.036 ms; longer filters and 1-2 wave launches are mixed (wave
    // quantisation) and keep the image path.  SC_FS_SMALL=0 disables (A/B).
    static const bool fs_small = [] {
        const char *v = getenv("SC_FS_SMALL");
        return !(v && atoi(v) == 0);
    }();
    const int64_t tiles_all = cdiv(n_len, (int64_t)TR * G::TN) * channels;
    const bool small_ok = fs_small && s_needed > 4 && s8 <= 10 && 4 * tiles_all >= (int64_t)sm_count() &&
                          tiles_all <= (int64_t)sm_count();
    if (s8 > fs_max_s8 || (2 * tiles_all < fs_min_tiles_x2 * (int64_t)sm_count() && !small_ok)) return SC_ERR_STATE;
    const int64_t ngroups = KG * s8 + KG - 1;
    const int64_t h8_ch = ngroups * 64;
    const int64_t tiles_per_ch = cdiv(n_len, (int64_t)TR * G::TN);
    const int64_t n_tiles = tiles_per_ch * channels;
    // shift-range splits when the tiles leave SMs idle (fixed-order reduce)
    const int sms = sm_count();
    const int64_t stages = s8 / SSH;
    int64_t nsplit = 1;
    {
        double best = 0.0;
        for (int64_t sp = 1; sp <= 16 && sp <= stages; ++sp) {
            const int64_t units = n_tiles * sp;
            const int64_t waves = (units + sms - 1) / sms;
            const double eff = (double)units / (double)(waves * sms);
            if (eff > best + 0.03) best = eff, nsplit = sp;
            if (best > 0.95) break;
        }
    }
    const int64_t sps = cdiv(stages, nsplit) * SSH;
    nsplit = cdiv(s8, sps);
    // One-stage, one-channel launches fold the H8 build and the non-finite
    // fallback into the tensor-core kernel (one launch instead of three;
    // a cooperative launch, for the grid barrier before the fallback).
    // SC_FS_FOLD=0 keeps the three launches.
    static const bool fold_on = [] {
        const char *v = getenv("SC_FS_FOLD");
        return !(v && atoi(v) == 0);
    }();
    const bool one = nsplit == 1 && s8 == SSH;
    bool fold = fold_on && one && channels == 1 && !pre && !getenv("SC_FS_TRACE");
    FsArgs a;
    a.fold = 0, a.h = h, a.nh = nh, a.gbar = nullptr;
    int err = 0;
    if (fold) {
        FsCtl *ctl = fs_ctl(stream, &err);
        if (err) return err;
        if (nonfinite_out) *nonfinite_out = &ctl->flag;
        if (fallback_folded) *fallback_folded = true;
        a.x = x, a.ldx = ldx, a.x_base = x_base, a.x_lo = x_lo, a.x_hi = x_hi;
        a.h8[0] = a.h8[1] = nullptr, a.h8_ch = 0, a.eh = nullptr;
        a.s8 = s8, a.tiles_per_ch = tiles_per_ch, a.n_tiles = n_tiles, a.n_begin = n_begin, a.n_end = n_end;
        a.channels = channels, a.y = y, a.ldy = ldy, a.flag = &ctl->flag;
        a.nsplit = nsplit, a.sps = sps, a.n_units = n_tiles * nsplit;
        SC_REQUIRE(a.n_units < (int64_t)INT32_MAX, "fir: too many work units");
        a.ws = nullptr, a.trace = nullptr, a.fold = 1, a.gbar = &ctl->gbar;
        using G1 = FsGeo<SSH, true>;
        SC_CHECK_CUDA(cudaFuncSetAttribute(k_tc_fir_fs<SSH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           G1::SM_TOTAL));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)std::min<int64_t>(a.n_units, sms));
        cfg.blockDim = dim3(G1::THREADS);
        cfg.dynamicSmemBytes = G1::SM_TOTAL;
        cfg.stream = stream;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        const cudaError_t le = cudaLaunchKernelEx(&cfg, k_tc_fir_fs<SSH, true>, a);
        if (le == cudaSuccess) {
            note_launch();
            note_tc_launch(SSH, G::TN, n_tiles * (int64_t)TR * G::TN * (int64_t)TR * s8, SC_TC_KERNEL_FUSED_SPLIT);
            return SC_OK;
        }
        // the grid cannot be co-resident here (e.g. a partitioned device):
        // the three-launch form below
        cudaGetLastError();
        if (fallback_folded) *fallback_folded = false;
        a.fold = 0;
    }
    // scratch: [flag u32 | eh i32 x C] [h8 hi | h8 lo]
    const size_t head = (size_t)cdiv(4 * channels + 64, 256) * 256;
    char *ws = static_cast<char *>(scratch(head + 2 * (size_t)h8_ch * channels * 2 + 1024, 3, stream, &err));
    if (err) return err;
    unsigned *flag = pre ? pre->flag : reinterpret_cast<unsigned *>(ws);
    int *eh = reinterpret_cast<int *>(ws + 16);
    __half *h8_hi = reinterpret_cast<__half *>(ws + head);
    __half *h8_lo = h8_hi + h8_ch * channels;
    if (nonfinite_out) *nonfinite_out = flag;
    // one channel: k_h8_fs stores the flag itself (no memset node in the chain)
    const bool set_flag = !pre && channels == 1;
    if (!pre && !set_flag) SC_CHECK_CUDA(cudaMemsetAsync(flag, 0, 4, stream));
    {
        dim3 g((unsigned)cdiv(ngroups * 8, 256), (unsigned)channels);
        SC_LAUNCH_PDL(k_h8_fs, g, dim3(256), 0, stream, h, ldh, nh, s8, ngroups, h8_hi, h8_lo, h8_ch, eh, flag,
                      set_flag);
    }
    a.x = x, a.ldx = ldx, a.x_base = x_base, a.x_lo = x_lo, a.x_hi = x_hi;
    a.h8[0] = h8_hi, a.h8[1] = h8_lo, a.h8_ch = h8_ch, a.eh = eh;
    a.s8 = s8, a.tiles_per_ch = tiles_per_ch, a.n_tiles = n_tiles, a.n_begin = n_begin, a.n_end = n_end;
    a.channels = channels, a.y = y, a.ldy = ldy, a.flag = flag;
    a.nsplit = nsplit, a.sps = sps, a.n_units = n_tiles * nsplit;
    SC_REQUIRE(a.n_units < (int64_t)INT32_MAX && a.s8 < (int64_t)INT32_MAX, "fir: too many work units");
    a.ws = nullptr;
    static const bool trace = getenv("SC_FS_TRACE") != nullptr;
    a.trace = nullptr;
    if (trace) {
        SC_CHECK_CUDA(cudaMalloc(&a.trace, 32 * 8 * 8));
        SC_CHECK_CUDA(cudaMemset(a.trace, 0, 32 * 8 * 8));
    }
    if (nsplit > 1) {
        a.ws = static_cast<float *>(scratch(sizeof(float) * (size_t)n_len * channels * nsplit, 4, stream, &err));
        if (err) return err;
    }
    const int grid = (int)std::min<int64_t>(a.n_units, sms);
    if (nsplit == 1 && s8 == SSH) {
        using G1 = FsGeo<SSH, true>;
        SC_CHECK_CUDA(cudaFuncSetAttribute(k_tc_fir_fs<SSH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           G1::SM_TOTAL));
        SC_LAUNCH_PDL(k_tc_fir_fs<SSH, true>, dim3(grid), dim3(G1::THREADS), G1::SM_TOTAL, stream, a);
    } else {
        SC_CHECK_CUDA(cudaFuncSetAttribute(k_tc_fir_fs<SSH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           G::SM_TOTAL));
        SC_LAUNCH_PDL(k_tc_fir_fs<SSH, false>, dim3(grid), dim3(G::THREADS), G::SM_TOTAL, stream, a);
    }
    if (a.trace) {
        unsigned long long h[32 * 8];
        cudaMemcpy(h, a.trace, sizeof h, cudaMemcpyDeviceToHost);
        cudaFree(a.trace);
        const unsigned long long t0 = h[0];
        for (int k = 0; k < 32 && h[k * 8]; ++k)
            fprintf(stderr, "[fs] unit %2d conv %7.2f load %7.2f ready %7.2f | mma %7.2f issued %7.2f | epi %7.2f store %7.2f done %7.2f us\n",
                    k, (h[k * 8 + 0] - t0) * 1e-3, (h[k * 8 + 1] - t0) * 1e-3, (h[k * 8 + 2] - t0) * 1e-3,
                    (h[k * 8 + 3] - t0) * 1e-3, (h[k * 8 + 4] - t0) * 1e-3, (h[k * 8 + 5] - t0) * 1e-3,
                    h[k * 8 + 7] ? (h[k * 8 + 7] - t0) * 1e-3 : 0.0, (h[k * 8 + 6] - t0) * 1e-3);
    }
    note_tc_launch(SSH, G::TN, n_tiles * (int64_t)TR * G::TN * (int64_t)TR * s8, SC_TC_KERNEL_FUSED_SPLIT);
    if (nsplit > 1) {
        dim3 g((unsigned)cdiv(n_len, 256), (unsigned)channels);
        SC_LAUNCH_PDL(k_tc_split_reduce, g, dim3(256), 0, stream, static_cast<const float *>(a.ws), (int)nsplit,
                      (int)channels, n_len, y, ldy, static_cast<const unsigned *>(flag),
                      TcFallback{x, ldx, x_base, x_lo, x_hi, h, ldh, nh, n_begin});
        if (fallback_folded) *fallback_folded = true;
    }
    return SC_OK;
}

namespace {
}  // namespace

bool tc_fir_supported(int64_t nh) { return nh >= 2 * TR; }

// Filters of 3-4 shifts (256-511 taps) run one-stage units with 4-shift
// drains (k_tc_fir_fs<4, true>: one accumulator per unit, the streaming
// epilogue); shorter ones 2-shift drains; 5-72 shifts the multi-stage units.
int launch_fir_f32_tc_fs(const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi, const float *h,
                         int64_t ldh, int64_t nh, float *y, int64_t ldy, int64_t n_begin, int64_t n_end,
                         int64_t channels, cudaStream_t stream, const unsigned **nonfinite_out, const TcPre *pre,
                         bool *fallback_folded) {
    const int64_t s_needed = (nh + TR - 2) / TR + 1;
    static const bool one4 = [] {
        const char *v = getenv("SC_FS_SSH4");  // 0: 3-4 shift filters keep the multi-stage units (A/B)
        return !(v && atoi(v) == 0);
    }();
    if (one4 && s_needed > 2 && s_needed <= 4)
        return launch_fs_impl<4>(x, ldx, x_base, x_lo, x_hi, h, ldh, nh, y, ldy, n_begin, n_end, channels, stream,
                                 nonfinite_out, pre, fallback_folded);
    return launch_fs_impl<2>(x, ldx, x_base, x_lo, x_hi, h, ldh, nh, y, ldy, n_begin, n_end, channels, stream,
                             nonfinite_out, pre, fallback_folded);
}

int launch_fir_f32_tc(const float *x, int64_t ldx, int64_t x_base, int64_t x_lo, int64_t x_hi,
                      const float *h, int64_t ldh, int64_t nh, float *y, int64_t ldy, int64_t n_begin,
                      int64_t n_end, int64_t channels, cudaStream_t stream, const unsigned **nonfinite_out,
                      const TcPre *pre, bool *fallback_folded) {
    if (nonfinite_out) *nonfinite_out = nullptr;
    if (fallback_folded) *fallback_folded = false;
    const int64_t n_len = n_end - n_begin;
    if (n_len <= 0 || channels <= 0) return SC_OK;
    SC_REQUIRE(nh >= 1, "tc fir: empty impulse response");
    SC_REQUIRE(channels < 65536, "tc fir: too many channels");
    // Filters whose shifts fit one converter window skip the split image
    // (k_tc_fir_fs); SC_TC_FUSED=0 forces the image path.
    static const bool fused = [] {
        const char *v = getenv("SC_TC_FUSED");
        return !(v && atoi(v) == 0);
    }();
    if (fused) {
        const int rc = launch_fir_f32_tc_fs(x, ldx, x_base, x_lo, x_hi, h, ldh, nh, y, ldy, n_begin, n_end, channels,
                                            stream, nonfinite_out, pre, fallback_folded);
        if (rc != SC_ERR_STATE) return rc;
    }
    const int64_t s_needed = (nh + TR - 2) / TR + 1;
    static const int wide_ssh_env = [] {
        const char *v = getenv("SC_TC_WIDE_SSH");  // experiment knob: 2, 4 or 8 (0 = by padding)
        const int k = v ? atoi(v) : 0;
        return k == 2 || k == 4 || k == 8 ? k : 0;
    }();
    // Drain period at 256-row tiles: 4 shifts, unless draining every 2 saves
    // >= 3 % of the padded shifts (short filters: 9 shifts pad to 12 vs 10).
    // Measured on 2^26-sample launches (profiles/r02_medium_ssh.txt): 2-shift
    // drains cost ~2 % of MMA throughput, so 1,024 taps 0.529 -> 0.485 ms,
    // 2,048 taps 0.740 -> 0.697, 4,096 taps 1.175 -> 1.128; cfg3/cfg4/cfg5
    // (751 / 129 / 2,049 shifts: <= 1.5 % padding either way) keep 4.
    const int wide_ssh = wide_ssh_env ? wide_ssh_env
                                      : (cdiv(s_needed, 4) * 4 * 100 >= cdiv(s_needed, 2) * 2 * 103 ? 2 : 4);
    // 256 output rows per tile (measured +2 % on cfg5, +2.7 % on cfg4, +3 %
    // on cfg3 end to end over 128: half the A-operand reads per FLOP) unless
    // the launch is too small to fill the SMs with 256-row work units (tiles
    // x shift-range splits of >= 48 shifts): cfg2's 19 short segments keep
    // 128-row tiles (0.18 ms vs 0.22 ms).  SC_TC_N=128|256 forces one.
    static const int tnv_env = [] {
        const char *v = getenv("SC_TC_N");
        return v ? atoi(v) : 0;
    }();
    const int ssh_wide = s_needed <= 2 ? 2 : wide_ssh;
    const int wp_wide = ssh_wide == 2 ? TcStage<2, 256>::WP : ssh_wide == 4 ? TcStage<4, 256>::WP : TcStage<8, 256>::WP;
    const int64_t s8_wide = cdiv(s_needed, ssh_wide) * ssh_wide;
    const int64_t wide_units = cdiv(n_len, (int64_t)TR * 256) * channels * std::max<int64_t>(1, s8_wide / wp_wide);
    const int TNV = tnv_env == 128 ? 128 : tnv_env == 256 ? 256 : (wide_units >= sm_count() ? 256 : 128);
    // 128-row tiles (small launches, e.g. cfg2's 19 segments) drain every 8
    // shifts; SC_TC_SSH128=4 drains every 4 (less shift padding, but measured
    // slower on cfg2: 0.102 vs 0.095 ms)
    static const int ssh128 = [] {
        const char *v = getenv("SC_TC_SSH128");
        return v && atoi(v) == 4 ? 4 : 8;
    }();
    const int SSH = TNV == 256 ? ssh_wide : (s_needed <= 2 ? 2 : ssh128);  // drain period: see TcStage
    const int64_t s8 = cdiv(s_needed, SSH) * SSH;
    const int64_t TN = TNV, TTILE = (int64_t)TR * TNV;
    const int WP = TNV == 128 ? (SSH == 2 ? TcStage<2, 128>::WP : SSH == 4 ? TcStage<4, 128>::WP : TcStage<8, 128>::WP)
                              : (SSH == 2 ? TcStage<2, 256>::WP : SSH == 4 ? TcStage<4, 256>::WP : TcStage<8, 256>::WP);
    const int64_t tiles_per_ch = cdiv(n_len, TTILE);
    const int64_t row_min = -((s8 + WP + 7) / 8) * 8;
    const int64_t nrows = tiles_per_ch * TN - row_min;
    const int64_t ngroups = KG * s8 + KG - 1;

    // scratch: [amax 2C u32 | scales 3C f32] [xt hi | xt lo] [h8 hi | h8 lo]
    const int64_t xt_ch = nrows * KG * 8;
    const int64_t h8_ch = ngroups * 64;
    const size_t head = (size_t)cdiv(20 * channels + 64, 256) * 256;
    const size_t bytes = head + 2 * (size_t)(xt_ch + h8_ch) * channels * 2 + 1024;
    int err = 0;
    char *ws = static_cast<char *>(scratch(bytes, 3, stream, &err));
    if (err) return err;
    unsigned *amax_own = reinterpret_cast<unsigned *>(ws);
    const unsigned *amax = pre ? pre->amax : amax_own;
    unsigned *flag = pre ? pre->flag : reinterpret_cast<unsigned *>(ws + 8 * channels);
    float *scales = reinterpret_cast<float *>(ws + 8 * channels + 16);
    if (nonfinite_out) *nonfinite_out = flag;
    __half *xt_hi = reinterpret_cast<__half *>(ws + head);
    __half *xt_lo = xt_hi + xt_ch * channels;
    __half *h8_hi = xt_lo + xt_ch * channels;
    __half *h8_lo = h8_hi + h8_ch * channels;

    if (!pre) {  // the caller's pass already took the maxima and the flag
    SC_CHECK_CUDA(cudaMemsetAsync(amax_own, 0, 8 * channels + 4, stream));
    {
        // ~8 resident CTAs per SM across all channels for x, float4 per thread
        const int64_t xn = x_hi - x_lo;
        const int64_t per_ch = std::max<int64_t>(1, 8 * (int64_t)sm_count() / channels);
        const int gx = xn > 0 ? (int)std::min<int64_t>(cdiv(xn, 1024), per_ch) : 0;
        const int gh = (int)std::min<int64_t>(cdiv(nh, 1024), std::max<int64_t>(1, per_ch / 4));
        dim3 g((unsigned)(gx + gh), (unsigned)channels);
        k_amax2<<<g, 256, 0, stream>>>(x + (x_lo - x_base), ldx, xn, gx, h, ldh, nh, amax_own, flag);
        SC_CHECK_LAUNCH();
    }
    }
    {
        const int gsplit = (int)cdiv(nrows, 32);
        const int gh8 = (int)cdiv(ngroups * 8, 256);
        dim3 g((unsigned)(gsplit + gh8), (unsigned)channels);
        SC_LAUNCH_PDL(k_tc_prep, g, dim3(256), 0, stream, x, ldx, x_base, x_lo, x_hi, n_begin, row_min, nrows, gsplit,
                      h, ldh, nh, s8, ngroups, amax, scales, xt_hi, xt_lo, xt_ch, h8_hi, h8_lo, h8_ch, flag);
    }
    // function attributes are per device (context): set on every launch so
    // multi-GPU drivers (one host thread per device) never miss it
#define SC_TC_ATTR(S, N) \
    SC_CHECK_CUDA(cudaFuncSetAttribute(k_tc_fir<S, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                       TcStage<S, N>::SM_TOTAL))
    if (TNV == 128 && SSH == 2) SC_TC_ATTR(2, 128);
    else if (TNV == 128 && SSH == 4) SC_TC_ATTR(4, 128);
    else if (TNV == 128) SC_TC_ATTR(8, 128);
    else if (SSH == 2) SC_TC_ATTR(2, 256);
    else if (SSH == 4) SC_TC_ATTR(4, 256);
    else SC_TC_ATTR(8, 256);
#undef SC_TC_ATTR
    TcArgs a;
    a.xt[0] = xt_hi;
    a.xt[1] = xt_lo;
    a.h8[0] = h8_hi;
    a.h8[1] = h8_lo;
    a.xt_ch = xt_ch;
    a.h8_ch = h8_ch;
    a.nrows = nrows;
    a.row_min = row_min;
    a.s8 = s8;
    a.tiles_per_ch = tiles_per_ch;
    a.n_tiles = tiles_per_ch * channels;
    a.n_begin = n_begin;
    a.n_end = n_end;
    a.y = y;
    a.ldy = ldy;
    a.scales = scales;
    a.nonfinite = flag;
    a.channels = channels;
    // Shift-range splits fill idle SMs when whole tiles leave the last wave
    // mostly empty (cfg3: 182 tiles on 148 SMs); each split keeps >= 2 X
    // windows so its window load stays amortised -- unless the tiles alone
    // leave more than half the SMs idle (cfg2's 19 short segments: 38 tiles
    // of a 40-shift filter), where splits down to one drain period pay.
    const int sms = sm_count();
    const int64_t stages = s8 / SSH;
    static const bool small_split = [] {
        const char *v = getenv("SC_TC_SMALL_SPLIT");  // experiment knob: 0 disables
        return !(v && atoi(v) == 0);
    }();
    const int64_t min_stages = (small_split && a.n_tiles * 2 <= sms) ? 1 : WP / SSH;
    int64_t nsplit = 1;
    {
        double best = 0.0;
        for (int64_t s = 1; s <= 16 && s * min_stages <= stages; ++s) {
            const int64_t units = a.n_tiles * s;
            const int64_t waves = (units + sms - 1) / sms;
            const double eff = (double)units / (double)(waves * sms);
            if (eff > best + 0.03) {
                best = eff;
                nsplit = s;
            }
            if (best > 0.95) break;
        }
    }
    const int64_t sps = cdiv(stages, nsplit) * SSH;
    nsplit = cdiv(s8, sps);
    a.nsplit = nsplit;
    a.sps = sps;
    a.n_units = a.n_tiles * nsplit;
    SC_REQUIRE(a.n_units < (int64_t)INT32_MAX && a.s8 < (int64_t)INT32_MAX, "fir: too many work units");
    a.ws = nullptr;
    if (nsplit > 1) {
        a.ws = static_cast<float *>(scratch(sizeof(float) * (size_t)n_len * channels * nsplit, 4, stream, &err));
        if (err) return err;
    }
    const int grid = (int)std::min<int64_t>(a.n_units, sms);
#define SC_TC_LAUNCH(S, N) \
    SC_LAUNCH_PDL(k_tc_fir<S, N>, dim3(grid), dim3(TcGeo<N>::THREADS), TcStage<S, N>::SM_TOTAL, stream, a)
    if (TNV == 128 && SSH == 2) SC_TC_LAUNCH(2, 128);
    else if (TNV == 128 && SSH == 4) SC_TC_LAUNCH(4, 128);
    else if (TNV == 128) SC_TC_LAUNCH(8, 128);
    else if (SSH == 2) SC_TC_LAUNCH(2, 256);
    else if (SSH == 4) SC_TC_LAUNCH(4, 256);
    else SC_TC_LAUNCH(8, 256);
#undef SC_TC_LAUNCH
    note_tc_launch(SSH, TNV, a.n_tiles * TTILE * (int64_t)TR * s8, SC_TC_KERNEL_IMAGE);
    if (nsplit > 1) {
        dim3 g((unsigned)cdiv(n_len, 256), (unsigned)channels);
        SC_LAUNCH_PDL(k_tc_split_reduce, g, dim3(256), 0, stream, static_cast<const float *>(a.ws), (int)nsplit,
                      (int)channels, n_len, y, ldy, static_cast<const unsigned *>(flag),
                      TcFallback{x, ldx, x_base, x_lo, x_hi, h, ldh, nh, n_begin});
        if (fallback_folded) *fallback_folded = true;
    }
    return SC_OK;
}

}  // namespace sc
