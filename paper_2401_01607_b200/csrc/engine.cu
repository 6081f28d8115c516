// engine.cu -- device-resident streaming engine (ScatterEngine,
// pkg/src/scatterconv/engine.py:60-214), its multichannel batch (SURVEY.md
// 8(f)1: one engine per channel, engine.py:60-66 / cli.py:186-202, in ONE
// launch per block), and the literal scatter_block drop-in (_kernels.py:14-52).
//
// Residue layout.  The reference keeps a circular ring of cap slots and a
// read index (engine.py:75-79).  On the device we keep the same residue in
// SCHEDULE ORDER (index 0 = next slot to emit, engine.py:211-214) in two
// ping-pong buffers.  A block of n samples is one ordered gather launch:
//   for slot t in [0, n + cap):  acc = res_in[t] (if t < cap) + sum over
//   block samples m ascending of x[m]*h[t-m];  t < n -> out[t], else
//   res_out[t-n]
// which continues each slot's chain exactly where the reference's per-sample
// loop would (_kernels.py:31-51), and avoids the ring's slot aliasing
// (slots t and t+cap of one block) that would be a race in parallel.
//
// State that the reference updates data-dependently -- `live` (engine.py
// :78-79 / _kernels.py:43-51), and through it `cap` on a swap
// (engine.py:179) and `read_index` -- lives in device memory and is updated
// by small epilogue kernels, so process_block, swap_ir and the deferred
// swap never wait on the host.  The host keeps only an upper bound of cap
// (to size launches and buffers) and the sample counter.
//
// Channels: every per-engine array is [C][ld] (ld = its capacity) and every
// kernel runs grid.y = C (or one thread per channel), so C engines that share
// block size, IR length and swap times -- the reference CLI's per-channel
// loop -- advance together.  Each channel keeps its own live/cap/read_index.

#include <algorithm>
#include <map>
#include <cstring>
#include <new>
#include <vector>

#include "sc_common.cuh"

namespace sc {
namespace {

// per-channel device state: live, cap, read_index, and the channel's current
// IR length (channels may hold IRs of different lengths: one engine per
// channel, engine.py:60-66)
enum { ST_LIVE = 0, ST_CAP = 1, ST_RI = 2, ST_NH = 3, ST_N = 4 };

// live/read_index after a block (derivation in DESIGN.md): with J = last
// index whose sample scatters (-1 if none),
//   live' = max(0, live - n, J >= 0 ? nh - n + J : 0);  ri' = (ri + n) % cap.
// One CTA per channel.
template <typename T, int SKIP>
__global__ void k_block_epilogue(const T *__restrict__ x, int64_t ldx, int64_t n, double thr, int64_t nh,
                                 int64_t *__restrict__ st) {
    const T *xc = x + blockIdx.x * ldx;
    int64_t *s = st + blockIdx.x * ST_N;
    __shared__ long long sj[32];
    long long J = -1;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (!skipped<SKIP>(xc[i], thr)) J = i > J ? i : J;
    for (int o = 16; o > 0; o >>= 1) {
        const long long v = __shfl_xor_sync(0xffffffffu, J, o);
        J = v > J ? v : J;
    }
    if ((threadIdx.x & 31) == 0) sj[threadIdx.x >> 5] = J;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) J = sj[w] > J ? sj[w] : J;
        if (nh <= 0) nh = s[ST_NH];  // channels with their own IR lengths
        int64_t live = s[ST_LIVE] - n;
        if (live < 0) live = 0;
        if (J >= 0 && nh - n + J > live) live = nh - n + J;
        s[ST_LIVE] = live;
        s[ST_RI] = (s[ST_RI] + n) % s[ST_CAP];
    }
}

__global__ void k_swap_state(int64_t *st, int64_t nh_new, int64_t C) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    int64_t *s = st + c * ST_N;
    const int64_t live = s[ST_LIVE];
    s[ST_CAP] = nh_new > live ? nh_new : live;  // engine.py:179
    s[ST_RI] = 0;                               // engine.py:184
    s[ST_NH] = nh_new;
}

// per-channel swap: channels with nh_new[c] > 0 swap (to that length), the
// others keep their IR and state untouched
__global__ void k_swap_state_ch(int64_t *st, const int64_t *__restrict__ nh_new, int64_t C) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C || nh_new[c] <= 0) return;
    int64_t *s = st + c * ST_N;
    const int64_t live = s[ST_LIVE];
    s[ST_CAP] = nh_new[c] > live ? nh_new[c] : live;
    s[ST_RI] = 0;
    s[ST_NH] = nh_new[c];
}

// nh <= 0: every channel keeps its own IR length (cap = that length)
__global__ void k_reset_state(int64_t *st, int64_t nh, int64_t C) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    int64_t *s = st + c * ST_N;
    s[ST_LIVE] = 0;
    if (nh > 0) s[ST_NH] = nh;
    s[ST_CAP] = s[ST_NH];
    s[ST_RI] = 0;
}

template <typename T>
__global__ void k_ring_to_sched(const T *__restrict__ ring, int64_t cap, int64_t ri,
                                T *__restrict__ sched) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap) sched[i] = ring[(ri + i) % cap];
}

template <typename T>
__global__ void k_sched_to_ring(const T *__restrict__ sched, int64_t cap, int64_t ri,
                                T *__restrict__ ring) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap) ring[(ri + i) % cap] = sched[i];
}

size_t esize(int dtype) { return dtype == SC_F64 ? 8 : 4; }

int launch_epilogue(int dtype, const void *x, int64_t ldx, int64_t n, double thr, int64_t nh, int64_t *st,
                    int64_t C, cudaStream_t s) {
    if (dtype == SC_F64)
        k_block_epilogue<double, SC_SKIP_NOT_GT><<<(unsigned)C, 1024, 0, s>>>(static_cast<const double *>(x), ldx,
                                                                             n, thr, nh, st);
    else
        k_block_epilogue<float, SC_SKIP_NOT_GT><<<(unsigned)C, 1024, 0, s>>>(static_cast<const float *>(x), ldx, n,
                                                                            thr, nh, st);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

// ---- one block in one launch (process_block / process_sample, small blocks)
// Latency path of the block engine (engine.py:118-146): slots t in
// [0, n + cap_ub) of the block, one thread per slot, each one ordered chain
// acc = residue[t] (t < logical cap) then + x[m]*h[t-m] for m ascending over
// the block's scattering samples -- the exact chain k_chain_w forms, so the
// results are bit-identical to it (and to the reference in float64).  The
// block and the taps a CTA's slots touch are staged in shared memory; the
// scatter decision is one bit per sample.  The grid's last CTA of each
// channel row is the epilogue: it finds the block's last scattering index J
// (backward scan) and updates live / read_index (k_block_epilogue's
// recurrence).  It only touches live and read_index, the slot CTAs only read
// cap, so the two run side by side: one launch per block instead of two.
constexpr int BS_TB = 64;        // slots per CTA
constexpr int BS_MAX_N = 2048;   // largest block this path takes

struct BlockStepArgs {
    const void *x;
    int64_t ldx, n;
    const void *h;
    int64_t ldh, nh;
    const void *rin;
    void *rout;
    int64_t res_ld;
    void *out;
    int64_t ldo;
    int64_t n_slots;
    int64_t *st;
    double thr;
    int slot_ctas;
    int ragged;  // channels hold IRs of different lengths: nh = st[ST_NH] per channel
};

__device__ __forceinline__ void cp_async_elem(void *smem, const void *gmem, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}

template <typename T, bool FUSED>
__global__ void __launch_bounds__(BS_TB) k_block_step(BlockStepArgs a) {
    extern __shared__ __align__(16) unsigned char bs_smem[];
    const int c = blockIdx.y;
    const T *__restrict__ xc = static_cast<const T *>(a.x) + (int64_t)c * a.ldx;
    const int n = (int)a.n;
    int64_t *st = a.st + (int64_t)c * ST_N;
    if ((int)blockIdx.x == a.slot_ctas) {
        // epilogue CTA: live' = max(0, live - n, J >= 0 ? nh - n + J : 0), ri' = (ri + n) % cap
        asm volatile("griddepcontrol.launch_dependents;\n" ::);
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        long long J = -1;
        for (int top = n; top > 0; top -= BS_TB) {
            const int i = top - 1 - (int)threadIdx.x;
            if (i >= 0 && !skipped<SC_SKIP_NOT_GT>(xc[i], a.thr)) J = i;
            if (__syncthreads_or(J >= 0)) break;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const long long v = __shfl_xor_sync(0xffffffffu, J, o);
            J = v > J ? v : J;
        }
        __shared__ long long sj[BS_TB / 32];
        if ((threadIdx.x & 31) == 0) sj[threadIdx.x >> 5] = J;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < BS_TB / 32; ++w) J = sj[w] > J ? sj[w] : J;
            const int64_t nh = a.ragged ? st[ST_NH] : a.nh;
            int64_t live = st[ST_LIVE] - a.n;
            if (live < 0) live = 0;
            if (J >= 0 && nh - a.n + J > live) live = nh - a.n + J;
            st[ST_LIVE] = live;
            st[ST_RI] = (st[ST_RI] + a.n) % st[ST_CAP];
        }
        return;
    }
    T *xs = reinterpret_cast<T *>(bs_smem);
    unsigned *xm = reinterpret_cast<unsigned *>(xs + BS_MAX_N);
    T *hs = reinterpret_cast<T *>(xm + BS_MAX_N / 32);
    const int64_t t0 = (int64_t)blockIdx.x * BS_TB;
    const int64_t t = t0 + threadIdx.x;
    asm volatile("griddepcontrol.launch_dependents;\n" ::);
    // a ragged engine's per-channel IR length lives in the device state:
    // read after this grid's predecessors are done
    if (a.ragged) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const int64_t nhc = a.ragged ? st[ST_NH] : a.nh;
    // taps k = t - m for this CTA's slots: [k0, k1)
    const int64_t k0 = t0 - (n - 1) > 0 ? t0 - (n - 1) : 0;
    const int64_t k1 = t0 + BS_TB < nhc ? t0 + BS_TB : nhc;
    const T *__restrict__ hc = static_cast<const T *>(a.h) + (int64_t)c * a.ldh;
    // Programmatic dependent launch: the next block's kernel may start now
    // (its CTAs fit beside ours); it stages its taps -- engine-owned, only
    // ever written by swaps, which are stream-ordered before any kernel they
    // precede -- and then waits for this grid before touching the residue,
    // the state or its block.
    for (int64_t k = k0 + threadIdx.x; k < k1; k += BS_TB) cp_async_elem(hs + (k - k0), hc + k, (int)sizeof(T));
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    // one round trip: the block goes to shared memory as async copies while
    // the residue slot and the logical cap load to registers
    for (int i = threadIdx.x; i < n; i += BS_TB) cp_async_elem(xs + i, xc + i, (int)sizeof(T));
    asm volatile("cp.async.commit_group;\n" ::);
    const T *rin = static_cast<const T *>(a.rin) + (int64_t)c * a.res_ld;
    const T r0 = t < a.res_ld ? rin[t] : T(0);
    const int64_t cap = st[ST_CAP];  // the residue's logical length, on the device
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    // scatter decisions (_kernels.py:33): one bit per sample, and skipped
    // samples zeroed; whether this CTA's taps are all finite
    bool finite = true;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += BS_TB) finite &= (bool)isfinite((double)hs[k - k0]);
    for (int w = threadIdx.x >> 5; w * 32 < n; w += BS_TB / 32) {
        const int i = w * 32 + (threadIdx.x & 31);
        const bool keep = i < n && !skipped<SC_SKIP_NOT_GT>(xs[i < n ? i : 0], a.thr);
        const unsigned bits = __ballot_sync(0xffffffffu, keep);
        if ((threadIdx.x & 31) == 0) xm[w] = bits;
        if (i < n && !keep) xs[i] = T(0);
    }
    finite = __syncthreads_and(finite);
    if (t >= a.n_slots) return;
    T acc = t < cap ? r0 : T(0);
    // m in [max(0, t - nh + 1), min(n - 1, t)]
    const int64_t mlo64 = t - nhc + 1 > 0 ? t - nhc + 1 : 0;
    const int mlo = (int)(mlo64 < n ? mlo64 : n);
    const int mhi = (int)(t < n - 1 ? t : n - 1);
    const T *hb = hs + (t - k0);  // tap k = t - m at hb[-m]
    int m = mlo;
    if (finite) {
        // every tap finite: a skipped (zeroed) sample adds exactly +-0, which
        // leaves the chain's value unchanged (it is never -0): no tests
        for (; m + 7 <= mhi; m += 8) {
            T xv[8], hv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) xv[u] = xs[m + u], hv[u] = hb[-(m + u)];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = mac_step<FUSED>(acc, xv[u], hv[u]);
        }
        for (; m <= mhi; ++m) acc = mac_step<FUSED>(acc, xs[m], hb[-m]);
    } else {
        for (; m <= mhi; ++m)
            if ((xm[m >> 5] >> (m & 31)) & 1u) acc = mac_step<FUSED>(acc, xs[m], hb[-m]);
    }
    if (t < a.n)
        static_cast<T *>(a.out)[(int64_t)c * a.ldo + t] = acc;
    else
        static_cast<T *>(a.rout)[(int64_t)c * a.res_ld + (t - a.n)] = acc;
}

constexpr size_t block_step_smem(size_t es) { return es * BS_MAX_N + 4 * (BS_MAX_N / 32) + es * (BS_TB + BS_MAX_N - 1); }
static_assert(block_step_smem(8) <= 48 * 1024, "k_block_step stays under the default dynamic smem limit");

int launch_block_step(const BlockStepArgs &a, int dtype, bool fused, int64_t C, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(a.slot_ctas + 1), (unsigned)C);
    cfg.blockDim = dim3(BS_TB);
    cfg.dynamicSmemBytes = block_step_smem(dtype == SC_F64 ? 8 : 4);  // < 48 KB: no opt-in attribute
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (dtype == SC_F64 && fused)
        e = cudaLaunchKernelEx(&cfg, k_block_step<double, true>, a);
    else if (dtype == SC_F64)
        e = cudaLaunchKernelEx(&cfg, k_block_step<double, false>, a);
    else
        e = cudaLaunchKernelEx(&cfg, k_block_step<float, false>, a);
    if (e != cudaSuccess) {
        set_error("k_block_step launch failed: %s", cudaGetErrorString(e));
        return SC_ERR_CUDA;
    }
    SC_CHECK_LAUNCH();
    return SC_OK;
}

// ---- fused multi-block streaming (sc_engine_process_blocks)

constexpr int kMaxEvents = kMaxSegs - 1;  // IR changes per fused launch

struct StreamEvents {
    int64_t n;                     // number of events
    int64_t block[kMaxEvents];     // block index the swap precedes (ascending)
    int64_t nh[kMaxEvents];        // new IR length
};

// J[c*n_blocks + b] = last index (within block b of channel c) whose sample
// scatters, -1 if none.  grid (n_blocks, C).
template <typename T>
__global__ void k_blocks_last_scatter(const T *__restrict__ x, int64_t ldx, int64_t n_total, int64_t nb,
                                      double thr, int64_t n_blocks, int64_t *__restrict__ J) {
    // The last scattering index: walk the block backwards one CTA-wide tile
    // at a time and stop at the first tile holding a scattering sample (a
    // dense drive stops after one tile; only skip-heavy blocks scan further).
    const int64_t b = blockIdx.x;
    const T *xc = x + blockIdx.y * ldx;
    const int64_t s = b * nb;
    const int64_t n = n_total - s < nb ? n_total - s : nb;
    long long j = -1;
    for (int64_t top = n; top > 0; top -= blockDim.x) {
        const int64_t i = top - 1 - threadIdx.x;
        if (i >= 0 && !skipped<SC_SKIP_NOT_GT>(xc[s + i], thr)) j = i;
        if (__syncthreads_or(j >= 0)) break;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const long long v = __shfl_xor_sync(0xffffffffu, j, o);
        j = v > j ? v : j;
    }
    __shared__ long long sj[32];
    if ((threadIdx.x & 31) == 0) sj[threadIdx.x >> 5] = j;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) j = sj[w] > j ? sj[w] : j;
        J[blockIdx.y * n_blocks + b] = j;
    }
}

// flush (engine.py:148-161) in one launch: per channel row c, copy the
// schedule prefix [0, n_copy) of the current residue into the tail and zero
// both residue buffers (each element is read before the same thread zeroes
// it); CTA (0, c) thread 0 writes channel c's state to the pinned host
// read-back and resets it (live = ri = 0, cap = nh).
template <typename T>
__global__ void k_flush(T *__restrict__ cur, T *__restrict__ other, int64_t res_ld, T *__restrict__ tail,
                        int64_t tail_ld, int64_t n_copy, int64_t *__restrict__ st, int64_t nh,
                        int64_t *__restrict__ st_host) {
    const int64_t c = blockIdx.y;
    T *rc = cur + c * res_ld;
    T *ro = other + c * res_ld;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < res_ld; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n_copy) tail[c * tail_ld + i] = rc[i];
        rc[i] = T(0);
        ro[i] = T(0);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t *sc = st + c * ST_N;
        for (int k = 0; k < ST_N; ++k) st_host[c * ST_N + k] = sc[k];
        sc[ST_LIVE] = 0;
        sc[ST_CAP] = nh > 0 ? nh : sc[ST_NH];  // ring of len(ir) (engine.py:157), per channel when ragged
        sc[ST_RI] = 0;
    }
}

// ---- FAST fused streams (float32, tensor cores)
// The fused stream is  out/res_out[t] = res_in[t] (t < cap) + sum over IR
// segments j of conv(x masked to segment j, h_j)[t]  -- the same sum the
// ordered chain forms, in another order.  Each segment's convolution runs on
// the FAST FIR path (tcgen05 kernel from 256 taps) into its own region of fy;
// k_fast_combine adds the regions that cover each slot in segment order and
// splits the result into the block outputs and the next residue.  Samples the
// engine would skip (|x| <= thr, NaN) are zeroed in the masked drive.
struct FastSegs {
    int n;
    int64_t m_lo[kMaxSegs], m_hi[kMaxSegs], nh[kMaxSegs], off[kMaxSegs];
};

// One CTA per (engine block, channel): zero the samples the engine skips and
// record the block's last scattering index J (the k_blocks_last_scatter
// result, from the same pass over x).  The engine's test !(|x| > thr) is done
// in float against keep = the smallest float above thr (|x| > thr  <=>
// |x| >= keep for float x; NaN fails both), float4-wide when aligned.
// Segment remap of the masked copy: block b of segment j (sm.m_lo[j] <=
// b*nb) lands at sm.dst[j] + (b*nb - sm.m_lo[j]); sm.n == 0 keeps the layout.
struct SegMap {
    int n;
    int64_t m_lo[kMaxSegs], dst[kMaxSegs];
};

// Staging of every IR of a fused call in ONE launch (instead of one
// cudaMemcpy2DAsync per IR): copy j moves [C][nh_j] from src_j (row pitch
// sld_j) to stage + off_j (row pitch dld).  grid (x: 256-sample chunks of
// the longest IR, y: copy, z: channel).
struct StageCopies {
    int n;
    const void *src[kMaxSegs];
    int64_t sld[kMaxSegs], off[kMaxSegs], nh[kMaxSegs];
};

// Extras of the mask pass for the batched tensor-core FIR: per (channel,
// segment) max |masked x| into amax[2*(c*nseg + j)] (the TC kernel's power-
// of-two scales; float bits, atomicMax), a flag for Inf samples (NaN is
// skipped by the engine rule, so masked samples are otherwise finite), the
// residue length (cap) of every channel snapshotted before the state replay
// -- which runs concurrently on a side stream -- rewrites it, and the zero
// padding of the shorter segments (grid.x CTAs past the blocks).
struct MaskExtras {
    unsigned *amax;    // nullptr: no amax (per-segment FIR path)
    unsigned *flag;
    int64_t *cap_snap;
    const int64_t *st;
    int nseg;
    int64_t L;         // padded segment length (batched layout)
    int64_t len[kMaxSegs];
    // the batched FIR's IR staging (one copy per segment, taking max |h|), CTAs past the
    // zero-padding ones: copy j of `stage` in `parts` 256-sample strides
    float *fh;
    int64_t fh_ld;
    int parts;
};

// Blocks of at most kMaskWarpNb samples take one WARP each (8 per CTA):
// with a CTA per 256-sample block, cfg2's 1,875 blocks were 2 waves of
// CTAs that each did one load, two barriers and an atomic (~10 us).
constexpr int64_t kMaskWarpNb = 1024;
constexpr int kMaskBpc = 8;  // blocks per CTA in warp mode (256 threads)

__device__ __forceinline__ void mask_block_warp(const float *__restrict__ x, int64_t ldx, int64_t n_total, int64_t nb,
                                                float keep, float *__restrict__ xm, int64_t ldm, int64_t n_blocks,
                                                int64_t *__restrict__ J, bool vec4, const SegMap &sm,
                                                const MaskExtras &mx, int64_t b) {
    const int lane = threadIdx.x & 31;
    if (b == 0 && lane == 0 && mx.cap_snap) mx.cap_snap[blockIdx.y] = mx.st[blockIdx.y * ST_N + ST_CAP];
    const float *xc = x + blockIdx.y * ldx + b * nb;
    int64_t dst = b * nb;
    int seg = 0;
    if (sm.n > 0) {
        while (seg + 1 < sm.n && sm.m_lo[seg + 1] <= b * nb) ++seg;
        dst = sm.dst[seg] + (b * nb - sm.m_lo[seg]);
    }
    float *mc = xm + blockIdx.y * ldm + dst;
    const int64_t n = n_total - b * nb < nb ? n_total - b * nb : nb;
    long long j = -1;
    float amx = 0.0f;
    bool inf = false;
    int64_t i0 = 0;
    if (vec4) {
        const int64_t n4 = n >> 2;
        for (int64_t q = lane; q < n4; q += 32) {
            float4 v = reinterpret_cast<const float4 *>(xc)[q];
            const bool k0 = fabsf(v.x) >= keep, k1 = fabsf(v.y) >= keep, k2 = fabsf(v.z) >= keep,
                       k3 = fabsf(v.w) >= keep;
            v.x = k0 ? v.x : 0.0f, v.y = k1 ? v.y : 0.0f, v.z = k2 ? v.z : 0.0f, v.w = k3 ? v.w : 0.0f;
            reinterpret_cast<float4 *>(mc)[q] = v;
            amx = fmaxf(amx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
            inf |= isinf(v.x) || isinf(v.y) || isinf(v.z) || isinf(v.w);
            const long long base = 4 * q;
            if (k3) j = base + 3;
            else if (k2) j = base + 2;
            else if (k1) j = base + 1;
            else if (k0) j = base;
        }
        i0 = n4 << 2;
    }
    for (int64_t i = i0 + lane; i < n; i += 32) {
        const float v = xc[i];
        const bool keepv = fabsf(v) >= keep;
        const float w = keepv ? v : 0.0f;
        mc[i] = w;
        amx = fmaxf(amx, fabsf(w));
        inf |= isinf(w);
        if (keepv) j = i;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const long long v = __shfl_xor_sync(0xffffffffu, j, o);
        j = v > j ? v : j;
        amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
    }
    if (mx.amax && __any_sync(0xffffffffu, inf) && lane == 0) atomicOr(mx.flag, 1u);
    if (lane == 0) {
        J[blockIdx.y * n_blocks + b] = j;
        if (mx.amax) atomicMax(mx.amax + 2 * (blockIdx.y * mx.nseg + seg), __float_as_uint(amx));
    }
}

__global__ void k_mask_skip(const float *__restrict__ x, int64_t ldx, int64_t n_total, int64_t nb, float keep,
                            float *__restrict__ xm, int64_t ldm, int64_t n_blocks, int64_t *__restrict__ J,
                            bool vec4, SegMap sm, MaskExtras mx, StageCopies stage, int bpc) {
    pdl_begin();
    // CTAs: [0, nbc) blocks (bpc per CTA), then nseg zero-padding CTAs, then
    // the IR staging CTAs
    const int64_t nbc = (n_blocks + bpc - 1) / bpc;
    const int64_t bx = blockIdx.x;
    const int64_t n_stage = mx.fh ? (int64_t)mx.parts * stage.n : 0;
    if (bx >= (int64_t)gridDim.x - n_stage) {
        // IR staging for the batched FIR, taking max |h| and flagging non-finite taps
        const int64_t q = bx - ((int64_t)gridDim.x - n_stage);
        const int j = (int)(q / mx.parts), part = (int)(q % mx.parts);
        const int64_t ch = blockIdx.y;
        const float *src = static_cast<const float *>(stage.src[j]) + ch * stage.sld[j];
        float *dst = mx.fh + ch * mx.fh_ld + stage.off[j];
        float amx = 0.0f;
        bool bad = false;
        for (int64_t i = (int64_t)part * blockDim.x + threadIdx.x; i < stage.nh[j]; i += (int64_t)mx.parts * blockDim.x) {
            const float v = src[i];
            dst[i] = v;
            amx = fmaxf(amx, fabsf(v));
            bad |= !isfinite(v);
        }
        for (int o = 16; o > 0; o >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
        if ((threadIdx.x & 31) == 0) atomicMax(mx.amax + 2 * (ch * stage.n + j) + 1, __float_as_uint(amx));
        if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(mx.flag, 1u);
        return;
    }
    if (bx >= nbc) {
        // zero [len_j, L) of segment j's padded row
        const int j = (int)(bx - nbc);
        float *row = xm + blockIdx.y * ldm + (int64_t)j * mx.L;
        for (int64_t i = mx.len[j] + threadIdx.x; i < mx.L; i += blockDim.x) row[i] = 0.0f;
        return;
    }
    if (bpc > 1) {
        const int64_t bw = bx * bpc + (threadIdx.x >> 5);
        if (bw < n_blocks) mask_block_warp(x, ldx, n_total, nb, keep, xm, ldm, n_blocks, J, vec4, sm, mx, bw);
        return;
    }
    const int64_t b = bx;
    if (b == 0 && threadIdx.x == 0 && mx.cap_snap) mx.cap_snap[blockIdx.y] = mx.st[blockIdx.y * ST_N + ST_CAP];
    const float *xc = x + blockIdx.y * ldx + b * nb;
    int64_t dst = b * nb;
    int seg = 0;
    if (sm.n > 0) {
        while (seg + 1 < sm.n && sm.m_lo[seg + 1] <= b * nb) ++seg;
        dst = sm.dst[seg] + (b * nb - sm.m_lo[seg]);
    }
    float *mc = xm + blockIdx.y * ldm + dst;
    const int64_t n = n_total - b * nb < nb ? n_total - b * nb : nb;
    long long j = -1;
    float amx = 0.0f;
    bool inf = false;
    int64_t i0 = 0;
    if (vec4) {
        const int64_t n4 = n >> 2;
        for (int64_t q = threadIdx.x; q < n4; q += blockDim.x) {
            float4 v = reinterpret_cast<const float4 *>(xc)[q];
            const bool k0 = fabsf(v.x) >= keep, k1 = fabsf(v.y) >= keep, k2 = fabsf(v.z) >= keep,
                       k3 = fabsf(v.w) >= keep;
            v.x = k0 ? v.x : 0.0f, v.y = k1 ? v.y : 0.0f, v.z = k2 ? v.z : 0.0f, v.w = k3 ? v.w : 0.0f;
            reinterpret_cast<float4 *>(mc)[q] = v;
            amx = fmaxf(amx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
            inf |= isinf(v.x) || isinf(v.y) || isinf(v.z) || isinf(v.w);
            const long long base = 4 * q;
            if (k3) j = base + 3;
            else if (k2) j = base + 2;
            else if (k1) j = base + 1;
            else if (k0) j = base;
        }
        i0 = n4 << 2;
    }
    for (int64_t i = i0 + threadIdx.x; i < n; i += blockDim.x) {
        const float v = xc[i];
        const bool keepv = fabsf(v) >= keep;
        const float w = keepv ? v : 0.0f;
        mc[i] = w;
        amx = fmaxf(amx, fabsf(w));
        inf |= isinf(w);
        if (keepv) j = i;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const long long v = __shfl_xor_sync(0xffffffffu, j, o);
        j = v > j ? v : j;
        amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
    }
    __shared__ long long sj[32];
    __shared__ float sa[32];
    if ((threadIdx.x & 31) == 0) sj[threadIdx.x >> 5] = j, sa[threadIdx.x >> 5] = amx;
    if (mx.amax && __syncthreads_or(inf) && threadIdx.x == 0) atomicOr(mx.flag, 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) j = sj[w] > j ? sj[w] : j, amx = fmaxf(amx, sa[w]);
        J[blockIdx.y * n_blocks + b] = j;
        // IEEE order of non-negative floats == order of their bit patterns
        if (mx.amax) atomicMax(mx.amax + 2 * (blockIdx.y * mx.nseg + seg), __float_as_uint(amx));
    }
}


// 4 consecutive slots per thread; segments that miss the 4 slots are skipped
// with one test.
__global__ void k_fast_combine(FastSegs sg, const float *__restrict__ fy, int64_t fy_ld,
                               const float *__restrict__ rin, int64_t res_ld, const int64_t *__restrict__ cap_snap,
                               int64_t n_total, int64_t n_slots, float *__restrict__ out, int64_t ldo,
                               float *__restrict__ rout, unsigned *zero_next, int64_t zero_words) {
    pdl_begin();
    const int64_t c = blockIdx.y;
    const int64_t cap = cap_snap[c];
    // the next call's max / flag words start at zero (they were consumed by
    // this call's FIR, which precedes this kernel)
    if (zero_next && blockIdx.y == 0)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < zero_words; i += (int64_t)gridDim.x * blockDim.x)
            zero_next[i] = 0u;
    const float *yc = fy + c * fy_ld;
    for (int64_t t4 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; t4 < n_slots;
         t4 += (int64_t)gridDim.x * blockDim.x * 4) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = t4 + q < cap && t4 + q < n_slots ? rin[c * res_ld + t4 + q] : 0.0f;
        for (int j = 0; j < sg.n; ++j) {
            const int64_t lo = sg.m_lo[j], hi = sg.m_hi[j] + sg.nh[j] - 1;
            if (t4 + 3 < lo || t4 >= hi) continue;
            const float *src = yc + sg.off[j] - lo;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (t4 + q >= lo && t4 + q < hi) v[q] += src[t4 + q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t t = t4 + q;
            if (t < n_total)
                out[c * ldo + t] = v[q];
            else if (t < n_slots)
                rout[c * res_ld + (t - n_total)] = v[q];
        }
    }
}


template <typename T>
__global__ void k_stage_irs(StageCopies c, T *__restrict__ stage, int64_t dld) {
    const int j = blockIdx.y;
    const int64_t ch = blockIdx.z;
    const T *src = static_cast<const T *>(c.src[j]) + ch * c.sld[j];
    T *dst = stage + ch * dld + c.off[j];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.nh[j]; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}


// Replays engine.py's bookkeeping over all blocks of the call: each swap
// (cap = max(nh, live), ri = 0; engine.py:179-184) and each block
// (live' = max(0, live - n, J >= 0 ? nh - n + J : 0), ri' = (ri + n) % cap).
// Per block b the live-length update is  live' = max(live - n_b, c_b)  with
// c_b = max(0, J_b >= 0 ? nh_b - n_b + J_b : 0): a max-plus map
// l -> max(l + A, B).  Such maps compose associatively,
// (A1,B1) then (A2,B2) = (A1 + A2, max(B1 + A2, B2)), so the state after n
// blocks is an ordered reduction, not a serial walk.  Swaps only reset cap
// (= max(nh, live at the swap)) and read_index (= 0), so the final state
// needs live at the LAST swap and at the end:
//   cap = max(nh_last, live(b_last)),  ri = (samples since b_last) mod cap,
// or, without swaps, ri = (ri0 + n_total) mod cap.  One CTA per channel.
constexpr int64_t kMaxPlusNegInf = INT64_MIN / 4;
constexpr int SS_TB = 256;
constexpr int64_t kFoldLastScatter = 64;  // streams of at most this many blocks: J inside k_stream_state

__device__ __forceinline__ void mp_then(int64_t &A, int64_t &B, int64_t A2, int64_t B2) {
    const int64_t b1 = B <= kMaxPlusNegInf ? kMaxPlusNegInf : B + A2;
    A += A2;
    B = b1 > B2 ? b1 : B2;
}

// ordered composition of the maps of blocks [lo, hi) across the CTA
__device__ void mp_reduce(const int64_t *__restrict__ Jc, int64_t lo, int64_t hi, int64_t nb, int64_t n_total,
                          int64_t nh0, const StreamEvents &ev, int64_t &A_out, int64_t &B_out) {
    __shared__ int64_t sA[SS_TB / 32], sB[SS_TB / 32];
    const int64_t cnt = hi - lo;
    const int64_t per = (cnt + SS_TB - 1) / SS_TB;
    const int64_t b0 = lo + threadIdx.x * per;
    const int64_t b1 = b0 + per < hi ? b0 + per : hi;
    int64_t A = 0, B = kMaxPlusNegInf;
    if (b0 < b1) {
        // IR length in force at block b0: the last event at or before it
        int64_t nh = nh0;
        int k = 0;
        while (k < ev.n && ev.block[k] <= b0) nh = ev.nh[k++];
        for (int64_t b = b0; b < b1; ++b) {
            while (k < ev.n && ev.block[k] == b) nh = ev.nh[k++];
            const int64_t n = n_total - b * nb < nb ? n_total - b * nb : nb;
            const int64_t j = Jc[b];
            int64_t c = j >= 0 ? nh - n + j : 0;
            c = c > 0 ? c : 0;
            mp_then(A, B, -n, c);
        }
    }
    // in-order tree over lanes, then over warps
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t A2 = __shfl_down_sync(0xffffffffu, A, o);
        const int64_t B2 = __shfl_down_sync(0xffffffffu, B, o);
        if ((lane & (2 * o - 1)) == 0) mp_then(A, B, A2, B2);
    }
    if (lane == 0) {
        sA[warp] = A;
        sB[warp] = B;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        A = sA[0];
        B = sB[0];
        for (int w = 1; w < SS_TB / 32; ++w) mp_then(A, B, sA[w], sB[w]);
        A_out = A;
        B_out = B;
    }
    __syncthreads();
}

// Last scattering index of every block, by this CTA's warps: each warp takes
// blocks in turn and scans one backwards 32 samples per ballot (a dense drive
// is decided by the first ballot).  For the few-block streams where a
// separate grid-wide pass would cost more launch than work.
template <typename T>
__device__ void blocks_last_scatter_cta(const T *__restrict__ xc, int64_t n_total, int64_t nb, int64_t n_blocks,
                                        double thr, int64_t *__restrict__ Jc) {
    const int lane = threadIdx.x & 31;
    for (int64_t b = threadIdx.x >> 5; b < n_blocks; b += SS_TB / 32) {
        const int64_t base = b * nb;
        const int64_t n = n_total - base < nb ? n_total - base : nb;
        long long j = -1;
        for (int64_t top = n; top > 0; top -= 32) {
            const int64_t i = top - 1 - lane;
            const unsigned bits = __ballot_sync(0xffffffffu, i >= 0 && !skipped<SC_SKIP_NOT_GT>(xc[base + i], thr));
            if (bits) {
                j = top - 1 - (__ffs(bits) - 1);  // lowest set lane = highest index
                break;
            }
        }
        if (lane == 0) Jc[b] = j;
    }
}

__global__ void __launch_bounds__(SS_TB) k_stream_state(int64_t *__restrict__ J, int64_t n_blocks, int64_t nb,
                                                        int64_t n_total, int64_t nh0, StreamEvents ev, int64_t *st,
                                                        const void *x, int64_t ldx, double thr, int x_dtype) {
    const int64_t c = blockIdx.x;
    int64_t *s = st + c * ST_N;
    int64_t *Jc = J + c * n_blocks;
    if (x) {  // J not computed by an earlier pass: find it here first
        if (x_dtype == SC_F64)
            blocks_last_scatter_cta(static_cast<const double *>(x) + c * ldx, n_total, nb, n_blocks, thr, Jc);
        else
            blocks_last_scatter_cta(static_cast<const float *>(x) + c * ldx, n_total, nb, n_blocks, thr, Jc);
        __syncthreads();
    }
    int last = -1;  // last event that precedes a processed block
    for (int k = 0; k < ev.n; ++k)
        if (ev.block[k] < n_blocks) last = k;
    const int64_t b_last = last >= 0 ? ev.block[last] : 0;
    __shared__ int64_t red[2];
    int64_t A, B;
    mp_reduce(Jc, 0, b_last, nb, n_total, nh0, ev, A, B);
    if (threadIdx.x == 0) {
        red[0] = A;
        red[1] = B;
    }
    mp_reduce(Jc, b_last, n_blocks, nb, n_total, nh0, ev, A, B);
    if (threadIdx.x == 0) {
        const int64_t live0 = s[ST_LIVE];
        int64_t live = live0 + red[0];
        live = live > red[1] ? live : red[1];
        int64_t cap = s[ST_CAP], ri = s[ST_RI];
        const int64_t since = n_total - b_last * nb;
        if (last >= 0) {
            const int64_t nh_last = ev.nh[last];
            cap = nh_last > live ? nh_last : live;
            ri = since % cap;
            s[ST_NH] = nh_last;
        } else {
            ri = (ri + since) % cap;
        }
        int64_t fin = live + A;
        s[ST_LIVE] = fin > B ? fin : B;
        s[ST_CAP] = cap;
        s[ST_RI] = ri;
    }
}

}  // namespace
}  // namespace sc

using namespace sc;

struct sc_engine {
    int dtype = SC_F32;
    size_t es = 4;
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t C = 1;  // channels
    int64_t nb = 8192;
    double thr = 0.0;
    // current impulse response, engine-owned copy: [C][ir_ld]
    void *ir = nullptr;
    int64_t nh = 0, ir_ld = 0;
    // pending impulse response (swap_ir_at_next_block): [C][pend_ld]
    void *pend = nullptr;
    int64_t pend_nh = 0, pend_ld = 0;
    bool has_pending = false;
    // residue in schedule order, ping-pong: [C][res_ld]
    void *res[2] = {nullptr, nullptr};
    int cur = 0;
    int64_t res_ld = 0;
    int64_t cap_ub = 0;     // host upper bound of every channel's logical cap
    int64_t *st = nullptr;  // device [C][ST_N]: live, cap, read_index
    int64_t consumed = 0;
    // staging copies of the IRs of one fused process_blocks call: [C][stage_ld]
    void *stage = nullptr;
    int64_t stage_ld = 0;
    int64_t *jbuf = nullptr;  // [C][n_blocks] last-scatter index per block
    // FAST fused streams (float32): masked drive [C][fx_ld] and the per-segment
    // convolutions [C][fy_ld] (segment j at column offset fy_off[j])
    // (flat buffers; the row pitch is chosen per call)
    int mode = SC_MODE_ORDERED;
    void *fx = nullptr, *fy = nullptr, *fh = nullptr;
    int64_t fx_cap = 0, fy_cap = 0, fh_cap = 0;
    int64_t jbuf_ld = 0;
    // host-pipelined streams (sc_engine_process_blocks_host): device copies of
    // the call's input and output [C][n], and the upload / download streams
    void *hx = nullptr, *hy = nullptr;
    int64_t h_cap = 0;
    cudaStream_t up = nullptr, down = nullptr;
    // pinned host copy of the state a flush reads back ([C][ST_N]); the
    // flush enqueues all of its device work before the one host wait
    int64_t *st_host = nullptr;
    struct GraphCache *gc = nullptr;  // CUDA graphs of repeated process_blocks calls
    cudaStream_t cap_stream = nullptr;  // private stream the graphs are captured on
    // FAST fused streams: side stream for the state replay (overlaps the FIR)
    // and the per-call scratch of the mask pass (amax / flag / cap snapshot)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    void *tcpre = nullptr;
    int64_t tcpre_cap = 0;
    bool flush_open = false;
    int64_t flush_cap = 0, flush_nh = 0;
    // Channels with IRs of their own (per-channel swaps, engine.py:60-66's one
    // engine per channel): host copy of every channel's IR length; `ragged`
    // when they differ (the kernels then read each channel's length from the
    // device state).  A per-channel pending swap keeps its lengths in pend_nh_c
    // (<= 0: that channel has none).  nh_arg: device copy of one swap's
    // per-channel lengths for k_swap_state_ch.
    int64_t *nh_host = nullptr;
    bool ragged = false;
    int64_t *pend_nh_c = nullptr;
    bool pend_ch = false;
    int64_t *nh_arg = nullptr;
};

namespace {

// Grow a [C][ld] buffer to [C][want], keeping the first keep_n samples of
// every row; new samples are zero.
int ensure_2d(void **p, int64_t *ld, int64_t want, size_t es, int64_t C, int64_t keep_n, cudaStream_t s) {
    if (*ld >= want) return SC_OK;
    void *np = nullptr;
    if (cudaMalloc(&np, (size_t)want * es * C) != cudaSuccess) {
        cudaGetLastError();
        set_error("engine: cudaMalloc(%lld x %lld samples) failed", (long long)C, (long long)want);
        return SC_ERR_ALLOC;
    }
    SC_CHECK_CUDA(cudaMemsetAsync(np, 0, (size_t)want * es * C, s));
    if (*p) {
        if (keep_n > 0)
            SC_CHECK_CUDA(cudaMemcpy2DAsync(np, (size_t)want * es, *p, (size_t)(*ld) * es, (size_t)keep_n * es,
                                            (size_t)C, cudaMemcpyDeviceToDevice, s));
        SC_CHECK_CUDA(cudaStreamSynchronize(s));  // old buffer may still be read
        cudaFree(*p);
    }
    *p = np;
    *ld = want;
    return SC_OK;
}

// rows of n samples: dst[c*dld + i] = src[c*sld + i]
int copy_rows(sc_engine *e, void *dst, int64_t dld, const void *src, int64_t sld, int64_t n) {
    if (n <= 0) return SC_OK;
    SC_CHECK_CUDA(cudaMemcpy2DAsync(dst, (size_t)dld * e->es, src, (size_t)sld * e->es, (size_t)n * e->es,
                                    (size_t)e->C, cudaMemcpyDeviceToDevice, e->stream));
    return SC_OK;
}

unsigned cgrid(int64_t C) { return (unsigned)cdiv(C, 128); }

int grow_residue(sc_engine *e, int64_t want) {
    if (e->res_ld >= want) return SC_OK;
    int64_t ld0 = e->res_ld, ld1 = e->res_ld;
    int rc = ensure_2d(&e->res[e->cur], &ld0, want, e->es, e->C, e->cap_ub, e->stream);
    if (rc) return rc;
    rc = ensure_2d(&e->res[1 - e->cur], &ld1, want, e->es, e->C, 0, e->stream);
    if (rc) return rc;
    e->res_ld = want;
    return SC_OK;
}

// swap_ir core (engine.py:163-186): h is [C][h_ld] in device memory.
int do_swap(sc_engine *e, const void *h, int64_t h_ld, int64_t nh) {
    if (h != e->ir) {
        int rc = ensure_2d(&e->ir, &e->ir_ld, nh, e->es, e->C, 0, e->stream);
        if (rc) return rc;
        rc = copy_rows(e, e->ir, e->ir_ld, h, h_ld, nh);
        if (rc) return rc;
    }
    // new cap = max(nh, live) <= max(nh, cap_ub): grow buffers on the host bound only
    const int64_t ub = nh > e->cap_ub ? nh : e->cap_ub;
    int rc = grow_residue(e, ub);
    if (rc) return rc;
    e->cap_ub = ub;
    e->nh = nh;
    for (int64_t c = 0; c < e->C; ++c) e->nh_host[c] = nh;
    e->ragged = false;
    k_swap_state<<<cgrid(e->C), 128, 0, e->stream>>>(e->st, nh, e->C);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

// Per-channel swap_ir: channel c with nh_new[c] > 0 takes row c of h (pitch
// h_ld) as its new IR, the others keep theirs (one engine per channel,
// engine.py:163-186 each).  Rows are zero-padded past their length.
int do_swap_ch(sc_engine *e, const void *h, int64_t h_ld, const int64_t *nh_new) {
    int64_t mx = 0;
    for (int64_t c = 0; c < e->C; ++c) {
        const int64_t keep = nh_new[c] > 0 ? nh_new[c] : e->nh_host[c];
        mx = keep > mx ? keep : mx;
    }
    int rc = SC_OK;
    if (h != e->ir) {
        // the untouched channels' taps must survive a wider buffer
        rc = ensure_2d(&e->ir, &e->ir_ld, mx, e->es, e->C, e->nh, e->stream);
        if (rc) return rc;
        for (int64_t c = 0; c < e->C; ++c) {
            if (nh_new[c] <= 0) continue;
            char *dst = static_cast<char *>(e->ir) + (size_t)(c * e->ir_ld) * e->es;
            SC_CHECK_CUDA(cudaMemcpyAsync(dst, static_cast<const char *>(h) + (size_t)(c * h_ld) * e->es,
                                          (size_t)nh_new[c] * e->es, cudaMemcpyDeviceToDevice, e->stream));
            if (e->ir_ld > nh_new[c])
                SC_CHECK_CUDA(cudaMemsetAsync(dst + (size_t)nh_new[c] * e->es, 0,
                                              (size_t)(e->ir_ld - nh_new[c]) * e->es, e->stream));
        }
    }
    const int64_t ub = mx > e->cap_ub ? mx : e->cap_ub;
    rc = grow_residue(e, ub);
    if (rc) return rc;
    e->cap_ub = ub;
    // the lengths go to the device in stream order (a pageable source is
    // staged by the copy call itself, so nh_new need not outlive it)
    SC_CHECK_CUDA(cudaMemcpyAsync(e->nh_arg, nh_new, sizeof(int64_t) * e->C, cudaMemcpyHostToDevice, e->stream));
    bool uniform = true;
    for (int64_t c = 0; c < e->C; ++c) {
        if (nh_new[c] > 0) e->nh_host[c] = nh_new[c];
        uniform = uniform && e->nh_host[c] == e->nh_host[0];
    }
    e->nh = mx;
    e->ragged = !uniform;
    k_swap_state_ch<<<cgrid(e->C), 128, 0, e->stream>>>(e->st, e->nh_arg, e->C);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

int run_pending_swap(sc_engine *e) {
    e->has_pending = false;
    if (e->pend_ch) {
        e->pend_ch = false;
        return do_swap_ch(e, e->pend, e->pend_ld, e->pend_nh_c);
    }
    return do_swap(e, e->pend, e->pend_ld, e->pend_nh);
}

// One block of n samples per channel: block/out are [C][ld].
// float64 engines in FAST mode run the ordered chain with fused multiply-adds
bool fused_chain(const sc_engine *e) { return e->dtype == SC_F64 && e->mode == SC_MODE_FAST; }

int do_block(sc_engine *e, const void *block, int64_t ldx, int64_t n, void *out, int64_t ldo, bool apply_pending) {
    if (apply_pending && e->has_pending) {
        int rc = run_pending_swap(e);
        if (rc) return rc;
    }
    SC_REQUIRE(n <= e->nb, "block of %lld samples exceeds block_size_nb=%lld", (long long)n,
               (long long)e->nb);
    if (n == 0) return SC_OK;
    void *rin = e->res[e->cur], *rout = e->res[1 - e->cur];
    if (n <= BS_MAX_N && e->C < 65536) {
        // latency path: slots + state epilogue in one launch
        BlockStepArgs a{};
        a.x = block, a.ldx = ldx, a.n = n;
        a.h = e->ir, a.ldh = e->ir_ld, a.nh = e->nh;
        a.rin = rin, a.rout = rout, a.res_ld = e->res_ld;
        a.out = out, a.ldo = ldo;
        a.n_slots = n + e->cap_ub;
        a.st = e->st;
        a.thr = e->thr;
        a.slot_ctas = (int)cdiv(a.n_slots, BS_TB);
        a.ragged = e->ragged ? 1 : 0;
        int rc = launch_block_step(a, e->dtype, fused_chain(e), e->C, e->stream);
        if (rc) return rc;
        e->cur = 1 - e->cur;
        e->consumed += n;
        return SC_OK;
    }
    int rc = SC_OK;
    if (e->ragged) {
        // channels with their own IR lengths: one ordered launch per channel
        for (int64_t c = 0; c < e->C; ++c) {
            const size_t es = e->es;
            ChainSeg seg{static_cast<const char *>(e->ir) + (size_t)(c * e->ir_ld) * es, e->nh_host[c], 0, n};
            ChainBatch batch{1, ldx, e->ir_ld, ldo, e->res_ld, e->res_ld, ST_N};
            rc = launch_chain(e->dtype, SC_SKIP_NOT_GT, e->thr, static_cast<const char *>(block) + (size_t)(c * ldx) * es,
                              0, &seg, 1, static_cast<const char *>(rin) + (size_t)(c * e->res_ld) * es, 0,
                              e->st + c * ST_N + ST_CAP, 0, n + e->cap_ub, static_cast<char *>(out) + (size_t)(c * ldo) * es,
                              n, static_cast<char *>(rout) + (size_t)(c * e->res_ld) * es, e->stream, nullptr, &batch,
                              fused_chain(e));
            if (rc) return rc;
        }
    } else {
        ChainSeg seg{e->ir, e->nh, 0, n};
        ChainBatch batch{e->C, ldx, e->ir_ld, ldo, e->res_ld, e->res_ld, ST_N};
        rc = launch_chain(e->dtype, SC_SKIP_NOT_GT, e->thr, block, 0, &seg, 1, rin, 0, e->st + ST_CAP, 0,
                          n + e->cap_ub, out, n, rout, e->stream, nullptr, &batch, fused_chain(e));
    }
    if (rc) return rc;
    rc = launch_epilogue(e->dtype, block, ldx, n, e->thr, e->ragged ? 0 : e->nh, e->st, e->C, e->stream);
    if (rc) return rc;
    e->cur = 1 - e->cur;
    e->consumed += n;
    return SC_OK;
}

int read_state(sc_engine *e, std::vector<int64_t> &host) {
    host.assign((size_t)(ST_N * e->C), 0);
    SC_CHECK_CUDA(cudaMemcpyAsync(host.data(), e->st, sizeof(int64_t) * ST_N * e->C, cudaMemcpyDeviceToHost,
                                  e->stream));
    SC_CHECK_CUDA(cudaStreamSynchronize(e->stream));
    return SC_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int now = -1;
        cudaGetDevice(&now);
        if (prev >= 0 && now != prev) cudaSetDevice(prev);
    }
};

// Fused back-to-back blocks (see sc_engine_process_blocks); x/out are
// [C][ldx]/[C][ldo] rows of n_total samples.
// Segments sharing one IR length NH (periodic swaps -- the CLI's, cfg2's and
// mstream's pattern) are convolved in ONE batched FIR launch: each segment is
// padded with zeros to the longest length L, batch (channel c, segment j)
// reads the masked drive at (c*S + j)*L (row pitch S*L), its IR staged at
// (c*S + j)*NH and writes (c*S + j)*(L + NH - 1).
bool uniform_segs(const ChainSeg *segs, int nseg, int64_t *L, int64_t *NH) {
    // one IR length; segments padded to the longest, <= 25 % padding
    *NH = segs[0].nh;
    *L = 0;
    int64_t total = 0;
    for (int j = 0; j < nseg; ++j) {
        const int64_t len = segs[j].m_hi - segs[j].m_lo;
        if (segs[j].nh != *NH) return false;
        *L = len > *L ? len : *L;
        total += len;
    }
    return nseg >= 2 && 4 * (*L * nseg - total) <= total;
}

// FAST fused streams go to the FIR kernels when the work amortises their
// set-up: a batched launch (uniform segments) from 2^28 MACs in total,
// otherwise ~6 launches per segment, so every segment needs >= 2^30 MACs
// over the channels (the ordered chain needs >= ~30 us for that much work).
bool fast_stream_worth(const sc_engine *e, const ChainSeg *segs, int nseg) {
    if (e->mode != SC_MODE_FAST || e->dtype != SC_F32) return false;
    int64_t L, NH;
    double total = 0.0;
    bool each = true;
    for (int j = 0; j < nseg; ++j) {
        const double w = (double)e->C * (double)(segs[j].m_hi - segs[j].m_lo) * (double)segs[j].nh;
        total += w;
        each = each && w >= 1073741824.0;
    }
    if (uniform_segs(segs, nseg, &L, &NH) && (double)e->C * nseg < 65536.0 && total >= 268435456.0) return true;
    return each;
}

// Also fills e->jbuf (last scattering index per block) from its mask pass and
// replays the engine state (k_stream_state) on a side stream that overlaps
// the FIR: the combine reads each channel's residue length from the mask
// pass's snapshot, so the replay may rewrite the state meanwhile.
int fast_stream(sc_engine *e, const void *x, int64_t ldx, int64_t n_total, int64_t nb, int64_t ub,
                const ChainSeg *segs, const int64_t *seg_ld, int nseg, void *rin, void *rout, void *out, int64_t ldo,
                const StreamEvents &sev) {
    const int64_t n_blocks = cdiv(n_total, nb);
    int64_t L, NH;
    const bool batched = uniform_segs(segs, nseg, &L, &NH) && e->C * nseg < 65536;
    const int64_t Lo = L + NH - 1;
    FastSegs sg{};
    sg.n = nseg;
    int64_t tot = 0;
    for (int j = 0; j < nseg; ++j) {
        sg.m_lo[j] = segs[j].m_lo;
        sg.m_hi[j] = segs[j].m_hi;
        sg.nh[j] = segs[j].nh;
        sg.off[j] = batched ? j * Lo : tot;
        tot += segs[j].m_hi - segs[j].m_lo + segs[j].nh - 1;
    }
    const int64_t xpitch = batched ? nseg * L : n_total;  // per channel
    const int64_t ypitch = batched ? nseg * Lo : tot;
    int rc = ensure_2d(&e->fx, &e->fx_cap, e->C * xpitch, 4, 1, 0, e->stream);
    if (rc) return rc;
    rc = ensure_2d(&e->fy, &e->fy_cap, e->C * ypitch, 4, 1, 0, e->stream);
    if (rc) return rc;
    // [amax 2*C*nseg u32 | flag u32 | pad] [cap snapshot C x i64]
    const int64_t amax_bytes = ((8 * e->C * nseg + 4 + 15) / 16) * 16;
    rc = ensure_2d(&e->tcpre, &e->tcpre_cap, amax_bytes + 8 * e->C, 1, 1, 0, e->stream);
    if (rc) return rc;
    if (!e->side) {
        SC_CHECK_CUDA(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
        SC_CHECK_CUDA(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
        SC_CHECK_CUDA(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
    }
    unsigned *amax = static_cast<unsigned *>(e->tcpre);
    unsigned *flag = amax + 2 * e->C * nseg;
    int64_t *cap_snap = reinterpret_cast<int64_t *>(static_cast<char *>(e->tcpre) + amax_bytes);
    float *xm = static_cast<float *>(e->fx), *fy = static_cast<float *>(e->fy);
    {
        // amax / flag are zero here: a fresh buffer is zero-filled, and every
        // batched call's combine zeroes them for the next one
        // smallest float strictly above thr (thr >= 0): |x| > thr <=> |x| >= keep
        float keep = (float)e->thr;
        if ((double)keep <= e->thr) keep = nextafterf(keep, INFINITY);
        SegMap sm{};
        MaskExtras mx{};
        mx.cap_snap = cap_snap;
        mx.st = e->st;
        mx.nseg = nseg;
        int tails = 0;
        if (batched) {
            sm.n = nseg;
            for (int j = 0; j < nseg; ++j) sm.m_lo[j] = segs[j].m_lo, sm.dst[j] = j * L;
            mx.amax = amax;
            mx.flag = flag;
            mx.L = L;
            for (int j = 0; j < nseg; ++j) mx.len[j] = segs[j].m_hi - segs[j].m_lo;
            if (xpitch > n_total) tails = nseg;  // zero padding of the shorter segments
        }
        const bool vec4 = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(xm)) & 15) == 0 &&
                          ldx % 4 == 0 && xpitch % 4 == 0 && nb % 4 == 0 && (!batched || L % 4 == 0);
        // the batched FIR's IR staging rides in the same launch (extra CTAs)
        StageCopies cp{};
        int parts = 0;
        if (batched) {
            rc = ensure_2d(&e->fh, &e->fh_cap, e->C * nseg * NH, 4, 1, 0, e->stream);
            if (rc) return rc;
            cp.n = nseg;
            for (int j = 0; j < nseg; ++j)
                cp.src[j] = segs[j].h, cp.sld[j] = seg_ld[j], cp.off[j] = j * NH, cp.nh[j] = NH;
            parts = (int)std::min<int64_t>(cdiv(NH, 256), 64);
            mx.fh = static_cast<float *>(e->fh);
            mx.fh_ld = nseg * NH;
            mx.parts = parts;
        }
        const int bpc = nb <= kMaskWarpNb ? kMaskBpc : 1;
        const dim3 g((unsigned)(cdiv(n_blocks, (int64_t)bpc) + tails + (int64_t)parts * (batched ? nseg : 0)),
                     (unsigned)e->C);
        SC_LAUNCH_PDL(k_mask_skip, g, dim3(256), 0, e->stream, static_cast<const float *>(x), ldx, n_total, nb, keep,
                      xm, xpitch, n_blocks, e->jbuf, vec4, sm, mx, cp, bpc);
    }
    // the state replay needs only J (and the state): fork it off
    SC_CHECK_CUDA(cudaEventRecord(e->ev_fork, e->stream));
    SC_CHECK_CUDA(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
    k_stream_state<<<(unsigned)e->C, SS_TB, 0, e->side>>>(e->jbuf, n_blocks, nb, n_total, e->nh, sev, e->st, nullptr,
                                                          ldx, e->thr, e->dtype);
    SC_CHECK_LAUNCH();
    SC_CHECK_CUDA(cudaEventRecord(e->ev_join, e->side));
    // NaN/Inf in x or h: launch_fir_f32's device-gated ordered fallback
    if (batched) {
        const TcPre pre{amax, flag};
        rc = launch_fir_f32(SC_MODE_FAST, xm, L, 0, 0, L, static_cast<const float *>(e->fh), NH, NH, fy, Lo, 0, Lo,
                            e->C * nseg, e->stream, &pre);
        if (rc) return rc;
    } else {
        for (int j = 0; j < nseg; ++j) {
            // outputs [m_lo, m_hi + nh - 1) of segment j's drive samples
            rc = launch_fir_f32(SC_MODE_FAST, xm, xpitch, 0, segs[j].m_lo, segs[j].m_hi,
                                static_cast<const float *>(segs[j].h), seg_ld[j], segs[j].nh, fy + sg.off[j],
                                ypitch, segs[j].m_lo, segs[j].m_hi + segs[j].nh - 1, e->C, e->stream);
            if (rc) return rc;
        }
    }
    const int64_t n_slots = n_total + ub;
    const dim3 g((unsigned)std::min<int64_t>(cdiv(n_slots, 1024), 4096), (unsigned)e->C);
    SC_LAUNCH_PDL(k_fast_combine, g, dim3(256), 0, e->stream, sg, static_cast<const float *>(fy), ypitch,
                  static_cast<const float *>(rin), e->res_ld, static_cast<const int64_t *>(cap_snap), n_total, n_slots,
                  static_cast<float *>(out), ldo, static_cast<float *>(rout), batched ? amax : nullptr,
                  (int64_t)(batched ? 2 * e->C * nseg + 1 : 0));
    SC_CHECK_CUDA(cudaStreamWaitEvent(e->stream, e->ev_join, 0));
    return SC_OK;
}

int process_blocks_stepwise(sc_engine *e, const void *x, int64_t ldx, int64_t n_total, int64_t nb,
                            const int64_t *swap_blocks, const void *const *swap_irs, const int64_t *swap_ld,
                            const int64_t *swap_nh, int64_t nh_stride, int64_t n_swaps, void *out, int64_t ldo) {
    const int64_t n_blocks = cdiv(n_total, nb);
    std::vector<int64_t> order;
    for (int64_t i = 0; i < n_swaps; ++i)
        if (swap_blocks[i] >= 0 && swap_blocks[i] < n_blocks) order.push_back(i);
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return swap_blocks[a] < swap_blocks[b]; });
    size_t k = 0;
    for (int64_t b = 0; b < n_blocks; ++b) {
        for (; k < order.size() && swap_blocks[order[k]] == b; ++k) {
            const int64_t i = order[k];
            const int64_t ld = swap_ld ? swap_ld[i] : (nh_stride ? 0 : swap_nh[i]);
            int rc;
            if (nh_stride) {
                int64_t ldm = ld;
                if (!ldm)
                    for (int64_t c = 0; c < e->C; ++c) ldm = swap_nh[i * nh_stride + c] > ldm ? swap_nh[i * nh_stride + c] : ldm;
                rc = do_swap_ch(e, swap_irs[i], ldm, swap_nh + i * nh_stride);
            } else {
                rc = do_swap(e, swap_irs[i], ld, swap_nh[i]);
            }
            if (rc) return rc;
        }
        const int64_t s0 = b * nb, n = n_total - s0 < nb ? n_total - s0 : nb;
        int rc = do_block(e, static_cast<const char *>(x) + (size_t)s0 * e->es, ldx, n,
                          static_cast<char *>(out) + (size_t)s0 * e->es, ldo, b == 0);
        if (rc) return rc;
    }
    return SC_OK;
}

int process_blocks_impl(sc_engine *e, const void *x, int64_t ldx, int64_t n_total, int64_t nb,
                        const int64_t *swap_blocks, const void *const *swap_irs, const int64_t *swap_nh,
                        const int64_t *swap_ld, int64_t n_swaps, void *out, int64_t ldo) {
    if (n_total == 0) return SC_OK;
    if (e->ragged || e->pend_ch)
        return process_blocks_stepwise(e, x, ldx, n_total, nb, swap_blocks, swap_irs, swap_ld, swap_nh, 0, n_swaps,
                                       out, ldo);
    const int64_t n_blocks = cdiv(n_total, nb);
    // IR timeline: (block, h [C][nh], nh); a pending deferred swap acts right
    // before block 0, after any explicit swap scheduled there (engine.py:124-126).
    struct Ev {
        int64_t block;
        const void *h;
        int64_t ld, nh;
    };
    std::vector<Ev> ev;
    for (int64_t i = 0; i < n_swaps; ++i)
        if (swap_blocks[i] >= 0 && swap_blocks[i] < n_blocks)
            ev.push_back({swap_blocks[i], swap_irs[i], swap_ld ? swap_ld[i] : swap_nh[i], swap_nh[i]});
    std::stable_sort(ev.begin(), ev.end(), [](const Ev &a, const Ev &b) { return a.block < b.block; });
    if (e->has_pending) {
        size_t pos = 0;
        while (pos < ev.size() && ev[pos].block == 0) ++pos;
        ev.insert(ev.begin() + pos, Ev{0, e->pend, e->pend_ld, e->pend_nh});
        e->has_pending = false;
    }
    // Swaps before the same block: only the last one's IR and cap matter
    // (swap_ir keeps every live residue sample whatever the cap, engine.py:
    // 178-183, and live does not change between them), so keep the last.
    // Afterwards every event has its own block, which bounds the split below.
    {
        size_t w = 0;
        for (size_t r = 0; r < ev.size(); ++r) {
            if (w > 0 && ev[w - 1].block == ev[r].block) ev[w - 1] = ev[r];
            else ev[w++] = ev[r];
        }
        ev.resize(w);
    }
    // Too many IR changes for one launch: process consecutive block ranges
    // (each range holds <= kMaxEvents events at distinct blocks, so the
    // recursive call never splits again).
    if ((int64_t)ev.size() > kMaxEvents) {
        int64_t b0 = 0;
        size_t k = 0;
        while (b0 < n_blocks) {
            const size_t k1 = std::min(ev.size(), k + kMaxEvents);
            int64_t b1 = k1 < ev.size() ? ev[k1].block : n_blocks;
            if (b1 <= b0) b1 = b0 + 1;
            std::vector<int64_t> sb, sn, sl;
            std::vector<const void *> sh;
            for (; k < ev.size() && ev[k].block < b1; ++k) {
                sb.push_back(ev[k].block - b0);
                sh.push_back(ev[k].h);
                sn.push_back(ev[k].nh);
                sl.push_back(ev[k].ld);  // the pending IR lives in a pitched buffer
            }
            const int64_t s0 = b0 * nb, s1 = std::min(n_total, b1 * nb);
            int rc = process_blocks_impl(e, static_cast<const char *>(x) + (size_t)s0 * e->es, ldx, s1 - s0, nb,
                                         sb.data(), sh.data(), sn.data(), sl.data(), (int64_t)sb.size(),
                                         static_cast<char *>(out) + (size_t)s0 * e->es, ldo);
            if (rc) return rc;
            b0 = b1;
        }
        return SC_OK;
    }
    // The IR timeline as segments of drive samples, each with its taps' source
    // (the engine's copy, the pending buffer or the caller's IR; row pitch
    // seg_ld).  The FAST path reads the sources directly (stream-ordered, like
    // any kernel given the caller's buffers); the ordered chain wants one row
    // pitch for all segments, so it stages them in engine memory [C][stage_ld].
    int64_t max_nh = e->nh;
    ChainSeg segs[kMaxSegs];
    int64_t seg_ld[kMaxSegs];
    int nseg = 0;
    segs[nseg] = ChainSeg{e->ir, e->nh, 0, n_total};
    seg_ld[nseg++] = e->ir_ld;
    int64_t ub = e->cap_ub;
    StreamEvents sev{};
    sev.n = 0;
    for (const Ev &v : ev) {
        max_nh = v.nh > max_nh ? v.nh : max_nh;
        const int64_t m = v.block * nb;
        if (segs[nseg - 1].m_lo == m) {
            segs[nseg - 1].h = v.h;  // a later swap before the same block wins
            segs[nseg - 1].nh = v.nh;
            seg_ld[nseg - 1] = v.ld;
        } else {
            segs[nseg - 1].m_hi = m;
            segs[nseg] = ChainSeg{v.h, v.nh, m, n_total};
            seg_ld[nseg++] = v.ld;
        }
        sev.block[sev.n] = v.block;
        sev.nh[sev.n] = v.nh;
        ++sev.n;
        ub = v.nh > ub ? v.nh : ub;
    }
    int rc = ensure_2d(reinterpret_cast<void **>(&e->jbuf), &e->jbuf_ld, n_blocks * e->C, 8, 1, 0, e->stream);
    if (rc) return rc;
    rc = grow_residue(e, ub);
    if (rc) return rc;
    const bool fast = fast_stream_worth(e, segs, nseg);
    int64_t hld = e->ir_ld;  // ordered path: the common row pitch of the segments' taps
    if (!fast && !(nseg == 1 && segs[0].h == e->ir)) {
        int64_t tot = 0;
        for (int j = 0; j < nseg; ++j) tot += segs[j].nh;
        rc = ensure_2d(&e->stage, &e->stage_ld, tot, e->es, e->C, 0, e->stream);
        if (rc) return rc;
        StageCopies cp{};
        int64_t off = 0;
        for (int j = 0; j < nseg; ++j) {
            cp.src[j] = segs[j].h, cp.sld[j] = seg_ld[j], cp.off[j] = off, cp.nh[j] = segs[j].nh;
            segs[j].h = static_cast<char *>(e->stage) + (size_t)off * e->es;
            off += segs[j].nh;
        }
        cp.n = nseg;
        const dim3 gs((unsigned)std::min<int64_t>(cdiv(max_nh, 256), 64), (unsigned)cp.n, (unsigned)e->C);
        if (e->dtype == SC_F64)
            k_stage_irs<double><<<gs, 256, 0, e->stream>>>(cp, static_cast<double *>(e->stage), e->stage_ld);
        else
            k_stage_irs<float><<<gs, 256, 0, e->stream>>>(cp, static_cast<float *>(e->stage), e->stage_ld);
        SC_CHECK_LAUNCH();
        hld = e->stage_ld;
    }
    // the IR in force after the call (becomes the engine's copy)
    const void *last_src = fast ? ev.empty() ? e->ir : ev.back().h : segs[nseg - 1].h;
    const int64_t last_ld = fast ? ev.empty() ? e->ir_ld : ev.back().ld : hld;
    const int64_t last_nh = segs[nseg - 1].nh;
    // One ordered launch for every block: slot t accumulates its drive samples
    // in ascending order across blocks and IR segments -- the same chain as
    // block-by-block processing (bit-identical), continued from the residue.
    void *rin = e->res[e->cur], *rout = e->res[1 - e->cur];
    bool j_from_x = false;
    if (fast) {
        // (the FAST path also replays the state, on a side stream)
        rc = fast_stream(e, x, ldx, n_total, nb, ub, segs, seg_ld, nseg, rin, rout, out, ldo, sev);
        if (rc) return rc;
    } else {
        ChainBatch batch{e->C, ldx, hld, ldo, e->res_ld, e->res_ld, ST_N};
        rc = launch_chain(e->dtype, SC_SKIP_NOT_GT, e->thr, x, 0, segs, nseg, rin, 0, e->st + ST_CAP, 0,
                          n_total + ub, out, n_total, rout, e->stream, nullptr, &batch, fused_chain(e));
        if (rc) return rc;
        if (n_blocks <= kFoldLastScatter) {
            j_from_x = true;  // the state kernel finds J itself
        } else {
        const dim3 gj((unsigned)n_blocks, (unsigned)e->C);
        if (e->dtype == SC_F64)
            k_blocks_last_scatter<double><<<gj, 256, 0, e->stream>>>(static_cast<const double *>(x), ldx, n_total,
                                                                    nb, e->thr, n_blocks, e->jbuf);
        else
            k_blocks_last_scatter<float><<<gj, 256, 0, e->stream>>>(static_cast<const float *>(x), ldx, n_total,
                                                                   nb, e->thr, n_blocks, e->jbuf);
        SC_CHECK_LAUNCH();
        }
    }
    if (!fast) {
    k_stream_state<<<(unsigned)e->C, SS_TB, 0, e->stream>>>(e->jbuf, n_blocks, nb, n_total, e->nh, sev, e->st,
                                                            j_from_x ? x : nullptr, ldx, e->thr, e->dtype);
    SC_CHECK_LAUNCH();
    }
    // host-side bookkeeping: the last IR becomes current (engine-owned copy)
    if (last_src != e->ir) {
        rc = ensure_2d(&e->ir, &e->ir_ld, last_nh, e->es, e->C, 0, e->stream);
        if (rc) return rc;
        rc = copy_rows(e, e->ir, e->ir_ld, last_src, last_ld, last_nh);
        if (rc) return rc;
        e->nh = last_nh;
    }
    e->cap_ub = ub;
    for (int64_t c = 0; c < e->C; ++c) e->nh_host[c] = e->nh;
    e->cur = 1 - e->cur;
    e->consumed += n_total;
    return SC_OK;
}

// ---- CUDA graphs for repeated fused calls
// A streaming application calls process_blocks with the same shapes, buffers
// and swap schedule over and over (cfg2's bench step; a render loop): the
// ~12-launch sequence costs tens of microseconds of host enqueue for a
// ~0.1 ms device step.  Every host decision process_blocks_impl takes is a
// function of its arguments and of the engine's host-side state, and every
// address its kernels touch is among them -- so the call is memoised as a
// CUDA graph keyed by all of it (plus the library's scratch generation, which
// moves whenever a scratch buffer is reallocated).  A key seen for the
// second time is captured (its first occurrence ran normally and already
// grew every buffer the call needs, so the capture never allocates or
// synchronises) and replayed from then on: one cudaGraphLaunch, then the
// recorded host-state transition.  Graph replay and direct launches enqueue
// the same kernels with the same arguments: results are identical.
}  // namespace

// (at namespace scope: sc_engine holds a GraphCache *)
struct GraphEntry {
    int seen = 0;
    bool bad = false;  // capture failed once: always run directly
    cudaGraphExec_t exec = nullptr;
    // the host-state transition of the call (a replayed call never grows a
    // buffer, so these are all it changes besides consumed += n_total)
    int64_t post_nh = 0, post_cap_ub = 0;
    int post_cur = 0;
    // what the captured call counted (sc_launch_count, sc_tc_stats)
    int64_t launches = 0, tc_launches = 0, tc_padded = 0;
    int tc_ssh = 0, tc_tn = 0;
};

struct GraphCache {
    std::map<std::vector<int64_t>, GraphEntry> entries;
    int64_t hits = 0, captures = 0, failures = 0;
    ~GraphCache() {
        for (auto &kv : entries)
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    }
};

namespace {

bool graphs_enabled() {
    static const bool on = [] {
        const char *v = getenv("SC_ENGINE_GRAPHS");  // 0 disables (A/B)
        return !(v && atoi(v) == 0);
    }();
    return on;
}

std::vector<int64_t> graph_key(const sc_engine *e, const void *x, int64_t ldx, int64_t n_total, int64_t nb,
                               const int64_t *swap_blocks, const void *const *swap_irs, const int64_t *swap_nh,
                               int64_t n_swaps, const void *out, int64_t ldo) {
    auto P = [](const void *p) { return (int64_t) reinterpret_cast<uintptr_t>(p); };
    std::vector<int64_t> k;
    k.reserve(48 + 3 * (size_t)n_swaps);
    k.insert(k.end(), {P(x), ldx, n_total, nb, P(out), ldo, n_swaps, scratch_generation(),
                       (int64_t)e->dtype, e->C, e->nb, (int64_t)e->mode, P(e->stream), (int64_t)e->device,
                       P(e->ir), e->nh, e->ir_ld, (int64_t)e->has_pending, e->has_pending ? P(e->pend) : 0,
                       e->has_pending ? e->pend_nh : 0, e->has_pending ? e->pend_ld : 0, P(e->res[0]), P(e->res[1]),
                       (int64_t)e->cur, e->res_ld, e->cap_ub, P(e->st), P(e->stage), e->stage_ld, P(e->jbuf),
                       e->jbuf_ld, P(e->fx), P(e->fy), P(e->fh), e->fx_cap, e->fy_cap, e->fh_cap, P(e->tcpre),
                       e->tcpre_cap, P(e->side)});
    int64_t thr_bits;
    std::memcpy(&thr_bits, &e->thr, sizeof thr_bits);
    k.push_back(thr_bits);
    for (int64_t i = 0; i < n_swaps; ++i) {
        k.push_back(swap_blocks[i]);
        k.push_back(P(swap_irs[i]));
        k.push_back(swap_nh[i]);
    }
    return k;
}

int process_blocks_graphed(sc_engine *e, const void *x, int64_t n_total, int64_t nb, const int64_t *swap_blocks,
                           const void *const *swap_irs, const int64_t *swap_nh, int64_t n_swaps, void *out) {
    auto direct = [&] {
        return process_blocks_impl(e, x, n_total, n_total, nb, swap_blocks, swap_irs, swap_nh, nullptr, n_swaps, out,
                                   n_total);
    };
    if (!graphs_enabled() || n_total == 0 || e->ragged || e->pend_ch) return direct();
    if (!e->gc) e->gc = new GraphCache();
    GraphCache *gc = e->gc;
    const int64_t key_gen = scratch_generation();
    std::vector<int64_t> key = graph_key(e, x, n_total, n_total, nb, swap_blocks, swap_irs, swap_nh, n_swaps, out,
                                         n_total);
    static const bool dbg = getenv("SC_GRAPH_DEBUG") != nullptr;
    if (dbg) {
        fprintf(stderr, "[graph key]");
        for (int64_t v : key) fprintf(stderr, " %lld", (long long)v);
        fprintf(stderr, "\n");
    }
    auto it = gc->entries.find(key);
    if (it == gc->entries.end()) {
        if (gc->entries.size() >= 16) {  // bound the cache
            for (auto &kv : gc->entries)
                if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
            gc->entries.clear();
        }
        it = gc->entries.emplace(std::move(key), GraphEntry{}).first;
    }
    GraphEntry &g = it->second;
    const int64_t consumed = e->consumed;
    if (g.exec) {
        SC_CHECK_CUDA(cudaGraphLaunch(g.exec, e->stream));
        ++gc->hits;
        note_launches(g.launches);
        note_tc_replay(g.tc_launches, g.tc_padded, g.tc_ssh, g.tc_tn);
        e->has_pending = false;
        e->nh = g.post_nh;
        for (int64_t c = 0; c < e->C; ++c) e->nh_host[c] = e->nh;
        e->cap_ub = g.post_cap_ub;
        e->cur = g.post_cur;
        e->consumed = consumed + n_total;
        return SC_OK;
    }
    if (g.bad || ++g.seen < 2) return direct();
    // second occurrence: capture this call, then launch it
    const sc_engine pre = *e;
    auto same_buffers = [&] {  // the capture must not have grown anything
        return e->ir == pre.ir && e->ir_ld == pre.ir_ld && e->stage == pre.stage && e->jbuf == pre.jbuf &&
               e->res[0] == pre.res[0] && e->res[1] == pre.res[1] && e->res_ld == pre.res_ld && e->fx == pre.fx &&
               e->fy == pre.fy && e->fh == pre.fh && scratch_generation() == key_gen;
    };
    // Capture on a private stream (the caller's may be the legacy default
    // stream, which cannot capture) with the engine pointed at it; the graph
    // is then launched on the caller's stream.
    if (!e->cap_stream && cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        g.bad = true;
        return direct();
    }
    const cudaStream_t orig = e->stream;
    e->stream = e->cap_stream;
    scratch_capture_alias(e->cap_stream, orig, true);
    if (cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        scratch_capture_alias(nullptr, nullptr, false);
        e->stream = orig;
        g.bad = true;
        ++gc->failures;
        return direct();
    }
    const int64_t l0 = launches_so_far();
    int64_t tl0, tp0;
    int ts0, tn0;
    tc_stats_now(&tl0, &tp0, &ts0, &tn0);
    const int rc = direct();
    int64_t tl1, tp1;
    int ts1, tn1;
    tc_stats_now(&tl1, &tp1, &ts1, &tn1);
    g.launches = launches_so_far() - l0;
    g.tc_launches = tl1 - tl0, g.tc_padded = tp1 - tp0, g.tc_ssh = ts1, g.tc_tn = tn1;
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(e->stream, &graph);
    scratch_capture_alias(nullptr, nullptr, false);
    e->stream = orig;
    cudaGraphExec_t exec = nullptr;
    if (rc == SC_OK && ce == cudaSuccess && graph && same_buffers() &&
        cudaGraphInstantiateWithFlags(&exec, graph, 0) == cudaSuccess) {
        cudaGraphDestroy(graph);
        g.exec = exec;
        g.post_nh = e->nh;
        g.post_cap_ub = e->cap_ub;
        g.post_cur = e->cur;
        ++gc->captures;
        SC_CHECK_CUDA(cudaGraphLaunch(exec, e->stream));
        return SC_OK;
    }
    // capture did not work out: nothing ran; undo the host-side effects and run directly
    if (dbg)
        fprintf(stderr, "[graph capture failed] rc=%d capture=%s same_buffers=%d err=%s\n", rc, cudaGetErrorString(ce),
                (int)same_buffers(), rc ? sc_last_error() : "");
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    const int64_t consumed_now = pre.consumed;
    e->has_pending = pre.has_pending;
    e->nh = pre.nh;
    for (int64_t c = 0; c < e->C; ++c) e->nh_host[c] = e->nh;
    e->cap_ub = pre.cap_ub;
    e->cur = pre.cur;
    e->consumed = consumed_now;
    g.bad = true;
    ++gc->failures;
    return direct();
}

}  // namespace

extern "C" {

int sc_engine_create_multi(int dtype, const void *h, int64_t nh, int64_t channels, int64_t block_size_nb,
                           double threshold, void *stream, sc_engine **out) {
    SC_REQUIRE(dtype == SC_F32 || dtype == SC_F64, "sc_engine_create: bad dtype %d", dtype);
    SC_REQUIRE(nh >= 1, "impulse response is empty");
    SC_REQUIRE(channels >= 1 && channels < 65536, "channels must be in [1, 65535], got %lld", (long long)channels);
    SC_REQUIRE(block_size_nb >= 1, "block_size_nb must be >= 1, got %lld", (long long)block_size_nb);
    SC_REQUIRE(threshold >= 0.0, "zero_skip_threshold must be >= 0, got %g", threshold);
    SC_REQUIRE(h && out, "sc_engine_create: null pointer");
    sc_engine *e = new (std::nothrow) sc_engine();
    if (!e) {
        set_error("sc_engine_create: out of host memory");
        return SC_ERR_ALLOC;
    }
    e->dtype = dtype;
    e->es = esize(dtype);
    cudaGetDevice(&e->device);
    e->stream = as_stream(stream);
    e->C = channels;
    e->nb = block_size_nb;
    e->thr = threshold;
    int rc = SC_OK;
    if (cudaMalloc(&e->st, sizeof(int64_t) * ST_N * channels) != cudaSuccess) {
        cudaGetLastError();
        set_error("sc_engine_create: cudaMalloc failed");
        rc = SC_ERR_ALLOC;
    }
    e->nh_host = new (std::nothrow) int64_t[channels];
    e->pend_nh_c = new (std::nothrow) int64_t[channels];
    if (!e->nh_host || !e->pend_nh_c) {
        set_error("sc_engine_create: out of host memory");
        rc = SC_ERR_ALLOC;
    } else {
        for (int64_t c = 0; c < channels; ++c) e->nh_host[c] = nh, e->pend_nh_c[c] = 0;
    }
    if (!rc && cudaMalloc(reinterpret_cast<void **>(&e->nh_arg), sizeof(int64_t) * channels) != cudaSuccess) {
        cudaGetLastError();
        set_error("sc_engine_create: cudaMalloc failed");
        rc = SC_ERR_ALLOC;
    }
    if (!rc) rc = ensure_2d(&e->ir, &e->ir_ld, nh, e->es, e->C, 0, e->stream);
    if (!rc) rc = grow_residue(e, nh);
    if (!rc) rc = copy_rows(e, e->ir, e->ir_ld, h, nh, nh);
    if (!rc) {
        e->nh = nh;
        e->cap_ub = nh;
        k_reset_state<<<cgrid(channels), 128, 0, e->stream>>>(e->st, nh, channels);
        if (cudaGetLastError() != cudaSuccess) rc = SC_ERR_CUDA;
    }
    if (rc) {
        sc_engine_destroy(e);
        return rc;
    }
    *out = e;
    return SC_OK;
}

int sc_engine_create(int dtype, const void *h, int64_t nh, int64_t block_size_nb, double threshold,
                     void *stream, sc_engine **out) {
    return sc_engine_create_multi(dtype, h, nh, 1, block_size_nb, threshold, stream, out);
}

int sc_engine_channels(sc_engine *e, int64_t *channels) {
    SC_REQUIRE(e && channels, "null pointer");
    *channels = e->C;
    return SC_OK;
}

int sc_engine_destroy(sc_engine *e) {
    if (!e) return SC_OK;
    DeviceGuard g(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    cudaFree(e->ir);
    cudaFree(e->pend);
    cudaFree(e->res[0]);
    cudaFree(e->res[1]);
    cudaFree(e->st);
    pinned_small_free(e->st_host);
    cudaFree(e->nh_arg);
    delete[] e->nh_host;
    delete[] e->pend_nh_c;
    delete e->gc;
    if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
    if (e->side) cudaStreamDestroy(e->side);
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    if (e->ev_join) cudaEventDestroy(e->ev_join);
    cudaFree(e->tcpre);
    cudaFree(e->stage);
    cudaFree(e->jbuf);
    cudaFree(e->fx);
    cudaFree(e->fy);
    cudaFree(e->fh);
    cudaFree(e->hx);
    cudaFree(e->hy);
    if (e->up) cudaStreamDestroy(e->up);
    if (e->down) cudaStreamDestroy(e->down);
    delete e;
    return SC_OK;
}

int sc_engine_set_mode(sc_engine *e, int mode) {
    SC_REQUIRE(e, "null engine");
    SC_REQUIRE(mode == SC_MODE_ORDERED || mode == SC_MODE_FAST, "engine mode must be ORDERED or FAST, got %d", mode);
    e->mode = mode;
    return SC_OK;
}

int sc_engine_set_stream(sc_engine *e, void *stream) {
    SC_REQUIRE(e, "null engine");
    e->stream = as_stream(stream);
    return SC_OK;
}

int sc_engine_process_block(sc_engine *e, const void *block, int64_t n, void *out) {
    SC_REQUIRE(e, "null engine");
    SC_REQUIRE(n >= 0 && (n == 0 || (block && out)), "sc_engine_process_block: bad block");
    DeviceGuard g(e->device);
    // FAST mode: a block big enough for the tensor-core FIR (>= 2^30 MACs over
    // the channels, with the IR that will be in force) goes through the fused
    // path as a one-block stream (same state updates, pending swap included)
    const int64_t nh_next = e->has_pending ? e->pend_nh : e->nh;
    if (n > 0 && n <= e->nb && e->mode == SC_MODE_FAST && e->dtype == SC_F32 && !e->ragged && !e->pend_ch &&
        (double)e->C * (double)n * (double)nh_next >= 1073741824.0)
        return process_blocks_impl(e, block, n, n, n, nullptr, nullptr, nullptr, nullptr, 0, out, n);
    return do_block(e, block, n, n, out, n, true);
}

int sc_engine_process_sample(sc_engine *e, const void *x, void *out) {
    SC_REQUIRE(e && x && out, "sc_engine_process_sample: null pointer");
    DeviceGuard g(e->device);
    // engine.py:99-116: one sample per channel; a pending swap is NOT applied
    return do_block(e, x, 1, 1, out, 1, false);
}

int sc_engine_swap_ir(sc_engine *e, const void *h, int64_t nh) {
    SC_REQUIRE(e && h, "sc_engine_swap_ir: null pointer");
    SC_REQUIRE(nh >= 1, "impulse response is empty");
    DeviceGuard g(e->device);
    return do_swap(e, h, nh, nh);
}

int sc_engine_swap_ir_at_next_block(sc_engine *e, const void *h, int64_t nh) {
    SC_REQUIRE(e && h, "sc_engine_swap_ir_at_next_block: null pointer");
    SC_REQUIRE(nh >= 1, "impulse response is empty");
    DeviceGuard g(e->device);
    int rc = ensure_2d(&e->pend, &e->pend_ld, nh, e->es, e->C, 0, e->stream);
    if (rc) return rc;
    rc = copy_rows(e, e->pend, e->pend_ld, h, nh, nh);
    if (rc) return rc;
    e->pend_nh = nh;
    e->has_pending = true;
    e->pend_ch = false;
    return SC_OK;
}

int sc_engine_swap_ir_channels(sc_engine *e, const void *h, int64_t ldh, const int64_t *nh_per_channel) {
    SC_REQUIRE(e && h && nh_per_channel, "sc_engine_swap_ir_channels: null pointer");
    DeviceGuard g(e->device);
    int64_t mx = 0;
    for (int64_t c = 0; c < e->C; ++c) mx = nh_per_channel[c] > mx ? nh_per_channel[c] : mx;
    SC_REQUIRE(mx >= 1, "sc_engine_swap_ir_channels: no channel swaps");
    SC_REQUIRE(ldh >= mx, "sc_engine_swap_ir_channels: row pitch below the longest IR");
    return do_swap_ch(e, h, ldh, nh_per_channel);
}

int sc_engine_swap_ir_at_next_block_channels(sc_engine *e, const void *h, int64_t ldh,
                                             const int64_t *nh_per_channel) {
    SC_REQUIRE(e && h && nh_per_channel, "sc_engine_swap_ir_at_next_block_channels: null pointer");
    DeviceGuard g(e->device);
    int64_t mx = 0;
    for (int64_t c = 0; c < e->C; ++c) mx = nh_per_channel[c] > mx ? nh_per_channel[c] : mx;
    SC_REQUIRE(mx >= 1, "sc_engine_swap_ir_at_next_block_channels: no channel swaps");
    SC_REQUIRE(ldh >= mx, "sc_engine_swap_ir_at_next_block_channels: row pitch below the longest IR");
    // a uniform pending swap becomes per-channel: the channels named here
    // replace theirs (engine.py:188-192, per channel)
    if (e->has_pending && !e->pend_ch)
        for (int64_t c = 0; c < e->C; ++c) e->pend_nh_c[c] = e->pend_nh;
    if (!e->has_pending)
        for (int64_t c = 0; c < e->C; ++c) e->pend_nh_c[c] = 0;
    const int64_t keep_n = e->has_pending ? e->pend_ld : 0;
    int rc = ensure_2d(&e->pend, &e->pend_ld, mx, e->es, e->C, keep_n, e->stream);
    if (rc) return rc;
    for (int64_t c = 0; c < e->C; ++c) {
        if (nh_per_channel[c] <= 0) continue;
        SC_CHECK_CUDA(cudaMemcpyAsync(static_cast<char *>(e->pend) + (size_t)(c * e->pend_ld) * e->es,
                                      static_cast<const char *>(h) + (size_t)(c * ldh) * e->es,
                                      (size_t)nh_per_channel[c] * e->es, cudaMemcpyDeviceToDevice, e->stream));
        e->pend_nh_c[c] = nh_per_channel[c];
    }
    e->has_pending = true;
    e->pend_ch = true;
    return SC_OK;
}

int sc_engine_channel_nh(sc_engine *e, int64_t *nh_per_channel) {
    SC_REQUIRE(e && nh_per_channel, "sc_engine_channel_nh: null pointer");
    for (int64_t c = 0; c < e->C; ++c) nh_per_channel[c] = e->nh_host[c];
    return SC_OK;
}

int sc_engine_process_blocks_channels(sc_engine *e, const void *x, int64_t n_total, int64_t nb,
                                      const int64_t *swap_blocks, const void *const *swap_irs,
                                      const int64_t *swap_ld, const int64_t *swap_nh, int64_t n_swaps, void *out) {
    SC_REQUIRE(e, "null engine");
    SC_REQUIRE(nb >= 1 && nb <= e->nb, "sc_engine_process_blocks_channels: nb must be in [1, block_size_nb]");
    SC_REQUIRE(n_total >= 0 && (n_total == 0 || (x && out)), "sc_engine_process_blocks_channels: bad input");
    SC_REQUIRE(n_swaps == 0 || (swap_blocks && swap_irs && swap_nh), "sc_engine_process_blocks_channels: bad swaps");
    DeviceGuard g(e->device);
    if (n_total == 0) return SC_OK;
    return process_blocks_stepwise(e, x, n_total, n_total, nb, swap_blocks, swap_irs, swap_ld, swap_nh, e->C, n_swaps,
                                   out, n_total);
}

int sc_engine_flush_begin(sc_engine *e, void *tail, int64_t tail_capacity) {
    SC_REQUIRE(e, "sc_engine_flush_begin: null pointer");
    SC_REQUIRE(!e->flush_open, "sc_engine_flush_begin: previous flush not finished (sc_engine_flush_end)");
    DeviceGuard g(e->device);
    // Every channel's tail (max(nh - 1, live) samples, engine.py:155-156) is
    // a prefix of its schedule; entries past it are zero (beyond its live
    // slots), so copying the bound cap_ub >= every tail needs no host read of
    // live first.  The state goes to pinned memory in the same stream order.
    const int64_t n_copy = e->cap_ub;
    SC_REQUIRE(tail_capacity >= n_copy && (n_copy <= 0 || tail),
               "sc_engine_flush_begin: tail buffer below sc_engine_tail_bound (%lld < %lld)",
               (long long)tail_capacity, (long long)n_copy);
    if (!e->st_host) {
        e->st_host = static_cast<int64_t *>(pinned_small(sizeof(int64_t) * ST_N * e->C));
        SC_REQUIRE(e->st_host, "sc_engine_flush_begin: pinned host allocation failed");
    }
    {
        const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(e->res_ld, 256), 2 * sm_count()));
        const dim3 g(gx, (unsigned)e->C);
        if (e->dtype == SC_F64)
            k_flush<double><<<g, 256, 0, e->stream>>>(static_cast<double *>(e->res[e->cur]),
                                                      static_cast<double *>(e->res[1 - e->cur]), e->res_ld,
                                                      static_cast<double *>(tail), tail_capacity, n_copy, e->st,
                                                      e->ragged ? 0 : e->nh, e->st_host);
        else
            k_flush<float><<<g, 256, 0, e->stream>>>(static_cast<float *>(e->res[e->cur]),
                                                     static_cast<float *>(e->res[1 - e->cur]), e->res_ld,
                                                     static_cast<float *>(tail), tail_capacity, n_copy, e->st,
                                                     e->ragged ? 0 : e->nh, e->st_host);
        SC_CHECK_LAUNCH();
    }
    e->flush_cap = tail_capacity;
    e->flush_nh = e->nh;
    e->cap_ub = e->nh;
    e->consumed = 0;
    e->flush_open = true;
    return SC_OK;
}

int sc_engine_flush_end(sc_engine *e, int64_t *n_tail) {
    SC_REQUIRE(e && n_tail, "sc_engine_flush_end: null pointer");
    SC_REQUIRE(e->flush_open, "sc_engine_flush_end: no flush in flight");
    DeviceGuard g(e->device);
    e->flush_open = false;
    SC_CHECK_CUDA(cudaStreamSynchronize(e->stream));
    int64_t nt_max = 0;
    for (int64_t c = 0; c < e->C; ++c) {
        const int64_t live = e->st_host[c * ST_N + ST_LIVE];
        const int64_t nhc = e->nh_host[c];
        n_tail[c] = (nhc - 1 > live) ? nhc - 1 : live;  // engine.py:155
        nt_max = std::max(nt_max, n_tail[c]);
    }
    SC_REQUIRE(e->flush_cap >= nt_max, "sc_engine_flush: tail buffer too small (%lld < %lld)",
               (long long)e->flush_cap, (long long)nt_max);
    return SC_OK;
}

int sc_engine_flush(sc_engine *e, void *tail, int64_t tail_capacity, int64_t *n_tail) {
    SC_REQUIRE(e && n_tail, "sc_engine_flush: null pointer");
    SC_REQUIRE(!e->flush_open, "sc_engine_flush: a split flush is in flight (sc_engine_flush_end)");
    if (tail_capacity >= e->cap_ub) {  // one launch, one host wait
        const int rc = sc_engine_flush_begin(e, tail, tail_capacity);
        return rc ? rc : sc_engine_flush_end(e, n_tail);
    }
    // a buffer sized to the exact tail: read live first, copy only the tail
    DeviceGuard g(e->device);
    std::vector<int64_t> hs;
    int rc = read_state(e, hs);
    if (rc) return rc;
    int64_t nt_max = 0;
    for (int64_t c = 0; c < e->C; ++c) {
        const int64_t live = hs[c * ST_N + ST_LIVE];
        const int64_t nhc = e->nh_host[c];
        n_tail[c] = (nhc - 1 > live) ? nhc - 1 : live;  // engine.py:155
        nt_max = std::max(nt_max, n_tail[c]);
    }
    SC_REQUIRE(tail_capacity >= nt_max && (nt_max == 0 || tail), "sc_engine_flush: tail buffer too small (%lld < %lld)",
               (long long)tail_capacity, (long long)nt_max);
    // entries past a channel's own tail length are zero (beyond its live slots)
    rc = copy_rows(e, tail, tail_capacity, e->res[e->cur], e->res_ld, nt_max);
    if (rc) return rc;
    // reset (engine.py:157-160): zero ring of len(ir), ri = live = consumed = 0
    SC_CHECK_CUDA(cudaMemsetAsync(e->res[0], 0, (size_t)e->res_ld * e->es * e->C, e->stream));
    SC_CHECK_CUDA(cudaMemsetAsync(e->res[1], 0, (size_t)e->res_ld * e->es * e->C, e->stream));
    k_reset_state<<<cgrid(e->C), 128, 0, e->stream>>>(e->st, e->ragged ? 0 : e->nh, e->C);
    SC_CHECK_LAUNCH();
    e->cap_ub = e->nh;
    e->consumed = 0;
    return SC_OK;
}

int sc_engine_tail_bound(sc_engine *e, int64_t *bound) {
    SC_REQUIRE(e && bound, "sc_engine_tail_bound: null pointer");
    *bound = std::max<int64_t>(e->cap_ub, 1);  // live <= cap <= cap_ub; nh - 1 < cap_ub
    return SC_OK;
}

int sc_engine_state(sc_engine *e, int64_t *read_index, int64_t *live, int64_t *cap, int64_t *consumed,
                    int64_t *nh, int *has_pending) {
    SC_REQUIRE(e, "null engine");
    DeviceGuard g(e->device);
    std::vector<int64_t> hs;
    int rc = read_state(e, hs);
    if (rc) return rc;
    for (int64_t c = 0; c < e->C; ++c) {
        if (read_index) read_index[c] = hs[c * ST_N + ST_RI];
        if (live) live[c] = hs[c * ST_N + ST_LIVE];
        if (cap) cap[c] = hs[c * ST_N + ST_CAP];
    }
    if (consumed) *consumed = e->consumed;
    if (nh) *nh = e->nh;
    if (has_pending) *has_pending = e->has_pending ? 1 : 0;
    return SC_OK;
}

int sc_engine_schedule(sc_engine *e, void *dst, int64_t n, int64_t *n_written) {
    SC_REQUIRE(e && n_written, "null pointer");
    DeviceGuard g(e->device);
    std::vector<int64_t> hs;
    int rc = read_state(e, hs);
    if (rc) return rc;
    int64_t kmax = 0;
    for (int64_t c = 0; c < e->C; ++c) {
        n_written[c] = std::min(n, hs[c * ST_N + ST_CAP]);
        kmax = std::max(kmax, n_written[c]);
    }
    if (kmax > 0) {
        SC_REQUIRE(dst, "null destination");
        rc = copy_rows(e, dst, n, e->res[e->cur], e->res_ld, kmax);
        if (rc) return rc;
        SC_CHECK_CUDA(cudaStreamSynchronize(e->stream));
    }
    return SC_OK;
}

int sc_engine_current_ir(sc_engine *e, void *dst, int64_t capacity, int64_t *nh) {
    SC_REQUIRE(e && nh, "null pointer");
    DeviceGuard g(e->device);
    *nh = e->nh;
    if (dst) {
        SC_REQUIRE(capacity >= e->nh, "sc_engine_current_ir: buffer too small");
        return copy_rows(e, dst, capacity, e->ir, e->ir_ld, e->nh);
    }
    return SC_OK;
}

int sc_engine_graph_stats(sc_engine *e, int64_t *hits, int64_t *captures, int64_t *failures) {
    SC_REQUIRE(e, "null engine");
    if (hits) *hits = e->gc ? e->gc->hits : 0;
    if (captures) *captures = e->gc ? e->gc->captures : 0;
    if (failures) *failures = e->gc ? e->gc->failures : 0;
    return SC_OK;
}

int sc_engine_process_blocks(sc_engine *e, const void *x, int64_t n_total, int64_t nb,
                             const int64_t *swap_blocks, const void *const *swap_irs,
                             const int64_t *swap_nh, int64_t n_swaps, void *out) {
    SC_REQUIRE(e, "null engine");
    SC_REQUIRE(nb >= 1 && nb <= e->nb, "sc_engine_process_blocks: nb must be in [1, block_size_nb]");
    SC_REQUIRE(n_total >= 0 && (n_total == 0 || (x && out)), "sc_engine_process_blocks: bad input");
    SC_REQUIRE(n_swaps == 0 || (swap_blocks && swap_irs && swap_nh), "sc_engine_process_blocks: bad swaps");
    for (int64_t i = 0; i < n_swaps; ++i) {
        SC_REQUIRE(swap_nh[i] >= 1, "impulse response is empty");
        SC_REQUIRE(i == 0 || swap_blocks[i] >= swap_blocks[i - 1], "swap_blocks must be ascending");
    }
    DeviceGuard g(e->device);
    return process_blocks_graphed(e, x, n_total, nb, swap_blocks, swap_irs, swap_nh, n_swaps, out);
}

// Host-resident stream: the same call as sc_engine_process_blocks with x and
// out in host memory.  The stream is cut into `chunks` runs of whole blocks;
// run k's upload (upload stream, one 2-D copy of the [C][run] columns),
// blocks (engine stream) and download (download stream) are event-chained,
// so the upload of run k+1 and the download of run k-1 overlap the blocks of
// run k.  Same engine state transitions as one call (a swap schedule is cut
// at the run boundaries; swaps are relative to the run's first block).
int sc_engine_process_blocks_host(sc_engine *e, const void *x_host, int64_t n_total, int64_t nb,
                                  const int64_t *swap_blocks, const void *const *swap_irs, const int64_t *swap_nh,
                                  int64_t n_swaps, void *out_host, int chunks) {
    SC_REQUIRE(e, "null engine");
    SC_REQUIRE(nb >= 1 && nb <= e->nb, "sc_engine_process_blocks_host: nb must be in [1, block_size_nb]");
    SC_REQUIRE(n_total >= 0 && (n_total == 0 || (x_host && out_host)), "sc_engine_process_blocks_host: bad input");
    SC_REQUIRE(n_swaps == 0 || (swap_blocks && swap_irs && swap_nh), "sc_engine_process_blocks_host: bad swaps");
    for (int64_t i = 0; i < n_swaps; ++i) {
        SC_REQUIRE(swap_nh[i] >= 1, "impulse response is empty");
        SC_REQUIRE(i == 0 || swap_blocks[i] >= swap_blocks[i - 1], "swap_blocks must be ascending");
    }
    if (n_total == 0) return SC_OK;
    DeviceGuard g(e->device);
    const size_t es = e->es, row = (size_t)n_total * es;
    if (e->h_cap < n_total * e->C) {
        cudaFree(e->hx);
        cudaFree(e->hy);
        e->hx = e->hy = nullptr;
        e->h_cap = 0;
        if (cudaMalloc(&e->hx, row * e->C) != cudaSuccess || cudaMalloc(&e->hy, row * e->C) != cudaSuccess) {
            cudaGetLastError();
            set_error("sc_engine_process_blocks_host: cudaMalloc of %lld bytes failed", (long long)(2 * row * e->C));
            return SC_ERR_ALLOC;
        }
        e->h_cap = n_total * e->C;
    }
    if (!e->up) SC_CHECK_CUDA(cudaStreamCreateWithFlags(&e->up, cudaStreamNonBlocking));
    if (!e->down) SC_CHECK_CUDA(cudaStreamCreateWithFlags(&e->down, cudaStreamNonBlocking));
    const int64_t n_blocks = cdiv(n_total, nb);
    // automatic: 2..4 runs (each extra run adds an IR-length halo of work to
    // FAST segments; mstream measured best at 4: 5.4 ms vs 5.9 at 7, 7.7 at 1)
    if (chunks <= 0) chunks = (int)std::max<int64_t>(2, std::min<int64_t>(4, (int64_t)(row * e->C >> 24)));
    chunks = (int)std::min<int64_t>(chunks, n_blocks);
    const int64_t per = cdiv(n_blocks, (int64_t)chunks);
    std::vector<cudaEvent_t> evs;
    auto event = [&](cudaStream_t st) {
        cudaEvent_t ev = nullptr;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return (cudaEvent_t) nullptr;
        evs.push_back(ev);
        cudaEventRecord(ev, st);
        return ev;
    };
    int rc = SC_OK;
    // the caller's earlier work on the engine stream precedes the first upload
    cudaEvent_t start = event(e->stream);
    if (!start || cudaStreamWaitEvent(e->up, start, 0) != cudaSuccess) rc = SC_ERR_CUDA;
    // every upload is queued first (the copy engine never waits on the host),
    // then each run's blocks wait for their upload and its download for them
    std::vector<cudaEvent_t> uploaded;
    for (int64_t b0 = 0; b0 < n_blocks && !rc; b0 += per) {
        const int64_t a0 = b0 * nb, a1 = std::min(n_total, std::min(n_blocks, b0 + per) * nb);
        const size_t off = (size_t)a0 * es;
        if (cudaMemcpy2DAsync(static_cast<char *>(e->hx) + off, row, static_cast<const char *>(x_host) + off, row,
                              (size_t)(a1 - a0) * es, (size_t)e->C, cudaMemcpyHostToDevice, e->up) != cudaSuccess) {
            rc = SC_ERR_CUDA;
            break;
        }
        uploaded.push_back(event(e->up));
        if (!uploaded.back()) rc = SC_ERR_CUDA;
    }
    size_t k = 0, run = 0;
    for (int64_t b0 = 0; b0 < n_blocks && !rc; b0 += per, ++run) {
        const int64_t b1 = std::min(n_blocks, b0 + per);
        const int64_t a0 = b0 * nb, a1 = std::min(n_total, b1 * nb), w = a1 - a0;
        const size_t off = (size_t)a0 * es;
        if (cudaStreamWaitEvent(e->stream, uploaded[run], 0) != cudaSuccess) {
            rc = SC_ERR_CUDA;
            break;
        }
        std::vector<int64_t> sb, sn;
        std::vector<const void *> sh;
        for (; k < (size_t)n_swaps && swap_blocks[k] < b1; ++k)
            if (swap_blocks[k] >= b0) {
                sb.push_back(swap_blocks[k] - b0);
                sh.push_back(swap_irs[k]);
                sn.push_back(swap_nh[k]);
            }
        rc = process_blocks_impl(e, static_cast<char *>(e->hx) + off, n_total, w, nb, sb.data(), sh.data(), sn.data(),
                                 nullptr, (int64_t)sb.size(), static_cast<char *>(e->hy) + off, n_total);
        if (rc) break;
        cudaEvent_t done = event(e->stream);
        if (!done || cudaStreamWaitEvent(e->down, done, 0) != cudaSuccess ||
            cudaMemcpy2DAsync(static_cast<char *>(out_host) + off, row, static_cast<char *>(e->hy) + off, row,
                              (size_t)w * es, (size_t)e->C, cudaMemcpyDeviceToHost, e->down) != cudaSuccess) {
            rc = SC_ERR_CUDA;
            break;
        }
    }
    if (rc == SC_ERR_CUDA) set_error("sc_engine_process_blocks_host: %s", cudaGetErrorString(cudaGetLastError()));
    // the result is in host memory when the call returns; later engine work
    // waits for the last download (the device buffers are reused)
    cudaEvent_t fin = event(e->down);
    if (fin) cudaStreamWaitEvent(e->stream, fin, 0);
    if (cudaStreamSynchronize(e->down) != cudaSuccess && !rc) {
        set_error("sc_engine_process_blocks_host: %s", cudaGetErrorString(cudaGetLastError()));
        rc = SC_ERR_CUDA;
    }
    cudaStreamSynchronize(e->up);
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
    return rc;
}

// ---------------------------------------------------------------- literal kernel

int sc_scatter_block(int dtype, void *ring, int64_t cap, const void *ir, int64_t nh,
                     const void *block, int64_t n, void *out, int64_t read_index, int64_t live,
                     double threshold, int64_t *read_index_out, int64_t *live_out, void *stream) {
    SC_REQUIRE(dtype == SC_F32 || dtype == SC_F64, "sc_scatter_block: bad dtype %d", dtype);
    SC_REQUIRE(cap >= 1 && nh >= 1 && nh <= cap, "sc_scatter_block: need 1 <= len(ir) <= len(ring)");
    SC_REQUIRE(read_index >= 0 && read_index < cap, "sc_scatter_block: read_index out of range");
    SC_REQUIRE(ring && ir && read_index_out && live_out, "sc_scatter_block: null pointer");
    SC_REQUIRE(n == 0 || (block && out), "sc_scatter_block: null block/out");
    cudaStream_t s = as_stream(stream);
    if (n == 0) {
        *read_index_out = read_index;
        *live_out = live;
        return SC_OK;
    }
    const size_t es = esize(dtype);
    int err = 0;
    char *ws = static_cast<char *>(scratch(es * (size_t)cap * 2 + 64, 2, s, &err));
    if (err) return err;
    void *sched_in = ws, *sched_out = ws + es * (size_t)cap;
    int64_t *st = reinterpret_cast<int64_t *>(ws + es * (size_t)cap * 2);
    int64_t hs[ST_N] = {live, cap, read_index, 0};
    SC_CHECK_CUDA(cudaMemcpyAsync(st, hs, sizeof(hs), cudaMemcpyHostToDevice, s));
    const unsigned g = (unsigned)cdiv(cap, 256);
    if (dtype == SC_F64)
        k_ring_to_sched<double><<<g, 256, 0, s>>>(static_cast<double *>(ring), cap, read_index,
                                                  static_cast<double *>(sched_in));
    else
        k_ring_to_sched<float><<<g, 256, 0, s>>>(static_cast<float *>(ring), cap, read_index,
                                                 static_cast<float *>(sched_in));
    SC_CHECK_LAUNCH();
    ChainSeg seg{ir, nh, 0, n};
    int rc = launch_chain(dtype, SC_SKIP_NOT_GT, threshold, block, 0, &seg, 1, sched_in, cap,
                          nullptr, 0, n + cap, out, n, sched_out, s);
    if (rc) return rc;
    rc = launch_epilogue(dtype, block, n, n, threshold, nh, st, 1, s);
    if (rc) return rc;
    const int64_t ri2 = (read_index + n) % cap;
    if (dtype == SC_F64)
        k_sched_to_ring<double><<<g, 256, 0, s>>>(static_cast<double *>(sched_out), cap, ri2,
                                                  static_cast<double *>(ring));
    else
        k_sched_to_ring<float><<<g, 256, 0, s>>>(static_cast<float *>(sched_out), cap, ri2,
                                                 static_cast<float *>(ring));
    SC_CHECK_LAUNCH();
    SC_CHECK_CUDA(cudaMemcpyAsync(hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    SC_CHECK_CUDA(cudaStreamSynchronize(s));
    *read_index_out = ri2;
    *live_out = hs[ST_LIVE];
    return SC_OK;
}

}  // extern "C"
