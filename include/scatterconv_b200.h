/*
 * scatterconv_b200.h -- C ABI of the B200 (sm_100a) scatter-convolution library.
 *
 * This is the drop-in boundary for the reference package `scatterconv`
 * (/root/reference/pkg/src/scatterconv).  The reference's only native call is
 * the numba kernel `_kernels.scatter_block` (_kernels.py:14-52); its Python
 * entry points (core.py:122-167, engine.py:60-214) are what users call.  Each
 * entry point below names the reference interface it replaces.  The Python
 * mirror `paper_2401_01607_b200` binds these with ctypes (INTEGRATION.md shows
 * the binding a scatterconv maintainer would add).
 *
 * Conventions
 *  - Return 0 on success, a negative SC_ERR_* code otherwise; no C++
 *    exception crosses this boundary.  sc_last_error() returns a thread-local
 *    message for the last failure on the calling thread.
 *  - Unless stated otherwise every sample pointer is a DEVICE pointer (e.g.
 *    torch.Tensor.data_ptr() of a CUDA tensor) on the current CUDA device, and
 *    every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream).  Calls documented "synchronous" wait on the stream.
 *  - dtype: SC_F32 or SC_F64 for every sample array of a call.
 *  - Engine handles are single-threaded (engine.py:60-66: one engine per
 *    channel); distinct handles may be used concurrently from different
 *    threads.  The engine owns copies of every impulse response it is given
 *    (engine.py:72, :185); callers own inputs and outputs.
 *
 * Precision modes
 *  - SC_MODE_ORDERED: every output is ONE chain over input index m ascending,
 *    starting at +0.0, each step `acc = acc + x[m]*h[n-m]` -- the reference's
 *    order (_kernels.py:1-8, core.py:83-86).  float64: product and sum rounded
 *    separately (no FMA), bit-identical to the reference.  float32: one fused
 *    multiply-add per step.  In both dtypes stream == batch for any block
 *    partition.
 *  - SC_MODE_FAST: float32 -- the fastest kernel for the shape, SC_MODE_TC
 *    for long filters, SC_MODE_FFMA otherwise; fixed (deterministic) order,
 *    within 1e-5*max|x|*||h||_1 of the reference.  float64 (any non-ORDERED
 *    mode) -- the ordered chain with one fused multiply-add per step: same
 *    order, one rounding fewer per MAC, twice the FP64 throughput, within
 *    1e-12*max|x|*||h||_1 (north_star's FP64 bar); stream == batch still
 *    holds within the mode.
 *  - SC_MODE_FFMA: register-tiled CUDA-core kernel (FFMA2 = fma.rn.f32x2).
 *  - SC_MODE_TC: tcgen05 tensor-core block-Toeplitz GEMM with an fp16 hi/lo
 *    split of x and h (3 MMAs per K-step, FP32 accumulation in TMEM); requires
 *    finite inputs.
 *
 * Skip rules (zero skipping)
 *  - SC_SKIP_NONE     every input sample scatters (scatter_convolve, core.py:90)
 *  - SC_SKIP_LE       skip |x| <= threshold; NaN is not skipped (core.py:164)
 *  - SC_SKIP_NOT_GT   skip unless |x| > threshold; NaN is skipped (_kernels.py:33)
 */
#ifndef SCATTERCONV_B200_H
#define SCATTERCONV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_ABI_VERSION 1

#define SC_OK 0
#define SC_ERR_ARG (-1)    /* invalid argument (sizes, dtype, null pointers) */
#define SC_ERR_CUDA (-2)   /* CUDA runtime error (message has cudaGetErrorString) */
#define SC_ERR_ALLOC (-3)  /* device/host allocation failed */
#define SC_ERR_STATE (-4)  /* engine used in an invalid state */

enum { SC_F32 = 0, SC_F64 = 1 };
enum { SC_MODE_FAST = 0, SC_MODE_ORDERED = 1, SC_MODE_FFMA = 2, SC_MODE_TC = 3 };
enum { SC_SKIP_NONE = 0, SC_SKIP_LE = 1, SC_SKIP_NOT_GT = 2 };

int sc_abi_version(void);
const char *sc_last_error(void);

/* Number of CUDA kernels this library has launched in this process (all
 * threads, all devices).  Benchmarks read it around a timed region to report
 * how many of the library's kernels ran there. */
int64_t sc_launch_count(void);

/* Tensor-core bookkeeping for the roofline (bench.py): cumulative k_tc_fir
 * launches and the MACs their MMAs issue over the PADDED block-Toeplitz GEMM
 * (whole tiles of 128*tile_n outputs x 128 taps x every drain-padded shift;
 * each padded MAC is 3 fp16 MMA MACs: hi*hi, lo*hi, hi*lo), plus the last
 * launch's template (drain period in shifts, tile width in output rows).
 * No reference counterpart (bench instrumentation). */
int sc_tc_stats(int64_t *launches, int64_t *padded_macs, int *last_ssh, int *last_tile_n);
void sc_tc_stats_reset(void);
/* Which tensor-core kernel issued the last counted launch (graph replays keep
 * the kernel their capture recorded): SC_TC_KERNEL_IMAGE = k_tc_fir (fp16
 * hi/lo operand image in HBM), SC_TC_KERNEL_FUSED_SPLIT = k_tc_fir_fs (x
 * read as FP32 and split in shared memory), SC_TC_KERNEL_NONE before any.
 * Not reset by sc_tc_stats_reset.  No reference counterpart (bench
 * instrumentation: the roofline names the kernel the library ran). */
#define SC_TC_KERNEL_NONE 0
#define SC_TC_KERNEL_IMAGE 1
#define SC_TC_KERNEL_FUSED_SPLIT 2
int sc_tc_last_kernel(void);

/* ---------------------------------------------------------------- whole signal */

/* Full linear convolution y[0 : ne+nh-1] = x (*) h.
 * Replaces core._scatter_full (core.py:80-92) and therefore
 * scatter_convolve (core.py:122-131), commuted_convolve (core.py:134-147:
 * pass the shorter signal as `x` to drive) and scatter_convolve_skip_zeros
 * (core.py:150-167, skip_mode = SC_SKIP_LE).  The FAST/FFMA/TC modes need
 * SC_F32 and skip_mode SC_SKIP_NONE; otherwise the ORDERED kernel runs. */
int sc_fir_full(int dtype, int mode, const void *x, int64_t ne, const void *h, int64_t nh,
                void *y, int skip_mode, double threshold, void *stream);

/* Output-range convolution for time sharding (north_star (4)):
 * y[i] = sum_k h[k] * X(n_begin + i - k) for i in [0, n_end - n_begin), where
 * X(m) = x[m - x_begin] for m in [x_begin, x_end) and 0 elsewhere.  A shard
 * owning outputs [a, b) passes x_begin = max(0, a-nh+1), x_end = min(ne, b):
 * its input slice plus the (nh-1)-sample halo.  float32; mode FAST, FFMA or TC. */
int sc_fir_range(int dtype, int mode, const void *x, int64_t x_begin, int64_t x_end, const void *h,
                 int64_t nh, void *y, int64_t n_begin, int64_t n_end, void *stream);

/* Batched multichannel (replaces one engine per channel, engine.py:60-66,
 * cli.py:186-202, bench.py:200-202): for c in [0, channels):
 * y[c*ldy : c*ldy + ne+nh-1] = x[c*ldx : c*ldx+ne] (*) h[c*ldh : c*ldh+nh].
 * One launch of the FIR kernel.  float32; mode FAST, FFMA or TC. */
int sc_fir_batched(int dtype, int mode, const void *x, int64_t ldx, const void *h, int64_t ldh,
                   void *y, int64_t ldy, int64_t channels, int64_t ne, int64_t nh, void *stream);

/* Gather form with an exactly rounded accumulator: y[n] = math.fsum of the
 * individually rounded products e[m]*h[n-m] (direct_form, core.py:102-119),
 * bit-identical to CPython's fsum (Shewchuk partials + its half-even
 * fix-up).  float64 only.  `status` (device pointer to one unsigned, may be
 * NULL) receives bit 0 for an intermediate overflow of finite products and
 * bit 1 for -inf + inf -- the two cases where math.fsum raises
 * (OverflowError / ValueError) -- OR-ed in by the kernel. */
int sc_direct_form(const double *e, int64_t ne, const double *h, int64_t nh, double *y, unsigned *status,
                   void *stream);

/* ---------------------------------------------------------------- literal kernel */

/* Exact drop-in for _kernels.scatter_block (_kernels.py:14-52) on device
 * arrays: ring[cap] (the reference's physical ring layout, read_index),
 * ir[nh] (nh <= cap), block[n], out[n].  Mutates ring and out.
 * Synchronous (it returns the data-dependent `live` through live_out). */
int sc_scatter_block(int dtype, void *ring, int64_t cap, const void *ir, int64_t nh,
                     const void *block, int64_t n, void *out, int64_t read_index, int64_t live,
                     double threshold, int64_t *read_index_out, int64_t *live_out, void *stream);

/* ---------------------------------------------------------------- streaming engine */

/* Device-resident ScatterEngine (engine.py:60-214).  The residue (the
 * reference's ring in schedule order), the current and pending impulse
 * responses, read_index, live and cap all live in device memory; no call
 * below except _flush / _state / _schedule waits on the device. */
typedef struct sc_engine sc_engine;

/* engine.py:68-81 (+ EngineConfig block_size_nb / zero_skip_threshold).
 * h is a device pointer; it is copied. */
int sc_engine_create(int dtype, const void *h, int64_t nh, int64_t block_size_nb,
                     double threshold, void *stream, sc_engine **out);

/* C engines that advance together (one per channel -- the reference's
 * multichannel pattern, engine.py:60-66, cli.py:186-202 -- in one launch per
 * block).  h is [channels][nh] row-major.  Every
 * sample array of the calls below is then [channels][n] row-major, and the
 * per-channel outputs of _flush / _state / _schedule (n_tail, read_index,
 * live, cap, n_written) are arrays of `channels` entries; each channel keeps
 * its own live / cap / read_index.  channels = 1 is sc_engine_create. */
int sc_engine_create_multi(int dtype, const void *h, int64_t nh, int64_t channels,
                           int64_t block_size_nb, double threshold, void *stream, sc_engine **out);
int sc_engine_channels(sc_engine *e, int64_t *channels);
int sc_engine_destroy(sc_engine *e);
int sc_engine_set_stream(sc_engine *e, void *stream);

/* Kernel family: SC_MODE_ORDERED (default; bit-identical to block-by-block
 * calls and, in float64, to the reference) or SC_MODE_FAST.  float64 FAST:
 * every launch uses the fused-multiply-add chain (see SC_MODE_FAST above).
 * float32 FAST, fused streams (sc_engine_process_blocks): when the IR
 * segments of a call carry enough work (one batched launch for equal
 * segments from 2^28 MACs; otherwise >= 2^30 MACs per segment) over the
 * channels, each segment's convolution runs on the FAST FIR path (tensor
 * cores from 256 taps) and a combine kernel adds the segments and the
 * residue -- results within the FP32 tolerance, not bit-identical.  A single
 * block (sc_engine_process_block) with >= 2^30 MACs takes the same path;
 * smaller blocks and samples stay on the ordered chain. */
int sc_engine_set_mode(sc_engine *e, int mode);

/* process_block (engine.py:118-146): applies a pending swap first, then
 * consumes block[n] (n <= block_size_nb) and writes out[n].  Async. */
int sc_engine_process_block(sc_engine *e, const void *block, int64_t n, void *out);

/* process_sample (engine.py:99-116): like a 1-sample block but never applies
 * a pending swap.  Async; out is one device sample. */
int sc_engine_process_sample(sc_engine *e, const void *x, void *out);

/* swap_ir (engine.py:163-186): effective for the very next sample; residue
 * keeps its schedule; cap = max(nh_new, live) is computed on device. Async. */
int sc_engine_swap_ir(sc_engine *e, const void *h, int64_t nh);

/* swap_ir_at_next_block (engine.py:188-192).  Async (h is copied). */
int sc_engine_swap_ir_at_next_block(sc_engine *e, const void *h, int64_t nh);

/* Independent channels (engine.py:60-66: one ScatterEngine per channel, each
 * with its own IR, length and swap times).  h is [C][ldh] (device);
 * channel c swaps to its row's first nh_per_channel[c] taps when that is
 * >= 1 and keeps its IR otherwise (nh_per_channel is a HOST array of C
 * lengths).  Channels may then hold IRs of different lengths: every
 * channel's live / cap / read_index / tail length follows its own
 * (engine.py:163-192 per channel).  _at_next_block is the per-channel
 * pending swap (a uniform pending swap becomes per-channel, the named
 * channels replacing theirs). */
int sc_engine_swap_ir_channels(sc_engine *e, const void *h, int64_t ldh, const int64_t *nh_per_channel);
int sc_engine_swap_ir_at_next_block_channels(sc_engine *e, const void *h, int64_t ldh,
                                             const int64_t *nh_per_channel);
/* Host copy of every channel's current IR length (C values). */
int sc_engine_channel_nh(sc_engine *e, int64_t *nh_per_channel);

/* flush (engine.py:148-161): writes max(nh-1, live) tail samples in emission
 * order to tail (device, capacity tail_capacity; per channel for a
 * multichannel engine), returns the count(s) in n_tail and resets the engine
 * (pending swap survives).  Waits for the state read (the tail length is
 * data dependent); the tail itself is written asynchronously on the engine
 * stream. */
int sc_engine_flush(sc_engine *e, void *tail, int64_t tail_capacity, int64_t *n_tail);

/* Host-side upper bound of every channel's tail length (no synchronisation):
 * a tail_capacity that always suffices for sc_engine_flush. */
int sc_engine_tail_bound(sc_engine *e, int64_t *bound);

/* flush (engine.py:148-161) split in two so that all of its device work is
 * queued before its only host wait: _begin enqueues the tail copy (the
 * sc_engine_tail_bound prefix of the schedule; samples past a channel's tail
 * are zero), the state read-back into pinned memory and the reset; _end
 * waits for the stream and returns each channel's tail length
 * max(len(ir) - 1, live).  tail_capacity must be >= sc_engine_tail_bound.
 * No other engine call may come between the two. */
int sc_engine_flush_begin(sc_engine *e, void *tail, int64_t tail_capacity);
int sc_engine_flush_end(sc_engine *e, int64_t *n_tail);

/* State (engine.py:83-97): read_index, live, cap (= len(ring)), consumed,
 * current nh, has_pending.  Synchronous. */
int sc_engine_state(sc_engine *e, int64_t *read_index, int64_t *live, int64_t *cap,
                    int64_t *consumed, int64_t *nh, int *has_pending);

/* Residue in schedule order (_schedule_order, engine.py:211-214): copies
 * min(n, cap) samples to dst (device).  Synchronous. */
int sc_engine_schedule(sc_engine *e, void *dst, int64_t n, int64_t *n_written);

/* Current impulse response (engine.py:91-93) copied to dst (device, nh). Async. */
int sc_engine_current_ir(sc_engine *e, void *dst, int64_t capacity, int64_t *nh);

/* Back-to-back blocks with no host synchronisation (render, engine.py:194-209,
 * plus an IR swap schedule): x[n_total] is cut into blocks of nb; before block
 * b = swap_blocks[i] the engine performs swap_ir(swap_irs[i], swap_nh[i]).
 * Bit-identical to the equivalent sequence of process_block/swap_ir calls.
 * A call repeated with the same arguments, buffers and engine host state is
 * captured as a CUDA graph on its second occurrence and replayed from then
 * on (same kernels, same arguments; SC_ENGINE_GRAPHS=0 disables). */
int sc_engine_process_blocks(sc_engine *e, const void *x, int64_t n_total, int64_t nb,
                             const int64_t *swap_blocks, const void *const *swap_irs,
                             const int64_t *swap_nh, int64_t n_swaps, void *out);

/* Graph-replay bookkeeping of sc_engine_process_blocks: replays, captures,
 * and captures that failed (those keys then always run directly). */
int sc_engine_graph_stats(sc_engine *e, int64_t *hits, int64_t *captures, int64_t *failures);

/* process_blocks with a per-channel swap schedule: before block
 * swap_blocks[i], channel c swaps to row c of swap_irs[i] ([C][swap_ld[i]],
 * swap_ld may be NULL = the longest length of that swap) with length
 * swap_nh[i*C + c], or keeps its IR when that is <= 0.  Blocks run one
 * launch each (one engine per channel semantics; bit-identical to the
 * equivalent sequence of per-channel swaps and process_block calls). */
int sc_engine_process_blocks_channels(sc_engine *e, const void *x, int64_t n_total, int64_t nb,
                                      const int64_t *swap_blocks, const void *const *swap_irs,
                                      const int64_t *swap_ld, const int64_t *swap_nh, int64_t n_swaps, void *out);

/* The same with x[C][n_total] and out[C][n_total] in HOST memory (pinned for
 * full PCIe rate; swap IRs on the device).  The stream is processed in
 * `chunks` runs of whole blocks (0 = automatic: 2..4 by size) whose uploads,
 * blocks and downloads overlap on three streams; the engine state, and in
 * ORDERED mode the results bit for bit, are those of one
 * sc_engine_process_blocks call (FAST: within the FP32 tolerance).  Synchronous: out is filled on
 * return.  (No reference counterpart: render, engine.py:194-209, over a host
 * signal, with the transfers hidden behind the blocks.) */
int sc_engine_process_blocks_host(sc_engine *e, const void *x_host, int64_t n_total, int64_t nb,
                                  const int64_t *swap_blocks, const void *const *swap_irs,
                                  const int64_t *swap_nh, int64_t n_swaps, void *out_host, int chunks);

/* ---------------------------------------------------------------- multi-GPU */

/* Outputs [n_begin, n_end) of the convolution of a HOST signal x[ne] with
 * h[nh] (host, or a device pointer on `device`), computed on `device` and
 * written to the host buffer y_host[n_end - n_begin].  Only inputs
 * [max(0, n_begin-nh+1), min(ne, n_end)) are uploaded (the range's slice plus
 * its halo).  The range is cut into `chunks` output chunks (0 = by size:
 * one per >= 2^36 MACs or 16 MiB of input, 2..12) whose upload, FIR and
 * download run on three persistent streams, so transfers in both directions
 * overlap the kernels of neighbouring chunks; device buffers persist across
 * calls.  Pinned x_host / y_host overlap fully; pageable ones are correct
 * but serialise.  Synchronous.  mode as sc_fir_full.  The host-I/O leg of
 * scatter_convolve (core.py:122-131) on one GPU, and one rank's shard in
 * the time-sharded multi-GPU path. */
int sc_fir_range_host(int dtype, int mode, const void *x_host, int64_t ne, const void *h, int64_t nh,
                      void *y_host, int64_t n_begin, int64_t n_end, int device, int chunks);

/* Whole-signal convolution of a HOST signal x[ne] with h[nh] (host),
 * partitioned by output time segment over ngpu devices (devices[]; repeats
 * allowed): device g computes outputs [a_g, b_g) from its input slice plus
 * the (nh-1)-sample halo -- no MAC repeated, no partial sums exchanged, no
 * reduction (SURVEY.md 8(b) sc_fir_sharded, north_star (4)).  Each device
 * runs the chunk-pipelined range engine of sc_fir_range_host on its own host
 * thread.  y[ne+nh-1] is a host pointer when gather_device < 0; else a
 * device pointer on gather_device that the FIR epilogues store into directly
 * (peer stores over NVLink; peer copies when peer access is unavailable).
 * Synchronous.  mode as sc_fir_full; ORDERED float64 stays bit-identical to
 * the reference at any device count (every output's chain runs on one
 * device). */
int sc_fir_sharded(int dtype, int mode, const void *x_host, int64_t ne, const void *h_host, int64_t nh, void *y,
                   int ngpu, const int *devices, int gather_device);

/* ---------------------------------------------------------------- WAV on device */

/* SURVEY.md 8(f) row 3.  encoding: 0 pcm16, 1 pcm24, 2 float32 (the three
 * encodings of wavio.py).  Decode the raw interleaved data-chunk bytes
 * (device) into out[channels][frames] (wavio.py:118-130: PCM / 2^(bits-1)). */
int sc_wav_decode(int encoding, const void *raw, int64_t frames, int64_t channels, int out_dtype,
                  void *out, void *stream);

/* Encode in[channels][ld] * gain into interleaved bytes (device); integer PCM
 * rounds half-to-even and saturates, adding the number of clipped samples to
 * *clipped (a device counter) -- wavio.py:133-198 semantics. */
int sc_wav_encode(int encoding, int in_dtype, const void *in, int64_t ld, int64_t frames,
                  int64_t channels, double gain, void *raw, unsigned long long *clipped, void *stream);

/* max |x| over n samples into *peak_bits (device; the float64 bit pattern,
 * initialise to 0) -- the --normalize peak of cli.py:204-210. */
int sc_peak_abs(int dtype, const void *x, int64_t n, unsigned long long *peak_bits, void *stream);

/* ---------------------------------------------------------------- fixed point */

/* bit-true fixed-point simulation (quantize.py).
 * Quantise n float64 samples (device) to a word_bits two's-complement
 * fractional grid: k = clamp(rint(x * 2^(word_bits-1))), NaN -> INT64_MIN
 * (quantize.py:137-143).  xq (optional) receives k / 2^(word_bits-1)
 * (quantize.py:146-147).  stats[0] += samples outside [-1, 1) (the caller
 * raises ValueError), stats[1] = max(stats[1], max |k|); both device
 * counters, initialise to 0.  word_bits in [2, 64]. */
int sc_fixed_quantize(const double *x, int64_t n, int word_bits, int64_t *k, double *xq,
                      unsigned long long *stats, void *stream);

/* t[i] / 2^shift rounded to nearest, ties to even, for int64 device arrays
 * (0 <= shift <= 63) -- replaces the scalar helper _round_shift_half_even,
 * quantize.py:145-154 (the requantisation step of both schemes). */
int sc_fixed_round_shift(const int64_t *t, int64_t n, int shift, int64_t *out, void *stream);

/* Exact-integer convolution of quantised ke[ne], kh[nh] (device) under one
 * requantisation scheme (0 "ideal": one half-even rounding per output;
 * 1 "mac": rounding after every multiply-accumulate), y[ne+nh-1] = result /
 * 2^(word_bits-1) in float64 -- fixed_point_convolve, quantize.py:163-195.
 * Intermediates are __int128; the caller guarantees bitlen(max|ke|) +
 * bitlen(max|kh|) + ceil(log2(min(ne, nh))) <= 126.  wide != 0 selects
 * 64x64->128 products (needed once max|k| > 2^31). */
int sc_fixed_convolve(const int64_t *ke, int64_t ne, const int64_t *kh, int64_t nh, int word_bits, int scheme,
                      int wide, double *y, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SCATTERCONV_B200_H */
