/*
 * scatter_oracle.c -- CPU restatement of the reference's convolution arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the
 * `cpu_baseline` / `--impl reference` arm of bench.py).  Nothing in the
 * product package `paper_2401_01607_b200` links, loads or calls it; the
 * product path is the CUDA library under paper_2401_01607_b200/csrc.
 *
 * Pinned against the reference package itself: tests/golden/make_golden.py
 * imports /root/reference/pkg/src/scatterconv in the build container and
 * writes fixtures; tests/test_oracle_golden.py checks this file reproduces
 * them bit-for-bit.
 *
 * Every function cites the reference code it restates.  Arithmetic is plain
 * IEEE binary64, multiply then add as two separately rounded operations.  The
 * Makefile compiles with -O2 -ffp-contract=off -fno-fast-math so gcc never
 * fuses or reassociates, matching numba's strict default
 * (pkg/src/scatterconv/_kernels.py:1-8).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------
 * scatter_block -- pkg/src/scatterconv/_kernels.py:14-52
 *
 * Per input sample x (in order): when |x| > threshold scatter x*ir[i] into
 * ring slot (ri+i) mod cap, split into a head run and a wrapped run
 * (:34-42); raise live to nh (:43-44).  Then for every sample emit
 * ring[ri], zero it, advance ri mod cap and decrement live (:45-51).
 * NaN input is skipped because !(|NaN| > thr).  Returns through the out
 * pointers the updated (read_index, live) (:52).
 * ---------------------------------------------------------------------- */
void oracle_scatter_block(double *ring, int64_t cap, const double *ir, int64_t nh,
                          const double *block, int64_t n, double *out,
                          int64_t read_index, int64_t live, double threshold,
                          int64_t *read_index_out, int64_t *live_out)
{
    int64_t ri = read_index;
    for (int64_t s = 0; s < n; ++s) {
        const double x = block[s];
        if (fabs(x) > threshold) {
            const int64_t head = cap - ri;
            if (nh <= head) {
                double *dst = ring + ri;
                for (int64_t i = 0; i < nh; ++i) {
                    const double p = x * ir[i];
                    dst[i] = dst[i] + p;
                }
            } else {
                double *dst = ring + ri;
                for (int64_t i = 0; i < head; ++i) {
                    const double p = x * ir[i];
                    dst[i] = dst[i] + p;
                }
                const double *ir2 = ir + head;
                for (int64_t i = 0; i < nh - head; ++i) {
                    const double p = x * ir2[i];
                    ring[i] = ring[i] + p;
                }
            }
            if (live < nh) live = nh;
        }
        out[s] = ring[ri];
        ring[ri] = 0.0;
        ri += 1;
        if (ri == cap) ri = 0;
        if (live > 0) live -= 1;
    }
    *read_index_out = ri;
    *live_out = live;
}

/* ------------------------------------------------------------------------
 * _scatter_full -- pkg/src/scatterconv/core.py:80-92
 *
 * out = zeros(nd+nk-1); for each drive sample n (ascending), out[n:n+nk] +=
 * x * kern.  Every slot therefore accumulates its products in increasing
 * drive index, starting from +0.0.  skip_mode:
 *   0  no skipping                         (core.py:90-91, scatter_convolve)
 *   1  skip when |x| <= threshold          (core.py:163-165, skip_zeros; NaN
 *                                           is NOT skipped there)
 *   2  skip unless |x| > threshold         (_kernels.py:33, engine rule;
 *                                           NaN IS skipped)
 * ---------------------------------------------------------------------- */
void oracle_scatter_full(const double *drive, int64_t nd, const double *kern, int64_t nk,
                         double *out, int skip_mode, double threshold)
{
    const int64_t nout = nd + nk - 1;
    for (int64_t i = 0; i < nout; ++i) out[i] = 0.0;
    for (int64_t n = 0; n < nd; ++n) {
        const double x = drive[n];
        if (skip_mode == 1 && fabs(x) <= threshold) continue;
        if (skip_mode == 2 && !(fabs(x) > threshold)) continue;
        double *dst = out + n;
        for (int64_t i = 0; i < nk; ++i) {
            const double p = x * kern[i];
            dst[i] = dst[i] + p;
        }
    }
}

/* ------------------------------------------------------------------------
 * Exactly rounded sum -- the math.fsum used by direct_form
 * (pkg/src/scatterconv/core.py:115-118).  Restates the published
 * Shewchuk "partials" algorithm with the half-even fix-up across partials
 * that CPython's fsum applies, so the result is the correctly rounded sum of
 * the (individually rounded) products.  Non-finite handling: NaN/Inf
 * summands short-circuit to their IEEE sum (CPython raises on inf-inf; we
 * return NaN there).
 * ---------------------------------------------------------------------- */
typedef struct {
    double *p;
    int64_t n, cap;
    double special, inf_sum;
} fsum_state;

static void fsum_init(fsum_state *s, double *buf, int64_t cap)
{
    s->p = buf;
    s->n = 0;
    s->cap = cap;
    s->special = 0.0;
    s->inf_sum = 0.0;
}

static void fsum_add(fsum_state *s, double x)
{
    const double xsave = x;
    int64_t i = 0;
    for (int64_t j = 0; j < s->n; ++j) {
        double y = s->p[j];
        if (fabs(x) < fabs(y)) {
            const double t = x;
            x = y;
            y = t;
        }
        const double hi = x + y;
        const double yr = hi - x;
        const double lo = y - yr;
        if (lo != 0.0) s->p[i++] = lo;
        x = hi;
    }
    s->n = i;
    if (x != 0.0) {
        if (!isfinite(x)) {
            if (isinf(xsave)) s->inf_sum += xsave;
            s->special += xsave;
            s->n = 0;
        } else {
            s->p[s->n++] = x; /* cap is >= number of terms + 1 */
        }
    }
}

static double fsum_result(fsum_state *s)
{
    if (s->special != 0.0 || isnan(s->special)) {
        if (isnan(s->inf_sum)) return NAN;
        return s->special;
    }
    double hi = 0.0, lo = 0.0;
    int64_t n = s->n;
    if (n > 0) {
        hi = s->p[--n];
        while (n > 0) {
            const double x = hi;
            const double y = s->p[--n];
            hi = x + y;
            const double yr = hi - x;
            lo = y - yr;
            if (lo != 0.0) break;
        }
        if (n > 0 && ((lo < 0.0 && s->p[n - 1] < 0.0) || (lo > 0.0 && s->p[n - 1] > 0.0))) {
            const double y = lo * 2.0;
            const double x = hi + y;
            const double yr = x - hi;
            if (y == yr) hi = x;
        }
    }
    return hi;
}

/* direct_form -- pkg/src/scatterconv/core.py:102-119: gather form, each output
 * n is fsum(e[m]*h[n-m] for m in [max(0,n-nh+1), min(n,ne-1)]).  Computes
 * outputs [n_begin, n_end) only (spot windows for very long filters). */
void oracle_direct_form(const double *e, int64_t ne, const double *h, int64_t nh,
                        double *out, int64_t n_begin, int64_t n_end)
{
    const int64_t maxterms = (ne < nh ? ne : nh) + 2;
    double *buf = (double *)malloc(sizeof(double) * (size_t)maxterms);
    for (int64_t n = n_begin; n < n_end; ++n) {
        fsum_state s;
        fsum_init(&s, buf, maxterms);
        const int64_t lo = n - nh + 1 > 0 ? n - nh + 1 : 0;
        const int64_t hi = n < ne - 1 ? n : ne - 1;
        for (int64_t m = lo; m <= hi; ++m) fsum_add(&s, e[m] * h[n - m]);
        out[n - n_begin] = fsum_result(&s);
    }
    free(buf);
}

/* ------------------------------------------------------------------------
 * Parallel engine driver (CPU baseline and large-config oracle).
 *
 * The reference parallelises only by running independent engines on
 * separate threads (engine.py:60-66; bench.py:200-202, relying on the
 * nogil kernel).  For one long signal we run one engine per contiguous
 * input segment, each exactly as engine.render + flush does (engine.py:
 * 118-161, 194-209: blocks of nb through scatter_block, then the ring in
 * schedule order), and overlap-add the segment outputs at their offsets
 * (linearity).  Per segment the arithmetic is the reference's; the
 * cross-segment add changes summation order at the 1e-16 relative level.
 * ---------------------------------------------------------------------- */
typedef struct {
    const double *x;
    int64_t a, b; /* input segment [a, b) */
    const double *h;
    int64_t nh, nb;
    double *seg_out; /* (b-a)+nh-1 */
} seg_job;

static void run_engine_segment(const seg_job *j)
{
    const int64_t nh = j->nh, len = j->b - j->a;
    double *ring = (double *)calloc((size_t)nh, sizeof(double));
    int64_t ri = 0, live = 0;
    for (int64_t s = 0; s < len; s += j->nb) {
        const int64_t n = (len - s) < j->nb ? (len - s) : j->nb;
        oracle_scatter_block(ring, nh, j->h, nh, j->x + j->a + s, n, j->seg_out + s, ri, live,
                             0.0, &ri, &live);
    }
    /* flush: schedule order ring[ri:] + ring[:ri], first nh-1 (engine.py:148-161) */
    double *tail = j->seg_out + len;
    int64_t k = 0;
    for (int64_t i = ri; i < nh && k < nh - 1; ++i) tail[k++] = ring[i];
    for (int64_t i = 0; i < ri && k < nh - 1; ++i) tail[k++] = ring[i];
    free(ring);
}

static void *seg_thread(void *arg)
{
    run_engine_segment((const seg_job *)arg);
    return NULL;
}

/* y[0:ne+nh-1] = conv(x, h) with n_threads engines over input segments.
 * Returns 0 on success. */
int oracle_conv_parallel(const double *x, int64_t ne, const double *h, int64_t nh,
                         double *y, int64_t nb, int n_threads)
{
    if (n_threads < 1) n_threads = 1;
    if (n_threads > ne) n_threads = (int)ne;
    seg_job *jobs = (seg_job *)calloc((size_t)n_threads, sizeof(seg_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    const int64_t per = (ne + n_threads - 1) / n_threads;
    int used = 0;
    for (int t = 0; t < n_threads; ++t) {
        const int64_t a = (int64_t)t * per;
        if (a >= ne) break;
        const int64_t b = a + per < ne ? a + per : ne;
        jobs[t].x = x;
        jobs[t].a = a;
        jobs[t].b = b;
        jobs[t].h = h;
        jobs[t].nh = nh;
        jobs[t].nb = nb;
        jobs[t].seg_out = (double *)malloc(sizeof(double) * (size_t)(b - a + nh - 1));
        used++;
    }
    for (int t = 1; t < used; ++t) pthread_create(&th[t], NULL, seg_thread, &jobs[t]);
    run_engine_segment(&jobs[0]);
    for (int t = 1; t < used; ++t) pthread_join(th[t], NULL);
    const int64_t nout = ne + nh - 1;
    for (int64_t i = 0; i < nout; ++i) y[i] = 0.0;
    for (int t = 0; t < used; ++t) {
        const int64_t len = jobs[t].b - jobs[t].a + nh - 1;
        double *dst = y + jobs[t].a;
        for (int64_t i = 0; i < len; ++i) dst[i] = dst[i] + jobs[t].seg_out[i];
        free(jobs[t].seg_out);
    }
    free(jobs);
    free(th);
    return 0;
}

/* Many independent channels, one engine each, spread over n_threads
 * (the reference's one-engine-per-channel pattern, engine.py:60-66). */
typedef struct {
    const double *x;
    const double *h;
    double *y;
    int64_t channels, ne, nh, nb;
    int64_t next;
    pthread_mutex_t mu;
} chan_pool;

static void *chan_thread(void *arg)
{
    chan_pool *p = (chan_pool *)arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        const int64_t c = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (c >= p->channels) break;
        seg_job j;
        j.x = p->x + c * p->ne;
        j.a = 0;
        j.b = p->ne;
        j.h = p->h + c * p->nh;
        j.nh = p->nh;
        j.nb = p->nb;
        j.seg_out = p->y + c * (p->ne + p->nh - 1);
        run_engine_segment(&j);
    }
    return NULL;
}

int oracle_conv_channels(const double *x, const double *h, double *y, int64_t channels,
                         int64_t ne, int64_t nh, int64_t nb, int n_threads)
{
    chan_pool p;
    p.x = x;
    p.h = h;
    p.y = y;
    p.channels = channels;
    p.ne = ne;
    p.nh = nh;
    p.nb = nb;
    p.next = 0;
    pthread_mutex_init(&p.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    for (int t = 1; t < n_threads; ++t) pthread_create(&th[t], NULL, chan_thread, &p);
    chan_thread(&p);
    for (int t = 1; t < n_threads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&p.mu);
    return 0;
}

/* ------------------------------------------------------------------------
 * Output window of _scatter_full -- core.py:80-92 restricted to outputs
 * [n_begin, n_end): for each drive sample m in ascending order add x*kern
 * into the window slots it reaches.  Every slot sees exactly the reference's
 * chain (ascending m, mul then add), so the window is bit-identical to the
 * same slots of the full reference result.  Threads split the WINDOW (never a
 * slot's chain).  skip_mode as in oracle_scatter_full.
 * ---------------------------------------------------------------------- */
typedef struct {
    const double *x;
    int64_t ne;
    const double *h;
    int64_t nh;
    double *out;
    int64_t n_begin, n_end;
    int skip_mode;
    double threshold;
} win_job;

static void run_window(const win_job *w)
{
    for (int64_t n = w->n_begin; n < w->n_end; ++n) w->out[n - w->n_begin] = 0.0;
    int64_t m_lo = w->n_begin - w->nh + 1;
    if (m_lo < 0) m_lo = 0;
    int64_t m_hi = w->n_end - 1;
    if (m_hi > w->ne - 1) m_hi = w->ne - 1;
    for (int64_t m = m_lo; m <= m_hi; ++m) {
        const double x = w->x[m];
        if (w->skip_mode == 1 && fabs(x) <= w->threshold) continue;
        if (w->skip_mode == 2 && !(fabs(x) > w->threshold)) continue;
        int64_t a = m > w->n_begin ? m : w->n_begin;           /* slots n in [a, b) */
        int64_t b = m + w->nh < w->n_end ? m + w->nh : w->n_end;
        double *dst = w->out - w->n_begin;
        const double *hk = w->h - m;
        for (int64_t n = a; n < b; ++n) {
            const double p = x * hk[n];
            dst[n] = dst[n] + p;
        }
    }
}

static void *win_thread(void *arg)
{
    run_window((const win_job *)arg);
    return NULL;
}

void oracle_scatter_window(const double *x, int64_t ne, const double *h, int64_t nh, double *out,
                           int64_t n_begin, int64_t n_end, int skip_mode, double threshold,
                           int n_threads)
{
    const int64_t len = n_end - n_begin;
    if (len <= 0) return;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > len) n_threads = (int)len;
    win_job *jobs = (win_job *)calloc((size_t)n_threads, sizeof(win_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    const int64_t per = (len + n_threads - 1) / n_threads;
    int used = 0;
    for (int t = 0; t < n_threads; ++t) {
        const int64_t a = n_begin + (int64_t)t * per;
        if (a >= n_end) break;
        const int64_t b = a + per < n_end ? a + per : n_end;
        jobs[t] = (win_job){x, ne, h, nh, out + (a - n_begin), a, b, skip_mode, threshold};
        used++;
    }
    for (int t = 1; t < used; ++t) pthread_create(&th[t], NULL, win_thread, &jobs[t]);
    run_window(&jobs[0]);
    for (int t = 1; t < used; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

/* ------------------------------------------------------------------ fixed point
 * Bit-true fixed-point simulation, restating quantize.py:137-195.  Samples
 * quantise to k = clamp(round_half_even(x * 2^frac)), NaN -> INT64_MIN (what
 * numpy's float->int64 cast gives on x86).  Convolution is exact in __int128;
 * "ideal" (scheme 0) rounds the exact sum once, "mac" (scheme 1) rounds after
 * every multiply-accumulate with the first product kept exact until it joins
 * the second.  Valid while every intermediate fits 127 bits (the callers'
 * word lengths are <= 32 bits). */

int64_t oracle_fixed_quantize(const double *x, int64_t n, int frac, int64_t *k)
{
    const double scale = ldexp(1.0, frac);
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double v = x[i];
        if (v < -1.0 || v >= 1.0) bad++;
        if (isnan(v)) {
            k[i] = INT64_MIN;
            continue;
        }
        double r = nearbyint(v * scale); /* default rounding mode: half to even */
        if (r < -scale) r = -scale;
        if (r > scale - 1.0) r = scale - 1.0;
        k[i] = (int64_t)r;
    }
    return bad;
}

static __int128 rshe(__int128 t, int s)
{
    const __int128 q = t >> s;
    const unsigned __int128 r = (unsigned __int128)t & (((unsigned __int128)1 << s) - 1);
    const unsigned __int128 half = (unsigned __int128)1 << (s - 1);
    return q + ((r > half || (r == half && (q & 1))) ? 1 : 0);
}

void oracle_fixed_conv(const int64_t *ke, int64_t ne, const int64_t *kh, int64_t nh, int frac, int scheme,
                       double *out)
{
    for (int64_t n = 0; n < ne + nh - 1; ++n) {
        const int64_t lo = n - nh + 1 > 0 ? n - nh + 1 : 0;
        const int64_t hi = n < ne - 1 ? n : ne - 1;
        __int128 c;
        if (scheme == 0) {
            __int128 acc = 0;
            for (int64_t m = lo; m <= hi; ++m) acc += (__int128)ke[m] * kh[n - m];
            c = rshe(acc, frac);
        } else if (lo == hi) {
            c = rshe((__int128)ke[lo] * kh[n - lo], frac);
        } else {
            c = rshe((__int128)ke[lo] * kh[n - lo] + (__int128)ke[lo + 1] * kh[n - lo - 1], frac);
            for (int64_t m = lo + 2; m <= hi; ++m)
                c = rshe((__int128)((unsigned __int128)c << frac) + (__int128)ke[m] * kh[n - m], frac);
        }
        out[n] = ldexp((double)c, -frac); /* libgcc int128->double rounds to nearest */
    }
}
