// k_fixed.cu -- bit-true fixed-point FIR simulation on the device (SURVEY.md
// 8(f) row 4).
//
// The reference runs this in pure Python with unbounded integers
// (pkg/src/scatterconv/quantize.py:137-147 quantisation, :150-160 the
// half-even right shift, :163-195 the two requantisation schemes).  Here:
//   * k_fixed_quantize: one thread per sample -- x*2^frac (exact), rint
//     (round half to even), saturate to [-2^frac, 2^frac-1]; counts samples
//     outside [-1, 1) (the host raises the reference's ValueError) and keeps
//     max|k| so the host can prove the 128-bit accumulator is wide enough.
//     NaN maps to INT64_MIN, which is what numpy's float->int64 cast yields
//     on x86 for the reference.
//   * k_fixed_conv<SCHEME, WIDE>: one thread per output sample n walking
//     m = lo..hi in the reference's order.  Products are exact (int64 when
//     both operands fit 32 bits, else 64x64->128); the "ideal" accumulator and
//     the "mac" running value live in __int128, so every intermediate the
//     Python reference forms is represented exactly as long as
//     bitlen(max|ke|) + bitlen(max|kh|) + ceil(log2(terms)) <= 126, which the
//     host checks before launching.  Output = correctly rounded
//     int128 -> double, then an exact scale by 2^-frac (Python's int / int).
// Warp lanes take consecutive n, so ke[m] is a broadcast and kh[n-m] a
// coalesced (reversed) read; both inputs stay L1/L2 resident.

#include <algorithm>
#include <cstdint>

#include "sc_common.cuh"

namespace sc {
namespace {

typedef __int128 i128;
typedef unsigned __int128 u128;

__global__ void k_fixed_quantize(const double *__restrict__ x, int64_t n, int frac, int64_t *__restrict__ k,
                                 double *__restrict__ xq, unsigned long long *__restrict__ stats) {
    // stats[0] = samples outside [-1, 1), stats[1] = max |k| (as unsigned)
    const double scale = ldexp(1.0, frac);
    unsigned long long bad = 0, mx = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        bad += (v < -1.0 || v >= 1.0) ? 1ull : 0ull;
        int64_t q;
        if (v != v) {
            q = INT64_MIN;
        } else {
            double r = rint(__dmul_rn(v, scale));
            r = r < -scale ? -scale : (r > scale - 1.0 ? scale - 1.0 : r);
            q = (int64_t)r;
        }
        k[i] = q;
        if (xq) xq[i] = __dmul_rn(__ll2double_rn(q), ldexp(1.0, -frac));  // numpy: k / scale
        const unsigned long long a = q < 0 ? 0ull - (unsigned long long)q : (unsigned long long)q;
        mx = a > mx ? a : mx;
    }
    for (int o = 16; o; o >>= 1) {
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = t > mx ? t : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicAdd(&stats[0], bad);
        atomicMax(&stats[1], mx);
    }
}

// t / 2^s rounded to nearest, ties to even (quantize.py:150-160); s >= 1.
__device__ __forceinline__ i128 rshift_half_even(i128 t, int s) {
    const i128 q = t >> s;  // arithmetic: floor for negatives too
    const u128 r = (u128)t & (((u128)1 << s) - 1);
    const u128 half = (u128)1 << (s - 1);
    return q + ((r > half || (r == half && (q & 1))) ? 1 : 0);
}

// Correctly rounded (nearest-even) int128 -> double, times 2^-frac.
__device__ __forceinline__ double i128_to_double_scaled(i128 v, int frac) {
    const bool neg = v < 0;
    u128 u = neg ? (u128)0 - (u128)v : (u128)v;
    double d;
    if ((u >> 53) == 0) {
        d = (double)(unsigned long long)u;
    } else {
        const unsigned long long hi = (unsigned long long)(u >> 64);
        const int bits = hi ? 128 - __clzll((long long)hi) : 64 - __clzll((long long)(unsigned long long)u);
        const int sh = bits - 53;
        u128 q = u >> sh;
        const u128 r = u & (((u128)1 << sh) - 1);
        const u128 half = (u128)1 << (sh - 1);
        if (r > half || (r == half && (q & 1))) q += 1;
        d = ldexp((double)(unsigned long long)q, sh);
    }
    d = ldexp(d, -frac);
    return neg ? -d : d;
}

template <bool WIDE>
__device__ __forceinline__ i128 prod(int64_t a, int64_t b) {
    if (WIDE) return (i128)a * (i128)b;
    return (i128)(a * b);  // |a|,|b| <= 2^31: exact in int64
}

template <int SCHEME, bool WIDE>  // SCHEME 0 = ideal, 1 = mac
__global__ void __launch_bounds__(256) k_fixed_conv(const int64_t *__restrict__ ke, int64_t ne,
                                                    const int64_t *__restrict__ kh, int64_t nh, int frac,
                                                    double *__restrict__ y) {
    const int64_t total = ne + nh - 1;
    for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < total;
         n += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = n - nh + 1 > 0 ? n - nh + 1 : 0;
        const int64_t hi = n < ne - 1 ? n : ne - 1;
        i128 c;
        if (SCHEME == 0) {
            i128 acc = 0;
            for (int64_t m = lo; m <= hi; ++m) acc += prod<WIDE>(ke[m], kh[n - m]);
            c = rshift_half_even(acc, frac);
        } else {
            // the first product joins the second before its first rounding;
            // a lone product is only store-rounded (quantize.py:184-192)
            const i128 fine = prod<WIDE>(ke[lo], kh[n - lo]);
            if (lo == hi) {
                c = rshift_half_even(fine, frac);
            } else {
                c = rshift_half_even(fine + prod<WIDE>(ke[lo + 1], kh[n - lo - 1]), frac);
                for (int64_t m = lo + 2; m <= hi; ++m)
                    c = rshift_half_even((i128)((u128)c << frac) + prod<WIDE>(ke[m], kh[n - m]), frac);
            }
        }
        y[n] = i128_to_double_scaled(c, frac);
    }
}

// Element-wise t / 2^s, half-even (the scalar helper _round_shift_half_even,
// quantize.py:145-154), through the same rshift_half_even the schemes use.
__global__ void k_round_shift(const int64_t *__restrict__ t, int64_t n, int s, int64_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = s == 0 ? t[i] : (int64_t)rshift_half_even((i128)t[i], s);
}

}  // namespace
}  // namespace sc

using namespace sc;

extern "C" {

int sc_fixed_quantize(const double *x, int64_t n, int word_bits, int64_t *k, double *xq,
                      unsigned long long *stats, void *stream) {
    SC_REQUIRE(word_bits >= 2 && word_bits <= 64, "word_bits must be in [2, 64] on the device, got %d", word_bits);
    SC_REQUIRE(n >= 0 && stats, "sc_fixed_quantize: bad arguments");
    if (n == 0) return SC_OK;
    SC_REQUIRE(x && k, "sc_fixed_quantize: null pointer");
    const unsigned g = (unsigned)std::min<int64_t>(cdiv(n, 256), 4 * (int64_t)sm_count());
    k_fixed_quantize<<<g, 256, 0, as_stream(stream)>>>(x, n, word_bits - 1, k, xq, stats);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

int sc_fixed_round_shift(const int64_t *t, int64_t n, int shift, int64_t *out, void *stream) {
    SC_REQUIRE(shift >= 0 && shift <= 63, "shift must be in [0, 63], got %d", shift);
    SC_REQUIRE(n >= 0, "sc_fixed_round_shift: bad arguments");
    if (n == 0) return SC_OK;
    SC_REQUIRE(t && out, "sc_fixed_round_shift: null pointer");
    const unsigned g = (unsigned)std::min<int64_t>(cdiv(n, 256), 4 * (int64_t)sm_count());
    k_round_shift<<<g, 256, 0, as_stream(stream)>>>(t, n, shift, out);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

int sc_fixed_convolve(const int64_t *ke, int64_t ne, const int64_t *kh, int64_t nh, int word_bits, int scheme,
                      int wide, double *y, void *stream) {
    SC_REQUIRE(word_bits >= 2 && word_bits <= 64, "word_bits must be in [2, 64] on the device, got %d", word_bits);
    SC_REQUIRE(scheme == 0 || scheme == 1, "scheme must be 0 (ideal) or 1 (mac), got %d", scheme);
    SC_REQUIRE(ne > 0 && nh > 0 && ke && kh && y, "sc_fixed_convolve: empty signal or null pointer");
    const int frac = word_bits - 1;
    const int64_t total = ne + nh - 1;
    const unsigned g = (unsigned)std::min<int64_t>(cdiv(total, 256), 16 * (int64_t)sm_count());
    cudaStream_t s = as_stream(stream);
    if (scheme == 0) {
        if (wide) k_fixed_conv<0, true><<<g, 256, 0, s>>>(ke, ne, kh, nh, frac, y);
        else k_fixed_conv<0, false><<<g, 256, 0, s>>>(ke, ne, kh, nh, frac, y);
    } else {
        if (wide) k_fixed_conv<1, true><<<g, 256, 0, s>>>(ke, ne, kh, nh, frac, y);
        else k_fixed_conv<1, false><<<g, 256, 0, s>>>(ke, ne, kh, nh, frac, y);
    }
    SC_CHECK_LAUNCH();
    return SC_OK;
}

}  // extern "C"
