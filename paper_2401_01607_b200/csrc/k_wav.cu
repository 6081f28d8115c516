// k_wav.cu -- WAV sample codecs and reductions on the device (SURVEY.md 8(f)
// row 3: "WAV -> device pipeline").
//
// The reference decodes and encodes on the host with numpy
// (pkg/src/scatterconv/wavio.py:118-130 decoders, :133-198 writer) and
// normalises with a host max (cli.py:204-210).  Here the raw interleaved
// bytes of the data chunk are uploaded once and de-interleaved/decoded by a
// kernel straight into the [channels][frames] layout the multichannel engine
// consumes; encoding (gain, round-half-even, saturation, clip counting) and
// the peak for --normalize are device kernels too.  Arithmetic matches the
// reference bit for bit: integer PCM / 2^(bits-1) in float64, rint() for
// numpy's round-half-even, v = y*gain as one float64 multiply.

#include <algorithm>
#include <cstdint>

#include "sc_common.cuh"

namespace sc {
namespace {

enum { ENC_PCM16 = 0, ENC_PCM24 = 1, ENC_F32 = 2 };

__device__ __forceinline__ double decode_one(const uint8_t *p, int enc) {
    if (enc == ENC_PCM16) {
        const int16_t v = (int16_t)((uint16_t)p[0] | ((uint16_t)p[1] << 8));
        return (double)v / 32768.0;
    }
    if (enc == ENC_PCM24) {
        int32_t v = (int32_t)p[0] | ((int32_t)p[1] << 8) | ((int32_t)p[2] << 16);
        v -= (v & 0x800000) << 1;  // sign-extend bit 23
        return (double)v / (double)(1 << 23);
    }
    uint32_t u = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    return (double)__uint_as_float(u);
}

template <typename T>
__global__ void k_wav_decode(const uint8_t *__restrict__ raw, int64_t frames, int channels, int enc, int bps,
                             T *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // interleaved sample index
    if (i >= frames * channels) return;
    const int64_t f = i / channels;
    const int c = (int)(i - f * channels);
    out[(int64_t)c * frames + f] = (T)decode_one(raw + i * bps, enc);
}

template <typename T>
__global__ void k_wav_encode(const T *__restrict__ in, int64_t ld, int64_t frames, int channels, int enc, int bps,
                             double gain, uint8_t *__restrict__ raw, unsigned long long *clipped) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool clip = false;
    if (i < frames * channels) {
        const int64_t f = i / channels;
        const int c = (int)(i - f * channels);
        const double v = __dmul_rn((double)in[(int64_t)c * ld + f], gain);
        uint8_t *p = raw + i * bps;
        if (enc == ENC_F32) {
            const uint32_t u = __float_as_uint(__double2float_rn(v));
            p[0] = u & 0xFF;
            p[1] = (u >> 8) & 0xFF;
            p[2] = (u >> 16) & 0xFF;
            p[3] = (u >> 24) & 0xFF;
        } else {
            const int bits = enc == ENC_PCM16 ? 16 : 24;
            const double scale = (double)(1 << (bits - 1));
            double q = rint(__dmul_rn(v, scale));  // numpy round(): half to even
            clip = (q < -scale) || (q > scale - 1.0);
            q = q < -scale ? -scale : (q > scale - 1.0 ? scale - 1.0 : q);
            const uint32_t u = (uint32_t)(int32_t)q;
            p[0] = u & 0xFF;
            p[1] = (u >> 8) & 0xFF;
            if (bits == 24) p[2] = (u >> 16) & 0xFF;
        }
    }
    const unsigned n = __popc(__ballot_sync(0xffffffffu, clip));
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(clipped, (unsigned long long)n);
}

// max |x| over n samples as the bit pattern of a non-negative double
// (ordered like the value); NaN propagates as the largest pattern.
template <typename T>
__global__ void k_peak_abs(const T *__restrict__ x, int64_t n, unsigned long long *peak) {
    double m = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = fabs((double)x[i]);
        m = (v > m || v != v) ? v : m;
    }
    unsigned long long b = (unsigned long long)__double_as_longlong(m);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, b, o);
        b = v > b ? v : b;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(peak, b);
}

int bytes_per_sample(int enc) { return enc == ENC_PCM16 ? 2 : (enc == ENC_PCM24 ? 3 : 4); }

}  // namespace
}  // namespace sc

using namespace sc;

extern "C" {

int sc_wav_decode(int encoding, const void *raw, int64_t frames, int64_t channels, int out_dtype, void *out,
                  void *stream) {
    SC_REQUIRE(encoding >= 0 && encoding <= 2, "sc_wav_decode: bad encoding %d", encoding);
    SC_REQUIRE(out_dtype == SC_F32 || out_dtype == SC_F64, "sc_wav_decode: bad dtype");
    SC_REQUIRE(channels >= 1 && frames >= 0, "sc_wav_decode: bad shape");
    const int64_t n = frames * channels;
    if (n == 0) return SC_OK;
    SC_REQUIRE(raw && out, "sc_wav_decode: null pointer");
    const unsigned g = (unsigned)cdiv(n, 256);
    if (out_dtype == SC_F64)
        k_wav_decode<double><<<g, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t *>(raw), frames,
                                                                 (int)channels, encoding, bytes_per_sample(encoding),
                                                                 static_cast<double *>(out));
    else
        k_wav_decode<float><<<g, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t *>(raw), frames,
                                                                (int)channels, encoding, bytes_per_sample(encoding),
                                                                static_cast<float *>(out));
    SC_CHECK_LAUNCH();
    return SC_OK;
}

int sc_wav_encode(int encoding, int in_dtype, const void *in, int64_t ld, int64_t frames, int64_t channels,
                  double gain, void *raw, unsigned long long *clipped, void *stream) {
    SC_REQUIRE(encoding >= 0 && encoding <= 2, "sc_wav_encode: bad encoding %d", encoding);
    SC_REQUIRE(in_dtype == SC_F32 || in_dtype == SC_F64, "sc_wav_encode: bad dtype");
    SC_REQUIRE(channels >= 1 && frames >= 0 && ld >= frames, "sc_wav_encode: bad shape");
    const int64_t n = frames * channels;
    if (n == 0) return SC_OK;
    SC_REQUIRE(in && raw && clipped, "sc_wav_encode: null pointer");
    const unsigned g = (unsigned)cdiv(n, 256);
    if (in_dtype == SC_F64)
        k_wav_encode<double><<<g, 256, 0, as_stream(stream)>>>(static_cast<const double *>(in), ld, frames,
                                                                 (int)channels, encoding, bytes_per_sample(encoding),
                                                                 gain, static_cast<uint8_t *>(raw), clipped);
    else
        k_wav_encode<float><<<g, 256, 0, as_stream(stream)>>>(static_cast<const float *>(in), ld, frames,
                                                                (int)channels, encoding, bytes_per_sample(encoding),
                                                                gain, static_cast<uint8_t *>(raw), clipped);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

int sc_peak_abs(int dtype, const void *x, int64_t n, unsigned long long *peak_bits, void *stream) {
    SC_REQUIRE(dtype == SC_F32 || dtype == SC_F64, "sc_peak_abs: bad dtype");
    SC_REQUIRE(n >= 0 && peak_bits, "sc_peak_abs: bad arguments");
    if (n == 0) return SC_OK;
    SC_REQUIRE(x, "sc_peak_abs: null pointer");
    const unsigned g = (unsigned)std::min<int64_t>(cdiv(n, 256), 8 * (int64_t)sm_count());
    if (dtype == SC_F64)
        k_peak_abs<double><<<g, 256, 0, as_stream(stream)>>>(static_cast<const double *>(x), n, peak_bits);
    else
        k_peak_abs<float><<<g, 256, 0, as_stream(stream)>>>(static_cast<const float *>(x), n, peak_bits);
    SC_CHECK_LAUNCH();
    return SC_OK;
}

}  // extern "C"
