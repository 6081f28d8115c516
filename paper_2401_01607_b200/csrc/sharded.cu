// sharded.cu -- host-resident signals: the chunk-pipelined output-range
// engine (sc_fir_range_host) and the one-call multi-GPU driver built on it
// (sc_fir_sharded; north_star (4), SURVEY.md 8(b) `sc_fir_sharded`, 8(e)).
//
// A range job computes outputs [a, b) of y = x (*) h from the host signal:
// it needs only inputs [max(0, a-Nh+1), min(Ne, b)) -- its slice plus the
// (Nh-1)-sample halo.  The range is cut into chunks of outputs; per chunk the
// input still missing is uploaded on an upload stream, the chunk's FIR runs on
// a compute stream once its input has landed, and its outputs are downloaded
// on a third stream -- so PCIe/C2C transfers in both directions overlap the
// tensor-core work of neighbouring chunks.  Streams, device buffers and the
// library's scratch (keyed by stream) persist per (device, slot): no
// cudaMalloc/cudaFree (which synchronise) in steady state.
//
// sc_fir_sharded partitions the whole output into equal contiguous segments,
// one per listed device, and runs one range job per device on its own host
// thread.  No MAC is repeated and no partial sum crosses devices, so there is
// no reduction: each device writes its segment into the host result or, with
// a gather device, straight into that device's buffer -- the FIR epilogue
// stores over NVLink when peer access is available (compute and gather in one
// pass).  Output-segment sharding keeps every output's whole chain on one
// device: ORDERED float64 stays bit-identical to the reference at any device
// count.

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sc_common.cuh"

using namespace sc;

namespace {

// Persistent per (device, slot) resources.  Two jobs on one device must use
// different slots: the library's scratch is keyed by stream, so their set-up
// kernels would otherwise share it.
struct Pipe {
    std::mutex mu;  // one job at a time
    int device = -1;
    cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
    cudaEvent_t e_in = nullptr, e_cmp = nullptr;
    void *xd = nullptr, *yd = nullptr, *hd = nullptr;
    size_t xcap = 0, ycap = 0, hcap = 0;
};

Pipe *pipe_for(int device, int slot) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, std::unique_ptr<Pipe>> pipes;
    std::lock_guard<std::mutex> lk(mu);
    auto &p = pipes[{device, slot}];
    if (!p) {
        p.reset(new Pipe());
        p->device = device;
    }
    return p.get();
}

int pipe_init(Pipe &p) {
    if (p.s_in) return SC_OK;
    SC_CHECK_CUDA(cudaStreamCreateWithFlags(&p.s_in, cudaStreamNonBlocking));
    SC_CHECK_CUDA(cudaStreamCreateWithFlags(&p.s_cmp, cudaStreamNonBlocking));
    SC_CHECK_CUDA(cudaStreamCreateWithFlags(&p.s_out, cudaStreamNonBlocking));
    SC_CHECK_CUDA(cudaEventCreateWithFlags(&p.e_in, cudaEventDisableTiming));
    SC_CHECK_CUDA(cudaEventCreateWithFlags(&p.e_cmp, cudaEventDisableTiming));
    return SC_OK;
}

// grow-only device buffer of the pipe (its streams are idle between jobs)
int grow(void **buf, size_t *cap, size_t want) {
    if (*cap >= want) return SC_OK;
    cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    const size_t n = std::max<size_t>(want + want / 8, 256);
    if (cudaMalloc(buf, n) != cudaSuccess) {
        cudaGetLastError();
        set_error("fir range: cudaMalloc(%zu) failed", n);
        return SC_ERR_ALLOC;
    }
    *cap = n;
    return SC_OK;
}

bool is_device_ptr(const void *p, int device) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice && at.device == device;
}

// Chunks per range: one per >= 2^36 MACs (each chunk's tensor-core launch
// still fills the SMs: cfg5 on one GPU -> 12) or per >= 16 MiB of input for
// transfer-bound short filters; 2..12; a single chunk below 2^30 MACs and
// 32 MiB (nothing worth overlapping).
int64_t pick_chunks(int64_t nx, int64_t ny, int64_t nh, size_t es) {
    const double macs = (double)ny * (double)nh;
    const int64_t bytes = nx * (int64_t)es;
    if (macs < 1073741824.0 && bytes < (32ll << 20)) return 1;
    const int64_t by_macs = (int64_t)(macs / 68719476736.0);
    const int64_t by_bytes = bytes >> 24;
    return std::max<int64_t>(2, std::min<int64_t>(12, std::max(by_macs, by_bytes)));
}

struct RangeJob {
    int device;
    int slot;
    int64_t a, b;  // outputs [a, b)
    int64_t chunks = 0;  // 0 = pick_chunks
    // y_dev: the device buffer (on `gather_device`) that receives outputs
    // [a, b) at y_dev + (a - y_origin); nullptr = host y + (a - y_origin)
    void *y_host = nullptr;
    void *y_dev = nullptr;
    int gather_device = -1;
    int64_t y_origin = 0;
    int rc = 0;
    std::string err;
};

int run_range(RangeJob &j, int dtype, int mode, const void *x_host, int64_t ne, const void *h, int64_t nh) {
    const size_t es = dtype == SC_F64 ? 8 : 4;
    SC_CHECK_CUDA(cudaSetDevice(j.device));
    Pipe &p = *pipe_for(j.device, j.slot);
    std::lock_guard<std::mutex> lk(p.mu);
    int rc = pipe_init(p);
    if (rc) return rc;
    const int64_t xb = std::max<int64_t>(0, j.a - nh + 1);
    const int64_t xe = std::max<int64_t>(xb, std::min<int64_t>(ne, j.b));
    const int64_t nx = xe - xb, ny = j.b - j.a;
    if (ny <= 0) return SC_OK;
    // outputs go to the gather device directly when this device can store
    // there (same device, or peer access over NVLink); else staged in yd
    char *direct = nullptr;
    if (j.y_dev) {
        int can = j.gather_device == j.device;
        if (!can) cudaDeviceCanAccessPeer(&can, j.device, j.gather_device);
        if (can && j.gather_device != j.device) {
            const cudaError_t pe = cudaDeviceEnablePeerAccess(j.gather_device, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) can = 0;
            cudaGetLastError();
        }
        if (can) direct = static_cast<char *>(j.y_dev) + (size_t)(j.a - j.y_origin) * es;
    }
    rc = grow(&p.xd, &p.xcap, (size_t)std::max<int64_t>(nx, 1) * es);
    if (!rc && !direct) rc = grow(&p.yd, &p.ycap, (size_t)ny * es);
    if (rc) return rc;
    const void *hd = h;
    if (!is_device_ptr(h, j.device)) {
        rc = grow(&p.hd, &p.hcap, (size_t)nh * es);
        if (rc) return rc;
        SC_CHECK_CUDA(cudaMemcpyAsync(p.hd, h, (size_t)nh * es, cudaMemcpyDefault, p.s_in));
        hd = p.hd;
    }
    char *ybuf = direct ? direct : static_cast<char *>(p.yd);
    const int64_t chunks = j.chunks > 0 ? j.chunks : pick_chunks(nx, ny, nh, es);
    const int64_t per = (ny + chunks - 1) / chunks;
    int64_t uploaded = xb;
    for (int64_t c0 = j.a; c0 < j.b; c0 += per) {
        const int64_t c1 = std::min(j.b, c0 + per);
        const int64_t need = std::min(xe, c1);  // outputs < c1 read inputs < c1
        if (need > uploaded) {
            SC_CHECK_CUDA(cudaMemcpyAsync(static_cast<char *>(p.xd) + (size_t)(uploaded - xb) * es,
                                          static_cast<const char *>(x_host) + (size_t)uploaded * es,
                                          (size_t)(need - uploaded) * es, cudaMemcpyHostToDevice, p.s_in));
            uploaded = need;
        }
        SC_CHECK_CUDA(cudaEventRecord(p.e_in, p.s_in));
        SC_CHECK_CUDA(cudaStreamWaitEvent(p.s_cmp, p.e_in, 0));
        char *yc = ybuf + (size_t)(c0 - j.a) * es;
        const int64_t lo = std::max(xb, c0 - nh + 1);  // this chunk's inputs: [lo, need)
        if (dtype == SC_F32 && mode != SC_MODE_ORDERED) {
            rc = launch_fir_f32(mode, static_cast<const float *>(p.xd), 0, xb, lo, need,
                                static_cast<const float *>(hd), 0, nh, reinterpret_cast<float *>(yc), 0, c0, c1, 1,
                                p.s_cmp);
        } else {
            // the ordered chain of every output of [c0, c1) reads only [lo, need)
            ChainSeg seg{hd, nh, lo, need};
            rc = launch_chain(dtype, SC_SKIP_NONE, 0.0, p.xd, xb, &seg, 1, nullptr, 0, nullptr, c0, c1 - c0, yc,
                              c1 - c0, nullptr, p.s_cmp, nullptr, nullptr, dtype == SC_F64 && mode != SC_MODE_ORDERED);
        }
        if (rc) return rc;
        if (direct) continue;
        SC_CHECK_CUDA(cudaEventRecord(p.e_cmp, p.s_cmp));
        SC_CHECK_CUDA(cudaStreamWaitEvent(p.s_out, p.e_cmp, 0));
        if (j.y_dev)  // gather device not reachable by peer stores: peer copy
            SC_CHECK_CUDA(cudaMemcpyPeerAsync(static_cast<char *>(j.y_dev) + (size_t)(c0 - j.y_origin) * es,
                                              j.gather_device, yc, j.device, (size_t)(c1 - c0) * es, p.s_out));
        else
            SC_CHECK_CUDA(cudaMemcpyAsync(static_cast<char *>(j.y_host) + (size_t)(c0 - j.y_origin) * es, yc,
                                          (size_t)(c1 - c0) * es, cudaMemcpyDeviceToHost, p.s_out));
    }
    const cudaError_t e1 = cudaStreamSynchronize(p.s_cmp);
    const cudaError_t e2 = cudaStreamSynchronize(p.s_out);
    const cudaError_t e3 = cudaStreamSynchronize(p.s_in);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
        set_error("fir range on device %d failed: %s", j.device,
                  cudaGetErrorString(e1 != cudaSuccess ? e1 : e2 != cudaSuccess ? e2 : e3));
        return SC_ERR_CUDA;
    }
    return SC_OK;
}

int check_common(int dtype, int64_t ne, int64_t nh, const void *x_host, const void *h) {
    SC_REQUIRE(dtype == SC_F32 || dtype == SC_F64, "fir range: bad dtype %d", dtype);
    SC_REQUIRE(ne >= 1, "input signal is empty");
    SC_REQUIRE(nh >= 1, "impulse response is empty");
    SC_REQUIRE(x_host && h, "fir range: null pointer");
    return SC_OK;
}

}  // namespace

extern "C" int sc_fir_range_host(int dtype, int mode, const void *x_host, int64_t ne, const void *h, int64_t nh,
                                 void *y_host, int64_t n_begin, int64_t n_end, int device, int chunks) {
    int rc = check_common(dtype, ne, nh, x_host, h);
    if (rc) return rc;
    SC_REQUIRE(0 <= n_begin && n_begin <= n_end && n_end <= ne + nh - 1, "sc_fir_range_host: bad output range");
    SC_REQUIRE(y_host || n_end == n_begin, "sc_fir_range_host: null output");
    int count = 0, prev = 0;
    SC_CHECK_CUDA(cudaGetDeviceCount(&count));
    SC_REQUIRE(device >= 0 && device < count, "sc_fir_range_host: no device %d", device);
    cudaGetDevice(&prev);
    RangeJob j;
    j.device = device;
    j.slot = 0;
    j.a = n_begin;
    j.b = n_end;
    j.chunks = chunks;
    j.y_host = y_host;
    j.y_origin = n_begin;
    rc = run_range(j, dtype, mode, x_host, ne, h, nh);
    cudaSetDevice(prev);
    return rc;
}

extern "C" int sc_fir_sharded(int dtype, int mode, const void *x_host, int64_t ne, const void *h_host, int64_t nh,
                              void *y, int ngpu, const int *devices, int gather_device) {
    int rc = check_common(dtype, ne, nh, x_host, h_host);
    if (rc) return rc;
    SC_REQUIRE(y, "sc_fir_sharded: null pointer");
    SC_REQUIRE(ngpu >= 1 && devices, "sc_fir_sharded: need at least one device");
    int count = 0;
    SC_CHECK_CUDA(cudaGetDeviceCount(&count));
    for (int g = 0; g < ngpu; ++g)
        SC_REQUIRE(devices[g] >= 0 && devices[g] < count, "sc_fir_sharded: no device %d", devices[g]);
    SC_REQUIRE(gather_device < count, "sc_fir_sharded: no gather device %d", gather_device);
    int prev = 0;
    cudaGetDevice(&prev);
    const int64_t nout = ne + nh - 1;
    const int64_t per = (nout + ngpu - 1) / ngpu;
    std::vector<RangeJob> jobs((size_t)ngpu);
    for (int g = 0; g < ngpu; ++g) {
        RangeJob &j = jobs[(size_t)g];
        j.device = devices[g];
        j.slot = g;  // repeated devices get distinct pipes
        j.a = std::min<int64_t>((int64_t)g * per, nout);
        j.b = std::min<int64_t>(j.a + per, nout);
        if (gather_device >= 0) {
            j.y_dev = y;
            j.gather_device = gather_device;
        } else {
            j.y_host = y;
        }
    }
    std::vector<std::thread> threads;
    for (int g = 0; g < ngpu; ++g) {
        RangeJob &j = jobs[(size_t)g];
        if (j.b <= j.a) continue;
        threads.emplace_back([&j, dtype, mode, x_host, ne, h_host, nh] {
            j.rc = run_range(j, dtype, mode, x_host, ne, h_host, nh);
            if (j.rc) j.err = sc_last_error();  // the message is thread-local
        });
    }
    for (auto &t : threads) t.join();
    cudaSetDevice(prev);
    for (auto &j : jobs)
        if (j.rc) {
            set_error("%s", j.err.c_str());
            return j.rc;
        }
    return SC_OK;
}
