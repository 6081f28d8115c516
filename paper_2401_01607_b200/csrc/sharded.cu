// sharded.cu -- one call, several GPUs: the whole-signal convolution of a
// host-resident signal partitioned by OUTPUT time segment (north_star (4),
// SURVEY.md 8(b) `sc_fir_sharded`, 8(e)).
//
// Device g of the list owns outputs [a_g, b_g) (equal contiguous segments)
// and receives only its input slice plus the (Nh-1)-sample halo,
// [max(0, a_g-Nh+1), min(Ne, b_g)).  No MAC is repeated and no partial sum
// crosses devices, so there is no reduction: each device writes its segment
// straight into the host result or, with a gather device, into that
// device's buffer: the FIR epilogue stores there directly over NVLink when
// peer access is available (compute and gather in one pass), else through a
// peer copy.  One host thread per shard
// drives its device (upload on its own stream, FIR, download), so the
// uploads and kernels of all devices overlap.  Output-segment sharding keeps
// every output's whole chain on one device: ORDERED float64 stays
// bit-identical to the reference at any device count.

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sc_common.cuh"

using namespace sc;

namespace {

struct ShardJob {
    int device;
    int64_t a, b, xb, xe;  // outputs [a, b), inputs [xb, xe)
    int rc = 0;
    std::string err;
};

// Persistent stream per (device, shard slot): the library's scratch buffers
// are keyed by stream, so per-call streams would leak scratch, and two shards
// on one device must not share a stream (their set-up kernels would
// interleave on the shared scratch).
cudaStream_t shard_stream(int device, int slot) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, cudaStream_t> streams;
    std::lock_guard<std::mutex> lk(mu);
    auto it = streams.find({device, slot});
    if (it != streams.end()) return it->second;
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    streams[{device, slot}] = s;
    return s;
}

int run_shard(ShardJob &j, int slot, int dtype, int mode, const void *x_host, const void *h_host, int64_t nh,
              void *y, int gather_device) {
    const size_t es = dtype == SC_F64 ? 8 : 4;
    SC_CHECK_CUDA(cudaSetDevice(j.device));
    cudaStream_t s = shard_stream(j.device, slot);
    if (!s) {
        set_error("sc_fir_sharded: cannot create a stream on device %d", j.device);
        return SC_ERR_CUDA;
    }
    void *xd = nullptr, *hd = nullptr, *yd = nullptr;
    const int64_t nx = j.xe - j.xb, ny = j.b - j.a;
    int rc = SC_OK;
    auto fail = [&](int code) {
        rc = code;
        return code;
    };
    do {
        if (cudaMalloc(&xd, (size_t)std::max<int64_t>(nx, 1) * es) != cudaSuccess ||
            cudaMalloc(&hd, (size_t)nh * es) != cudaSuccess || cudaMalloc(&yd, (size_t)ny * es) != cudaSuccess) {
            cudaGetLastError();
            set_error("sc_fir_sharded: cudaMalloc on device %d failed", j.device);
            fail(SC_ERR_ALLOC);
            break;
        }
        if (nx > 0 && cudaMemcpyAsync(xd, static_cast<const char *>(x_host) + (size_t)j.xb * es, (size_t)nx * es,
                                      cudaMemcpyHostToDevice, s) != cudaSuccess) {
            set_error("sc_fir_sharded: upload to device %d failed", j.device);
            fail(SC_ERR_CUDA);
            break;
        }
        if (cudaMemcpyAsync(hd, h_host, (size_t)nh * es, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            set_error("sc_fir_sharded: upload to device %d failed", j.device);
            fail(SC_ERR_CUDA);
            break;
        }
        // With a gather device reachable by peer access (or the same device),
        // the kernel's epilogue stores its segment straight into the gather
        // buffer -- over NVLink for a peer -- so compute and gather are one
        // pass; otherwise the segment is staged and copied.
        void *dst = yd;
        bool direct = false;
        if (gather_device >= 0) {
            int can = gather_device == j.device;
            if (!can) cudaDeviceCanAccessPeer(&can, j.device, gather_device);
            if (can && gather_device != j.device) {
                const cudaError_t pe = cudaDeviceEnablePeerAccess(gather_device, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) can = 0;
                cudaGetLastError();
            }
            if (can) {
                dst = static_cast<char *>(y) + (size_t)j.a * es;
                direct = true;
            }
        }
        if (dtype == SC_F32 && mode != SC_MODE_ORDERED) {
            rc = launch_fir_f32(mode, static_cast<const float *>(xd), 0, j.xb, j.xb, j.xe,
                                static_cast<const float *>(hd), 0, nh, static_cast<float *>(dst), 0, j.a, j.b, 1, s);
        } else {
            // the ordered chain of every output of [a, b) reads only [xb, xe)
            ChainSeg seg{hd, nh, j.xb, j.xe};
            rc = launch_chain(dtype, SC_SKIP_NONE, 0.0, xd, j.xb, &seg, 1, nullptr, 0, nullptr, j.a, ny, dst, ny,
                              nullptr, s, nullptr, nullptr, dtype == SC_F64 && mode != SC_MODE_ORDERED);
        }
        if (rc) break;
        cudaError_t e = cudaSuccess;
        if (gather_device < 0)
            e = cudaMemcpyAsync(static_cast<char *>(y) + (size_t)j.a * es, yd, (size_t)ny * es,
                                cudaMemcpyDeviceToHost, s);
        else if (!direct)
            e = cudaMemcpyPeerAsync(static_cast<char *>(y) + (size_t)j.a * es, gather_device, yd, j.device,
                                    (size_t)ny * es, s);
        if (e != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) {
            set_error("sc_fir_sharded: result copy from device %d failed: %s", j.device,
                      cudaGetErrorString(cudaGetLastError()));
            fail(SC_ERR_CUDA);
            break;
        }
    } while (false);
    cudaStreamSynchronize(s);
    cudaFree(xd);
    cudaFree(hd);
    cudaFree(yd);
    return rc;
}

}  // namespace

extern "C" int sc_fir_sharded(int dtype, int mode, const void *x_host, int64_t ne, const void *h_host, int64_t nh,
                              void *y, int ngpu, const int *devices, int gather_device) {
    SC_REQUIRE(dtype == SC_F32 || dtype == SC_F64, "sc_fir_sharded: bad dtype %d", dtype);
    SC_REQUIRE(ne >= 1, "sc_fir_sharded: input signal is empty");
    SC_REQUIRE(nh >= 1, "sc_fir_sharded: impulse response is empty");
    SC_REQUIRE(x_host && h_host && y, "sc_fir_sharded: null pointer");
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
    std::vector<ShardJob> jobs((size_t)ngpu);
    for (int g = 0; g < ngpu; ++g) {
        ShardJob &j = jobs[(size_t)g];
        j.device = devices[g];
        j.a = std::min<int64_t>((int64_t)g * per, nout);
        j.b = std::min<int64_t>(j.a + per, nout);
        j.xb = std::max<int64_t>(0, j.a - nh + 1);
        j.xe = std::max<int64_t>(j.xb, std::min<int64_t>(ne, j.b));
    }
    std::vector<std::thread> threads;
    for (int g = 0; g < ngpu; ++g) {
        ShardJob &j = jobs[(size_t)g];
        if (j.b <= j.a) continue;
        threads.emplace_back([&j, g, dtype, mode, x_host, h_host, nh, y, gather_device] {
            j.rc = run_shard(j, g, dtype, mode, x_host, h_host, nh, y, gather_device);
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
