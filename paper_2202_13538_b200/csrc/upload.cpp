// Host -> device upload of large pageable host arrays (the graph CSR of a
// host-input preprocess, sampler.preprocess / DeviceGraph.from_graph).
//
// A plain cudaMemcpy from pageable memory is staged by the driver through
// its own small pinned bounce buffer on one thread (~8-10 GB/s here).  This
// splits the array into one contiguous part per worker thread; each worker
// copies its part in chunks into its own pair of pinned buffers and issues
// the H2D of each chunk on its own stream, so host copies and DMA overlap and
// several cores feed the copy engines.  The pinned buffers are allocated
// once and kept (later calls reuse them).  On return every copy is complete
// (the call is synchronous, like the pageable cudaMemcpy it replaces).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/walkjoin_b200.h"

namespace wj {
void set_error(const char *fmt, ...);
}

namespace {

constexpr size_t kChunk = 8u << 20;  // bytes per staged chunk
constexpr int kMaxWorkers = 16;

struct Worker {
    void *buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    int dev = -1;
};

std::mutex g_mu;
Worker g_workers[kMaxWorkers];

bool ready(Worker &w, int dev) {
    if (w.dev == dev && w.st) return true;
    if (w.st) return false;  // set up on another device: not reused
    for (int k = 0; k < 2; ++k) {
        if (cudaHostAlloc(&w.buf[k], kChunk, cudaHostAllocPortable) != cudaSuccess) return false;
        if (cudaEventCreateWithFlags(&w.ev[k], cudaEventDisableTiming) != cudaSuccess) return false;
    }
    if (cudaStreamCreateWithFlags(&w.st, cudaStreamNonBlocking) != cudaSuccess) return false;
    w.dev = dev;
    return true;
}

// worker t: bytes [lo, hi) of src -> dst, chunk by chunk through its two buffers
cudaError_t run_part(Worker &w, char *dst, const char *src, size_t lo, size_t hi) {
    int k = 0;
    for (size_t off = lo; off < hi; off += kChunk, k ^= 1) {
        const size_t n = hi - off < kChunk ? hi - off : kChunk;
        cudaError_t e = cudaEventSynchronize(w.ev[k]);  // the buffer's previous H2D is done
        if (e != cudaSuccess) return e;
        std::memcpy(w.buf[k], src + off, n);
        e = cudaMemcpyAsync(dst + off, w.buf[k], n, cudaMemcpyHostToDevice, w.st);
        if (e != cudaSuccess) return e;
        e = cudaEventRecord(w.ev[k], w.st);
        if (e != cudaSuccess) return e;
    }
    return cudaStreamSynchronize(w.st);
}

}  // namespace

extern "C" int wj_upload(void *dst, const void *src, int64_t bytes, int32_t threads) {
    if (bytes < 0 || (bytes > 0 && (!dst || !src))) {
        wj::set_error("wj_upload: bad arguments");
        return WJ_ERR_ARG;
    }
    if (bytes == 0) return WJ_OK;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        wj::set_error("wj_upload: no CUDA device");
        return WJ_ERR_CUDA;
    }
    std::lock_guard<std::mutex> lock(g_mu);
    int T = threads < 1 ? 1 : (threads > kMaxWorkers ? kMaxWorkers : threads);
    const size_t nchunks = ((size_t)bytes + kChunk - 1) / kChunk;
    if ((size_t)T > nchunks) T = (int)nchunks;
    for (int t = 0; t < T; ++t)
        if (!ready(g_workers[t], dev)) {
            cudaGetLastError();
            // fall back to the driver's pageable copy (still correct)
            const cudaError_t e = cudaMemcpy(dst, src, (size_t)bytes, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) {
                wj::set_error("wj_upload: %s", cudaGetErrorString(e));
                return WJ_ERR_CUDA;
            }
            return WJ_OK;
        }
    // contiguous parts of whole chunks per worker
    std::vector<cudaError_t> err(T, cudaSuccess);
    std::vector<std::thread> pool;
    size_t c0 = 0;
    for (int t = 0; t < T; ++t) {
        const size_t c1 = nchunks * (size_t)(t + 1) / (size_t)T;
        const size_t lo = c0 * kChunk, hi = c1 * kChunk < (size_t)bytes ? c1 * kChunk : (size_t)bytes;
        c0 = c1;
        if (t == T - 1) {  // the caller's thread takes the last part
            err[t] = run_part(g_workers[t], (char *)dst, (const char *)src, lo, hi);
        } else {
            pool.emplace_back([&, t, lo, hi]() {
                cudaSetDevice(dev);
                err[t] = run_part(g_workers[t], (char *)dst, (const char *)src, lo, hi);
            });
        }
    }
    for (auto &th : pool) th.join();
    for (int t = 0; t < T; ++t)
        if (err[t] != cudaSuccess) {
            wj::set_error("wj_upload: %s", cudaGetErrorString(err[t]));
            return WJ_ERR_CUDA;
        }
    return WJ_OK;
}
