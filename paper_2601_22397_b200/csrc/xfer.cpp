// xfer.cpp -- large host->device copies from the caller's pageable memory.
//
// A pageable cudaMemcpyAsync is staged by the driver through one host thread
// (~10 GB/s on the test boxes: 6 ms of a 4M-tuple frontier batch's 6.5 ms).
// Here NT host threads copy 4 MB chunks into a process-wide pinned ring (two
// slots per thread) and queue each chunk's DMA as soon as it is staged, so the
// memcpys run in parallel and overlap the copy engine.
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace sair {

namespace {
constexpr size_t XCHUNK = 4u << 20;
constexpr size_t XSMALL = 8u << 20;  // below this the driver's own staging is as fast
std::mutex g_xmu;
char* g_ring = nullptr;
int g_nt = 0;

int ring_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(8u, hw ? hw / 2 : 1u));
}
}  // namespace

void copy_h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes < XSMALL) {
        SAIR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    std::lock_guard<std::mutex> lk(g_xmu);
    if (!g_ring) {
        g_nt = ring_threads();
        // portable: pinned for every device of the process (sharded callers)
        SAIR_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g_ring), (size_t)g_nt * 2 * XCHUNK,
                                cudaHostAllocPortable));
    }
    int dev = 0;
    SAIR_CUDA(cudaGetDevice(&dev));
    const int nt = g_nt;
    const size_t nch = (bytes + XCHUNK - 1) / XCHUNK;
    std::vector<cudaEvent_t> ev((size_t)nt * 2, nullptr);
    for (auto& e : ev) SAIR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    std::vector<cudaError_t> err((size_t)nt, cudaSuccess);
    auto work = [&](int t) {
        cudaError_t e = cudaSetDevice(dev);
        int use = 0;
        for (size_t k = (size_t)t; k < nch && e == cudaSuccess; k += (size_t)nt, ++use) {
            const int slot = 2 * t + (use & 1);
            char* buf = g_ring + (size_t)slot * XCHUNK;
            if (use >= 2) e = cudaEventSynchronize(ev[(size_t)slot]);  // the slot's last DMA
            if (e != cudaSuccess) break;
            const size_t off = k * XCHUNK, len = std::min(XCHUNK, bytes - off);
            std::memcpy(buf, static_cast<const char*>(src) + off, len);
            e = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf, len, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) e = cudaEventRecord(ev[(size_t)slot], st);
        }
        err[(size_t)t] = e;
    };
    std::vector<std::thread> th;
    const int used = (int)std::min<size_t>((size_t)nt, nch);
    for (int t = 1; t < used; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    // the ring is reused by the next call: its DMAs must have drained
    for (auto& e : ev) {
        cudaEventSynchronize(e);
        cudaEventDestroy(e);
    }
    for (cudaError_t e : err) SAIR_CUDA(e);
}

}  // namespace sair
