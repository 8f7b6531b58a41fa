// prism-b200 — WeightLoader (host/weight_load.hpp): chunked, multi-stream
// weight loading and the per-helper half of a staged NVLink fan-in.
// Copy-engine work only (no kernels): cudaMemcpyAsync with cudaMemcpyDefault
// (UVA resolves host / local / peer / IPC-opened pointers).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>

#include "common.cuh"
#include "host/weight_load.hpp"

namespace prism {

namespace {
cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }
cudaEvent_t E(void* p) { return static_cast<cudaEvent_t>(p); }

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int d) {
        PRISM_CUDA(cudaGetDevice(&prev));
        PRISM_CUDA(cudaSetDevice(d));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};
}  // namespace

WeightLoader::WeightLoader(int device, int n_streams, std::size_t chunk_bytes)
    : device_(device), chunk_(chunk_bytes) {
    if (n_streams < 1 || n_streams > 64) throw std::invalid_argument("WeightLoader: n_streams must be in 1..64");
    if (chunk_bytes == 0) throw std::invalid_argument("WeightLoader: chunk_bytes must be > 0");
    DeviceGuard g(device_);
    for (int i = 0; i < n_streams; ++i) {
        cudaStream_t s;
        PRISM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        streams_.push_back(s);
        cudaEvent_t e;
        PRISM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        done_.push_back(e);
    }
    cudaEvent_t a, b;
    PRISM_CUDA(cudaEventCreate(&a));
    PRISM_CUDA(cudaEventCreate(&b));
    start_ = a;
    end_ = b;
}

WeightLoader::~WeightLoader() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    for (void* s : streams_) cudaStreamSynchronize(S(s));
    for (void* p : staging_) cudaFree(p);
    for (void* e : done_) cudaEventDestroy(E(e));
    for (void* s : streams_) cudaStreamDestroy(S(s));
    cudaEventDestroy(E(start_));
    cudaEventDestroy(E(end_));
    cudaSetDevice(prev);
}

void WeightLoader::begin() {
    if (open_) return;
    // every stream starts after start_ (so the elapsed time covers them all)
    PRISM_CUDA(cudaEventRecord(E(start_), S(streams_[0])));
    for (std::size_t i = 1; i < streams_.size(); ++i) PRISM_CUDA(cudaStreamWaitEvent(S(streams_[i]), E(start_), 0));
    open_ = true;
}

void WeightLoader::load(const void* host, void* dst, std::size_t bytes) {
    if (!host || !dst) throw std::invalid_argument("WeightLoader::load: null pointer");
    DeviceGuard g(device_);
    begin();
    const auto* src = static_cast<const char*>(host);
    auto* out = static_cast<char*>(dst);
    const std::size_t n = streams_.size();
    std::size_t k = 0;
    for (std::size_t off = 0; off < bytes; off += chunk_, ++k) {
        const std::size_t len = std::min(chunk_, bytes - off);
        PRISM_CUDA(cudaMemcpyAsync(out + off, src + off, len, cudaMemcpyDefault, S(streams_[k % n])));
    }
}

void WeightLoader::load_naive(const void* host, void* dst, std::size_t bytes) {
    if (!host || !dst) throw std::invalid_argument("WeightLoader::load_naive: null pointer");
    DeviceGuard g(device_);
    begin();
    PRISM_CUDA(cudaMemcpyAsync(dst, host, bytes, cudaMemcpyDefault, S(streams_[0])));
}

void WeightLoader::load_part(const void* host, void* dst, std::size_t bytes, int part, int n_parts) {
    if (!host || !dst) throw std::invalid_argument("WeightLoader::load_part: null pointer");
    if (n_parts < 1 || part < 0 || part >= n_parts) throw std::invalid_argument("WeightLoader::load_part: bad part");
    DeviceGuard g(device_);
    const std::size_t n = streams_.size();
    if (staging_.empty()) {
        for (std::size_t i = 0; i < n; ++i) {
            void* p = nullptr;
            PRISM_CUDA(cudaMalloc(&p, chunk_));
            staging_.push_back(p);
        }
    }
    begin();
    const auto* src = static_cast<const char*>(host);
    auto* out = static_cast<char*>(dst);
    std::size_t k = 0;  // this part's chunk counter: stream and staging slot
    std::size_t idx = 0;
    for (std::size_t off = 0; off < bytes; off += chunk_, ++idx) {
        if (idx % static_cast<std::size_t>(n_parts) != static_cast<std::size_t>(part)) continue;
        const std::size_t len = std::min(chunk_, bytes - off);
        cudaStream_t s = S(streams_[k % n]);
        void* slot = staging_[k % n];
        PRISM_CUDA(cudaMemcpyAsync(slot, src + off, len, cudaMemcpyHostToDevice, s));
        PRISM_CUDA(cudaMemcpyAsync(out + off, slot, len, cudaMemcpyDefault, s));
        ++k;
    }
}

double WeightLoader::wait() {
    DeviceGuard g(device_);
    if (!open_) return 0.0;
    for (std::size_t i = 1; i < streams_.size(); ++i) {
        PRISM_CUDA(cudaEventRecord(E(done_[i]), S(streams_[i])));
        PRISM_CUDA(cudaStreamWaitEvent(S(streams_[0]), E(done_[i]), 0));
    }
    PRISM_CUDA(cudaEventRecord(E(end_), S(streams_[0])));
    PRISM_CUDA(cudaEventSynchronize(E(end_)));
    open_ = false;
    float ms = 0.0f;
    PRISM_CUDA(cudaEventElapsedTime(&ms, E(start_), E(end_)));
    return static_cast<double>(ms);
}

}  // namespace prism
