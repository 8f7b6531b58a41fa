// prism-b200 — model weight loading for activation.
//
// The reference models activation as a latency curve only
// (ActivationParams::load_latency_s, engine.hpp:68-74 here / reference
// engine.hpp:46-48, src/engine.cpp:44-51) after the paper's "parallel model
// weight loading": weights are chunked, loaded through
// several GPUs' host links in parallel, and gathered into the target GPU over
// NVLink, each helper keeping only a small staging buffer (~30 MB).
//
// WeightLoader is that data path, B200-first:
//   * load():      host -> target HBM, fixed-size chunks round-robin over
//                  n copy streams (the paper's observation: one cudaMemcpyAsync
//                  does not saturate the host link);
//   * load_part(): one helper's share of a fan-in — chunks i with
//                  i % n_parts == part go host -> this GPU's staging slot ->
//                  dst, where dst may be another GPU's memory (peer pointer or
//                  an IPC-opened pointer): H2D on this GPU's host link, then a
//                  copy-engine transfer over NVLink. Staging = n_streams
//                  chunks; chunk k uses stream and slot k % n_streams, so slot
//                  reuse is ordered by its stream (no events);
//   * load_naive(): the baseline, one cudaMemcpyAsync.
// All enqueue only; wait() synchronises and returns the device time from the
// first enqueue to the last copy (CUDA events). Host memory must be pinned
// (cudaHostAlloc / cudaHostRegister) for the copies to be asynchronous.
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

namespace prism {

class WeightLoader {
public:
    WeightLoader(int device, int n_streams, std::size_t chunk_bytes);
    ~WeightLoader();
    WeightLoader(const WeightLoader&) = delete;
    WeightLoader& operator=(const WeightLoader&) = delete;

    void load(const void* host, void* dst, std::size_t bytes);
    void load_part(const void* host, void* dst, std::size_t bytes, int part, int n_parts);
    void load_naive(const void* host, void* dst, std::size_t bytes);
    double wait();  // ms, device time of everything enqueued since the last wait()

    int device() const { return device_; }
    int streams() const { return static_cast<int>(streams_.size()); }
    std::size_t chunk_bytes() const { return chunk_; }

private:
    void begin();

    int device_ = 0;
    std::size_t chunk_ = 0;
    std::vector<void*> streams_;  // cudaStream_t
    std::vector<void*> done_;     // cudaEvent_t per stream
    void* start_ = nullptr;       // cudaEvent_t
    void* end_ = nullptr;
    std::vector<void*> staging_;  // device buffers, one chunk per stream (lazily allocated)
    bool open_ = false;           // start_ recorded, not yet waited
};

}  // namespace prism
