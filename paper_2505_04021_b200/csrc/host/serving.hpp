// prism::DeviceExecutor — simcore's IterationExecutor on the GPU data path
// (see serving.cpp): the two-level scheduler driving K1/K2/K3/K4.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "host/vmm.hpp"
#include "msim/simcore.hpp"

namespace prism {

struct ServingOptions {
    bool measured = false;           // charge the measured GPU time of each iteration (else the modelled one)
    std::uint64_t seed = 20251017;   // synthetic K/V content (K2)
    std::vector<int> owned;          // simulated GPUs run on a device (empty: all)
    int max_decode_batch = 512;      // requests decoding in one engine step
    std::uint64_t chunk_pages = 0;   // VMM chunk size (0: default)
};

struct ServingStats {
    std::uint64_t iterations = 0, attached = 0, detached = 0;
    std::uint64_t k2_launches = 0, k3_launches = 0, k4_launches = 0;
    std::uint64_t decode_tokens = 0, prefill_tokens = 0;
    std::uint64_t gpu_us = 0, modelled_us = 0;  // measured mode: charged GPU time vs the cost model's
};

class DeviceExecutor final : public msim::simcore::IterationExecutor {
public:
    // ordinals: physical CUDA devices; simulated GPU g runs on ordinals[g % n]
    // (one VmmDevice per simulated GPU).
    DeviceExecutor(std::vector<int> ordinals, ServingOptions opts);
    ~DeviceExecutor() override;
    DeviceExecutor(const DeviceExecutor&) = delete;
    DeviceExecutor& operator=(const DeviceExecutor&) = delete;

    void gpu_created(int gpu, msim::engine::GpuState& gs) override;
    void attached(int gpu, msim::engine::GpuState& gs, int engine_index) override;
    void detaching(int gpu, msim::engine::GpuState& gs, int engine_index) override;
    void before_step(int gpu, msim::engine::GpuState& gs, int engine_index) override;
    msim::SimTime iteration(int gpu, msim::engine::GpuState& gs, int engine_index,
                            const msim::engine::IterationOutcome& out, msim::SimTime modelled_us) override;

    void synchronize();
    const ServingStats& stats() const { return stats_; }
    VmmStats vmm_stats() const;

private:
    struct Buffers {
        void* q = nullptr;
        void* out = nullptr;
        int rows = 0;
        cudaEvent_t start = nullptr, stop = nullptr;
    };
    bool owns(int gpu) const;
    static void release(Buffers& b);

    std::vector<int> ordinals_;
    ServingOptions opts_;
    std::map<int, std::shared_ptr<VmmDevice>> devs_;
    std::map<std::pair<int, int>, Buffers> bufs_;
    ServingStats stats_;
};

}  // namespace prism
