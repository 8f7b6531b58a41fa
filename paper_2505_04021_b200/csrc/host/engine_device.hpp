// prism::EngineDevice — the GPU half of one msim::engine::Engine.
//
// Owns (per engine, on the engine's CUDA device):
//   * the device block table: one int32 arena; each admitted request gets a
//     row of prompt_tokens + output_tokens elements (its maximum live slot
//     count), holding slot ids page * tokens_per_page + slot in token order —
//     the device mirror of EngineRequest::kv (reference engine.hpp:64);
//   * the GPU-resident slot state of the engine's pool (DevicePool) that the
//     batched allocator kernel K1 updates from the pool's op log;
//   * the per-step descriptors the append (K2) and attention (K3) kernels read:
//     the slot ids allocated this step, and for every request that decoded this
//     step its row and context length.
// engine::step() (csrc/host/engine.cpp) calls the hooks below; everything is
// issued asynchronously on the engine's stream.
#pragma once
#include <cstdint>
#include <vector>

#include "msim/engine.hpp"

namespace prism {

struct StepDecode {
    std::uint64_t request_id;
    std::int64_t row;      // block-table element offset of the request's row
    std::int32_t ctx_len;  // live slots after this step's allocation
};

class EngineDevice {
public:
    virtual ~EngineDevice() = default;
    // Row arena (host bookkeeping; the rows live in device memory).
    virtual std::int64_t acquire_row(std::int64_t capacity) = 0;
    virtual void release_row(std::int64_t row) = 0;
    // Called by engine::step before any allocation / after the host logic.
    virtual void begin_step(msim::engine::Engine& eng) = 0;
    // prefill_*: the request whose chunk was allocated this step (id, row,
    // first position, slots incl. the first generated token), or row -1.
    virtual void end_step(msim::engine::Engine& eng, const msim::engine::IterationOutcome& out,
                          const std::vector<StepDecode>& decodes, std::uint64_t prefill_id, std::int64_t prefill_row,
                          std::int32_t prefill_first, std::int32_t prefill_tokens) = 0;
};

}  // namespace prism
