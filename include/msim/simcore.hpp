// prism-b200 — simcore: the deterministic discrete-event driver that composes
// the reference's pieces over a trace on N GPUs and measures SLO attainment.
//
// The reference specifies this module ("[MODULE] simcore")
// but ships no code for it: engine::step, place_models,
// eviction_tick, activate_on_arrival and the allocator exist, the loop that
// composes them does not. This implementation uses ONLY the public msim::
// API, so it is compiled twice — into the product library and into the
// oracle library built from the reference's own sources — and the two must
// produce identical metrics on the same inputs (tests/test_simcore.py).
//
// Event order: (timestamp, kind priority arrival <
// iteration_done < activation_done < scheduler_tick, sequence number); time
// is integer microseconds. Composition:
//   * t = 0: place_models (Algorithm 1) over all models with their demand
//     rates; every placed model is activated on its GPU (activation_done
//     after init + realign + load latency);
//   * arrival: the request joins its GPU's shared queue (Algorithm 2, see
//     LocalScheduler; FIFO: its model's engine queue); a model with no
//     engine is activated on the lowest-KVPR GPU whose free pages fit its
//     weights (activate_on_arrival), else it waits for a later tick;
//   * a GPU runs one iteration at a time (SPEC enginemodel, Open Questions):
//     when idle it steps its next serving engine with runnable work in
//     round-robin order (engine::step), then tops the pre-mapped buffer up
//     (refill_buffer, the buffer_refill event folded into iteration end);
//   * scheduler_tick every tick_s: eviction_tick over the GPUs (a resident
//     is idle while it has no queued or running request; a GPU is pressured
//     when its free pages fall below pressure_free_frac of capacity or a
//     model is waiting for activation), evicted engines are deactivated, and
//     waiting models retry activation.
// Metrics (SPEC SimMetrics): per request arrival / first token / completion
// (times when the producing iteration ends), preemption count; TTFT / TPOT
// attainment per model and overall at any SLO scale, recomputable without
// re-simulation.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "msim/engine.hpp"
#include "msim/time.hpp"
#include "msim/workload.hpp"

namespace msim::simcore {

struct ModelEntry {
    engine::ModelSpec spec;  // tp_degree must be 1
    double rate = 0.0;       // demand used by the initial placement (requests / s)
};

// Sharing policy ([MODULE] policies), same harness:
//   prism            Algorithm 1 placement, arrival activation, idle eviction,
//                    on-demand cross-model KV sharing through the ledger;
//   mux_flexible     MuxServe stand-in: place_models once at t = 0 (all
//                    models must fit), then frozen: no eviction, no arrival
//                    activation; colocated models share KV on demand;
//   static_partition the same frozen colocation, but each pool is hard-capped
//                    (KvPool::set_mapped_page_cap) at an equal share of its
//                    GPU's KV pages: no cross-model borrowing;
//   qlm_timeshare    QLM stand-in: one resident model per GPU; when a GPU's
//                    resident model has drained, the oldest waiting request's
//                    model is swapped in on the first such GPU (no residency
//                    awareness) at stop-and-restart cost (engine init + naive
//                    weight load).
enum class Policy { prism = 0, mux_flexible = 1, static_partition = 2, qlm_timeshare = 3 };

// Local (per-GPU) scheduler ([MODULE] local_sched):
//   moore_hodgson  Algorithm 2: every arrival for a resident model joins ONE
//                  shared queue per GPU; on every arrival, iteration boundary
//                  and activation the GPU runs admission::moore_hodgson over
//                  it, then admission::dispatch hands admitted requests to
//                  their engines in deadline order through a gate that only
//                  lets IMMEDIATELY-runnable requests through (the engine has
//                  no queued or in-flight prefill; the pool's
//                  allocatable_tokens covers the first chunk, next_chunk_need
//                  semantics, plus the engine's reserved_pages), and
//                  admission::requeue_deferred merges the rest back;
//   fifo           per-model FIFO: arrivals go straight into their engine's
//                  local queue (the baselines' admission; SPEC property 10's
//                  comparison point).
// Policy::prism uses `local`; the baseline policies always use fifo.
enum class LocalScheduler { moore_hodgson = 0, fifo = 1 };

// Optional executor behind the modelled iterations (product only; the
// reference has no device): with one attached, simcore is the serving loop
// of the GPU data path. It gives each simulated GPU's ledger its device
// (gpu_created, before any pool exists), gives every activated engine its
// GPU half (attached, after finish_activation) and takes it back before
// deactivate (detaching), brackets every engine::step — which, with a device
// attached, runs K1 (batched slot allocation + block-table update) — and
// then runs the iteration's kernels (iteration: K2 append, K4 chunked-prefill
// attention and K3 decode attention over all layers) and returns the
// duration to charge: the modelled one (decisions identical to the host-only
// run) or the measured GPU time of the iteration.
class IterationExecutor {
public:
    virtual ~IterationExecutor() = default;
    virtual void gpu_created(int gpu, engine::GpuState& gs) = 0;
    virtual void attached(int gpu, engine::GpuState& gs, int engine_index) = 0;
    virtual void detaching(int gpu, engine::GpuState& gs, int engine_index) = 0;
    virtual void before_step(int gpu, engine::GpuState& gs, int engine_index) = 0;
    virtual SimTime iteration(int gpu, engine::GpuState& gs, int engine_index, const engine::IterationOutcome& out,
                              SimTime modelled_us) = 0;
};

struct SimConfig {
    Policy policy = Policy::prism;
    LocalScheduler local = LocalScheduler::moore_hodgson;
    int n_gpus = 1;
    std::uint64_t capacity_pages = 0;  // per GPU
    std::uint64_t page_bytes = 2ull << 20;
    engine::EngineParams params;
    engine::ActivationParams activation;
    engine::ActivationMethod method = engine::ActivationMethod::parallel;
    double tau_per_gb = 0.05;
    double tick_s = 10.0;
    double idle_evict_s = 10.0;
    double pressure_free_frac = 0.10;
    std::uint64_t buffer_target_pages = 8;
    bool initial_placement = true;
    std::uint64_t max_events = 200'000'000;  // safety valve: the run stops (truncated) beyond it
    IterationExecutor* executor = nullptr;   // not owned; null = host-only simulation
};

struct RequestRecord {
    std::uint64_t id = 0;  // 1-based trace index
    std::string model_id;
    SimTime arrival_us = 0;
    SimTime first_token_us = -1;  // -1: never
    SimTime completion_us = -1;
    int prompt_tokens = 0;
    int output_tokens = 0;
    int preemptions = 0;
    int gpu = -1;
};

struct SimMetrics {
    std::vector<RequestRecord> requests;  // trace order
    SimTime end_us = 0;                   // time of the last event
    std::uint64_t events = 0;
    std::uint64_t iterations = 0;
    std::uint64_t activations = 0;
    std::uint64_t evictions = 0;
    std::uint64_t preemptions = 0;
    std::uint64_t dispatches = 0;         // Algorithm 2: requests handed to engines
    std::uint64_t schedule_rounds = 0;    // Algorithm 2: moore_hodgson invocations
    std::uint64_t output_tokens = 0;      // tokens of completed requests
    std::vector<SimTime> gpu_busy_us;     // per GPU, time inside iterations
    bool truncated = false;
};

// Runs the trace to completion. Throws msim::UsageError before the loop for an
// infeasible configuration (a model whose weights fit no GPU, tp_degree != 1,
// a trace event for an unknown model).
SimMetrics run(const SimConfig& cfg, const std::vector<ModelEntry>& models,
               const std::vector<workload::TraceEvent>& trace);

struct Attainment {
    std::uint64_t n = 0;         // requests of the model in the trace
    double ttft = 0.0;           // fraction with first_token - arrival <= scale * ttft_slo
    double tpot = 0.0;           // fraction with (completion - first) / (output - 1) <= scale * tpot_slo
    double both = 0.0;           // fraction meeting both
};

// Per model (by model_id) and overall ("" key); unfinished requests miss.
std::map<std::string, Attainment> attainment(const SimMetrics& m, const std::vector<ModelEntry>& models,
                                             double slo_scale);

}  // namespace msim::simcore
