// prism::DeviceExecutor — simcore's IterationExecutor on the GPU data path:
// the two-level scheduler (placement / eviction / arrival activation
// globally, Algorithm 2 per GPU, engine::step) driving the real kernels.
//
// Per simulated GPU the executor owns (if it runs that GPU on a device) one
// VmmDevice on a physical CUDA device, attached to the GPU's ledger before
// any pool exists, so every pool created by finish_activation reserves its
// VA (cuMemAddressReserve) and maps 2 MiB pages on demand, and every
// deactivate frees them (free_kvcache -> VmmDevice::release: VA freed,
// physical chunks back to the handle cache for the next model's pool).
// Per activated engine: attach_engine_device (device slot mirror, block
// table, step descriptors) and q / out buffers for its largest step.
// Per iteration (simcore step_next): engine::step runs K1 through the device
// hooks; iteration() then appends the step's K/V rows for all layers (K2,
// synthetic content), runs K4 over the prefill chunk and K3 over the decoded
// requests for every layer, and returns either the modelled duration (the
// decisions then equal the host-only simulation's) or the measured GPU time
// from before K1 to after the last K3 (CUDA events on the engine stream).
// Iterations of simulated GPUs the executor does not own stay modelled.
#include "host/serving.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "host/pool_state.hpp"
#include "host/vmm.hpp"
#include "msim/kvcache_device.hpp"

namespace prism {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

DeviceExecutor::DeviceExecutor(std::vector<int> ordinals, ServingOptions opts) : ordinals_(std::move(ordinals)),
                                                                                opts_(std::move(opts)) {
    if (ordinals_.empty()) throw std::runtime_error("DeviceExecutor: no CUDA device");
}

DeviceExecutor::~DeviceExecutor() {
    for (auto& [k, b] : bufs_) release(b);
    for (auto& [g, d] : devs_) {
        cudaSetDevice(d->ordinal());
        cudaStreamSynchronize(static_cast<cudaStream_t>(d->stream()));
    }
}

bool DeviceExecutor::owns(int gpu) const {
    return opts_.owned.empty() || std::find(opts_.owned.begin(), opts_.owned.end(), gpu) != opts_.owned.end();
}

void DeviceExecutor::release(Buffers& b) {
    if (b.q) cudaFree(b.q);
    if (b.out) cudaFree(b.out);
    if (b.start) cudaEventDestroy(b.start);
    if (b.stop) cudaEventDestroy(b.stop);
    b = Buffers{};
}

void DeviceExecutor::gpu_created(int gpu, msim::engine::GpuState& gs) {
    if (!owns(gpu)) return;
    const int ordinal = ordinals_[static_cast<std::size_t>(gpu) % ordinals_.size()];
    auto dev = VmmDevice::open(ordinal, gs.ledger.page_bytes(), opts_.chunk_pages);
    gs.ledger.attach_device(dev.get());
    devs_[gpu] = std::move(dev);
}

void DeviceExecutor::attached(int gpu, msim::engine::GpuState& gs, int engine_index) {
    if (!owns(gpu)) return;
    msim::engine::Engine& e = gs.engines.at(static_cast<std::size_t>(engine_index));
    const msim::engine::ModelSpec& m = *e.model;
    EngineDeviceOptions o;
    o.max_decode_batch = opts_.max_decode_batch;
    o.max_step_tokens = m.chunk_size + opts_.max_decode_batch + 1;
    attach_engine_device(e, gs.ledger, o);
    Buffers& b = bufs_[{gpu, engine_index}];
    release(b);
    const std::size_t row = static_cast<std::size_t>(m.n_q_heads) * m.head_dim * 2;
    b.rows = std::max(opts_.max_decode_batch, m.chunk_size);
    ck(cudaSetDevice(devs_.at(gpu)->ordinal()), "cudaSetDevice");
    ck(cudaMalloc(&b.q, row * b.rows), "cudaMalloc q");
    ck(cudaMalloc(&b.out, row * b.rows), "cudaMalloc out");
    // q content: small values (attention output magnitude is irrelevant to
    // the timing; numerics are checked by the parity tests)
    ck(cudaMemset(b.q, 0x20, row * b.rows), "cudaMemset q");
    ck(cudaEventCreate(&b.start), "cudaEventCreate");
    ck(cudaEventCreate(&b.stop), "cudaEventCreate");
    ++stats_.attached;
}

void DeviceExecutor::detaching(int gpu, msim::engine::GpuState& gs, int engine_index) {
    if (!owns(gpu)) return;
    const auto it = bufs_.find({gpu, engine_index});
    if (it != bufs_.end()) {
        // the engine's kernels read these buffers: drain its stream first
        ck(cudaStreamSynchronize(static_cast<cudaStream_t>(devs_.at(gpu)->stream())), "cudaStreamSynchronize");
        release(it->second);
        bufs_.erase(it);
    }
    (void)gs;
    ++stats_.detached;
}

void DeviceExecutor::before_step(int gpu, msim::engine::GpuState& gs, int engine_index) {
    if (!owns(gpu) || !opts_.measured) return;
    (void)gs;
    Buffers& b = bufs_.at({gpu, engine_index});
    ck(cudaEventRecord(b.start, static_cast<cudaStream_t>(devs_.at(gpu)->stream())), "cudaEventRecord");
}

msim::SimTime DeviceExecutor::iteration(int gpu, msim::engine::GpuState& gs, int engine_index,
                                        const msim::engine::IterationOutcome& out, msim::SimTime modelled_us) {
    if (!owns(gpu)) return modelled_us;
    (void)out;
    msim::engine::Engine& e = gs.engines.at(static_cast<std::size_t>(engine_index));
    const msim::engine::ModelSpec& m = *e.model;
    Buffers& b = bufs_.at({gpu, engine_index});
    const int n_tok = last_step_tokens(e), n_dec = last_step_decodes(e), n_pf = last_step_prefill_tokens(e);
    const float scale = 1.0f / std::sqrt(static_cast<float>(m.head_dim));
    // PRISM_SERVE_SYNC=1 (diagnosis): synchronise after every launch group
    // and name the one that failed
    static const bool dbg_sync = std::getenv("PRISM_SERVE_SYNC") != nullptr;
    const auto check = [&](const char* what, int layer) {
        if (!dbg_sync) return;
        const cudaError_t err = cudaStreamSynchronize(static_cast<cudaStream_t>(devs_.at(gpu)->stream()));
        if (err != cudaSuccess) {
            throw std::runtime_error(std::string("serving: ") + what + " layer " + std::to_string(layer) + " of " +
                                     m.model_id + " (iteration " + std::to_string(stats_.iterations) + ", tokens " +
                                     std::to_string(n_tok) + ", decodes " + std::to_string(n_dec) + ", prefill " +
                                     std::to_string(n_pf) + "): " + cudaGetErrorString(err));
        }
    };
    check("K1 (engine::step)", -1);
    if (dbg_sync && n_tok > 0) {
        // every slot K2 is about to write must lie in a mapped chunk (a page
        // may already be free again: completions free in the same step)
        const std::vector<std::int32_t> slots = last_step_slots(e);
        const auto* st = e.pools.at(0).state();
        for (const std::int32_t sid : slots) {
            const std::uint64_t page = static_cast<std::uint64_t>(sid) / st->tpp;
            const unsigned cs = devs_.at(gpu)->debug_chunk_state(st->va + page * gs.ledger.page_bytes());
            if (sid < 0 || page >= st->vpages || (cs & 2u) == 0) {
                throw std::runtime_error("serving: step slot " + std::to_string(sid) + " page " + std::to_string(page) +
                                         " occ " + std::to_string(page < st->vpages ? st->occ[page] : 0) +
                                         " chunk state " + std::to_string(cs) + " of " + m.model_id + " (iteration " +
                                         std::to_string(stats_.iterations) + ")");
            }
        }
    }
    if (n_tok > 0) append_step_kv_synthetic(e, 0, m.n_layers, opts_.seed);  // K2
    check("K2", -1);
    for (int layer = 0; layer < m.n_layers; ++layer) {
        if (n_pf > 0) prefill_attention(e, layer, b.q, b.out, scale);  // K4
        check("K4", layer);
        if (n_dec > 0) decode_attention(e, layer, b.q, b.out, scale);  // K3
        check("K3", layer);
    }
    ++stats_.iterations;
    stats_.k2_launches += n_tok > 0;
    stats_.k4_launches += n_pf > 0 ? m.n_layers : 0;
    stats_.k3_launches += n_dec > 0 ? m.n_layers : 0;
    stats_.decode_tokens += static_cast<std::uint64_t>(n_dec);
    stats_.prefill_tokens += static_cast<std::uint64_t>(n_pf);
    if (!opts_.measured) return modelled_us;
    const auto stream = static_cast<cudaStream_t>(devs_.at(gpu)->stream());
    ck(cudaEventRecord(b.stop, stream), "cudaEventRecord");
    ck(cudaEventSynchronize(b.stop), "cudaEventSynchronize");
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, b.start, b.stop), "cudaEventElapsedTime");
    const msim::SimTime us = std::max<msim::SimTime>(1, static_cast<msim::SimTime>(std::llround(ms * 1e3)));
    stats_.gpu_us += static_cast<std::uint64_t>(us);
    stats_.modelled_us += static_cast<std::uint64_t>(std::max<msim::SimTime>(modelled_us, 0));
    return us;
}

void DeviceExecutor::synchronize() {
    for (auto& [g, d] : devs_) {
        ck(cudaSetDevice(d->ordinal()), "cudaSetDevice");
        ck(cudaStreamSynchronize(static_cast<cudaStream_t>(d->stream())), "cudaStreamSynchronize");
    }
}

VmmStats DeviceExecutor::vmm_stats() const {
    VmmStats total;
    for (const auto& [g, d] : devs_) {
        const VmmStats s = d->stats();
        total.maps += s.maps;
        total.unmaps += s.unmaps;
        total.revived += s.revived;
        total.creates += s.creates;
        total.driver_unmaps += s.driver_unmaps;
        total.steals += s.steals;
        total.urgent += s.urgent;
        total.premaps += s.premaps;
        total.map_ns_total += s.map_ns_total;
        total.unmap_ns_total += s.unmap_ns_total;
        total.background_ns_total += s.background_ns_total;
    }
    return total;
}

}  // namespace prism
