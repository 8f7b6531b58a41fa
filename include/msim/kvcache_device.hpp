// prism-b200 — GPU data path of the elastic KV cache (new API; the reference
// has no counterpart: it writes no K/V and has no attention operator,
// SPEC.md:193 / :278).
//
//   attach_engine_device   give a serving engine (one TP part) its GPU half:
//                          device slot mirror of its pool, device block table,
//                          step descriptors, attention workspace.
//   engine::step()         unchanged API; with a device attached it also
//                          launches K1 (batched slot allocation / free on the
//                          GPU-resident slot state, block-table update).
//   append_step_kv         K2: scatter this step's new K/V rows into pages.
//   decode_attention       K3: paged GQA decode attention (bf16 in, fp32
//                          accumulation, split-K) for the requests that
//                          decoded in the last step, one layer per call.
// All device work is asynchronous on the GPU's stream (VmmDevice::stream(),
// engine_stream()); device buffers passed in (K/V, q) must be complete in that
// stream's order and outputs are ready in it — a caller producing them on
// another stream orders the two (event / stream wait), as with any library
// stream.
// Every function throws std::runtime_error when CUDA is unavailable — there
// is no CPU fallback.
#pragma once
#include <cstdint>
#include <vector>

#include "msim/engine.hpp"
#include "msim/pagealloc.hpp"

namespace prism {

class VmmDevice;

struct EngineDeviceOptions {
    std::int64_t table_capacity = 1 << 20;  // initial block-table arena (int32 elements); grows on demand
    int max_decode_batch = 1024;            // requests decoding in one step
    int max_step_tokens = 8192;             // slots allocated in one step (prefill chunk + decodes)
};

// Requires eng.model with the attention shape set, eng.pools.size() == 1 and
// the ledger's VmmDevice. Call right after finish_activation(), before step().
void attach_engine_device(msim::engine::Engine& eng, msim::pagealloc::PhysicalLedger& ledger,
                          const EngineDeviceOptions& opts = {});

// Number of slots allocated by the last step (prefill chunk tokens first, then
// one per decoded request in admission order) and number of decoded requests.
int last_step_tokens(const msim::engine::Engine& eng);
int last_step_decodes(const msim::engine::Engine& eng);
// Ids of the requests that decoded in the last step, in the order used by
// decode_attention's q / out rows.
const std::vector<std::uint64_t>& last_step_decode_ids(const msim::engine::Engine& eng);

// K2. k, v: device bf16 tensors [layer_end - layer_begin][last_step_tokens][n_kv][head_dim].
void append_step_kv(msim::engine::Engine& eng, int layer_begin, int layer_end, const void* k, const void* v);

// K2 with generated content: writes synth_value(seed, request, position, ...)
// for this step's slots (tests and benchmarks; oracle-checkable).
void append_step_kv_synthetic(msim::engine::Engine& eng, int layer_begin, int layer_end, std::uint64_t seed);

// K3. q, out: device bf16 [last_step_decodes][n_q_heads][head_dim]; scale is
// applied to q·k (pass 1/sqrt(head_dim) for standard attention).
void decode_attention(msim::engine::Engine& eng, int layer, const void* q, void* out, float scale);

// K4 (chunked-prefill attention, tcgen05/TMEM): causal attention of the last
// step's prefill chunk over its request's pages. q, out: device bf16
// [last_step_prefill_tokens][n_q_heads][head_dim]; query i sits at position
// last_step_prefill_first + i and attends keys 0..that position (the chunk's
// own K/V must have been appended, K2). head_dim 64 or 128.
void prefill_attention(msim::engine::Engine& eng, int layer, const void* q, void* out, float scale);
// Query tokens of the last step's prefill chunk (0: none, or it was preempted
// in the same step), the position of its first token and its request id.
int last_step_prefill_tokens(const msim::engine::Engine& eng);
int last_step_prefill_first(const msim::engine::Engine& eng);
std::uint64_t last_step_prefill_request(const msim::engine::Engine& eng);

// End-to-end decode with HOST buffers for the last step: H2D of the new K/V
// rows ([n_layers][last_step_tokens][n_kv][head_dim], may be null) and q
// ([n_layers][last_step_decodes][n_q][head_dim]) on the engine's copy
// stream, K2 + one K3 per layer on the compute stream, D2H of out (same shape
// as q) layer by layer as each K3 finishes. wait=false returns once enqueued
// (wait_host() blocks until `out` is complete).
void decode_host(msim::engine::Engine& eng, const void* new_k, const void* new_v, const void* q, void* out,
                 float scale, bool wait);
void wait_host(const msim::engine::Engine& eng);

// Fills q [last_step_decodes][n_q][head_dim] with synth content (kind = Q, at
// each request's newest position) times q_scale.
void synth_decode_q(msim::engine::Engine& eng, int layer, std::uint64_t seed, float q_scale, void* q);

// Test hooks (synchronous): device copies of the last step's slot ids and of
// the slot-state mirror.
std::vector<std::int32_t> last_step_slots(const msim::engine::Engine& eng);
std::vector<std::int32_t> read_table_row(const msim::engine::Engine& eng, std::int64_t row, int len);
void* engine_stream(const msim::engine::Engine& eng);

// Pool-level device mirror without an engine (C-ABI / tests): create the
// mirror, replay the pool's pending op log on the GPU (K1) and return the slot
// ids every logged allocation produced, in order.
void attach_pool_mirror(msim::pagealloc::KvPool& pool);
std::vector<std::int32_t> sync_pool_mirror(msim::pagealloc::KvPool& pool);
// Mirror state readback: occupancy per page and slot bitmaps (u32 words).
void read_pool_mirror(msim::pagealloc::KvPool& pool, std::vector<std::uint32_t>& occ,
                      std::vector<std::uint32_t>& bits);

}  // namespace prism
