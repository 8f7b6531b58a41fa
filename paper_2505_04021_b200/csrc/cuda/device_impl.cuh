// Private declarations shared by the prism-b200 CUDA translation units:
// the GPU-resident slot mirror of a pool (DevicePool) and the GPU half of an
// engine (EngineDeviceImpl).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <unordered_map>
#include <vector>

#include "cuda/common.cuh"
#include "host/engine_device.hpp"
#include "host/paged_op.hpp"
#include "host/pool_state.hpp"
#include "host/vmm.hpp"
#include "msim/kvcache_device.hpp"

namespace prism {

// Device copy of msim::pagealloc::detail::DeviceOp (same layout).
struct DevOp {
    std::uint32_t kind;
    std::uint32_t count;
    std::int64_t dest;
    std::int64_t first;
};
static_assert(sizeof(DevOp) == sizeof(msim::pagealloc::detail::DeviceOp), "DevOp layout");

// Host staging that can be reused only after the copy that read it finished.
template <typename T>
struct Staging {
    T* host = nullptr;    // pinned
    T* dev = nullptr;
    std::size_t cap = 0;
    cudaEvent_t done = nullptr;

    void ensure(std::size_t n) {
        if (done) PRISM_CUDA(cudaEventSynchronize(done));
        if (n <= cap) return;
        release();
        cap = std::max<std::size_t>(n, 256);
        PRISM_CUDA(cudaMallocHost(&host, cap * sizeof(T)));
        PRISM_CUDA(cudaMalloc(&dev, cap * sizeof(T)));
    }
    // Copies host[0, n) to dev on stream and marks the staging busy.
    void upload(std::size_t n, cudaStream_t s) {
        if (!done) PRISM_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        if (n) PRISM_CUDA(cudaMemcpyAsync(dev, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
        PRISM_CUDA(cudaEventRecord(done, s));
    }
    void release() {
        if (host) cudaFreeHost(host);
        if (dev) cudaFree(dev);
        host = nullptr;
        dev = nullptr;
        cap = 0;
    }
    ~Staging() {
        release();
        if (done) cudaEventDestroy(done);
    }
};

// GPU-resident slot state of one pool: occupancy per page and slot bitmaps
// (u32 words). Updated only by K1 from the pool's op log.
class DevicePool {
public:
    DevicePool(const msim::pagealloc::detail::PoolState& s, int device);
    ~DevicePool();
    DevicePool(const DevicePool&) = delete;
    DevicePool& operator=(const DevicePool&) = delete;

    // Replays and clears s.ops / s.freed_slots on `stream`. Slot ids of every
    // logged allocation are written, in order, to out[0 .. total) (out may be
    // null when total == 0) and, for ops with dest >= 0, to table[dest + i].
    // Returns the number of allocated slots.
    std::int64_t replay(msim::pagealloc::detail::PoolState& s, std::int32_t* table, std::int32_t* out,
                        std::int64_t out_cap, cudaStream_t stream);
    int status(cudaStream_t stream);  // 0 = consistent with the host allocator

    std::uint32_t vpages = 0, tpp = 0, words = 0;
    std::uint32_t* occ = nullptr;   // [vpages]
    std::uint32_t* bits = nullptr;  // [vpages * words]
    int* d_status = nullptr;
    Staging<DevOp> ops;
    Staging<std::int32_t> freed;
};

struct TokenMeta {
    std::uint64_t request;  // ~0ull: dead (its request was preempted in the same step)
    std::uint32_t pos;
    std::uint32_t pad;
};

struct DecodeDesc {
    std::int64_t row;
    std::int32_t ctx;
    std::int32_t pad;
    std::uint64_t request;
};


class EngineDeviceImpl final : public EngineDevice {
public:
    EngineDeviceImpl(msim::engine::Engine& eng, msim::pagealloc::PhysicalLedger& ledger,
                     const EngineDeviceOptions& opts);
    ~EngineDeviceImpl() override;

    std::int64_t acquire_row(std::int64_t capacity) override;
    void release_row(std::int64_t row) override;
    void begin_step(msim::engine::Engine& eng) override;
    void end_step(msim::engine::Engine& eng, const msim::engine::IterationOutcome& out,
                  const std::vector<StepDecode>& decodes, std::uint64_t prefill_id, std::int64_t prefill_row,
                  std::int32_t prefill_first, std::int32_t prefill_tokens) override;

    void grow_table(std::int64_t need);
    float* attn_workspace(std::size_t floats);
    int* attn_counters(std::size_t n);

    VmmDevice* vmm = nullptr;
    cudaStream_t stream = nullptr;
    msim::pagealloc::detail::PoolState* pool = nullptr;
    KvGeom geom{};
    int n_q = 0, n_kv = 0, head_dim = 0, group = 0, n_layers = 0;
    EngineDeviceOptions opts;

    // block table arena
    std::int32_t* table = nullptr;
    std::int64_t table_cap = 0;
    std::map<std::int64_t, std::int64_t> free_ranges;        // offset -> length
    std::unordered_map<std::int64_t, std::int64_t> row_len;  // offset -> length

    // last step
    std::int32_t* step_slots = nullptr;  // [max_step_tokens]
    int step_tokens = 0;
    int step_decodes = 0;
    std::vector<std::uint64_t> decode_ids;
    // the last step's prefill chunk (K4): block-table row, first position,
    // query tokens (0: no live chunk), request id
    std::int64_t prefill_row = -1;
    std::int32_t prefill_first = 0, prefill_chunk = 0;
    std::uint64_t prefill_request = 0;
    Staging<TokenMeta> token_meta;
    Staging<DecodeDesc> decode_desc;

    float* workspace = nullptr;
    std::size_t workspace_floats = 0;
    int* counters = nullptr;
    std::size_t counters_n = 0;

    // stream-K K3: pair-tile prefix of the current step (rebuilt once per step)
    std::uint64_t step_serial = 0;
    std::uint64_t sk_step = ~0ull;
    Staging<std::int32_t> sk_prefix;
    Staging<std::int32_t> sk_range_pair;  // first pair of each stream-K CTA range
    int sk_total = 0, sk_per_cta = 1, sk_max_parts = 1;
    std::uint64_t sk_launches = 0;  // selects the CTA range counter (alternate launches)
    // true while the last operation this engine put on `stream` is a
    // stream-K K3 launch (no K1 / K2 / upload / other kernel since): the next
    // K3 may then be launched as a programmatic dependent (PDL) of it.
    bool k3_chain = false;
    // the same for a K4 launch after this engine's own K4 (PDL chain of
    // consecutive prefill-attention layers)
    bool k4_chain = false;
    // K4: key-tile prefix over the Q-tile pairs of the last (first, chunk)
    Staging<std::int32_t> pf_prefix;
    int pf_first = -1, pf_chunk = -1, pf_per_head = 0;

    // host-buffer (end-to-end) path
    cudaStream_t copy_stream = nullptr;
    void* host_stage = nullptr;       // device staging for K/V/q/out: two sets
    int stage_parity = 0;             // set the next call uses
    bool stage_used[2] = {false, false};
    cudaEvent_t stage_free[2] = {nullptr, nullptr};  // recorded after a set's last reader
    std::size_t host_stage_bytes = 0;
    std::vector<cudaEvent_t> host_events;
    cudaEvent_t host_done = nullptr;
};

// K2 / K3 over CALLER-owned block tables (pool-level op, C-ABI
// prism_paged_*): an engine that keeps its own scheduler and slot tables
// (SURVEY §8b's suggested kv_append / decode_attn entry points) uses the
// pool's pages directly. Runs on the pool's VMM stream (so the VMM's release
// fences cover its reads); the same K3 scratch members as EngineDeviceImpl.
struct PagedCtx final : PagedOp {
    PagedCtx(const msim::pagealloc::KvPool& pool, int n_layers, int n_q, int n_kv, int head_dim);
    ~PagedCtx() override;
    PagedCtx(const PagedCtx&) = delete;
    PagedCtx& operator=(const PagedCtx&) = delete;

    // offsets: HOST int32 [n_seqs + 1], non-decreasing, offsets[0] = 0, every
    // sequence >= 1 token; slot_ids: DEVICE int32 [offsets[n_seqs]] (page *
    // tpp + slot, in token order); q / out: device bf16 [n_seqs][n_q][head_dim]
    void decode_attention(int layer, const std::int32_t* offsets, int n_seqs, const std::int32_t* slot_ids,
                          const void* q, void* out, float scale) override;
    // slots: DEVICE int32 [n_tok]; k / v: device bf16 [layer_end - layer_begin][n_tok][n_kv][head_dim]
    void kv_append(int layer_begin, int layer_end, const std::int32_t* slots, int n_tok, const void* k,
                   const void* v) override;
    void prefill_attention(int layer, const std::int32_t* slot_ids, int first, int n_tokens, const void* q, void* out,
                           float scale) override;

    float* attn_workspace(std::size_t floats);
    int* attn_counters(std::size_t n);

    VmmDevice* vmm = nullptr;
    cudaStream_t stream = nullptr;
    KvGeom geom{};
    int n_q = 0, n_kv = 0, head_dim = 0, group = 0, n_layers = 0;
    Staging<DecodeDesc> decode_desc;
    Staging<TokenMeta> token_meta;  // all live (K2 skips dead tokens only in engine steps)
    Staging<std::int32_t> sk_prefix;
    Staging<std::int32_t> sk_range_pair;  // first pair of each stream-K CTA range
    std::uint64_t step_serial = 0, sk_step = ~0ull;
    int sk_total = 0, sk_per_cta = 1, sk_max_parts = 1;
    std::uint64_t sk_launches = 0;  // selects the CTA range counter (alternate launches)
    bool k3_chain = false;
    // the same for a K4 launch after this engine's own K4 (PDL chain of
    // consecutive prefill-attention layers)
    bool k4_chain = false;
    // K4: key-tile prefix over the Q-tile pairs of the last (first, chunk)
    Staging<std::int32_t> pf_prefix;
    int pf_first = -1, pf_chunk = -1, pf_per_head = 0;
    float* workspace = nullptr;
    std::size_t workspace_floats = 0;
    int* counters = nullptr;
    std::size_t counters_n = 0;
};

EngineDeviceImpl& impl_of(const msim::engine::Engine& eng);

}  // namespace prism
