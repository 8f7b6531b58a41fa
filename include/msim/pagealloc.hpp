// prism-b200 — elastic KV memory: per-GPU page ledger + per-model virtual KV
// pools with token-slot allocation.
//
// Drop-in for reference proj/include/msim/pagealloc.hpp (same namespace,
// type names, public members and free-function signatures; the reference's
// own tests compile unchanged against it). What differs is underneath:
//   * pick_page is O(log V) (segment tree over page occupancy + hierarchical
//     bitsets) instead of the reference's O(V) scan (pagealloc.cpp:158-186);
//     the chosen (page, slot) sequence is identical.
//   * with a prism::VmmDevice attached to the ledger, every logical map /
//     unmap is a real CUDA VMM operation on the pool's reserved VA range
//     (2 MiB physical pages, cuMemCreate / cuMemMap / cuMemSetAccess /
//     cuMemUnmap), buffer pages are pre-created physical handles, and each
//     pool records an op log that the batched device allocator (K1) replays
//     against GPU-resident slot state.
// Without a device the ledger is pure accounting, exactly like the reference.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "msim/core.hpp"

namespace prism {
class VmmDevice;  // csrc/cuda/vmm.cu
}

namespace msim::pagealloc {

using PoolId = std::uint32_t;

// One token's KV slot: page index inside the pool's virtual range and slot
// index inside that page (reference pagealloc.hpp:16-24).
struct TokenSlotHandle {
    PoolId pool = 0;
    std::uint32_t page = 0;
    std::uint32_t slot = 0;
    friend bool operator==(const TokenSlotHandle& x, const TokenSlotHandle& y) {
        return x.pool == y.pool && x.page == y.page && x.slot == y.slot;
    }
};

enum class PagePlacement { most_occupied_first, lowest_index_first };

enum class AllocEventKind { map, unmap, buffer_hit, alloc_fail };
const char* to_string(AllocEventKind k);

struct AllocEvent {
    SimTime time_us = 0;
    int gpu_id = 0;
    std::string model_id;  // "" for buffer refills
    AllocEventKind kind = AllocEventKind::map;
    std::uint64_t pages = 0;
};

struct AllocResult {
    std::vector<TokenSlotHandle> handles;
    std::uint64_t shortfall_pages = 0;  // non-zero => nothing was committed
    std::uint64_t pages_mapped = 0;     // new pages not covered by the buffer
    std::uint64_t buffer_hits = 0;      // new pages served by the buffer
    bool ok() const { return shortfall_pages == 0; }
};

class KvPool;
namespace detail {
struct Access;     // the allocator internals (csrc/host/pagealloc.cpp)
struct PoolState;  // per-pool page/slot state (csrc/host/pool_state.hpp)
}  // namespace detail

// Page budget of one GPU. Weights, every model's mapped KV pages and the
// pre-mapped buffer draw from `capacity_pages`. One ledger (with its pools) is
// one serialization domain; different GPUs' ledgers are independent.
class PhysicalLedger {
public:
    PhysicalLedger(int gpu_id, std::uint64_t capacity_pages,
                   std::uint64_t page_bytes = defaults::kPageBytes);

    int gpu_id() const { return gpu_; }
    std::uint64_t page_bytes() const { return page_bytes_; }
    std::uint64_t capacity_pages() const { return capacity_; }
    std::uint64_t mapped_pages() const { return kv_pages_; }
    std::uint64_t buffer_pages() const { return buffer_; }
    std::uint64_t weight_pages() const { return weights_; }
    std::uint64_t free_pages() const { return capacity_ - kv_pages_ - buffer_ - weights_; }
    std::uint64_t pool_mapped_pages(PoolId id) const;

    std::uint64_t refill_buffer(std::uint64_t target_pages);

    bool reserve_weight_pages(const std::string& model_id, std::uint64_t pages);
    void release_weight_pages(const std::string& model_id);
    std::uint64_t weight_pages_of(const std::string& model_id) const;

    void set_time(SimTime now_us) { now_ = now_us; }
    void set_recording(bool on) { recording_ = on; }
    const std::vector<AllocEvent>& events() const { return log_; }
    void clear_events() { log_.clear(); }

    void check_invariants() const;

    // ---- prism-b200 extension: real memory behind the accounting ----------
    // Attach before creating pools. Not owned; must outlive the ledger's pools.
    void attach_device(prism::VmmDevice* dev);
    prism::VmmDevice* device() const { return dev_; }

private:
    friend struct detail::Access;

    struct PoolEntry {
        std::string model;
        std::uint64_t pages = 0;
    };

    void note(const std::string& model, AllocEventKind kind, std::uint64_t pages);

    int gpu_;
    std::uint64_t page_bytes_;
    std::uint64_t capacity_;
    std::uint64_t kv_pages_ = 0;
    std::uint64_t buffer_ = 0;
    std::uint64_t weights_ = 0;
    PoolId next_id_ = 1;
    std::map<PoolId, PoolEntry> pools_;
    std::map<std::string, std::uint64_t> weight_by_model_;
    SimTime now_ = 0;
    bool recording_ = false;
    std::vector<AllocEvent> log_;
    prism::VmmDevice* dev_ = nullptr;
    std::shared_ptr<prism::VmmDevice> dev_hold_;  // keeps the device alive
};

// One model's virtual KV range. Pages are mapped only when a token needs them
// and unmapped the moment their last token is freed. Move-only.
class KvPool {
public:
    KvPool(KvPool&&) noexcept;
    KvPool& operator=(KvPool&&) noexcept;
    KvPool(const KvPool&) = delete;
    KvPool& operator=(const KvPool&) = delete;
    ~KvPool();

    PoolId id() const;
    const std::string& model_id() const;
    std::uint64_t token_bytes() const;
    std::uint64_t tokens_per_page() const;
    std::uint64_t virtual_capacity_pages() const;
    std::uint64_t mapped_pages() const;
    std::uint64_t occupied_slots() const;
    std::uint64_t free_slots_in_mapped() const { return mapped_pages() * tokens_per_page() - occupied_slots(); }
    bool alive() const;

    void set_mapped_page_cap(std::optional<std::uint64_t> cap);
    std::optional<std::uint64_t> mapped_page_cap() const;

    std::uint64_t allocatable_tokens(const PhysicalLedger& ledger) const;
    bool can_alloc(const PhysicalLedger& ledger, std::uint64_t num_tokens) const {
        return num_tokens <= allocatable_tokens(ledger);
    }

    bool page_mapped(std::uint32_t page) const;
    std::uint64_t page_occupied(std::uint32_t page) const;

    // ---- prism-b200 extensions --------------------------------------------
    // Base device VA of page 0 (0 when the ledger has no device).
    std::uint64_t device_base() const;
    detail::PoolState* state() const { return st_.get(); }

private:
    friend struct detail::Access;
    KvPool();
    std::unique_ptr<detail::PoolState> st_;
};

KvPool alloc_kvcache(PhysicalLedger& ledger, const std::string& model_id,
                     std::uint64_t token_bytes, std::uint64_t virtual_capacity_pages,
                     PagePlacement placement = PagePlacement::most_occupied_first);
void free_kvcache(PhysicalLedger& ledger, KvPool& pool);
AllocResult alloc_kv(KvPool& pool, PhysicalLedger& ledger, std::uint64_t num_tokens);
void free_kv(KvPool& pool, PhysicalLedger& ledger, const std::vector<TokenSlotHandle>& handles);
std::uint64_t refill_buffer(PhysicalLedger& ledger, std::uint64_t target_pages);

}  // namespace msim::pagealloc
