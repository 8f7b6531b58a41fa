// prism::VmmDevice — CUDA virtual-memory backend of one GPU's page ledger.
//
// Implements the physical side of the kvcached-style elastic pool
// (§5.1; the reference only models it: SPEC.md:193 lists "real CUDA
// VMM calls" as a non-goal). One instance per GPU, attached to that GPU's
// PhysicalLedger; all calls come from the ledger's serialization domain (one
// host thread per GPU), so there are no locks.
//
// Physical pages (2 MiB cuMemCreate handles) are in exactly one state:
//   live     mapped at a pool VA page the ledger counts as mapped
//   parked   still mapped at a pool VA page the ledger has UNMAPPED: a later
//            map of the same page revives it with no driver call
//   buffer   pre-created, counted by the ledger's pre-mapped buffer
//   taken    left the buffer for a map() in progress
//   cached   created, not mapped anywhere
// A logical unmap only parks the page. Driver unmaps happen when a handle is
// needed elsewhere and the physical budget (ledger capacity minus weights) is
// exhausted — the page is then "stolen": cuMemUnmap at its old VA, cuMemMap at
// the new one — or when a pool's VA range is released. A parked page is only
// stolen once the fence recorded after its unmap has passed on the GPU stream
// (kernels issued before the unmap may still read it).
// Maps of fresh pages are batched: contiguous runs share one cuMemSetAccess.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

namespace prism {

struct VmmStats {
    std::uint64_t maps = 0;           // logical page maps requested
    std::uint64_t revived = 0;        // maps satisfied by a parked page at the same VA
    std::uint64_t creates = 0;        // cuMemCreate calls
    std::uint64_t unmaps = 0;         // logical unmaps (parks)
    std::uint64_t driver_unmaps = 0;  // cuMemUnmap calls actually issued
    std::uint64_t steals = 0;         // parked pages moved to another VA
    double map_ns_total = 0.0;        // host wall time of logical maps (incl. steals, creates, SetAccess)
    double unmap_ns_total = 0.0;      // host wall time of logical unmaps + explicit reclaims
    double steal_ns_total = 0.0;      // part of map_ns_total: cuMemUnmap of stolen parked pages
    double prefill_ns_total = 0.0;    // handle creation ahead of need (prefill_cache), off the map path
    std::vector<float> map_ns;        // per logical map (bounded)
    std::vector<float> unmap_ns;      // per logical unmap / driver unmap (bounded)
    double create_ns_total = 0.0;     // inside cuMemCreate
    double map_call_ns_total = 0.0;   // inside cuMemMap
    double access_ns_total = 0.0;     // inside cuMemSetAccess
    std::uint64_t access_calls = 0;
};

class VmmDevice : public std::enable_shared_from_this<VmmDevice> {
public:
    // Opens CUDA device `ordinal`; throws std::runtime_error (CUDA missing,
    // no such device, VMM unsupported, page size not a granularity multiple).
    // Shared ownership: ledgers and pools keep the device alive.
    static std::shared_ptr<VmmDevice> open(int ordinal, std::uint64_t page_bytes);
    ~VmmDevice();

    int ordinal() const { return ordinal_; }
    std::uint64_t page_bytes() const { return page_bytes_; }

    std::uint64_t reserve(std::uint64_t pages);
    void release(std::uint64_t va, std::uint64_t pages);

    void map(std::uint64_t page_va, bool from_buffer);
    void map_batch(const std::uint64_t* page_vas, std::size_t n, std::size_t n_from_buffer);
    void unmap(std::uint64_t page_va);
    // Between defer_access(true) and flush_access() fresh pages are cuMemMap'ed
    // but cuMemSetAccess is postponed and issued once per contiguous run at
    // the flush (the engine brackets a step with it; no kernel may touch the
    // pages before the flush).
    void defer_access(bool on);
    void flush_access();
    // Keep `n` created-but-unmapped handles ready so maps of fresh pages skip
    // cuMemCreate (bounded by the physical budget).
    void prefill_cache(std::uint64_t n);

    // Physically unmap every parked page (wait=true synchronizes first; with
    // wait=false only pages whose fence passed).
    void reclaim(bool wait);
    // The GPU's work stream (cudaStream_t); every engine on this GPU uses it.
    void* stream() const { return stream_; }
    // Record a fence: pages parked before it become stealable once it passes.
    void fence();

    void grow_buffer(std::uint64_t n);
    void take_buffer(std::uint64_t n);
    // Maximum physical pages this device may hold (ledger capacity - weights).
    void set_budget(std::uint64_t pages);
    std::uint64_t buffered_handles() const { return buffer_.size(); }
    std::uint64_t cached_handles() const { return cache_.size(); }
    std::uint64_t pending_unmaps() const { return parked_.size(); }
    std::uint64_t total_handles() const;

    const VmmStats& stats() const { return stats_; }
    void reset_stats();

    std::uint64_t capacity_pages(std::uint64_t reserve_bytes) const;

private:
    VmmDevice() = default;
    std::uint64_t acquire_handle(bool from_buffer);  // a handle not mapped anywhere
    std::uint64_t steal();                           // unmap a parked page, return its handle
    void drop_handle(std::uint64_t h);
    void driver_unmap(std::uint64_t va);
    void advance_fences(bool wait);
    void flush_now();  // issue the pending cuMemSetAccess calls

    struct Parked {
        std::uint64_t handle;
        std::uint64_t epoch;
    };

    int ordinal_ = 0;
    std::uint64_t page_bytes_ = 0;
    std::uint64_t budget_ = ~0ull;
    std::vector<std::uint64_t> buffer_;
    std::vector<std::uint64_t> taken_;
    std::vector<std::uint64_t> cache_;
    std::unordered_map<std::uint64_t, std::uint64_t> live_;  // va -> handle
    std::map<std::uint64_t, Parked> parked_;                // va -> handle (ordered: steal from the top)
    std::vector<std::uint64_t> unaccessed_;  // fresh VAs waiting for cuMemSetAccess
    bool defer_access_ = false;
    std::vector<void*> fences_;       // cudaEvent_t, oldest first; fences_[0] has index fenced_
    std::uint64_t epoch_ = 0;         // fences recorded so far
    std::uint64_t fenced_ = 0;        // fences known complete
    VmmStats stats_;
    void* access_desc_ = nullptr;     // CUmemAccessDesc
    void* prop_ = nullptr;            // CUmemAllocationProp
    void* stream_ = nullptr;          // cudaStream_t
};

}  // namespace prism
