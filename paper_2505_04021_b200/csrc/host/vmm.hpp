// prism::VmmDevice — CUDA virtual-memory backend of one GPU's page ledger.
//
// Implements the physical side of the kvcached-style elastic pool
// (§5.1, "maintains a buffer of pre-allocated and mapped memory
// pages ... overhead fully overlapped with inference computation"; the
// reference only models it: SPEC.md:193 lists real CUDA VMM calls as a
// non-goal). One instance per GPU, attached to that GPU's PhysicalLedger.
//
// Physical pages (2 MiB cuMemCreate handles) are in exactly one state:
//   live     mapped at a pool VA page the ledger counts as mapped
//   parked   still mapped (with access) at a pool VA page the ledger does not
//            count: either released by the pool (a logical unmap) or
//            pre-mapped by the background worker at a page the pool is about
//            to use. A logical map of a parked page is a revive: no driver call.
//   buffer / taken   pre-created handles counted by the ledger's buffer
//   cached   created, not mapped anywhere
// Driver work happens
//   * on the background worker thread: cuMemCreate of ready handles, and
//     cuMemMap + cuMemSetAccess of each active pool's next pages (the lowest
//     unmapped indices — exactly the pages the allocator maps next), taking
//     released (dirty parked) pages of other pools when the physical budget
//     (ledger capacity - weights) is exhausted;
//   * on the caller's thread only for maps the worker did not anticipate.
// Measured on B200: cuMemSetAccess ~170-200 us per 2 MiB page (the dominant
// cost), cuMemUnmap ~80-110 us, cuMemCreate ~70-90 us, cuMemMap ~2 us; VMM
// calls from a second host thread do not slow kernels or launches
// (tools/vmm_interference.py), so the worker hides them.
// A parked page released by a pool is stolen only after the fence recorded
// after its release has passed on the GPU stream.
#pragma once
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace prism {

struct VmmStats {
    std::uint64_t maps = 0;           // logical page maps requested
    std::uint64_t revived = 0;        // maps satisfied by a parked page (no driver call on the map path)
    std::uint64_t premapped_hits = 0; // ... of which the worker had pre-mapped
    std::uint64_t creates = 0;        // cuMemCreate calls (any thread)
    std::uint64_t unmaps = 0;         // logical unmaps (parks)
    std::uint64_t driver_unmaps = 0;  // cuMemUnmap calls (any thread)
    std::uint64_t steals = 0;         // parked pages moved to another VA (any thread)
    std::uint64_t batched_unmaps = 0; // cuMemUnmap calls that covered a run of >1 pages
    std::uint64_t premaps = 0;        // pages pre-mapped by the worker
    double map_ns_total = 0.0;        // caller-thread wall time of logical maps
    double unmap_ns_total = 0.0;      // caller-thread wall time of logical unmaps + reclaims
    double steal_ns_total = 0.0;      // caller-thread cuMemUnmap time of steals (inside map_ns_total)
    double background_ns_total = 0.0; // worker-thread driver time (create / map / access / steal)
    std::vector<float> map_ns;        // per logical map, caller thread (bounded)
    std::vector<float> unmap_ns;      // per logical unmap, caller thread (bounded)
    double create_ns_total = 0.0;     // inside cuMemCreate (any thread)
    double map_call_ns_total = 0.0;   // inside cuMemMap (any thread)
    double access_ns_total = 0.0;     // inside cuMemSetAccess (any thread)
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
    // Between defer_access(true) and defer_access(false) fresh caller-thread
    // maps postpone cuMemSetAccess to one call per contiguous run.
    void defer_access(bool on);
    void flush_access();
    // Ask the worker to pre-map these pages (a pool's next unmapped pages).
    // `owner` identifies the pool; a new hint replaces that pool's old one.
    void premap(std::uint64_t owner, const std::uint64_t* page_vas, std::size_t n);
    void forget(std::uint64_t owner);  // drop a pool's hint (pool released)
    // Keep `n` created-but-unmapped handles ready (worker).
    void prefill_cache(std::uint64_t n);

    // Physically unmap parked pages (wait=true: all, after draining the
    // stream; false: those whose fence passed).
    void reclaim(bool wait);
    void* stream() const { return stream_; }
    void fence();

    void grow_buffer(std::uint64_t n);
    void take_buffer(std::uint64_t n);
    void set_budget(std::uint64_t pages);
    std::uint64_t buffered_handles() const;
    std::uint64_t cached_handles() const;
    std::uint64_t pending_unmaps() const;
    std::uint64_t total_handles() const;
    // Wait until the worker has no queued / in-flight work (tests).
    void quiesce();

    VmmStats stats() const;
    void reset_stats();

    std::uint64_t capacity_pages(std::uint64_t reserve_bytes) const;

private:
    VmmDevice() = default;
    using Lock = std::unique_lock<std::mutex>;
    std::uint64_t total_locked() const;
    std::uint64_t acquire_handle(Lock& lk, bool from_buffer);
    std::uint64_t steal(Lock& lk);
    void steal_batch(Lock& lk, std::size_t k);
    void driver_unmap(std::uint64_t va);  // unlocked driver call + stats
    void advance_fences(bool wait);
    void flush_now(Lock& lk);
    void fence_locked();
    void wait_inflight(Lock& lk, std::uint64_t va);
    void worker_main();

    struct Parked {
        std::uint64_t handle;
        std::uint64_t epoch;  // fences recorded before its release
        bool clean;           // pre-mapped by the worker, never read by a kernel
    };

    int ordinal_ = 0;
    std::uint64_t page_bytes_ = 0;
    std::uint64_t budget_ = ~0ull;
    mutable std::mutex mu_;
    std::condition_variable cv_;       // worker wakeups
    std::condition_variable done_cv_;  // in-flight maps finished
    std::vector<std::uint64_t> buffer_;
    std::vector<std::uint64_t> taken_;
    std::vector<std::uint64_t> cache_;
    std::unordered_map<std::uint64_t, std::uint64_t> live_;
    std::map<std::uint64_t, Parked> parked_;
    std::unordered_set<std::uint64_t> inflight_;  // VAs the worker is mapping
    std::map<std::uint64_t, std::vector<std::uint64_t>> hints_;  // owner -> next VAs
    std::uint64_t cache_target_ = 0;
    std::uint64_t worker_busy_ = 0;
    std::uint64_t inflight_handles_ = 0;  // handles the worker holds outside every list
    bool stop_ = false;
    std::thread worker_;
    std::vector<std::uint64_t> unaccessed_;
    bool defer_access_ = false;
    std::vector<void*> fences_;
    std::uint64_t epoch_ = 0;
    std::uint64_t fenced_ = 0;
    VmmStats stats_;
    void* access_desc_ = nullptr;
    void* prop_ = nullptr;
    void* stream_ = nullptr;
};

}  // namespace prism
