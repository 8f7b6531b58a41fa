// prism::VmmDevice — CUDA virtual-memory backend of one GPU's page ledger.
//
// Implements the physical side of the kvcached-style elastic pool
// (§5.1, "maintains a buffer of pre-allocated and mapped memory
// pages ... overhead fully overlapped with inference computation"; the
// reference only models it: SPEC.md:193 lists real CUDA VMM calls as a
// non-goal). One instance per GPU, attached to that GPU's PhysicalLedger.
//
// Physical pages (2 MiB cuMemCreate handles) are in exactly one state:
//   live     mapped + accessible at a pool VA page the ledger counts as mapped
//   pending  the ledger counts the VA page as mapped, its physical map is
//            queued on the worker (the caller waits for it at sync points)
//   parked   still mapped (with access) at a pool VA page the ledger does not
//            count: either released by the pool (a logical unmap) or
//            pre-mapped by the worker at a page the pool is about to use. A
//            logical map of a parked page is a revive: no driver call.
//   buffer / taken   pre-created handles counted by the ledger's buffer
//   cached   created, not mapped anywhere
//
// Every per-page driver call (cuMemCreate, cuMemMap, cuMemSetAccess and the
// cuMemUnmap that moves a released page to another pool) runs on ONE
// background worker thread per GPU, in priority order:
//   1. urgent maps: pages a pool mapped that were not parked (FIFO),
//      taking a handle from the buffer / cache / new within the budget, else
//      moving a released page of another pool (fence-gated);
//   2. look-ahead: each growing pool's next lowest unmapped pages (exactly
//      the pages the allocator maps next), pre-mapped from free budget only;
//   3. keeping created handles ready.
// The engine thread never calls the VMM driver on the step path: it revives,
// queues, and waits once per step (defer_access(false)) for its urgent pages
// before launching kernels that touch them. Measured on B200: VMM calls
// usually take 0.1-0.4 ms per 2 MiB page (cuMemSetAccess dominates, per page
// not per call) but stall for 5-50 ms at random while kernels run, and two
// threads issuing them concurrently stall each other (tools/vmm_sync_probe.py,
// tools/e2e_probe.py); VMM calls from a second thread do not slow kernels or
// launches (tools/vmm_interference.py).
// Whole-range operations (release, reclaim, budget shrink) are rare and run
// on the caller after waiting for the worker's in-flight work in the range.
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
    std::uint64_t revived = 0;        // maps satisfied by a parked page (no driver call)
    std::uint64_t premapped_hits = 0; // ... of which the worker had pre-mapped
    std::uint64_t creates = 0;        // cuMemCreate calls
    std::uint64_t unmaps = 0;         // logical unmaps (parks)
    std::uint64_t driver_unmaps = 0;  // cuMemUnmap calls
    std::uint64_t steals = 0;         // parked pages moved to another VA
    std::uint64_t batched_unmaps = 0; // unused (kept for ABI)
    std::uint64_t premaps = 0;        // pages pre-mapped by the worker (look-ahead)
    std::uint64_t urgent = 0;         // pages the worker mapped on demand
    std::uint64_t caller_steals_clean = 0;  // steals that took a pre-mapped page
    double map_ns_total = 0.0;        // caller-thread time in logical maps, incl. waits for the worker
    double unmap_ns_total = 0.0;      // caller-thread time in logical unmaps + reclaims
    double steal_ns_total = 0.0;      // cuMemUnmap time of steals (worker)
    double background_ns_total = 0.0; // worker-thread driver time
    double wait_ns_total = 0.0;       // caller time waiting for the worker (inside map_ns_total)
    std::vector<float> map_ns;        // per logical map, caller thread (bounded)
    std::vector<float> unmap_ns;      // per logical unmap, caller thread (bounded)
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
    // Logical maps: parked pages revive at once; the rest are queued on the
    // worker. Outside a defer_access(true) window the call waits for them.
    void map_batch(const std::uint64_t* page_vas, std::size_t n, std::size_t n_from_buffer);
    void unmap(std::uint64_t page_va);
    // defer_access(true): maps return without waiting; defer_access(false):
    // wait until every queued page is mapped and accessible.
    void defer_access(bool on);
    void flush_access();
    // Ask the worker to pre-map these pages (a pool's next unmapped pages).
    // `owner` is the pool's VA base; a new hint replaces the pool's old one.
    void premap(std::uint64_t owner, const std::uint64_t* page_vas, std::size_t n);
    void forget(std::uint64_t owner);  // drop a pool's hint
    // Keep `n` created-but-unmapped handles ready (worker).
    void prefill_cache(std::uint64_t n);

    // Physically unmap parked pages (wait=true: all, after draining the
    // worker and the stream; false: released pages whose fence passed).
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
    // Wait until the worker has no queued / in-flight work.
    void quiesce();

    VmmStats stats() const;
    void reset_stats();

    std::uint64_t capacity_pages(std::uint64_t reserve_bytes) const;

private:
    VmmDevice() = default;
    using Lock = std::unique_lock<std::mutex>;

    struct Parked {
        std::uint64_t handle;
        std::uint64_t epoch;  // fences recorded before its release
        bool clean;           // pre-mapped by the worker, never read by a kernel
    };
    using ParkedMap = std::map<std::uint64_t, Parked>;
    void park(std::uint64_t va, const Parked& p) {
        if (p.clean) ++clean_;
        parked_.emplace(va, p);
    }
    ParkedMap::iterator unpark(ParkedMap::iterator it) {
        if (it->second.clean) --clean_;
        return parked_.erase(it);
    }

    std::uint64_t total_locked() const;
    bool in_window(std::uint64_t va) const;
    bool busy_in(std::uint64_t lo, std::uint64_t hi) const;  // pending / in flight in [lo, hi)
    void wait_pending(Lock& lk);
    void check_failed() const;
    void advance_fences(bool wait);
    void fence_locked();
    void driver_unmap(std::uint64_t va);       // caller-side, under mu_
    std::uint64_t steal_now(Lock& lk);         // caller-side (budget shrink)
    // worker
    void worker_main();
    bool take_handle(Lock& lk, std::uint64_t va, bool urgent, std::uint64_t& h);
    bool steal_for_worker(Lock& lk, std::uint64_t& h);
    void map_run(Lock& lk, std::vector<std::uint64_t>& run, std::vector<std::uint64_t>& hs, bool urgent);

    int ordinal_ = 0;
    std::uint64_t page_bytes_ = 0;
    std::uint64_t budget_ = ~0ull;
    mutable std::mutex mu_;
    std::condition_variable cv_;       // worker wakeups
    std::condition_variable done_cv_;  // worker progress
    std::vector<std::uint64_t> buffer_;
    std::vector<std::uint64_t> taken_;
    std::vector<std::uint64_t> cache_;
    std::unordered_map<std::uint64_t, std::uint64_t> live_;
    ParkedMap parked_;
    std::uint64_t clean_ = 0;                                  // parked pages with clean == true
    std::unordered_map<std::uint64_t, std::uint64_t> pending_; // va -> earmarked buffer handle (0: none)
    std::deque<std::uint64_t> urgent_;                         // pending VAs not yet taken by the worker
    std::unordered_set<std::uint64_t> inflight_;               // VAs the worker maps / unmaps right now
    std::uint64_t inflight_handles_ = 0;                       // handles the worker holds outside every list
    std::uint64_t earmarked_ = 0;                              // buffer handles held in pending_
    std::map<std::uint64_t, std::vector<std::uint64_t>> hints_;  // owner -> next VAs (reversed)
    std::map<std::uint64_t, std::uint64_t> ranges_;              // reserved VA base -> end
    std::map<std::uint64_t, std::pair<std::uint64_t, std::uint64_t>> window_;  // owner -> [lo, hi) of last hint
    std::uint64_t cache_target_ = 0;
    std::uint64_t worker_busy_ = 0;
    bool stop_ = false;
    std::string failed_;  // first driver error on the worker (reported to callers)
    std::thread worker_;
    bool defer_ = false;
    std::vector<void*> fences_;
    std::uint64_t epoch_ = 0;
    std::uint64_t fenced_ = 0;
    VmmStats stats_;
    void* access_desc_ = nullptr;
    void* prop_ = nullptr;
    void* stream_ = nullptr;
};

}  // namespace prism
