// prism::VmmDevice — CUDA virtual-memory backend of one GPU's page ledger.
//
// Implements the physical side of the kvcached-style elastic pool
// (§5.1, "maintains a buffer of pre-allocated and mapped memory
// pages ... overhead fully overlapped with inference computation"; the
// reference only models it: SPEC.md:193 lists real CUDA VMM calls as a
// non-goal). One instance per GPU, attached to that GPU's PhysicalLedger.
//
// Logical pages stay the reference's 2 MiB pages (the ledger, allocator and
// slot ids are bit-exact). Physical memory is managed in CHUNKS of K
// consecutive logical pages of one pool (one cuMemCreate handle of K x 2 MiB,
// mapped with one cuMemMap + one cuMemSetAccess), because every VMM call
// costs the same per handle regardless of its size (measured on B200,
// tools/vmm_granularity_probe.py: create ~70-100 us, map ~1 us, set-access
// ~150-190 us, unmap ~80 us for 2 MiB and for 64 MiB alike), so K = 8 cuts
// the driver time per 2 MiB by 8x. A chunk is
//   live     mapped; at least one of its pages is logically mapped (refs > 0)
//   idle     mapped; no page logically mapped: released by its pool, or
//            mapped ahead by the look-ahead ("clean", never referenced).
//            A logical map into an idle chunk is a revive: no driver call.
//   pending  refs > 0 but not mapped yet: queued on the worker (urgent)
// and handles not mapped anywhere sit in the cache.
//
// Every per-chunk driver call runs on ONE background worker thread per GPU,
// in priority order:
//   1. urgent chunks (FIFO): handle from the cache, a new one within the
//      physical budget, else an idle chunk moved from elsewhere (stolen:
//      cuMemUnmap at its old VA, fence-gated unless clean);
//   2. look-ahead: the chunks of each growing pool's next lowest unmapped
//      pages (exactly what the allocator maps next), from free budget only;
//   3. keeping created handles ready (the ledger's buffer lives here).
// The engine thread never calls the VMM driver on the step path: it revives,
// queues, and waits once per step (defer_access(false)) for its pending
// chunks before launching kernels that touch them. VMM calls stall for 5-50
// ms at random under load and two threads issuing them stall each other
// (tools/vmm_trace_summary.py, tools/e2e_probe.py), so one thread owns them;
// VMM calls on a second thread do not slow kernels or launches
// (tools/vmm_interference.py).
//
// Physical budget: ceil(budget_pages / K) + one partial chunk per reserved
// pool range (the ledger's budget is in pages: capacity - weights).
// Whole-range operations (release, reclaim, budget shrink) are rare and run
// on the caller after waiting for the worker's in-flight work.
#pragma once
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

namespace prism {

struct VmmStats {
    std::uint64_t maps = 0;           // logical page maps requested
    std::uint64_t revived = 0;        // page maps into an already mapped chunk (no driver call)
    std::uint64_t premapped_hits = 0; // ... that revived a chunk the look-ahead mapped
    std::uint64_t creates = 0;        // cuMemCreate calls (chunks)
    std::uint64_t unmaps = 0;         // logical page unmaps
    std::uint64_t driver_unmaps = 0;  // cuMemUnmap calls (chunks)
    std::uint64_t steals = 0;         // idle chunks moved to another VA
    std::uint64_t over_budget = 0;    // urgent maps that found no safe idle chunk and created past the budget
    std::uint64_t premaps = 0;        // chunks mapped by the look-ahead
    std::uint64_t urgent = 0;         // chunks mapped on demand
    std::uint64_t caller_steals_clean = 0;  // steals that took a look-ahead chunk
    std::uint64_t reserve_steals = 0;  // background steals into the handle reserve (PRISM_VMM_RESERVE_CHUNKS)
    double map_ns_total = 0.0;        // caller-thread time in logical maps, incl. waits for the worker
    double unmap_ns_total = 0.0;      // caller-thread time in logical unmaps + reclaims
    double steal_ns_total = 0.0;      // cuMemUnmap time of steals (worker)
    double background_ns_total = 0.0; // worker-thread driver time
    double wait_ns_total = 0.0;       // caller time waiting for the worker (inside map_ns_total)
    std::vector<float> map_ns;        // per logical map, caller thread (bounded)
    std::vector<float> unmap_ns;      // per logical unmap, caller thread (bounded)
    std::vector<float> drv_map_ns;    // per chunk cuMemMap + cuMemSetAccess, worker thread (bounded)
    std::vector<float> drv_create_ns; // per cuMemCreate (bounded)
    std::vector<float> drv_unmap_ns;  // per cuMemUnmap of a steal (bounded)
    double create_ns_total = 0.0;     // inside cuMemCreate
    double map_call_ns_total = 0.0;   // inside cuMemMap
    double access_ns_total = 0.0;     // inside cuMemSetAccess
    std::uint64_t access_calls = 0;
};

class VmmDevice : public std::enable_shared_from_this<VmmDevice> {
public:
    // Opens CUDA device `ordinal`; throws std::runtime_error (CUDA missing,
    // no such device, VMM unsupported, chunk size not a granularity multiple).
    // chunk_pages = 0: PRISM_CHUNK_PAGES or 8. Shared ownership: ledgers and
    // pools keep the device alive.
    static std::shared_ptr<VmmDevice> open(int ordinal, std::uint64_t page_bytes, std::uint64_t chunk_pages = 0);
    ~VmmDevice();

    int ordinal() const { return ordinal_; }
    std::uint64_t page_bytes() const { return page_bytes_; }
    std::uint64_t chunk_pages() const { return chunk_pages_; }

    // VA for `pages` logical pages (rounded up to whole chunks, chunk aligned).
    std::uint64_t reserve(std::uint64_t pages);
    void release(std::uint64_t va, std::uint64_t pages);

    void map(std::uint64_t page_va, bool from_buffer);
    // Logical page maps: pages in mapped chunks revive at once; the rest are
    // queued on the worker. Outside a defer_access(true) window the call
    // waits for them. (Buffer pages are chunks kept in the cache.)
    void map_batch(const std::uint64_t* page_vas, std::size_t n, std::size_t n_from_buffer);
    void unmap(std::uint64_t page_va);
    // defer_access(true): maps return without waiting; defer_access(false):
    // wait until every queued chunk is mapped and accessible.
    void defer_access(bool on);
    void flush_access();
    // Ask the worker to map these pages' chunks ahead of need (a pool's next
    // unmapped pages). `owner` is the pool's VA base; a new hint replaces the
    // pool's old one.
    void premap(std::uint64_t owner, const std::uint64_t* page_vas, std::size_t n);
    void forget(std::uint64_t owner);
    // Keep created handles for `pages` logical pages ready (worker).
    void prefill_cache(std::uint64_t pages);
    // Startup reservation: create physical handles for `pages` logical pages
    // (bounded by the budget) and keep that many ready from now on, so page
    // maps during serving never wait on cuMemCreate (the OS allocation).
    void reserve_physical(std::uint64_t pages);

    // Physically unmap idle chunks (wait=true: all, after draining the worker
    // and the stream; false: released chunks whose fence passed).
    void reclaim(bool wait);
    void* stream() const { return stream_; }
    void fence();

    void grow_buffer(std::uint64_t pages);
    void take_buffer(std::uint64_t pages);
    void set_budget(std::uint64_t pages);
    std::uint64_t buffered_handles() const;  // ledger buffer pages backed here
    std::uint64_t cached_handles() const;    // created, unmapped chunks
    std::uint64_t pending_unmaps() const;    // idle (mapped, unreferenced) chunks
    std::uint64_t total_handles() const;     // all chunks
    std::uint64_t pool_count() const;        // reserved VA ranges (KV pools on this device)
    // Wait until the worker has no queued / in-flight work.
    void quiesce();

    VmmStats stats() const;
    void reset_stats();

    std::uint64_t capacity_pages(std::uint64_t reserve_bytes) const;
    // Diagnosis: state of the chunk holding page_va (bit 0 known, 1 mapped,
    // 2 inflight, 3 queued, 4 referenced, 5 idle).
    unsigned debug_chunk_state(std::uint64_t page_va) const;

private:
    VmmDevice() = default;
    using Lock = std::unique_lock<std::mutex>;
    using Clock = std::chrono::steady_clock;

    struct Chunk {
        std::uint64_t handle = 0;  // physical handle while mapped / in flight
        std::uint32_t refs = 0;    // logically mapped pages
        std::uint64_t epoch = 0;   // fences recorded before its last page left
        bool mapped = false;       // mapped + accessible at this VA
        bool inflight = false;     // the worker is mapping / unmapping it now
        bool queued = false;       // in urgent_
        bool clean = false;        // mapped by the look-ahead, never referenced
        // counted in unready_: a page of it was mapped while the chunk was
        // not; it must be mapped before the step's kernels run even if its
        // pages leave again in the same step (completion frees, preemption):
        // K2 / K3 of that step still touch them
        bool owed = false;
        std::chrono::steady_clock::time_point idle_at{};  // when it last became idle
    };
    using ChunkMap = std::map<std::uint64_t, Chunk>;

    std::uint64_t chunk_of(std::uint64_t page_va) const;
    std::uint64_t total_locked() const;   // chunks holding physical memory
    std::uint64_t budget_chunks() const;  // physical budget in chunks
    bool in_window(std::uint64_t chunk_va) const;
    void set_idle(std::uint64_t va, Chunk& c);
    void drop_if_empty(ChunkMap::iterator it);
    void wait_pending(Lock& lk);
    void check_failed() const;
    void advance_fences(bool wait);
    void fence_locked();
    void unmap_chunk_caller(ChunkMap::iterator it);  // caller-side driver unmap, under mu_
    // worker
    void worker_main();
    bool take_handle(Lock& lk, bool urgent, std::uint64_t& h);
    enum class StealMode { urgent, premap, reserve };
    bool steal_for_worker(Lock& lk, std::uint64_t& h, StealMode mode);
    bool map_chunk(Lock& lk, std::uint64_t va, std::uint64_t h, bool urgent);
    void trace(char kind, std::uint32_t n, Clock::time_point t0, double ns);
    void dump_trace() const;

    int ordinal_ = 0;
    std::uint64_t page_bytes_ = 0;
    std::uint64_t chunk_pages_ = 8;
    std::uint64_t chunk_bytes_ = 0;
    std::uint64_t budget_pages_ = ~0ull >> 8;
    std::uint64_t buffer_pages_ = 0;  // ledger buffer (pages) backed by cached chunks
    mutable std::mutex mu_;
    std::condition_variable cv_;       // worker wakeups
    std::condition_variable done_cv_;  // worker progress
    ChunkMap chunks_;                  // every chunk with refs, a handle or a queue entry
    std::set<std::uint64_t> idle_;     // mapped chunks with refs == 0
    std::uint64_t clean_ = 0;          // idle chunks with clean == true
    std::uint64_t mapped_ = 0;         // chunks holding a handle (mapped or in flight)
    std::uint64_t unready_ = 0;        // chunks with refs > 0 and !mapped
    std::vector<std::uint64_t> cache_;
    std::uint64_t creating_ = 0;       // handles being created on the worker
    std::deque<std::uint64_t> urgent_;
    std::map<std::uint64_t, std::vector<std::uint64_t>> hints_;  // owner -> chunk VAs (reversed)
    std::map<std::uint64_t, std::uint64_t> ranges_;              // reserved VA base -> end
    std::map<std::uint64_t, std::pair<std::uint64_t, std::uint64_t>> window_;  // owner -> [lo, hi) chunk VAs
    std::uint64_t cache_target_ = 0;   // chunks
    std::uint64_t reserve_pending_ = 0; // chunks still to create for reserve_physical() (one-shot)
    std::uint64_t worker_busy_ = 0;
    bool reserve_wanted_ = false;      // an urgent map stole: keep reserve_chunks() handles cached
    bool stop_ = false;
    std::string failed_;  // first driver error on the worker (reported to callers)
    std::thread worker_;
    bool defer_ = false;
    std::vector<void*> fences_;
    std::uint64_t epoch_ = 0;
    std::uint64_t fenced_ = 0;
    VmmStats stats_;
    // PRISM_VMM_TRACE=<path>: every worker driver call and caller wait,
    // written by stats() and at close ("t_ns kind n us"; C create, M urgent
    // map+access, P look-ahead map+access, U steal unmap, W caller wait).
    struct TraceRec {
        std::int64_t t_ns;
        char kind;
        std::uint32_t n;
        float us;
    };
    bool tracing_ = false;
    std::vector<TraceRec> trace_;
    void* access_desc_ = nullptr;
    void* prop_ = nullptr;
    void* stream_ = nullptr;
};

}  // namespace prism
