// prism::VmmDevice implementation: CUDA VMM (driver API) behind the ledger,
// in chunks of K logical pages (see host/vmm.hpp).
// Driver entry points are resolved at run time through the runtime's
// cudaGetDriverEntryPoint, so the library loads on machines without a driver
// (the CPU build/test container) and only fails when a device is opened.
//
// Threading: every public method takes mu_. The worker drops mu_ around its
// driver calls and marks the chunk it works on `inflight`; callers never
// wait for an in-flight chunk except at sync points (wait_pending) and in
// whole-range operations.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cstring>

#include "cuda/common.cuh"
#include "host/vmm.hpp"

namespace prism {

namespace {

struct Driver {
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    decltype(&cuDeviceGetAttribute) attribute = nullptr;
    bool loaded = false;
};

Driver& drv() {
    static Driver d;
    return d;
}

template <typename F>
void resolve(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    PRISM_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw std::runtime_error(std::string("driver symbol missing: ") + name);
    fn = reinterpret_cast<F>(p);
}

void load_driver() {
    static std::mutex once;
    std::lock_guard<std::mutex> g(once);
    Driver& d = drv();
    if (d.loaded) return;
    resolve("cuMemAddressReserve", d.reserve);
    resolve("cuMemAddressFree", d.addr_free);
    resolve("cuMemCreate", d.create);
    resolve("cuMemRelease", d.release);
    resolve("cuMemMap", d.map);
    resolve("cuMemUnmap", d.unmap);
    resolve("cuMemSetAccess", d.set_access);
    resolve("cuMemGetAllocationGranularity", d.granularity);
    resolve("cuDeviceGetAttribute", d.attribute);
    d.loaded = true;
}

void cu_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw std::runtime_error(std::string("CUDA driver error ") + std::to_string(r) + " in " + what);
}

using Clock = std::chrono::steady_clock;
double ns_since(Clock::time_point t0) { return std::chrono::duration<double, std::nano>(Clock::now() - t0).count(); }

constexpr std::size_t kMaxSamples = 1 << 16;
void sample(std::vector<float>& ring, double ns) {
    if (ring.size() < kMaxSamples) ring.push_back(static_cast<float>(ns));
}

// Minimum idle time of a chunk a look-ahead map may steal.
std::chrono::steady_clock::duration premap_steal_age() {
    static const auto age = [] {
        const char* e = std::getenv("PRISM_VMM_PREMAP_STEAL_AGE_MS");
        return std::chrono::duration_cast<std::chrono::steady_clock::duration>(
            std::chrono::duration<double, std::milli>(e ? std::atof(e) : 200.0));
    }();
    return age;
}
// Idle chunks moved per steal (one cuMemUnmap over a contiguous run).
constexpr int kStealBatch = 8;
// ... and per steal an urgent map waits for (PRISM_VMM_URGENT_STEAL_BATCH).
int urgent_steal_batch() {
    static const int n = [] {
        const char* e = std::getenv("PRISM_VMM_URGENT_STEAL_BATCH");
        return e ? std::max(1, std::min(kStealBatch, std::atoi(e))) : kStealBatch;
    }();
    return n;
}
// Background reserve: once an urgent map had to steal (the budget is spent),
// the worker keeps up to PRISM_VMM_RESERVE_CHUNKS unmapped handles ready by
// stealing safe idle chunks outside every window while it has nothing else
// to do, PRISM_VMM_RESERVE_BATCH chunks per cuMemUnmap, so the next urgent
// maps take a cached handle instead of waiting for an unmap.
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
std::uint64_t reserve_chunks() {
    static const std::uint64_t n = static_cast<std::uint64_t>(std::max(0, env_int("PRISM_VMM_RESERVE_CHUNKS", 8)));
    return n;
}
int reserve_batch() {
    static const int n = std::max(1, std::min(kStealBatch, env_int("PRISM_VMM_RESERVE_BATCH", 2)));
    return n;
}
// How many in-window idle chunks a steal skips over looking for one outside
// every look-ahead window (bounds the scan).
constexpr int kStealScan = 256;
// At most this many logical pages are mapped ahead by the look-ahead (2 GiB).
constexpr std::uint64_t kMaxCleanPages = 1024;

CUmemAllocationProp& prop_of(void* p) { return *static_cast<CUmemAllocationProp*>(p); }
CUmemAccessDesc& access_of(void* p) { return *static_cast<CUmemAccessDesc*>(p); }

}  // namespace

std::shared_ptr<VmmDevice> VmmDevice::open(int ordinal, std::uint64_t page_bytes, std::uint64_t chunk_pages) {
    int count = 0;
    PRISM_CUDA(cudaGetDeviceCount(&count));
    if (ordinal < 0 || ordinal >= count) throw std::runtime_error("VmmDevice: no CUDA device " + std::to_string(ordinal));
    PRISM_CUDA(cudaSetDevice(ordinal));
    PRISM_CUDA(cudaFree(nullptr));  // create the primary context
    load_driver();
    int vmm = 0;
    cu_check(drv().attribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, ordinal),
             "cuDeviceGetAttribute");
    if (!vmm) throw std::runtime_error("VmmDevice: device does not support virtual memory management");
    if (chunk_pages == 0) {
        const char* e = std::getenv("PRISM_CHUNK_PAGES");
        chunk_pages = e ? static_cast<std::uint64_t>(std::max(1, std::atoi(e))) : 8;
    }

    std::shared_ptr<VmmDevice> dev(new VmmDevice());
    dev->ordinal_ = ordinal;
    dev->page_bytes_ = page_bytes;
    dev->chunk_pages_ = chunk_pages;
    dev->chunk_bytes_ = page_bytes * chunk_pages;
    auto* prop = new CUmemAllocationProp();
    std::memset(prop, 0, sizeof(*prop));
    prop->type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop->location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop->location.id = ordinal;
    dev->prop_ = prop;
    auto* acc = new CUmemAccessDesc();
    acc->location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc->location.id = ordinal;
    acc->flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    dev->access_desc_ = acc;
    std::size_t gran = 0;
    cu_check(drv().granularity(&gran, prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "cuMemGetAllocationGranularity");
    if (gran == 0 || page_bytes % gran != 0) {
        throw std::runtime_error("VmmDevice: page size is not a multiple of the VMM granularity (" +
                                 std::to_string(gran) + ")");
    }
    cudaStream_t s = nullptr;
    PRISM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    dev->stream_ = s;
    dev->tracing_ = std::getenv("PRISM_VMM_TRACE") != nullptr;
    dev->worker_ = std::thread([raw = dev.get()] { raw->worker_main(); });
    return dev;
}

void VmmDevice::trace(char kind, std::uint32_t n, Clock::time_point t0, double ns) {
    if (!tracing_ || trace_.size() >= (1u << 20)) return;
    const auto t = std::chrono::duration_cast<std::chrono::nanoseconds>(t0.time_since_epoch()).count();
    trace_.push_back(TraceRec{static_cast<std::int64_t>(t), kind, n, static_cast<float>(ns / 1e3)});
}

void VmmDevice::dump_trace() const {
    if (!tracing_) return;
    if (FILE* f = std::fopen(std::getenv("PRISM_VMM_TRACE"), "w")) {
        for (const TraceRec& r : trace_) {
            std::fprintf(f, "%lld %c %u %.1f\n", static_cast<long long>(r.t_ns), r.kind, r.n, r.us);
        }
        std::fclose(f);
    }
}

VmmDevice::~VmmDevice() {
    {
        Lock lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    if (worker_.joinable()) worker_.join();
    dump_trace();
    try {
        cudaSetDevice(ordinal_);
        cudaDeviceSynchronize();
        for (auto& [va, c] : chunks_) {
            if (c.mapped) drv().unmap(va, chunk_bytes_);
            if (c.handle) drv().release(c.handle);
        }
        for (auto h : cache_) drv().release(h);
        for (void* e : fences_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
        if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
    } catch (...) {
    }
    delete static_cast<CUmemAllocationProp*>(prop_);
    delete static_cast<CUmemAccessDesc*>(access_desc_);
}

// ---------------------------------------------------------------- bookkeeping

std::uint64_t VmmDevice::chunk_of(std::uint64_t page_va) const {
    auto r = ranges_.upper_bound(page_va);
    if (r == ranges_.begin()) throw std::runtime_error("VmmDevice: address outside every reserved range");
    --r;
    return r->first + (page_va - r->first) / chunk_bytes_ * chunk_bytes_;
}

std::uint64_t VmmDevice::total_locked() const { return mapped_ + cache_.size() + creating_; }

std::uint64_t VmmDevice::budget_chunks() const {
    return (budget_pages_ + chunk_pages_ - 1) / chunk_pages_ + ranges_.size();
}

bool VmmDevice::in_window(std::uint64_t chunk_va) const {
    auto r = ranges_.upper_bound(chunk_va);
    if (r == ranges_.begin()) return false;
    --r;
    const auto w = window_.find(r->first);
    return w != window_.end() && chunk_va >= w->second.first && chunk_va < w->second.second;
}

void VmmDevice::set_idle(std::uint64_t va, Chunk& c) {
    idle_.insert(va);
    c.idle_at = Clock::now();
    if (c.clean) ++clean_;
}

void VmmDevice::drop_if_empty(ChunkMap::iterator it) {
    const Chunk& c = it->second;
    if (!c.mapped && !c.inflight && !c.queued && !c.owed && c.refs == 0 && c.handle == 0) chunks_.erase(it);
}

void VmmDevice::check_failed() const {
    if (!failed_.empty()) throw std::runtime_error("VmmDevice worker: " + failed_);
}

void VmmDevice::wait_pending(Lock& lk) {
    if (unready_ == 0) return;
    const auto tw = Clock::now();
    cv_.notify_one();
    done_cv_.wait(lk, [&] { return unready_ == 0 || !failed_.empty(); });
    const double ns = ns_since(tw);
    stats_.wait_ns_total += ns;
    trace('W', 0, tw, ns);
    check_failed();
}

// ---------------------------------------------------------------- worker

bool VmmDevice::take_handle(Lock& lk, bool urgent, std::uint64_t& h) {
    // A handle for the chunk in flight: cached, new within the physical
    // budget, or (urgent only) moved from an idle chunk; counted in mapped_.
    if (!cache_.empty()) {
        h = cache_.back();
        cache_.pop_back();
        ++mapped_;
        return true;
    }
    const auto create = [&]() {
        ++creating_;
        lk.unlock();
        CUmemGenericAllocationHandle ch = 0;
        const auto tc = Clock::now();
        const CUresult r = drv().create(&ch, chunk_bytes_, &prop_of(prop_), 0);
        const double ns = ns_since(tc);
        lk.lock();
        --creating_;
        if (r != CUDA_SUCCESS) return false;
        h = static_cast<std::uint64_t>(ch);
        ++mapped_;
        ++stats_.creates;
        stats_.create_ns_total += ns;
        sample(stats_.drv_create_ns, ns);
        trace('C', 1, tc, ns);
        return true;
    };
    if (total_locked() < budget_chunks() && create()) return true;
    if (!urgent) {
        // Look-ahead steals move memory to growing pools ahead of need, but
        // only chunks idle for at least PRISM_VMM_PREMAP_STEAL_AGE_MS (a
        // model that went quiet): stealing recently released chunks moved
        // memory back and forth (C2 churn: ~40% more driver unmaps).
        // PRISM_VMM_PREMAP_STEAL=0 turns them off.
        static const bool premap_steal = [] {
            const char* e = std::getenv("PRISM_VMM_PREMAP_STEAL");
            return !(e && e[0] == '0');
        }();
        return premap_steal && steal_for_worker(lk, h, StealMode::premap);
    }
    if (reserve_chunks() > 0) reserve_wanted_ = true;  // the budget is spent: keep handles ready
    if (steal_for_worker(lk, h, StealMode::urgent)) return true;
    // Nothing idle is safe to move (the budget shrank under queued maps, or
    // every idle chunk was released inside the open step): past the budget.
    ++stats_.over_budget;
    return create();
}

bool VmmDevice::steal_for_worker(Lock& lk, std::uint64_t& h, StealMode mode) {
    // reserve: like premap (safe chunks outside every window only, no fence
    // waits) but without the idle-age rule
    const bool premap = mode != StealMode::urgent;
    const bool need_age = mode == StealMode::premap;
    // Move the highest idle chunk that is safe (look-ahead and never read,
    // or released before a fence that passed), preferring chunks outside
    // every pool's look-ahead window: allocation reuses the lowest unmapped
    // page indices, so high idle chunks are the least likely to be revived.
    // The handle keeps its mapped_ count (it moves from chunk to chunk).
    // premap: a look-ahead map may take only a safe chunk outside every
    // window, and never waits for a fence (memory moves to growing pools
    // ahead of need instead of on an urgent map the caller waits for).
    while (!stop_) {
        advance_fences(false);
        std::uint64_t pick = 0, fallback = 0;
        int scanned = 0;
        const auto now = Clock::now();
        const auto aged = [&](const Chunk& v) { return !need_age || now - v.idle_at >= premap_steal_age(); };
        for (auto it = idle_.rbegin(); it != idle_.rend(); ++it) {
            const Chunk& v = chunks_.find(*it)->second;
            if (!(v.clean || v.epoch < fenced_) || !aged(v)) continue;
            if (!fallback) fallback = *it;
            if (!in_window(*it)) {
                pick = *it;
                break;
            }
            if (++scanned >= kStealScan) break;
        }
        if (premap && !pick) return false;
        if (!pick) pick = fallback;
        if (pick) {
            // Take the pick and up to kStealBatch - 1 idle chunks directly
            // below it in the same reservation (safe and outside every
            // window) in ONE cuMemUnmap: the driver cost of an unmap is mostly
            // per call, and a pool that needed one stolen chunk needs more.
            // The extra handles go to the cache for the next maps.
            auto r = ranges_.upper_bound(pick);
            const std::uint64_t res_lo = r == ranges_.begin() ? pick : std::prev(r)->first;
            std::uint64_t lo = pick;
            int n = 1;
            const int batch = mode == StealMode::premap   ? kStealBatch
                              : mode == StealMode::reserve ? reserve_batch()
                                                           : urgent_steal_batch();
            while (n < batch && lo >= res_lo + chunk_bytes_) {
                const std::uint64_t va = lo - chunk_bytes_;
                if (!idle_.count(va)) break;
                const Chunk& c = chunks_.find(va)->second;
                if (!(c.clean || c.epoch < fenced_) || in_window(va) || !aged(c)) break;
                lo = va;
                ++n;
            }
            std::vector<std::uint64_t> handles;
            for (std::uint64_t va = lo; va <= pick; va += chunk_bytes_) {
                Chunk& v = chunks_.find(va)->second;
                idle_.erase(va);
                if (v.clean) {
                    --clean_;
                    ++stats_.caller_steals_clean;
                }
                handles.push_back(v.handle);
                v.handle = 0;
                v.mapped = false;
                v.clean = false;
                v.inflight = true;
            }
            lk.unlock();
            const auto t0 = Clock::now();
            const CUresult res = drv().unmap(static_cast<CUdeviceptr>(lo), chunk_bytes_ * static_cast<std::uint64_t>(n));
            const double ns = ns_since(t0);
            lk.lock();
            if (res != CUDA_SUCCESS) {
                std::size_t k = 0;
                for (std::uint64_t va = lo; va <= pick; va += chunk_bytes_, ++k) {
                    Chunk& v = chunks_.find(va)->second;
                    v.inflight = false;
                    v.handle = handles[k];
                    v.mapped = true;
                    if (v.owed) {
                        --unready_;  // a caller mapped a page in it meanwhile: still mapped
                        v.owed = false;
                    }
                    if (v.refs == 0) set_idle(va, v);
                }
                failed_ = "cuMemUnmap failed (" + std::to_string(res) + ")";
                done_cv_.notify_all();
                return false;
            }
            ++stats_.driver_unmaps;
            stats_.steals += static_cast<std::uint64_t>(n);
            stats_.steal_ns_total += ns;
            sample(stats_.drv_unmap_ns, ns);
            trace('U', n, t0, ns);
            // the pick's handle goes to the caller (keeps its mapped_ count);
            // the others become cached, unmapped handles
            h = handles.back();
            for (std::size_t k = 0; k + 1 < handles.size(); ++k) {
                cache_.push_back(handles[k]);
                --mapped_;
            }
            for (std::uint64_t va = lo; va <= pick; va += chunk_bytes_) {
                const auto vit = chunks_.find(va);
                Chunk& v = vit->second;
                v.inflight = false;
                if (v.owed) {
                    // its pool mapped a page in it again meanwhile: map it back
                    if (!v.queued) {
                        urgent_.push_back(va);
                        v.queued = true;
                    }
                } else {
                    drop_if_empty(vit);
                }
            }
            done_cv_.notify_all();
            return true;
        }
        if (idle_.empty() || premap) return false;
        // Every idle chunk may still be read by kernels. Only fences the
        // CALLER records can make one safe (the engine records one at
        // begin_step, after every kernel of the earlier steps was launched).
        // The worker never records a fence: one recorded mid-step, between
        // the step's completion frees and its K2/K3 launches, would pass at
        // once and let a chunk those launches still read be unmapped. Poll
        // while a pending fence covers some idle chunk; otherwise the caller
        // is inside a step waiting on this map: give up (take_handle then
        // creates past the budget, counted in stats_.over_budget).
        const std::uint64_t horizon = fenced_ + fences_.size();
        bool coverable = false;
        for (const std::uint64_t v : idle_) {
            if (chunks_.find(v)->second.epoch < horizon) {
                coverable = true;
                break;
            }
        }
        if (!coverable) return false;
        lk.unlock();
        std::this_thread::sleep_for(std::chrono::microseconds(20));
        lk.lock();
    }
    return false;
}

bool VmmDevice::map_chunk(Lock& lk, std::uint64_t va, std::uint64_t h, bool urgent) {
    // `va` is marked inflight and owns handle h (counted in mapped_).
    const auto it = chunks_.find(va);
    Chunk& c = it->second;
    c.handle = h;
    lk.unlock();
    const auto tm = Clock::now();
    CUresult r = drv().map(static_cast<CUdeviceptr>(va), chunk_bytes_, 0, static_cast<CUmemGenericAllocationHandle>(h), 0);
    const double map_ns = ns_since(tm);
    double acc_ns = 0.0;
    if (r == CUDA_SUCCESS) {
        const auto ta = Clock::now();
        r = drv().set_access(static_cast<CUdeviceptr>(va), chunk_bytes_, &access_of(access_desc_), 1);
        acc_ns = ns_since(ta);
        if (r != CUDA_SUCCESS) drv().unmap(static_cast<CUdeviceptr>(va), chunk_bytes_);
    }
    lk.lock();
    c.inflight = false;
    stats_.map_call_ns_total += map_ns;
    stats_.access_ns_total += acc_ns;
    sample(stats_.drv_map_ns, map_ns + acc_ns);
    if (acc_ns > 0.0) ++stats_.access_calls;
    trace(urgent ? 'M' : 'P', 1, tm, map_ns + acc_ns);
    if (r != CUDA_SUCCESS) {
        c.handle = 0;
        --mapped_;
        cache_.push_back(h);
        if (urgent) {
            failed_ = "cuMemMap/cuMemSetAccess failed (" + std::to_string(r) + ")";
        } else if (c.owed && !c.queued) {
            // a caller mapped a page into this look-ahead chunk meanwhile and
            // counts it in unready_: retry it as an urgent map
            urgent_.push_back(va);
            c.queued = true;
        }
        hints_.clear();
        drop_if_empty(it);
        return false;
    }
    c.mapped = true;
    const bool owed = c.owed;
    if (owed) {
        --unready_;
        c.owed = false;
    }
    if (c.refs > 0) {
        c.clean = false;
    } else {
        c.clean = !owed;  // a chunk whose pages all left meanwhile keeps its release epoch
        set_idle(va, c);
    }
    if (urgent) {
        ++stats_.urgent;
    } else {
        ++stats_.premaps;
    }
    return true;
}

void VmmDevice::worker_main() {
    if (cudaSetDevice(ordinal_) != cudaSuccess) return;
    const auto free_chunk = [&](std::uint64_t v) {
        const auto it = chunks_.find(v);
        return it == chunks_.end() ||
               (!it->second.mapped && !it->second.inflight && !it->second.queued && !it->second.owed &&
                it->second.refs == 0);
    };
    Lock lk(mu_);
    while (!stop_) {
        // 1. urgent chunks
        if (!urgent_.empty()) {
            const std::uint64_t va = urgent_.front();
            urgent_.pop_front();
            const auto it = chunks_.find(va);
            Chunk& c = it->second;
            c.queued = false;
            if (!c.owed || c.mapped || c.inflight) {  // mapped by the look-ahead, or in flight
                drop_if_empty(it);
                continue;
            }
            ++worker_busy_;
            const auto t0 = Clock::now();
            c.inflight = true;
            std::uint64_t h = 0;
            if (take_handle(lk, true, h)) {
                map_chunk(lk, va, h, true);
            } else {
                c.inflight = false;
                if (failed_.empty()) failed_ = "out of physical memory for a queued chunk";
            }
            stats_.background_ns_total += ns_since(t0);
            --worker_busy_;
            done_cv_.notify_all();
            continue;
        }
        // 2. look-ahead
        std::uint64_t va = 0;
        if (clean_ * chunk_pages_ >= kMaxCleanPages) hints_.clear();  // enough is mapped ahead
        for (auto it = hints_.begin(); it != hints_.end() && !va;) {
            auto& list = it->second;
            while (!list.empty() && !va) {
                const std::uint64_t v = list.back();
                list.pop_back();
                if (free_chunk(v)) va = v;
            }
            it = list.empty() ? hints_.erase(it) : std::next(it);
        }
        if (va) {
            ++worker_busy_;
            const auto t0 = Clock::now();
            const auto it = chunks_.emplace(va, Chunk{}).first;
            it->second.inflight = true;
            std::uint64_t h = 0;
            if (take_handle(lk, false, h)) {
                map_chunk(lk, va, h, false);
            } else {
                it->second.inflight = false;
                if (it->second.owed && !it->second.queued) {  // wanted meanwhile
                    urgent_.push_back(va);
                    it->second.queued = true;
                }
                drop_if_empty(it);
                hints_.clear();  // no free budget: wait for the next hint
            }
            stats_.background_ns_total += ns_since(t0);
            --worker_busy_;
            done_cv_.notify_all();
            continue;
        }
        // 2b. background reserve of unmapped handles (PRISM_VMM_RESERVE_CHUNKS)
        if (reserve_wanted_ && cache_.size() < reserve_chunks()) {
            ++worker_busy_;
            const auto t0 = Clock::now();
            std::uint64_t h = 0;
            if (steal_for_worker(lk, h, StealMode::reserve)) {
                cache_.push_back(h);  // the steal counted it in mapped_
                --mapped_;
                ++stats_.reserve_steals;
            } else {
                reserve_wanted_ = false;  // nothing safe to move: wait for the next urgent steal
            }
            stats_.background_ns_total += ns_since(t0);
            --worker_busy_;
            done_cv_.notify_all();
            continue;
        }
        // 3. ready handles
        if ((cache_.size() < cache_target_ || reserve_pending_ > 0) && total_locked() < budget_chunks()) {
            ++worker_busy_;
            ++creating_;
            lk.unlock();
            CUmemGenericAllocationHandle h = 0;
            const auto t0 = Clock::now();
            const CUresult r = drv().create(&h, chunk_bytes_, &prop_of(prop_), 0);
            const double ns = ns_since(t0);
            lk.lock();
            --creating_;
            if (r == CUDA_SUCCESS) {
                cache_.push_back(static_cast<std::uint64_t>(h));
                if (reserve_pending_ > 0) --reserve_pending_;
                ++stats_.creates;
                stats_.create_ns_total += ns;
                trace('C', 1, t0, ns);
            } else {
                cache_target_ = 0;  // out of memory: stop until asked again
                reserve_pending_ = 0;
            }
            stats_.background_ns_total += ns;
            --worker_busy_;
            done_cv_.notify_all();
            continue;
        }
        done_cv_.notify_all();  // idle: quiesce() waiters
        cv_.wait(lk);
    }
}

void VmmDevice::premap(std::uint64_t owner, const std::uint64_t* vas, std::size_t n) {
    {
        Lock lk(mu_);
        std::vector<std::uint64_t> chunks;
        for (std::size_t i = 0; i < n; ++i) {
            const std::uint64_t c = chunk_of(vas[i]);
            if (chunks.empty() || chunks.back() != c) chunks.push_back(c);
        }
        if (chunks.empty()) {
            hints_.erase(owner);
            return;
        }
        window_[owner] = {chunks.front(), chunks.back() + chunk_bytes_};
        // stored reversed: the worker pops from the back, lowest VA first
        hints_[owner].assign(chunks.rbegin(), chunks.rend());
    }
    cv_.notify_one();
}

void VmmDevice::forget(std::uint64_t owner) {
    Lock lk(mu_);
    hints_.erase(owner);
    window_.erase(owner);
}

void VmmDevice::prefill_cache(std::uint64_t pages) {
    {
        Lock lk(mu_);
        cache_target_ = (pages + chunk_pages_ - 1) / chunk_pages_;
    }
    cv_.notify_one();
}

void VmmDevice::reserve_physical(std::uint64_t pages) {
    {
        Lock lk(mu_);
        // one-shot: create handles until the cache holds `pages` worth; they
        // are consumed by later maps and NOT refilled (a standing refill
        // target would keep the worker creating handles while serving)
        const std::uint64_t want = (pages + chunk_pages_ - 1) / chunk_pages_;
        reserve_pending_ = want > cache_.size() ? want - cache_.size() : 0;
    }
    cv_.notify_one();
}

void VmmDevice::quiesce() {
    Lock lk(mu_);
    cv_.notify_one();
    done_cv_.wait(lk, [&] {
        return !failed_.empty() ||
               (worker_busy_ == 0 && urgent_.empty() && hints_.empty() &&
                !(reserve_wanted_ && cache_.size() < reserve_chunks()) &&
                !((cache_.size() < cache_target_ || reserve_pending_ > 0) && total_locked() < budget_chunks()));
    });
    check_failed();
}

// ---------------------------------------------------------------- caller side

std::uint64_t VmmDevice::total_handles() const {
    Lock lk(mu_);
    return total_locked();
}
std::uint64_t VmmDevice::pool_count() const {
    Lock lk(mu_);
    return ranges_.size();
}
std::uint64_t VmmDevice::buffered_handles() const {
    Lock lk(mu_);
    return buffer_pages_;
}
std::uint64_t VmmDevice::cached_handles() const {
    Lock lk(mu_);
    return cache_.size();
}
std::uint64_t VmmDevice::pending_unmaps() const {
    Lock lk(mu_);
    return idle_.size();
}

std::uint64_t VmmDevice::reserve(std::uint64_t pages) {
    const std::uint64_t chunks = (pages + chunk_pages_ - 1) / chunk_pages_;
    CUdeviceptr va = 0;
    cu_check(drv().reserve(&va, chunks * chunk_bytes_, page_bytes_, 0, 0), "cuMemAddressReserve");
    Lock lk(mu_);
    ranges_[static_cast<std::uint64_t>(va)] = static_cast<std::uint64_t>(va) + chunks * chunk_bytes_;
    return static_cast<std::uint64_t>(va);
}

void VmmDevice::unmap_chunk_caller(ChunkMap::iterator it) {
    Chunk& c = it->second;
    const auto t0 = Clock::now();
    cu_check(drv().unmap(static_cast<CUdeviceptr>(it->first), chunk_bytes_), "cuMemUnmap");
    ++stats_.driver_unmaps;
    sample(stats_.unmap_ns, ns_since(t0));
    if (idle_.erase(it->first) && c.clean) --clean_;
    c.mapped = false;
    c.clean = false;
    cache_.push_back(c.handle);
    c.handle = 0;
    --mapped_;
}

void VmmDevice::release(std::uint64_t va, std::uint64_t pages) {
    Lock lk(mu_);
    (void)pages;
    const auto r = ranges_.find(va);
    if (r == ranges_.end()) throw std::runtime_error("VmmDevice::release: unknown range");
    const std::uint64_t end = r->second;
    hints_.erase(va);
    window_.erase(va);
    // the worker may be mapping into (or moving a chunk out of) this range
    cv_.notify_one();
    done_cv_.wait(lk, [&] {
        if (!failed_.empty()) return true;
        for (auto it = chunks_.lower_bound(va); it != chunks_.end() && it->first < end; ++it) {
            if (it->second.inflight || it->second.queued) return false;
        }
        return true;
    });
    bool synced = false;
    for (auto it = chunks_.lower_bound(va); it != chunks_.end() && it->first < end;) {
        Chunk& c = it->second;
        if (c.mapped) {
            if (!c.clean && !synced) {
                PRISM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
                synced = true;
            }
            unmap_chunk_caller(it);
        } else if (c.owed) {
            --unready_;  // never mapped (worker failed): nothing to undo
        }
        it = chunks_.erase(it);
    }
    ranges_.erase(r);
    cu_check(drv().addr_free(static_cast<CUdeviceptr>(va), end - va), "cuMemAddressFree");
}

void VmmDevice::advance_fences(bool wait) {
    std::size_t done = 0;
    while (done < fences_.size()) {
        auto ev = static_cast<cudaEvent_t>(fences_[done]);
        const cudaError_t q = wait ? cudaEventSynchronize(ev) : cudaEventQuery(ev);
        if (q == cudaErrorNotReady) break;
        PRISM_CUDA(q);
        cudaEventDestroy(ev);
        ++done;
    }
    fences_.erase(fences_.begin(), fences_.begin() + static_cast<std::ptrdiff_t>(done));
    fenced_ += done;
}

void VmmDevice::map(std::uint64_t va, bool from_buffer) {
    const std::uint64_t one[1] = {va};
    map_batch(one, 1, from_buffer ? 1 : 0);
}

void VmmDevice::map_batch(const std::uint64_t* vas, std::size_t n, std::size_t n_from_buffer) {
    (void)n_from_buffer;  // buffer pages are cached chunks (take_buffer)
    if (n == 0) return;
    const auto t0 = Clock::now();
    Lock lk(mu_);
    check_failed();
    stats_.maps += n;
    bool queued = false;
    for (std::size_t i = 0; i < n; ++i) {
        const std::uint64_t cv = chunk_of(vas[i]);
        Chunk& c = chunks_[cv];
        if (c.mapped) {
            // no driver call: the chunk is mapped (live, or idle: revive)
            if (c.refs == 0) {
                idle_.erase(cv);
                if (c.clean) {
                    --clean_;
                    ++stats_.premapped_hits;
                    c.clean = false;
                }
            }
            ++stats_.revived;
        } else if (!c.owed) {
            ++unready_;
            c.owed = true;
            if (!c.inflight && !c.queued) {
                urgent_.push_back(cv);
                c.queued = true;
                queued = true;
            }
        }
        ++c.refs;
    }
    if (queued) cv_.notify_one();
    if (!defer_) wait_pending(lk);
    const double per = ns_since(t0) / static_cast<double>(n);
    stats_.map_ns_total += per * static_cast<double>(n);
    for (std::size_t i = 0; i < n; ++i) sample(stats_.map_ns, per);
}

void VmmDevice::defer_access(bool on) {
    const auto t0 = Clock::now();
    Lock lk(mu_);
    defer_ = on;
    if (!on && unready_ > 0) {
        wait_pending(lk);
        stats_.map_ns_total += ns_since(t0);
    }
}

void VmmDevice::flush_access() {
    const auto t0 = Clock::now();
    Lock lk(mu_);
    if (unready_ == 0) return;
    wait_pending(lk);
    stats_.map_ns_total += ns_since(t0);
}

void VmmDevice::unmap(std::uint64_t va) {
    const auto t0 = Clock::now();
    Lock lk(mu_);
    const auto it = chunks_.find(chunk_of(va));
    if (it == chunks_.end() || it->second.refs == 0) throw std::runtime_error("VmmDevice::unmap: page not mapped");
    Chunk& c = it->second;
    if (--c.refs == 0) {
        c.epoch = epoch_;  // kernels issued before the next fence may read it
        c.clean = false;
        // not mapped yet: it stays owed (this step's kernels may touch its
        // pages) and lands idle, with this epoch, once the worker mapped it
        if (c.mapped) set_idle(it->first, c);
    }
    ++stats_.unmaps;
    const double ns = ns_since(t0);
    stats_.unmap_ns_total += ns;
    sample(stats_.unmap_ns, ns);
}

void VmmDevice::fence() {
    Lock lk(mu_);
    fence_locked();
}

void VmmDevice::fence_locked() {
    cudaEvent_t ev = nullptr;
    PRISM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    PRISM_CUDA(cudaEventRecord(ev, static_cast<cudaStream_t>(stream_)));
    fences_.push_back(ev);
    ++epoch_;
    if (fences_.size() > 64) advance_fences(false);  // keep the queue short
}

void VmmDevice::reclaim(bool wait) {
    Lock lk(mu_);
    if (wait) {
        // Everything goes back: stop the look-ahead and drain the worker.
        hints_.clear();
        cv_.notify_one();
        done_cv_.wait(lk, [&] { return (urgent_.empty() && worker_busy_ == 0) || !failed_.empty(); });
        PRISM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
        fence_locked();
        advance_fences(true);
    } else {
        advance_fences(false);
    }
    const auto t0 = Clock::now();
    for (auto v = idle_.begin(); v != idle_.end();) {
        const auto it = chunks_.find(*v);
        ++v;  // unmap_chunk_caller erases the current entry
        const Chunk& c = it->second;
        if (wait || (!c.clean && c.epoch < fenced_)) {
            unmap_chunk_caller(it);
            drop_if_empty(it);
        }
    }
    stats_.unmap_ns_total += ns_since(t0);
}

void VmmDevice::grow_buffer(std::uint64_t pages) {
    Lock lk(mu_);
    buffer_pages_ += pages;
    const std::uint64_t need = (buffer_pages_ + chunk_pages_ - 1) / chunk_pages_;
    while (cache_.size() < need) {
        CUmemGenericAllocationHandle h = 0;
        const auto tc = Clock::now();
        cu_check(drv().create(&h, chunk_bytes_, &prop_of(prop_), 0), "cuMemCreate");
        ++stats_.creates;
        stats_.create_ns_total += ns_since(tc);
        cache_.push_back(static_cast<std::uint64_t>(h));
    }
}

void VmmDevice::take_buffer(std::uint64_t pages) {
    Lock lk(mu_);
    buffer_pages_ -= std::min(pages, buffer_pages_);
}

void VmmDevice::set_budget(std::uint64_t pages) {
    Lock lk(mu_);
    budget_pages_ = pages;
    // Shrink: free cached handles first, then physically release idle chunks.
    const auto over = [&] { return total_locked() > budget_chunks(); };
    while (over() && !cache_.empty()) {
        drv().release(static_cast<CUmemGenericAllocationHandle>(cache_.back()));
        cache_.pop_back();
    }
    while (over() && !idle_.empty()) {
        advance_fences(false);
        auto pick = idle_.end();
        for (auto v = idle_.rbegin(); v != idle_.rend(); ++v) {
            const Chunk& c = chunks_.find(*v)->second;
            if (c.clean || c.epoch < fenced_) {
                pick = std::prev(v.base());
                break;
            }
        }
        if (pick == idle_.end()) {
            fence_locked();
            advance_fences(true);
            pick = std::prev(idle_.end());
        }
        const auto it = chunks_.find(*pick);
        unmap_chunk_caller(it);
        drop_if_empty(it);
        drv().release(static_cast<CUmemGenericAllocationHandle>(cache_.back()));
        cache_.pop_back();
        ++stats_.steals;
    }
}

VmmStats VmmDevice::stats() const {
    Lock lk(mu_);
    dump_trace();  // PRISM_VMM_TRACE only
    return stats_;
}

void VmmDevice::reset_stats() {
    Lock lk(mu_);
    stats_ = VmmStats{};
}

unsigned VmmDevice::debug_chunk_state(std::uint64_t page_va) const {
    Lock lk(mu_);
    const std::uint64_t cv = chunk_of(page_va);
    const auto it = chunks_.find(cv);
    if (it == chunks_.end()) return 0;
    const Chunk& c = it->second;
    return 1u | (c.mapped ? 2u : 0u) | (c.inflight ? 4u : 0u) | (c.queued ? 8u : 0u) | (c.refs > 0 ? 16u : 0u) |
           (idle_.count(cv) ? 32u : 0u);
}

std::uint64_t VmmDevice::capacity_pages(std::uint64_t reserve_bytes) const {
    std::size_t free_b = 0, total_b = 0;
    PRISM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    return free_b > reserve_bytes ? (free_b - reserve_bytes) / page_bytes_ : 0;
}

}  // namespace prism
