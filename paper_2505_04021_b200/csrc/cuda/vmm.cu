// prism::VmmDevice implementation: CUDA VMM (driver API) behind the ledger.
// Driver entry points are resolved at run time through the runtime's
// cudaGetDriverEntryPoint, so the library loads on machines without a driver
// (the CPU build/test container) and only fails when a device is opened.
//
// Threading: every public method takes mu_. The caller's thread performs its
// driver calls while holding mu_ (those are the maps nobody anticipated); the
// background worker drops mu_ around its driver calls and marks the VAs it
// is working on in inflight_, which callers wait out on done_cv_.
#include <cuda.h>

#include <algorithm>
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

// How many in-window parked entries a steal skips over looking for a page
// outside every look-ahead window (bounds the scan).
constexpr int kStealScan = 256;
// Longest contiguous run the worker maps before one cuMemSetAccess.
constexpr std::size_t kPremapRun = 8;
// At most this many pre-mapped (clean parked) pages per device (1 GiB).
constexpr std::uint64_t kMaxClean = 512;


CUmemAllocationProp& prop_of(void* p) { return *static_cast<CUmemAllocationProp*>(p); }
CUmemAccessDesc& access_of(void* p) { return *static_cast<CUmemAccessDesc*>(p); }

}  // namespace

std::shared_ptr<VmmDevice> VmmDevice::open(int ordinal, std::uint64_t page_bytes) {
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

    std::shared_ptr<VmmDevice> dev(new VmmDevice());
    dev->ordinal_ = ordinal;
    dev->page_bytes_ = page_bytes;
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
    dev->worker_ = std::thread([raw = dev.get()] { raw->worker_main(); });
    return dev;
}

VmmDevice::~VmmDevice() {
    {
        Lock lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    if (worker_.joinable()) worker_.join();
    try {
        cudaSetDevice(ordinal_);
        cudaDeviceSynchronize();
        for (auto& [va, p] : parked_) {
            drv().unmap(va, page_bytes_);
            drv().release(p.handle);
        }
        for (auto& [va, h] : live_) {
            drv().unmap(va, page_bytes_);
            drv().release(h);
        }
        for (auto h : buffer_) drv().release(h);
        for (auto h : taken_) drv().release(h);
        for (auto h : cache_) drv().release(h);
        for (void* e : fences_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
        if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
    } catch (...) {
    }
    delete static_cast<CUmemAllocationProp*>(prop_);
    delete static_cast<CUmemAccessDesc*>(access_desc_);
}

// ---------------------------------------------------------------- worker

bool VmmDevice::take_handle(Lock& lk, std::uint64_t va, bool urgent, std::uint64_t& h) {
    // A handle for `va`; it stays counted in inflight_handles_ until it lands
    // in live_ / parked_ (or back in cache_). Urgent maps use the buffer
    // handle the caller earmarked, then the cache, a new handle within the
    // budget, and finally a released page moved from elsewhere; look-ahead
    // maps only use free budget.
    if (urgent) {
        const auto p = pending_.find(va);
        if (p != pending_.end() && p->second) {
            h = p->second;
            p->second = 0;
            --earmarked_;
            ++inflight_handles_;
            return true;
        }
    }
    if (!cache_.empty()) {
        h = cache_.back();
        cache_.pop_back();
        ++inflight_handles_;
        return true;
    }
    if (total_locked() < budget_) {
        ++inflight_handles_;
        lk.unlock();
        CUmemGenericAllocationHandle ch = 0;
        const auto tc = Clock::now();
        const CUresult r = drv().create(&ch, page_bytes_, &prop_of(prop_), 0);
        const double ns = ns_since(tc);
        lk.lock();
        if (r == CUDA_SUCCESS) {
            h = static_cast<std::uint64_t>(ch);
            ++stats_.creates;
            stats_.create_ns_total += ns;
            return true;
        }
        --inflight_handles_;
        if (!urgent) return false;
    }
    if (!urgent) return false;
    if (steal_for_worker(lk, h)) return true;
    // Nothing parked to move (the ledger never maps past the budget, so this
    // means the budget shrank under queued maps): create past it.
    ++inflight_handles_;
    CUmemGenericAllocationHandle ch = 0;
    const CUresult r = drv().create(&ch, page_bytes_, &prop_of(prop_), 0);
    if (r != CUDA_SUCCESS) {
        --inflight_handles_;
        return false;
    }
    ++stats_.creates;
    h = static_cast<std::uint64_t>(ch);
    return true;
}

bool VmmDevice::steal_for_worker(Lock& lk, std::uint64_t& h) {
    // Move the highest parked page that is safe (pre-mapped and never read,
    // or released before a fence that passed), preferring pages outside every
    // pool's look-ahead window: allocation reuses the lowest unmapped page
    // indices, so high parked pages are the least likely to be revived soon.
    while (!stop_) {
        advance_fences(false);
        auto pick = parked_.end(), fallback = parked_.end();
        int scanned = 0;
        for (auto it = parked_.rbegin(); it != parked_.rend(); ++it) {
            if (!(it->second.clean || it->second.epoch < fenced_)) continue;
            if (fallback == parked_.end()) fallback = std::prev(it.base());
            if (!in_window(it->first)) {
                pick = std::prev(it.base());
                break;
            }
            if (++scanned >= kStealScan) break;
        }
        if (pick == parked_.end()) pick = fallback;
        if (pick != parked_.end()) {
            const std::uint64_t victim = pick->first;
            const Parked saved = pick->second;
            if (saved.clean) ++stats_.caller_steals_clean;
            unpark(pick);
            inflight_.insert(victim);
            ++inflight_handles_;
            lk.unlock();
            const auto t0 = Clock::now();
            const CUresult r = drv().unmap(static_cast<CUdeviceptr>(victim), page_bytes_);
            const double ns = ns_since(t0);
            lk.lock();
            inflight_.erase(victim);
            if (r != CUDA_SUCCESS) {
                --inflight_handles_;
                park(victim, saved);
                failed_ = "cuMemUnmap failed (" + std::to_string(r) + ")";
                done_cv_.notify_all();
                return false;
            }
            ++stats_.driver_unmaps;
            ++stats_.steals;
            stats_.steal_ns_total += ns;
            // its owner may have mapped the page again meanwhile
            if (pending_.count(victim)) urgent_.push_back(victim);
            h = saved.handle;
            done_cv_.notify_all();
            return true;
        }
        if (parked_.empty()) return false;
        // Every parked page may still be read by queued kernels: fence and
        // poll until that fence passes.
        fence_locked();
        lk.unlock();
        std::this_thread::sleep_for(std::chrono::microseconds(50));
        lk.lock();
    }
    return false;
}

void VmmDevice::map_run(Lock& lk, std::vector<std::uint64_t>& run, std::vector<std::uint64_t>& hs, bool urgent) {
    // `run`: contiguous VAs already in inflight_, one handle each in hs.
    lk.unlock();
    std::size_t mapped = 0;
    CUresult r = CUDA_SUCCESS;
    const auto tm = Clock::now();
    for (; mapped < run.size(); ++mapped) {
        r = drv().map(static_cast<CUdeviceptr>(run[mapped]), page_bytes_, 0,
                      static_cast<CUmemGenericAllocationHandle>(hs[mapped]), 0);
        if (r != CUDA_SUCCESS) break;
    }
    const double map_ns = ns_since(tm);
    double acc_ns = 0.0;
    if (r == CUDA_SUCCESS) {
        const auto ta = Clock::now();
        r = drv().set_access(static_cast<CUdeviceptr>(run[0]), run.size() * page_bytes_, &access_of(access_desc_), 1);
        acc_ns = ns_since(ta);
    }
    if (r != CUDA_SUCCESS) {
        for (std::size_t i = 0; i < mapped; ++i) drv().unmap(static_cast<CUdeviceptr>(run[i]), page_bytes_);
    }
    lk.lock();
    inflight_handles_ -= run.size();
    for (std::size_t i = 0; i < run.size(); ++i) {
        inflight_.erase(run[i]);
        if (r != CUDA_SUCCESS) {
            cache_.push_back(hs[i]);
            continue;
        }
        const auto p = pending_.find(run[i]);
        if (p != pending_.end()) {
            // logically mapped meanwhile (or urgent): straight to live
            if (p->second) {
                cache_.push_back(p->second);
                --earmarked_;
            }
            pending_.erase(p);
            live_.emplace(run[i], hs[i]);
        } else {
            park(run[i], Parked{hs[i], 0, true});
        }
    }
    stats_.map_call_ns_total += map_ns;
    stats_.access_ns_total += acc_ns;
    if (acc_ns > 0.0) ++stats_.access_calls;
    if (r != CUDA_SUCCESS) {
        if (urgent) failed_ = "cuMemMap/cuMemSetAccess failed (" + std::to_string(r) + ")";
        hints_.clear();
    } else if (urgent) {
        stats_.urgent += run.size();
    } else {
        stats_.premaps += run.size();
    }
}

void VmmDevice::worker_main() {
    if (cudaSetDevice(ordinal_) != cudaSuccess) return;
    const auto free_va = [&](std::uint64_t v) {
        return !live_.count(v) && !parked_.count(v) && !inflight_.count(v) && !pending_.count(v);
    };
    Lock lk(mu_);
    while (!stop_) {
        // 1. urgent maps, in runs of contiguous VAs
        std::vector<std::uint64_t> run, hs;
        while (!urgent_.empty() && run.size() < kPremapRun) {
            const std::uint64_t v = urgent_.front();
            if (!pending_.count(v) || inflight_.count(v)) {  // resolved by a look-ahead map
                urgent_.pop_front();
                continue;
            }
            if (!run.empty() && v != run.back() + page_bytes_) break;
            run.push_back(v);
            urgent_.pop_front();
        }
        if (!run.empty()) {
            ++worker_busy_;
            const auto t0 = Clock::now();
            for (std::uint64_t v : run) inflight_.insert(v);
            for (std::uint64_t v : run) {
                std::uint64_t h = 0;
                if (!take_handle(lk, v, true, h)) break;
                hs.push_back(h);
            }
            if (hs.size() < run.size()) {
                for (std::size_t i = hs.size(); i < run.size(); ++i) inflight_.erase(run[i]);
                if (failed_.empty()) failed_ = "VmmDevice: out of physical memory for a queued map";
                run.resize(hs.size());
            }
            if (!run.empty()) map_run(lk, run, hs, true);
            stats_.background_ns_total += ns_since(t0);
            --worker_busy_;
            done_cv_.notify_all();
            continue;
        }
        // 2. look-ahead: a run of up to kPremapRun contiguous hinted VAs
        if (clean_ >= kMaxClean) hints_.clear();  // enough memory is pre-mapped already
        const std::size_t max_run =
            static_cast<std::size_t>(std::min<std::uint64_t>(kPremapRun, kMaxClean - std::min(clean_, kMaxClean)));
        for (auto it = hints_.begin(); it != hints_.end() && run.empty();) {
            auto& list = it->second;
            while (!list.empty() && run.empty()) {
                const std::uint64_t v = list.back();
                list.pop_back();
                if (free_va(v)) run.push_back(v);
            }
            while (!run.empty() && run.size() < max_run && !list.empty() && list.back() == run.back() + page_bytes_ &&
                   free_va(list.back())) {
                run.push_back(list.back());
                list.pop_back();
            }
            it = list.empty() ? hints_.erase(it) : std::next(it);
        }
        if (!run.empty()) {
            ++worker_busy_;
            const auto t0 = Clock::now();
            for (std::uint64_t v : run) {
                std::uint64_t h = 0;
                if (!take_handle(lk, v, false, h)) {
                    hints_.clear();  // no free budget: look-ahead waits for the next hint
                    break;
                }
                hs.push_back(h);
            }
            // creating handles may have dropped the lock: keep the prefix
            // that is still free (a caller may have queued one urgently)
            std::size_t keep = 0;
            while (keep < hs.size() && free_va(run[keep])) ++keep;
            for (std::size_t i = keep; i < hs.size(); ++i) {
                cache_.push_back(hs[i]);
                --inflight_handles_;
            }
            run.resize(keep);
            hs.resize(keep);
            for (std::uint64_t v : run) inflight_.insert(v);
            if (!run.empty()) map_run(lk, run, hs, false);
            stats_.background_ns_total += ns_since(t0);
            --worker_busy_;
            done_cv_.notify_all();
            continue;
        }
        // 3. ready handles
        if (cache_.size() < cache_target_ && total_locked() < budget_) {
            ++worker_busy_;
            const auto t0 = Clock::now();
            ++inflight_handles_;
            lk.unlock();
            CUmemGenericAllocationHandle h = 0;
            const CUresult r = drv().create(&h, page_bytes_, &prop_of(prop_), 0);
            const double ns = ns_since(t0);
            lk.lock();
            --inflight_handles_;
            if (r == CUDA_SUCCESS) {
                cache_.push_back(static_cast<std::uint64_t>(h));
                ++stats_.creates;
                stats_.create_ns_total += ns;
            } else {
                cache_target_ = 0;  // out of memory: stop until asked again
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
        if (n) window_[owner] = {vas[0], vas[n - 1] + page_bytes_};
        auto& list = hints_[owner];
        // stored reversed: the worker pops from the back, lowest VA first
        list.assign(std::make_reverse_iterator(vas + n), std::make_reverse_iterator(vas));
        if (list.empty()) hints_.erase(owner);
    }
    cv_.notify_one();
}

void VmmDevice::forget(std::uint64_t owner) {
    Lock lk(mu_);
    hints_.erase(owner);
    window_.erase(owner);
}

void VmmDevice::prefill_cache(std::uint64_t n) {
    {
        Lock lk(mu_);
        cache_target_ = n;
    }
    cv_.notify_one();
}

void VmmDevice::quiesce() {
    Lock lk(mu_);
    cv_.notify_one();
    done_cv_.wait(lk, [&] {
        return !failed_.empty() ||
               (worker_busy_ == 0 && hints_.empty() && urgent_.empty() && pending_.empty() &&
                !(cache_.size() < cache_target_ && total_locked() < budget_));
    });
    check_failed();
}

// ---------------------------------------------------------------- caller side

void VmmDevice::check_failed() const {
    if (!failed_.empty()) throw std::runtime_error("VmmDevice worker: " + failed_);
}

void VmmDevice::wait_pending(Lock& lk) {
    if (pending_.empty()) return;
    const auto tw = Clock::now();
    cv_.notify_one();
    done_cv_.wait(lk, [&] { return pending_.empty() || !failed_.empty(); });
    stats_.wait_ns_total += ns_since(tw);
    check_failed();
}

bool VmmDevice::busy_in(std::uint64_t lo, std::uint64_t hi) const {
    for (const auto& kv : pending_) {
        if (kv.first >= lo && kv.first < hi) return true;
    }
    for (std::uint64_t v : inflight_) {
        if (v >= lo && v < hi) return true;
    }
    return false;
}

std::uint64_t VmmDevice::total_locked() const {
    return live_.size() + parked_.size() + buffer_.size() + taken_.size() + cache_.size() + inflight_handles_ +
           earmarked_;
}

std::uint64_t VmmDevice::total_handles() const {
    Lock lk(mu_);
    return total_locked();
}
std::uint64_t VmmDevice::buffered_handles() const {
    Lock lk(mu_);
    return buffer_.size() + taken_.size();
}
std::uint64_t VmmDevice::cached_handles() const {
    Lock lk(mu_);
    return cache_.size();
}
std::uint64_t VmmDevice::pending_unmaps() const {
    Lock lk(mu_);
    return parked_.size();
}

bool VmmDevice::in_window(std::uint64_t va) const {
    auto r = ranges_.upper_bound(va);
    if (r == ranges_.begin()) return false;
    --r;
    if (va >= r->second) return false;
    const auto w = window_.find(r->first);
    return w != window_.end() && va >= w->second.first && va < w->second.second;
}

std::uint64_t VmmDevice::reserve(std::uint64_t pages) {
    CUdeviceptr va = 0;
    cu_check(drv().reserve(&va, pages * page_bytes_, page_bytes_, 0, 0), "cuMemAddressReserve");
    Lock lk(mu_);
    ranges_[static_cast<std::uint64_t>(va)] = static_cast<std::uint64_t>(va) + pages * page_bytes_;
    return static_cast<std::uint64_t>(va);
}

void VmmDevice::release(std::uint64_t va, std::uint64_t pages) {
    Lock lk(mu_);
    const std::uint64_t end = va + pages * page_bytes_;
    hints_.erase(va);
    window_.erase(va);
    // the worker may be mapping into (or moving a page out of) this range
    done_cv_.wait(lk, [&] { return !busy_in(va, end) || !failed_.empty(); });
    ranges_.erase(va);
    bool synced = false;
    const auto sync = [&] {
        if (!synced) PRISM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
        synced = true;
    };
    for (auto it = parked_.lower_bound(va); it != parked_.end() && it->first < end;) {
        if (!it->second.clean) sync();
        driver_unmap(it->first);
        cache_.push_back(it->second.handle);
        it = unpark(it);
    }
    for (auto it = live_.begin(); it != live_.end();) {
        if (it->first >= va && it->first < end) {
            sync();
            driver_unmap(it->first);
            cache_.push_back(it->second);
            it = live_.erase(it);
        } else {
            ++it;
        }
    }
    cu_check(drv().addr_free(static_cast<CUdeviceptr>(va), pages * page_bytes_), "cuMemAddressFree");
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

std::uint64_t VmmDevice::steal_now(Lock& lk) {
    // Caller-side move (budget shrink): the highest safe parked page, after
    // draining the stream if none is safe yet.
    (void)lk;
    advance_fences(false);
    auto pick = parked_.end();
    for (auto it = parked_.rbegin(); it != parked_.rend(); ++it) {
        if (it->second.clean || it->second.epoch < fenced_) {
            pick = std::prev(it.base());
            break;
        }
    }
    if (pick == parked_.end()) {
        fence_locked();
        advance_fences(true);
        pick = std::prev(parked_.end());
    }
    driver_unmap(pick->first);
    const std::uint64_t h = pick->second.handle;
    unpark(pick);
    ++stats_.steals;
    return h;
}

void VmmDevice::map(std::uint64_t va, bool from_buffer) {
    const std::uint64_t one[1] = {va};
    map_batch(one, 1, from_buffer ? 1 : 0);
}

void VmmDevice::map_batch(const std::uint64_t* vas, std::size_t n, std::size_t n_from_buffer) {
    if (n == 0) return;
    const auto t0 = Clock::now();
    Lock lk(mu_);
    check_failed();
    stats_.maps += n;
    bool queued = false;
    for (std::size_t i = 0; i < n; ++i) {
        const std::uint64_t va = vas[i];
        const bool from_buffer = i < n_from_buffer;
        const auto p = parked_.find(va);
        if (p != parked_.end()) {
            // Revive in place; a buffer handle earmarked for this map returns
            // to the cache (it stays counted as physical memory).
            if (p->second.clean) ++stats_.premapped_hits;
            live_.emplace(va, p->second.handle);
            unpark(p);
            if (from_buffer && !taken_.empty()) {
                cache_.push_back(taken_.back());
                taken_.pop_back();
            }
            ++stats_.revived;
            continue;
        }
        if (live_.count(va) || pending_.count(va)) throw std::runtime_error("VmmDevice::map: page already mapped");
        std::uint64_t earmark = 0;
        if (from_buffer && !taken_.empty()) {
            earmark = taken_.back();
            taken_.pop_back();
            ++earmarked_;
        }
        pending_.emplace(va, earmark);
        // a page the worker is pre-mapping right now goes live when it lands
        if (!inflight_.count(va)) {
            urgent_.push_back(va);
            queued = true;
        }
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
    if (!on && !pending_.empty()) {
        wait_pending(lk);
        stats_.map_ns_total += ns_since(t0);
    }
}

void VmmDevice::flush_access() {
    const auto t0 = Clock::now();
    Lock lk(mu_);
    if (pending_.empty()) return;
    wait_pending(lk);
    stats_.map_ns_total += ns_since(t0);
}

void VmmDevice::unmap(std::uint64_t va) {
    const auto t0 = Clock::now();
    Lock lk(mu_);
    if (pending_.count(va)) {
        // mapped and released within one step: let its map land first
        cv_.notify_one();
        done_cv_.wait(lk, [&] { return !pending_.count(va) || !failed_.empty(); });
        check_failed();
    }
    const auto it = live_.find(va);
    if (it == live_.end()) throw std::runtime_error("VmmDevice::unmap: page not mapped");
    park(va, Parked{it->second, epoch_, false});
    live_.erase(it);
    ++stats_.unmaps;
    const double ns = ns_since(t0);
    stats_.unmap_ns_total += ns;
    sample(stats_.unmap_ns, ns);
}

void VmmDevice::driver_unmap(std::uint64_t va) {
    const auto t0 = Clock::now();
    cu_check(drv().unmap(static_cast<CUdeviceptr>(va), page_bytes_), "cuMemUnmap");
    ++stats_.driver_unmaps;
    sample(stats_.unmap_ns, ns_since(t0));
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
        done_cv_.wait(lk, [&] {
            return (pending_.empty() && inflight_.empty() && urgent_.empty() && worker_busy_ == 0) || !failed_.empty();
        });
        PRISM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
        fence_locked();
        advance_fences(true);
    } else {
        advance_fences(false);
    }
    const auto t0 = Clock::now();
    for (auto it = parked_.begin(); it != parked_.end();) {
        if (wait || (!it->second.clean && it->second.epoch < fenced_)) {
            driver_unmap(it->first);
            cache_.push_back(it->second.handle);
            it = unpark(it);
        } else {
            ++it;
        }
    }
    stats_.unmap_ns_total += ns_since(t0);
}

void VmmDevice::grow_buffer(std::uint64_t n) {
    Lock lk(mu_);
    for (std::uint64_t i = 0; i < n; ++i) {
        if (!cache_.empty()) {
            buffer_.push_back(cache_.back());
            cache_.pop_back();
            continue;
        }
        CUmemGenericAllocationHandle h = 0;
        const auto tc = Clock::now();
        cu_check(drv().create(&h, page_bytes_, &prop_of(prop_), 0), "cuMemCreate");
        ++stats_.creates;
        stats_.create_ns_total += ns_since(tc);
        buffer_.push_back(static_cast<std::uint64_t>(h));
    }
}

void VmmDevice::take_buffer(std::uint64_t n) {
    Lock lk(mu_);
    for (std::uint64_t i = 0; i < n && !buffer_.empty(); ++i) {
        taken_.push_back(buffer_.back());
        buffer_.pop_back();
    }
}

void VmmDevice::set_budget(std::uint64_t pages) {
    Lock lk(mu_);
    budget_ = pages;
    // Shrink: free cached handles first, then physically release parked pages.
    while (total_locked() > budget_ && !cache_.empty()) {
        drv().release(static_cast<CUmemGenericAllocationHandle>(cache_.back()));
        cache_.pop_back();
    }
    while (total_locked() > budget_ && !parked_.empty()) {
        drv().release(static_cast<CUmemGenericAllocationHandle>(steal_now(lk)));
    }
}

VmmStats VmmDevice::stats() const {
    Lock lk(mu_);
    return stats_;
}

void VmmDevice::reset_stats() {
    Lock lk(mu_);
    stats_ = VmmStats{};
}

std::uint64_t VmmDevice::capacity_pages(std::uint64_t reserve_bytes) const {
    std::size_t free_b = 0, total_b = 0;
    PRISM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    return free_b > reserve_bytes ? (free_b - reserve_bytes) / page_bytes_ : 0;
}

}  // namespace prism
