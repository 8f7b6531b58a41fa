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

// How many parked entries the worker inspects when looking for released
// memory to move (bounds its time under mu_).
constexpr int kStealScan = 256;

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

void VmmDevice::worker_main() {
    if (cudaSetDevice(ordinal_) != cudaSuccess) return;
    Lock lk(mu_);
    for (;;) {
        // Next job: the first hinted VA that is neither live, parked nor in
        // flight; otherwise top up the created-handle cache.
        std::uint64_t va = 0;
        bool have_va = false;
        for (auto it = hints_.begin(); it != hints_.end() && !have_va;) {
            auto& list = it->second;
            while (!list.empty()) {
                const std::uint64_t v = list.back();
                list.pop_back();
                if (!live_.count(v) && !parked_.count(v) && !inflight_.count(v)) {
                    va = v;
                    have_va = true;
                    break;
                }
            }
            it = list.empty() ? hints_.erase(it) : std::next(it);
        }
        const bool want_cache = cache_.size() < cache_target_ && total_locked() < budget_;
        if (!have_va && !want_cache) {
            if (stop_) return;
            done_cv_.notify_all();  // quiesce() waiters
            cv_.wait(lk);
            if (stop_) return;
            continue;
        }
        ++worker_busy_;
        const auto t0 = Clock::now();
        if (!have_va) {
            // Create one handle for the cache.
            ++inflight_handles_;
            lk.unlock();
            CUmemGenericAllocationHandle h = 0;
            const auto tc = Clock::now();
            const CUresult r = drv().create(&h, page_bytes_, &prop_of(prop_), 0);
            const double ns = ns_since(tc);
            lk.lock();
            --inflight_handles_;
            if (r == CUDA_SUCCESS) {
                cache_.push_back(static_cast<std::uint64_t>(h));
                ++stats_.creates;
                stats_.create_ns_total += ns;
            } else {
                cache_target_ = 0;  // out of memory: stop trying until asked again
            }
            stats_.background_ns_total += ns_since(t0);
            --worker_busy_;
            done_cv_.notify_all();
            continue;
        }
        // Pre-map `va`: needs a handle — cached, newly created within the
        // budget, or moved from a released (dirty, fence-passed) parked page.
        inflight_.insert(va);
        std::uint64_t h = 0;
        bool ok = false;
        std::uint64_t stolen_va = 0;
        // A handle taken below stays counted in inflight_handles_ until it
        // lands in parked_ (or back in cache_).
        if (!cache_.empty()) {
            h = cache_.back();
            cache_.pop_back();
            ++inflight_handles_;
            ok = true;
        } else if (total_locked() < budget_) {
            ++inflight_handles_;
            lk.unlock();
            CUmemGenericAllocationHandle ch = 0;
            const auto tc = Clock::now();
            const CUresult r = drv().create(&ch, page_bytes_, &prop_of(prop_), 0);
            const double ns = ns_since(tc);
            lk.lock();
            if (r == CUDA_SUCCESS) {
                h = static_cast<std::uint64_t>(ch);
                ok = true;
                ++stats_.creates;
                stats_.create_ns_total += ns;
            } else {
                --inflight_handles_;
            }
        } else {
            advance_fences(false);
            int scanned = 0;
            for (auto it = parked_.rbegin(); it != parked_.rend() && scanned < kStealScan; ++it, ++scanned) {
                if (!it->second.clean && it->second.epoch < fenced_ && !inflight_.count(it->first)) {
                    stolen_va = it->first;
                    break;
                }
            }
            if (stolen_va) {
                const auto p = parked_.find(stolen_va);
                h = p->second.handle;
                parked_.erase(p);
                inflight_.insert(stolen_va);
                ++inflight_handles_;
                lk.unlock();
                const CUresult r = drv().unmap(static_cast<CUdeviceptr>(stolen_va), page_bytes_);
                lk.lock();
                inflight_.erase(stolen_va);
                ok = r == CUDA_SUCCESS;
                if (ok) {
                    ++stats_.driver_unmaps;
                    ++stats_.steals;
                } else {
                    --inflight_handles_;
                    parked_.emplace(stolen_va, Parked{h, 0, false});  // still mapped: leave it parked
                }
                done_cv_.notify_all();
            }
        }
        if (!ok) {
            // No physical memory to move: drop the remaining hints until the
            // next premap() call (they are best effort).
            inflight_.erase(va);
            hints_.clear();
            --worker_busy_;
            done_cv_.notify_all();
            continue;
        }
        lk.unlock();
        const auto tm = Clock::now();
        CUresult r = drv().map(static_cast<CUdeviceptr>(va), page_bytes_, 0, static_cast<CUmemGenericAllocationHandle>(h), 0);
        const double map_ns = ns_since(tm);
        double acc_ns = 0.0;
        if (r == CUDA_SUCCESS) {
            const auto ta = Clock::now();
            r = drv().set_access(static_cast<CUdeviceptr>(va), page_bytes_, &access_of(access_desc_), 1);
            acc_ns = ns_since(ta);
            if (r != CUDA_SUCCESS) drv().unmap(static_cast<CUdeviceptr>(va), page_bytes_);
        }
        lk.lock();
        --inflight_handles_;
        inflight_.erase(va);
        stats_.map_call_ns_total += map_ns;
        stats_.access_ns_total += acc_ns;
        ++stats_.access_calls;
        if (r == CUDA_SUCCESS) {
            parked_.emplace(va, Parked{h, 0, true});
            ++stats_.premaps;
        } else {
            cache_.push_back(h);
            hints_.clear();
        }
        stats_.background_ns_total += ns_since(t0);
        --worker_busy_;
        done_cv_.notify_all();
    }
}

void VmmDevice::premap(std::uint64_t owner, const std::uint64_t* vas, std::size_t n) {
    {
        Lock lk(mu_);
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
        return worker_busy_ == 0 && hints_.empty() &&
               !(cache_.size() < cache_target_ && total_locked() < budget_);
    });
}

void VmmDevice::wait_inflight(Lock& lk, std::uint64_t va) {
    while (inflight_.count(va)) done_cv_.wait(lk);
}

// ---------------------------------------------------------------- caller side

std::uint64_t VmmDevice::total_locked() const {
    return live_.size() + parked_.size() + buffer_.size() + taken_.size() + cache_.size() + inflight_handles_;
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

std::uint64_t VmmDevice::reserve(std::uint64_t pages) {
    CUdeviceptr va = 0;
    cu_check(drv().reserve(&va, pages * page_bytes_, page_bytes_, 0, 0), "cuMemAddressReserve");
    return static_cast<std::uint64_t>(va);
}

void VmmDevice::release(std::uint64_t va, std::uint64_t pages) {
    Lock lk(mu_);
    const std::uint64_t end = va + pages * page_bytes_;
    hints_.erase(va);
    // the worker may be mapping into (or stealing from) this range
    done_cv_.wait(lk, [&] {
        for (std::uint64_t v : inflight_) {
            if (v >= va && v < end) return false;
        }
        return true;
    });
    bool synced = false;
    const auto sync = [&] {
        if (!synced) PRISM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
        synced = true;
    };
    for (auto it = parked_.lower_bound(va); it != parked_.end() && it->first < end;) {
        if (!it->second.clean) sync();
        driver_unmap(it->first);
        cache_.push_back(it->second.handle);
        it = parked_.erase(it);
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

std::uint64_t VmmDevice::steal(Lock& lk) {
    // Prefer the highest parked VA that is safe to move (pre-mapped and never
    // read, or released before a fence that passed): allocation reuses the
    // lowest unmapped page indices, so high parked pages are least likely to
    // be revived soon.
    advance_fences(false);
    auto pick = parked_.end();
    for (auto it = parked_.rbegin(); it != parked_.rend(); ++it) {
        if (it->second.clean || it->second.epoch < fenced_) {
            pick = std::prev(it.base());
            break;
        }
    }
    if (pick == parked_.end()) {
        // Every parked page may still be read by in-flight kernels: fence
        // now and wait, after which all of them are safe.
        fence_locked();
        advance_fences(true);
        pick = std::prev(parked_.end());
    }
    const auto t0 = Clock::now();
    driver_unmap(pick->first);
    const std::uint64_t h = pick->second.handle;
    parked_.erase(pick);
    ++stats_.steals;
    stats_.steal_ns_total += ns_since(t0);  // inside a map: counted by map_ns_total
    (void)lk;
    return h;
}

void VmmDevice::steal_batch(Lock& lk, std::size_t k) {
    if (k == 0 || parked_.empty()) return;
    advance_fences(false);
    std::vector<std::uint64_t> vas;
    vas.reserve(k);
    for (auto it = parked_.rbegin(); it != parked_.rend() && vas.size() < k; ++it) {
        if (it->second.clean || it->second.epoch < fenced_) vas.push_back(it->first);
    }
    if (vas.size() < k) {
        fence_locked();
        advance_fences(true);  // every parked page is now safe
        vas.clear();
        for (auto it = parked_.rbegin(); it != parked_.rend() && vas.size() < k; ++it) vas.push_back(it->first);
    }
    const auto t0 = Clock::now();
    std::sort(vas.begin(), vas.end());
    for (std::size_t i = 0; i < vas.size();) {
        std::size_t j = i + 1;
        while (j < vas.size() && vas[j] == vas[j - 1] + page_bytes_) ++j;
        // One cuMemUnmap for a run of whole mappings; per page if refused.
        bool done = false;
        if (j - i > 1) {
            done = drv().unmap(static_cast<CUdeviceptr>(vas[i]), (j - i) * page_bytes_) == CUDA_SUCCESS;
            if (done) {
                ++stats_.driver_unmaps;
                ++stats_.batched_unmaps;
            }
        }
        for (std::size_t x = i; x < j; ++x) {
            if (!done) driver_unmap(vas[x]);
            const auto p = parked_.find(vas[x]);
            cache_.push_back(p->second.handle);
            parked_.erase(p);
            ++stats_.steals;
        }
        i = j;
    }
    stats_.steal_ns_total += ns_since(t0);
    (void)lk;
}

std::uint64_t VmmDevice::acquire_handle(Lock& lk, bool from_buffer) {
    if (from_buffer && !taken_.empty()) {
        const std::uint64_t h = taken_.back();
        taken_.pop_back();
        return h;
    }
    if (!cache_.empty()) {
        const std::uint64_t h = cache_.back();
        cache_.pop_back();
        return h;
    }
    if (total_locked() >= budget_ && !parked_.empty()) return steal(lk);
    const auto tc = Clock::now();
    CUmemGenericAllocationHandle h = 0;
    CUresult r = drv().create(&h, page_bytes_, &prop_of(prop_), 0);
    if (r == CUDA_ERROR_OUT_OF_MEMORY && !parked_.empty()) return steal(lk);
    cu_check(r, "cuMemCreate");
    ++stats_.creates;
    stats_.create_ns_total += ns_since(tc);
    return static_cast<std::uint64_t>(h);
}

void VmmDevice::map(std::uint64_t va, bool from_buffer) {
    const std::uint64_t one[1] = {va};
    map_batch(one, 1, from_buffer ? 1 : 0);
}

void VmmDevice::map_batch(const std::uint64_t* vas, std::size_t n, std::size_t n_from_buffer) {
    if (n == 0) return;
    const auto t0 = Clock::now();
    Lock lk(mu_);
    for (std::size_t i = 0; i < n; ++i) wait_inflight(lk, vas[i]);
    stats_.maps += n;
    {
        // Handles this batch must obtain by stealing (budget exhausted):
        // steal them together so contiguous parked runs share a cuMemUnmap.
        std::size_t fresh = 0, buffered = 0;
        for (std::size_t i = 0; i < n; ++i) {
            if (parked_.find(vas[i]) != parked_.end()) continue;
            ++fresh;
            if (i < n_from_buffer) ++buffered;
        }
        const std::size_t have = std::min(buffered, taken_.size()) + cache_.size();
        const std::uint64_t total = total_locked();
        const std::uint64_t room = budget_ > total ? budget_ - total : 0;
        if (fresh > have + room) {
            // never steal a page this batch is about to revive
            std::vector<std::pair<std::uint64_t, Parked>> keep;
            for (std::size_t i = 0; i < n; ++i) {
                const auto p = parked_.find(vas[i]);
                if (p != parked_.end()) {
                    keep.emplace_back(*p);
                    parked_.erase(p);
                }
            }
            steal_batch(lk, fresh - have - room);
            for (auto& kv : keep) parked_.emplace(kv.first, kv.second);
        }
    }
    for (std::size_t i = 0; i < n; ++i) {
        const bool from_buffer = i < n_from_buffer;
        const auto p = parked_.find(vas[i]);
        if (p != parked_.end()) {
            // Revive in place; a buffer handle earmarked for this map returns
            // to the cache (it stays counted as physical memory).
            if (p->second.clean) ++stats_.premapped_hits;
            live_.emplace(vas[i], p->second.handle);
            parked_.erase(p);
            if (from_buffer && !taken_.empty()) {
                cache_.push_back(taken_.back());
                taken_.pop_back();
            }
            ++stats_.revived;
            continue;
        }
        const std::uint64_t h = acquire_handle(lk, from_buffer);
        const auto tm = Clock::now();
        cu_check(drv().map(static_cast<CUdeviceptr>(vas[i]), page_bytes_, 0,
                           static_cast<CUmemGenericAllocationHandle>(h), 0),
                 "cuMemMap");
        stats_.map_call_ns_total += ns_since(tm);
        live_.emplace(vas[i], h);
        unaccessed_.push_back(vas[i]);
    }
    if (!defer_access_) flush_now(lk);
    const double per = ns_since(t0) / static_cast<double>(n);
    stats_.map_ns_total += per * static_cast<double>(n);
    for (std::size_t i = 0; i < n; ++i) sample(stats_.map_ns, per);
}

void VmmDevice::defer_access(bool on) {
    {
        Lock lk(mu_);
        defer_access_ = on;
    }
    if (!on) flush_access();
}

void VmmDevice::flush_access() {
    // Deferred flush (outside map_batch): its time belongs to the maps.
    const auto t0 = Clock::now();
    Lock lk(mu_);
    if (unaccessed_.empty()) return;
    flush_now(lk);
    stats_.map_ns_total += ns_since(t0);
}

void VmmDevice::flush_now(Lock& lk) {
    (void)lk;
    if (unaccessed_.empty()) return;
    std::sort(unaccessed_.begin(), unaccessed_.end());
    for (std::size_t i = 0; i < unaccessed_.size();) {
        std::size_t j = i + 1;
        while (j < unaccessed_.size() && unaccessed_[j] == unaccessed_[j - 1] + page_bytes_) ++j;
        const auto ta = Clock::now();
        cu_check(drv().set_access(static_cast<CUdeviceptr>(unaccessed_[i]), (j - i) * page_bytes_,
                                  &access_of(access_desc_), 1),
                 "cuMemSetAccess");
        stats_.access_ns_total += ns_since(ta);
        ++stats_.access_calls;
        i = j;
    }
    unaccessed_.clear();
}

void VmmDevice::unmap(std::uint64_t va) {
    const auto t0 = Clock::now();
    Lock lk(mu_);
    const auto it = live_.find(va);
    if (it == live_.end()) throw std::runtime_error("VmmDevice::unmap: page not mapped");
    parked_.emplace(va, Parked{it->second, epoch_, false});
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
        // Everything goes back: stop pre-mapping and wait for the worker.
        hints_.clear();
        done_cv_.wait(lk, [&] { return inflight_.empty(); });
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
            it = parked_.erase(it);
        } else {
            ++it;
        }
    }
    stats_.unmap_ns_total += ns_since(t0);
}

void VmmDevice::grow_buffer(std::uint64_t n) {
    Lock lk(mu_);
    for (std::uint64_t i = 0; i < n; ++i) buffer_.push_back(acquire_handle(lk, false));
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
        drv().release(static_cast<CUmemGenericAllocationHandle>(steal(lk)));
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
