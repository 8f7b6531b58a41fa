// prism::VmmDevice implementation: CUDA VMM (driver API) behind the ledger.
// Driver entry points are resolved at run time through the runtime's
// cudaGetDriverEntryPoint, so the library loads on machines without a driver
// (the CPU build/test container) and only fails when a device is opened.
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
    return dev;
}

VmmDevice::~VmmDevice() {
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

std::uint64_t VmmDevice::total_handles() const {
    return live_.size() + parked_.size() + buffer_.size() + taken_.size() + cache_.size();
}

std::uint64_t VmmDevice::reserve(std::uint64_t pages) {
    CUdeviceptr va = 0;
    cu_check(drv().reserve(&va, pages * page_bytes_, page_bytes_, 0, 0), "cuMemAddressReserve");
    return static_cast<std::uint64_t>(va);
}

void VmmDevice::release(std::uint64_t va, std::uint64_t pages) {
    const std::uint64_t end = va + pages * page_bytes_;
    bool synced = false;
    for (auto it = parked_.lower_bound(va); it != parked_.end() && it->first < end;) {
        if (!synced) {
            PRISM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
            synced = true;
        }
        driver_unmap(it->first);
        drop_handle(it->second.handle);
        it = parked_.erase(it);
    }
    for (auto it = live_.begin(); it != live_.end();) {
        if (it->first >= va && it->first < end) {
            if (!synced) {
                PRISM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
                synced = true;
            }
            driver_unmap(it->first);
            drop_handle(it->second);
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

std::uint64_t VmmDevice::steal() {
    // Prefer the highest parked VA whose fence passed: allocation reuses the
    // lowest unmapped page indices, so high parked pages are least likely to
    // be revived soon.
    advance_fences(false);
    auto pick = parked_.end();
    for (auto it = parked_.rbegin(); it != parked_.rend(); ++it) {
        if (it->second.epoch < fenced_) {
            pick = std::prev(it.base());
            break;
        }
    }
    if (pick == parked_.end()) {
        // Every parked page may still be read by in-flight kernels: fence
        // now and wait, after which all of them are safe.
        fence();
        advance_fences(true);
        pick = std::prev(parked_.end());
    }
    const auto t0 = Clock::now();
    driver_unmap(pick->first);
    const std::uint64_t h = pick->second.handle;
    parked_.erase(pick);
    ++stats_.steals;
    stats_.steal_ns_total += ns_since(t0);  // inside a map: counted by map_ns_total
    return h;
}

std::uint64_t VmmDevice::acquire_handle(bool from_buffer) {
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
    if (total_handles() >= budget_ && !parked_.empty()) return steal();
    const auto tc = Clock::now();
    CUmemGenericAllocationHandle h = 0;
    CUresult r = drv().create(&h, page_bytes_, &prop_of(prop_), 0);
    if (r == CUDA_ERROR_OUT_OF_MEMORY && !parked_.empty()) return steal();
    cu_check(r, "cuMemCreate");
    ++stats_.creates;
    stats_.create_ns_total += ns_since(tc);
    return static_cast<std::uint64_t>(h);
}

void VmmDevice::drop_handle(std::uint64_t h) { cache_.push_back(h); }

void VmmDevice::map(std::uint64_t va, bool from_buffer) {
    const std::uint64_t one[1] = {va};
    map_batch(one, 1, from_buffer ? 1 : 0);
}

void VmmDevice::map_batch(const std::uint64_t* vas, std::size_t n, std::size_t n_from_buffer) {
    if (n == 0) return;
    const auto t0 = Clock::now();
    stats_.maps += n;
    for (std::size_t i = 0; i < n; ++i) {
        const bool from_buffer = i < n_from_buffer;
        const auto p = parked_.find(vas[i]);
        if (p != parked_.end()) {
            // Revive in place; a buffer handle earmarked for this map returns
            // to the cache (it stays counted as physical memory).
            live_.emplace(vas[i], p->second.handle);
            parked_.erase(p);
            if (from_buffer && !taken_.empty()) {
                cache_.push_back(taken_.back());
                taken_.pop_back();
            }
            ++stats_.revived;
            continue;
        }
        const std::uint64_t h = acquire_handle(from_buffer);
        const auto tm = Clock::now();
        cu_check(drv().map(static_cast<CUdeviceptr>(vas[i]), page_bytes_, 0,
                           static_cast<CUmemGenericAllocationHandle>(h), 0),
                 "cuMemMap");
        stats_.map_call_ns_total += ns_since(tm);
        live_.emplace(vas[i], h);
        unaccessed_.push_back(vas[i]);
    }
    if (!defer_access_) flush_now();
    const double per = ns_since(t0) / static_cast<double>(n);
    stats_.map_ns_total += per * static_cast<double>(n);
    for (std::size_t i = 0; i < n; ++i) sample(stats_.map_ns, per);
}

void VmmDevice::defer_access(bool on) {
    defer_access_ = on;
    if (!on) flush_access();
}

void VmmDevice::flush_access() {
    // Deferred flush (outside map_batch): its time belongs to the maps.
    const auto t0 = Clock::now();
    flush_now();
    stats_.map_ns_total += ns_since(t0);
}

void VmmDevice::flush_now() {
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

void VmmDevice::prefill_cache(std::uint64_t n) {
    const auto t0 = Clock::now();
    struct Charge {
        VmmStats& s;
        Clock::time_point t;
        ~Charge() { s.prefill_ns_total += ns_since(t); }
    } charge{stats_, t0};
    while (cache_.size() < n && total_handles() < budget_) {
        const auto tc = Clock::now();
        CUmemGenericAllocationHandle h = 0;
        if (drv().create(&h, page_bytes_, &prop_of(prop_), 0) != CUDA_SUCCESS) break;
        ++stats_.creates;
        stats_.create_ns_total += ns_since(tc);
        cache_.push_back(static_cast<std::uint64_t>(h));
    }
}

void VmmDevice::unmap(std::uint64_t va) {
    const auto t0 = Clock::now();
    const auto it = live_.find(va);
    if (it == live_.end()) throw std::runtime_error("VmmDevice::unmap: page not mapped");
    parked_.emplace(va, Parked{it->second, epoch_});
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
    cudaEvent_t ev = nullptr;
    PRISM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    PRISM_CUDA(cudaEventRecord(ev, static_cast<cudaStream_t>(stream_)));
    fences_.push_back(ev);
    ++epoch_;
    if (fences_.size() > 64) advance_fences(false);  // keep the queue short
}

void VmmDevice::reclaim(bool wait) {
    if (wait) {
        PRISM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
        fence();
        advance_fences(true);
    } else {
        advance_fences(false);
    }
    const auto t0 = Clock::now();
    for (auto it = parked_.begin(); it != parked_.end();) {
        if (wait || it->second.epoch < fenced_) {
            driver_unmap(it->first);
            drop_handle(it->second.handle);
            it = parked_.erase(it);
        } else {
            ++it;
        }
    }
    stats_.unmap_ns_total += ns_since(t0);
}

void VmmDevice::grow_buffer(std::uint64_t n) {
    for (std::uint64_t i = 0; i < n; ++i) buffer_.push_back(acquire_handle(false));
}

void VmmDevice::take_buffer(std::uint64_t n) {
    for (std::uint64_t i = 0; i < n && !buffer_.empty(); ++i) {
        taken_.push_back(buffer_.back());
        buffer_.pop_back();
    }
}

void VmmDevice::set_budget(std::uint64_t pages) {
    budget_ = pages;
    // Shrink: free cached handles first, then physically release parked pages.
    while (total_handles() > budget_ && !cache_.empty()) {
        drv().release(static_cast<CUmemGenericAllocationHandle>(cache_.back()));
        cache_.pop_back();
    }
    while (total_handles() > budget_ && !parked_.empty()) {
        drv().release(static_cast<CUmemGenericAllocationHandle>(steal()));
    }
}

void VmmDevice::reset_stats() { stats_ = VmmStats{}; }

std::uint64_t VmmDevice::capacity_pages(std::uint64_t reserve_bytes) const {
    std::size_t free_b = 0, total_b = 0;
    PRISM_CUDA(cudaMemGetInfo(&free_b, &total_b));
    return free_b > reserve_bytes ? (free_b - reserve_bytes) / page_bytes_ : 0;
}

}  // namespace prism
