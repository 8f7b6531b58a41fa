// prism::VmmDevice — CUDA virtual-memory backend of one GPU's page ledger.
//
// Implements the physical side of the kvcached-style elastic pool
// (§5.1; the reference only models it: SPEC.md:193 lists "real CUDA
// VMM calls" as a non-goal). One instance per GPU, owned by the caller and
// attached to that GPU's PhysicalLedger. All calls come from the ledger's
// serialization domain (one host thread per GPU), so there are no locks.
//
//   reserve/release   cuMemAddressReserve / cuMemAddressFree of a pool's whole
//                     virtual range (V x 2 MiB), 2 MiB aligned.
//   map               back one 2 MiB VA page with a physical handle: from the
//                     pre-created buffer (ledger buffer hit), else the recycle
//                     cache, else cuMemCreate; then cuMemMap + cuMemSetAccess.
//   unmap             deferred: the page joins a pending list that is only
//                     cuMemUnmap'ed once the GPU work issued before it has
//                     drained (reclaim()), because cuMemUnmap is synchronous
//                     on the device. A pending page that is mapped again
//                     before that is revived in place with no driver call.
//   grow/shrink       keep `buffer` pre-created handles (ledger refill_buffer /
//                     take_buffer).
// Latencies of every driver call are recorded for the map/unmap metric.
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

namespace prism {

struct VmmStats {
    std::uint64_t maps = 0;           // logical page maps requested
    std::uint64_t revived = 0;        // maps satisfied by reviving a pending unmap
    std::uint64_t creates = 0;        // cuMemCreate calls
    std::uint64_t unmaps = 0;         // logical unmaps requested
    std::uint64_t driver_unmaps = 0;  // cuMemUnmap calls actually issued
    double map_ns_total = 0.0;        // host wall time inside map() (all paths)
    double unmap_ns_total = 0.0;      // host wall time inside unmap() + reclaim()
    std::vector<float> map_ns;        // per-map samples (bounded ring)
    std::vector<float> unmap_ns;      // per driver-unmap samples (bounded ring)
};

class VmmDevice {
public:
    // Opens CUDA device `ordinal`; throws std::runtime_error (CUDA missing,
    // no such device, VMM unsupported, 2 MiB not a multiple of granularity).
    static std::unique_ptr<VmmDevice> open(int ordinal, std::uint64_t page_bytes);
    ~VmmDevice();

    int ordinal() const { return ordinal_; }
    std::uint64_t page_bytes() const { return page_bytes_; }

    std::uint64_t reserve(std::uint64_t pages);
    void release(std::uint64_t va, std::uint64_t pages);  // all pages must be unmapped/pending

    void map(std::uint64_t page_va, bool from_buffer);
    void unmap(std::uint64_t page_va);
    // Issue cuMemUnmap for pending pages whose fence completed (wait=false) or
    // for all of them after synchronising the device (wait=true).
    void reclaim(bool wait);
    // The GPU's work stream (cudaStream_t). Every engine on this GPU issues its
    // kernels here, so one fence orders all readers of the pool pages.
    void* stream() const { return stream_; }
    // Record a fence on stream(): pages unmapped before this call become
    // reclaimable once the stream passes it.
    void fence();

    void grow_buffer(std::uint64_t n);
    void take_buffer(std::uint64_t n);  // handles leave the buffer for map(from_buffer=true)
    std::uint64_t buffered_handles() const { return buffer_.size(); }
    std::uint64_t cached_handles() const { return cache_.size(); }
    std::uint64_t pending_unmaps() const { return pending_.size(); }

    const VmmStats& stats() const { return stats_; }
    void reset_stats();

    // Free physical memory in bytes (cudaMemGetInfo) and the ledger capacity
    // in pages that leaves `reserve_bytes` for everything else.
    std::uint64_t capacity_pages(std::uint64_t reserve_bytes) const;

private:
    VmmDevice() = default;
    std::uint64_t new_handle();
    void drop_handle(std::uint64_t h);
    void driver_unmap(std::uint64_t va);

    struct Pending {
        std::uint64_t handle;
        std::uint64_t epoch;
    };

    int ordinal_ = 0;
    std::uint64_t page_bytes_ = 0;
    std::vector<std::uint64_t> buffer_;   // pre-created, counted by the ledger's buffer
    std::vector<std::uint64_t> taken_;    // taken from the buffer, waiting for map()
    std::vector<std::uint64_t> cache_;    // recycled after unmap, not counted by the ledger
    std::unordered_map<std::uint64_t, std::uint64_t> live_;     // va -> handle (mapped)
    std::unordered_map<std::uint64_t, Pending> pending_;        // va -> handle (logically unmapped)
    std::vector<void*> fences_;           // cudaEvent_t per epoch, oldest first
    std::uint64_t epoch_ = 0;             // current epoch (fences recorded so far)
    std::uint64_t fenced_epoch_ = 0;      // epochs <= this are known complete
    std::uint64_t cache_limit_ = 64;
    VmmStats stats_;
    void* access_desc_ = nullptr;         // CUmemAccessDesc
    void* prop_ = nullptr;                // CUmemAllocationProp
    void* stream_ = nullptr;              // cudaStream_t (non-blocking)
};

}  // namespace prism
