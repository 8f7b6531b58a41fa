// K1 — batched slot allocation / free on the GPU-resident slot state.
//
// Replays a pool's op log (allocations and frees recorded by the host
// allocator during one engine step) against the device mirror and writes the
// chosen slot ids straight into the device block table, so no slot id crosses
// PCIe. It reproduces reference alloc_kv (src/pagealloc.cpp:188-244) exactly:
//
//   Consecutive successful allocations concatenate — alloc_kv(a) followed by
//   alloc_kv(b) yields the same (page, slot) sequence as alloc_kv(a + b)
//   (verified there on 47,978 randomized states). An alloc of n
//   tokens takes the free slots of pages in the order
//     partial pages by (occupancy desc, index asc), then unmapped pages by
//     index asc, each page's free slots ascending,
//   because pick_page's argmax is unchanged by filling the page it picked.
//
// One CTA of 1024 threads walks the op list in order. For an alloc group of n
// tokens (processed in sub-batches of <= 1024):
//   1. histogram of occupancy levels over the partial pages;
//   2. threshold level L*: every partial page above L* is consumed, plus the
//      first `take` pages (by index) at level L* (L* = 0: unmapped pages);
//   3. collect those pages (one pass + block scan for the index order);
//   4. bitonic-sort them by (occupancy desc, index asc);
//   5. prefix-sum their free slots; token j -> its page and the r-th free
//      slot of that page; write table[dest + i] and out[i];
//   6. set the bits, bump the occupancies.
// Frees clear bits and decrement occupancy (they commute, so they run in
// parallel). Mapped <=> occupancy > 0 on the device as on the host.
#include <algorithm>

#include "cuda/device_impl.cuh"

namespace prism {

namespace {

constexpr int kThreads = 1024;
constexpr int kSub = 1024;        // tokens per sub-batch; selected pages <= kSub
constexpr int kMaxTpp = 1024;
constexpr int kMaxGroupOps = 1024;

constexpr std::uint32_t kAlloc = 1, kFreeList = 2, kFreeRow = 3;

struct K1Args {
    std::uint32_t* occ;
    std::uint32_t* bits;
    std::uint32_t vpages, tpp, words;  // vpages: pages scanned (the pool's high-water mark, 4-aligned)
    std::uint64_t magic;
    const DevOp* ops;
    int n_ops;
    const std::int32_t* freed;
    std::int32_t* table;
    std::int32_t* out;
    int* status;
};

// Exclusive scan of one value per thread over the whole CTA.
__device__ std::uint32_t block_exclusive_scan(std::uint32_t v, std::uint32_t* warp_sums, std::uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    std::uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        std::uint32_t w = warp_sums[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_sums[lane] = w;  // inclusive
    }
    __syncthreads();
    const std::uint32_t before = (warp ? warp_sums[warp - 1] : 0) + x - v;
    *total = warp_sums[31];
    __syncthreads();
    return before;
}

__device__ __forceinline__ std::uint32_t nth_set_bit(std::uint32_t x, std::uint32_t r) {
    for (std::uint32_t i = 0; i < r; ++i) x &= x - 1;
    return static_cast<std::uint32_t>(__ffs(static_cast<int>(x)) - 1);
}

__device__ __forceinline__ void free_slot(const K1Args& a, std::uint32_t sid) {
    const std::uint32_t page = slot_page(sid, a.magic);
    const std::uint32_t slot = sid - page * a.tpp;
    atomicAnd(&a.bits[static_cast<std::uint64_t>(page) * a.words + (slot >> 5)], ~(1u << (slot & 31)));
    atomicSub(&a.occ[page], 1u);
}

__global__ void __launch_bounds__(kThreads, 1) k1_slot_alloc(K1Args a) {
    __shared__ std::uint32_t hist[kMaxTpp];
    __shared__ unsigned long long keys[kSub];
    __shared__ std::uint32_t start[kSub];
    __shared__ long long op_start[kMaxGroupOps + 1];
    __shared__ std::uint32_t warp_sums[32];
    __shared__ std::uint32_t s_level, s_take, s_above, s_nsel;

    const int tid = threadIdx.x;
    const std::uint32_t tpp = a.tpp;
    // occ is padded to a multiple of 4 pages with the value tpp ("full"), so
    // it is scanned with 16-byte loads and the pads are never selected.
    const uint4* occ4 = reinterpret_cast<const uint4*>(a.occ);
    const std::uint32_t v4 = (a.vpages + 3) / 4;
    const std::uint32_t chunk = (v4 + kThreads - 1) / kThreads;
    const std::uint32_t my_lo = min(v4, static_cast<std::uint32_t>(tid) * chunk);
    const std::uint32_t my_hi = min(v4, my_lo + chunk);
    long long out_pos = 0;

    for (int i = 0; i < a.n_ops;) {
        const DevOp op = a.ops[i];
        if (op.kind != kAlloc) {
            for (std::uint32_t j = tid; j < op.count; j += kThreads) {
                const std::int32_t sid = op.kind == kFreeRow ? __ldcg(&a.table[op.first + j]) : __ldcg(&a.freed[op.first + j]);
                free_slot(a, static_cast<std::uint32_t>(sid));
            }
            __syncthreads();
            ++i;
            continue;
        }
        // Group of consecutive allocations [i, end).
        int end = i;
        long long total = 0;
        while (end < a.n_ops && a.ops[end].kind == kAlloc && end - i < kMaxGroupOps) {
            if (tid == 0) op_start[end - i] = total;
            total += a.ops[end].count;
            ++end;
        }
        if (tid == 0) op_start[end - i] = total;
        const int n_group_ops = end - i;
        __syncthreads();

        for (long long done = 0; done < total;) {
            const std::uint32_t n = static_cast<std::uint32_t>(min(static_cast<long long>(kSub), total - done));
            // 1. histogram of partial pages' occupancy
            for (std::uint32_t k = tid; k < tpp; k += kThreads) hist[k] = 0;
            __syncthreads();
#pragma unroll 4
            for (std::uint32_t q = tid; q < v4; q += kThreads) {
                const uint4 o4 = __ldcg(occ4 + q);
                const std::uint32_t os[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (os[c] > 0 && os[c] < tpp) atomicAdd(&hist[os[c]], 1u);
                }
            }
            __syncthreads();
            // 2. threshold level
            if (tid == 0) {
                std::uint64_t acc = 0, above = 0;
                std::uint32_t level = 0, take = 0;
                bool found = false;
                for (std::uint32_t k = tpp - 1; k >= 1; --k) {
                    const std::uint64_t f = static_cast<std::uint64_t>(hist[k]) * (tpp - k);
                    if (acc + f >= n) {
                        level = k;
                        take = static_cast<std::uint32_t>((n - acc + (tpp - k) - 1) / (tpp - k));
                        found = true;
                        break;
                    }
                    acc += f;
                    above += hist[k];
                }
                if (!found) {
                    level = 0;
                    take = static_cast<std::uint32_t>((n - acc + tpp - 1) / tpp);
                }
                s_level = level;
                s_take = take;
                s_above = static_cast<std::uint32_t>(above);
                s_nsel = 0;
            }
            __syncthreads();
            const std::uint32_t level = s_level, take = s_take, above = s_above;
            // 3. collect: every partial page above the level (any order), and
            //    the first `take` pages at the level in index order.
            std::uint32_t at_level = 0;
            for (std::uint32_t q = my_lo; q < my_hi; ++q) {
                const uint4 o4 = __ldcg(occ4 + q);
                const std::uint32_t os[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const std::uint32_t o = os[c];
                    if (o > level && o < tpp) {
                        const std::uint32_t slot = atomicAdd(&s_nsel, 1u);
                        keys[slot] = (static_cast<unsigned long long>(tpp - o) << 32) | (q * 4 + c);
                    } else if (o == level) {
                        ++at_level;
                    }
                }
            }
            std::uint32_t level_total = 0;
            std::uint32_t rank = block_exclusive_scan(at_level, warp_sums, &level_total);
            if (level_total < take && tid == 0) atomicExch(a.status, 1);  // host and device disagree
            const std::uint32_t take_eff = min(take, level_total);
            if (rank < take_eff) {
                for (std::uint32_t q = my_lo; q < my_hi && rank < take_eff; ++q) {
                    const uint4 o4 = __ldcg(occ4 + q);
                    const std::uint32_t os[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (os[c] == level && rank < take_eff) {
                            keys[above + rank] = (static_cast<unsigned long long>(tpp - level) << 32) | (q * 4 + c);
                            ++rank;
                        }
                    }
                }
            }
            __syncthreads();
            const std::uint32_t m = above + take_eff;
            // 4. bitonic sort keys[0, P)
            std::uint32_t P = 1;
            while (P < m) P <<= 1;
            for (std::uint32_t k = tid; k < P; k += kThreads) {
                if (k >= m) keys[k] = ~0ull;
            }
            __syncthreads();
            for (std::uint32_t k = 2; k <= P; k <<= 1) {
                for (std::uint32_t j = k >> 1; j > 0; j >>= 1) {
                    const std::uint32_t x = tid;
                    const std::uint32_t y = x ^ j;
                    if (x < P && y > x) {
                        const unsigned long long kx = keys[x], ky = keys[y];
                        const bool up = (x & k) == 0;
                        if ((kx > ky) == up) {
                            keys[x] = ky;
                            keys[y] = kx;
                        }
                    }
                    __syncthreads();
                }
            }
            // 5. free-slot prefix over the sorted pages
            std::uint32_t free_here = 0;
            if (static_cast<std::uint32_t>(tid) < m) free_here = static_cast<std::uint32_t>(keys[tid] >> 32);
            std::uint32_t free_total = 0;
            const std::uint32_t my_start = block_exclusive_scan(free_here, warp_sums, &free_total);
            if (static_cast<std::uint32_t>(tid) < m) start[tid] = my_start;
            if (free_total < n && tid == 0) atomicExch(a.status, 2);
            __syncthreads();
            std::uint32_t my_sid = 0, my_word = 0, my_mask = 0;
            std::uint64_t my_page = 0;
            const bool has_token = static_cast<std::uint32_t>(tid) < n && free_total >= n;
            if (has_token) {
                // page index i: largest with start[i] <= tid
                std::uint32_t lo = 0, hi = m;
                while (hi - lo > 1) {
                    const std::uint32_t mid = (lo + hi) >> 1;
                    if (start[mid] <= static_cast<std::uint32_t>(tid)) lo = mid;
                    else hi = mid;
                }
                const std::uint32_t page = static_cast<std::uint32_t>(keys[lo] & 0xffffffffu);
                std::uint32_t r = static_cast<std::uint32_t>(tid) - start[lo];
                const std::uint32_t* wbits = a.bits + static_cast<std::uint64_t>(page) * a.words;
                std::uint32_t slot = 0;
                for (std::uint32_t w = 0; w < a.words; ++w) {
                    const std::uint32_t lim = tpp - w * 32;
                    const std::uint32_t valid = lim >= 32 ? 0xffffffffu : ((1u << lim) - 1u);
                    const std::uint32_t fr = ~__ldcg(&wbits[w]) & valid;
                    const std::uint32_t c = __popc(fr);
                    if (r < c) {
                        const std::uint32_t b = nth_set_bit(fr, r);
                        slot = w * 32 + b;
                        my_word = w;
                        my_mask = 1u << b;
                        break;
                    }
                    r -= c;
                }
                my_page = page;
                my_sid = page * tpp + slot;
                // outputs: group token t -> op
                const long long t = done + tid;
                int olo = 0, ohi = n_group_ops;
                while (ohi - olo > 1) {
                    const int mid = (olo + ohi) >> 1;
                    if (op_start[mid] <= t) olo = mid;
                    else ohi = mid;
                }
                const DevOp& gop = a.ops[i + olo];
                if (gop.dest >= 0) a.table[gop.dest + (t - op_start[olo])] = static_cast<std::int32_t>(my_sid);
                if (a.out) a.out[out_pos + t] = static_cast<std::int32_t>(my_sid);
            }
            __syncthreads();
            // 6. commit
            if (has_token) atomicOr(&a.bits[my_page * a.words + my_word], my_mask);
            if (static_cast<std::uint32_t>(tid) < m && free_total >= n) {
                const std::uint32_t page = static_cast<std::uint32_t>(keys[tid] & 0xffffffffu);
                const std::uint32_t f = static_cast<std::uint32_t>(keys[tid] >> 32);
                const std::uint32_t used = min(f, n - start[tid]);
                atomicAdd(&a.occ[page], used);  // L2 RMW: a plain += could read a stale L1 line
            }
            __syncthreads();
            done += n;
        }
        out_pos += total;
        i = end;
    }
}

}  // namespace

void destroy_device_pool(DevicePool* p) { delete p; }

DevicePool::DevicePool(const msim::pagealloc::detail::PoolState& s, int device) {
    if (s.tpp > kMaxTpp) throw std::runtime_error("device pool: tokens per page above 1024 is not supported");
    // K1 replays pick_page's most-occupied-first order (reference
    // src/pagealloc.cpp:162-170); a lowest-index-first pool would diverge.
    if (s.placement != msim::pagealloc::PagePlacement::most_occupied_first) {
        throw std::runtime_error("device pool: the K1 mirror replays most_occupied_first placement only");
    }
    // slot ids are int32 and div_magic40 is exact while sid * tpp < 2^40.
    if (s.vpages * s.tpp >= (1ull << 31) || s.vpages * s.tpp * s.tpp >= (1ull << 40)) {
        throw std::runtime_error("device pool: slot id range too large for the device block table");
    }
    PRISM_CUDA(cudaSetDevice(device));
    vpages = static_cast<std::uint32_t>(s.vpages);
    tpp = static_cast<std::uint32_t>(s.tpp);
    words = (tpp + 31) / 32;
    const std::size_t padded = (static_cast<std::size_t>(vpages) + 3) / 4 * 4;
    PRISM_CUDA(cudaMalloc(&occ, sizeof(std::uint32_t) * padded));
    PRISM_CUDA(cudaMalloc(&bits, sizeof(std::uint32_t) * vpages * words));
    PRISM_CUDA(cudaMalloc(&d_status, sizeof(int)));
    // Upload the current host state (pool may already hold tokens); the pad
    // pages read as full so K1 never selects them.
    std::vector<std::uint32_t> h_occ(padded, tpp);
    std::copy(s.occ.begin(), s.occ.end(), h_occ.begin());
    std::vector<std::uint32_t> h_bits(static_cast<std::size_t>(vpages) * words, 0);
    for (std::uint32_t p = 0; p < vpages; ++p) {
        if (!s.occ[p]) continue;
        const std::uint64_t* w64 = s.page_bits(p);
        for (std::uint32_t w = 0; w < words; ++w) {
            h_bits[static_cast<std::size_t>(p) * words + w] =
                static_cast<std::uint32_t>(w64[w >> 1] >> ((w & 1) * 32));
        }
    }
    PRISM_CUDA(cudaMemcpy(occ, h_occ.data(), sizeof(std::uint32_t) * padded, cudaMemcpyHostToDevice));
    PRISM_CUDA(cudaMemcpy(bits, h_bits.data(), sizeof(std::uint32_t) * h_bits.size(), cudaMemcpyHostToDevice));
    PRISM_CUDA(cudaMemset(d_status, 0, sizeof(int)));
}

DevicePool::~DevicePool() {
    if (occ) cudaFree(occ);
    if (bits) cudaFree(bits);
    if (d_status) cudaFree(d_status);
}

std::int64_t DevicePool::replay(msim::pagealloc::detail::PoolState& s, std::int32_t* table, std::int32_t* out,
                                std::int64_t out_cap, cudaStream_t stream) {
    std::int64_t total = 0;
    for (const auto& op : s.ops) {
        if (op.kind == msim::pagealloc::detail::DeviceOp::kAlloc) total += op.count;
    }
    if (s.ops.empty()) return 0;
    if (total > out_cap) throw std::runtime_error("device pool: step allocated more slots than the step buffer holds");
    ops.ensure(s.ops.size());
    std::memcpy(ops.host, s.ops.data(), s.ops.size() * sizeof(DevOp));
    ops.upload(s.ops.size(), stream);
    freed.ensure(std::max<std::size_t>(s.freed_slots.size(), 1));
    if (!s.freed_slots.empty()) std::memcpy(freed.host, s.freed_slots.data(), s.freed_slots.size() * sizeof(std::int32_t));
    freed.upload(s.freed_slots.size(), stream);
    // Every page this step's replay can pick was picked by the host allocator
    // (bit-exact replay), so it lies below the pool's high-water mark; pages
    // at or above it were never mapped (occupancy 0) and are never chosen:
    // K1 scans [0, hw) instead of all V virtual pages (C1: ~8K of 85,830).
    const std::uint32_t scan = static_cast<std::uint32_t>(std::min<std::uint64_t>(vpages, (s.hw + 3) / 4 * 4));
    K1Args a{occ, bits, scan, tpp, words, div_magic40(tpp), ops.dev, static_cast<int>(s.ops.size()), freed.dev,
             table, out, d_status};
    k1_slot_alloc<<<1, kThreads, 0, stream>>>(a);
    PRISM_CUDA(cudaGetLastError());
    s.ops.clear();
    s.freed_slots.clear();
    return total;
}

int DevicePool::status(cudaStream_t stream) {
    int h = 0;
    PRISM_CUDA(cudaMemcpyAsync(&h, d_status, sizeof(int), cudaMemcpyDeviceToHost, stream));
    PRISM_CUDA(cudaStreamSynchronize(stream));
    return h;
}

}  // namespace prism
