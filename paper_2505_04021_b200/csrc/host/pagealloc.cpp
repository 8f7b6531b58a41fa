// prism-b200 host allocator: PhysicalLedger + KvPool + alloc/free.
//
// Semantics follow reference proj/src/pagealloc.cpp line by line (cited per
// function); the data structures are new (see pool_state.hpp). When the
// ledger has a prism::VmmDevice attached, logical maps/unmaps drive real CUDA
// VMM calls and every slot change is appended to the pool's device op log.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "host/pool_state.hpp"
#include "host/vmm.hpp"

namespace msim::pagealloc {

const char* to_string(AllocEventKind k) {
    static const char* const names[] = {"map", "unmap", "buffer_hit", "alloc_fail"};
    const auto i = static_cast<unsigned>(k);
    return i < 4 ? names[i] : "?";
}

// ------------------------------------------------------------------ ledger
// reference src/pagealloc.cpp:17-106

PhysicalLedger::PhysicalLedger(int gpu_id, std::uint64_t capacity_pages, std::uint64_t page_bytes)
    : gpu_(gpu_id), page_bytes_(page_bytes), capacity_(capacity_pages) {
    if (page_bytes_ == 0) throw UsageError("ledger: zero page size");
}

void PhysicalLedger::attach_device(prism::VmmDevice* dev) {
    if (dev && dev->page_bytes() != page_bytes_) {
        throw UsageError("ledger: device page size differs from the ledger's");
    }
    if (dev && !pools_.empty()) throw UsageError("ledger: attach the device before creating pools");
    dev_ = dev;
    dev_hold_ = dev ? dev->shared_from_this() : nullptr;
    if (dev_) dev_->set_budget(capacity_ - weights_);  // physical pages the KV side may hold
    if (dev_ && buffer_ > dev_->buffered_handles()) dev_->grow_buffer(buffer_ - dev_->buffered_handles());
}

std::uint64_t PhysicalLedger::pool_mapped_pages(PoolId id) const {
    const auto it = pools_.find(id);
    return it == pools_.end() ? 0 : it->second.pages;
}

std::uint64_t PhysicalLedger::refill_buffer(std::uint64_t target_pages) {  // :27-34
    if (target_pages <= buffer_) return 0;
    const std::uint64_t add = std::min(target_pages - buffer_, free_pages());
    if (add == 0) return 0;
    if (dev_) dev_->grow_buffer(add);
    buffer_ += add;
    note("", AllocEventKind::map, add);
    return add;
}

bool PhysicalLedger::reserve_weight_pages(const std::string& model_id, std::uint64_t pages) {  // :42-50
    if (weight_by_model_.find(model_id) != weight_by_model_.end()) {
        throw UsageError("ledger: weights already resident for model " + model_id);
    }
    if (pages > free_pages()) return false;
    weight_by_model_.emplace(model_id, pages);
    weights_ += pages;
    if (dev_) dev_->set_budget(capacity_ - weights_);
    return true;
}

void PhysicalLedger::release_weight_pages(const std::string& model_id) {  // :52-59
    const auto it = weight_by_model_.find(model_id);
    if (it == weight_by_model_.end()) throw UsageError("ledger: no resident weights for model " + model_id);
    weights_ -= it->second;
    weight_by_model_.erase(it);
    if (dev_) dev_->set_budget(capacity_ - weights_);
}

std::uint64_t PhysicalLedger::weight_pages_of(const std::string& model_id) const {
    const auto it = weight_by_model_.find(model_id);
    return it == weight_by_model_.end() ? 0 : it->second;
}

void PhysicalLedger::note(const std::string& model, AllocEventKind kind, std::uint64_t pages) {  // :94-97
    if (recording_) log_.push_back(AllocEvent{now_, gpu_, model, kind, pages});
}

void PhysicalLedger::check_invariants() const {  // :99-106
    std::uint64_t total = 0;
    for (const auto& kv : pools_) total += kv.second.pages;
    if (total != kv_pages_) throw UsageError("ledger: per-pool counts drifted from total");
    if (kv_pages_ + buffer_ + weights_ > capacity_) {
        throw UsageError("ledger: mapped + buffer + weights exceeds capacity");
    }
}

// ------------------------------------------------------------------ pool accessors

KvPool::KvPool() : st_(std::make_unique<detail::PoolState>()) {}
KvPool::KvPool(KvPool&&) noexcept = default;
KvPool& KvPool::operator=(KvPool&&) noexcept = default;
KvPool::~KvPool() {
    // A pool dropped while alive keeps its pages accounted in the ledger (the
    // reference's destructor does nothing either); only device VA is returned.
    if (st_ && st_->dev && st_->va) {
        try {
            st_->dev->release(st_->va, st_->vpages);  // unmaps live + parked pages in the range
        } catch (...) {
        }
        st_->va = 0;
    }
}

PoolId KvPool::id() const { return st_->id; }
const std::string& KvPool::model_id() const { return st_->model; }
std::uint64_t KvPool::token_bytes() const { return st_->token_bytes; }
std::uint64_t KvPool::tokens_per_page() const { return st_->tpp; }
std::uint64_t KvPool::virtual_capacity_pages() const { return st_->vpages; }
std::uint64_t KvPool::mapped_pages() const { return st_->mapped; }
std::uint64_t KvPool::occupied_slots() const { return st_->occupied; }
bool KvPool::alive() const { return st_->alive; }
void KvPool::set_mapped_page_cap(std::optional<std::uint64_t> cap) { st_->cap = cap; }
std::optional<std::uint64_t> KvPool::mapped_page_cap() const { return st_->cap; }
std::uint64_t KvPool::device_base() const { return st_->va; }

bool KvPool::page_mapped(std::uint32_t page) const {
    return page < st_->occ.size() && st_->occ[page] > 0;
}

std::uint64_t KvPool::page_occupied(std::uint32_t page) const {
    return page < st_->occ.size() ? st_->occ[page] : 0;
}

namespace {

// New pages the pool may still map: ledger headroom (free + buffer), the
// virtual range, and the optional static cap (reference :147-156, :201-208).
std::uint64_t new_page_budget(const detail::PoolState& s, const PhysicalLedger& ledger) {
    std::uint64_t budget = std::min(ledger.free_pages() + ledger.buffer_pages(), s.vpages - s.mapped);
    if (s.cap) budget = std::min(budget, *s.cap > s.mapped ? *s.cap - s.mapped : 0);
    return budget;
}

}  // namespace

std::uint64_t KvPool::allocatable_tokens(const PhysicalLedger& ledger) const {
    if (!st_->alive) return 0;
    return free_slots_in_mapped() + new_page_budget(*st_, ledger) * st_->tpp;
}

// ------------------------------------------------------------------ allocator core

struct detail::Access {
    static PoolId open_pool(PhysicalLedger& l, const std::string& model) {  // :66-76
        for (const auto& kv : l.pools_) {
            if (kv.second.model == model) throw UsageError("ledger: duplicate KV pool for model " + model);
        }
        const PoolId id = l.next_id_++;
        l.pools_[id] = PhysicalLedger::PoolEntry{model, 0};
        return id;
    }

    static void close_pool(PhysicalLedger& l, PoolId id, std::uint64_t mapped) {  // :78-83
        const auto it = l.pools_.find(id);
        if (it == l.pools_.end()) throw UsageError("ledger: unknown pool");
        l.kv_pages_ -= mapped;
        if (mapped > 0) l.note(it->second.model, AllocEventKind::unmap, mapped);
        l.pools_.erase(it);
    }

    static void pool_delta(PhysicalLedger& l, PoolId id, std::int64_t delta) {  // :85-90
        const auto it = l.pools_.find(id);
        if (it == l.pools_.end()) throw UsageError("ledger: unknown pool");
        it->second.pages = static_cast<std::uint64_t>(static_cast<std::int64_t>(it->second.pages) + delta);
        l.kv_pages_ = static_cast<std::uint64_t>(static_cast<std::int64_t>(l.kv_pages_) + delta);
    }

    static std::uint64_t take_buffer(PhysicalLedger& l, std::uint64_t pages) {  // :36-40
        const std::uint64_t n = std::min(pages, l.buffer_);
        l.buffer_ -= n;
        if (l.dev_ && n) l.dev_->take_buffer(n);
        return n;
    }

    static void note(PhysicalLedger& l, const std::string& m, AllocEventKind k, std::uint64_t p) { l.note(m, k, p); }

    static detail::PoolState& st(KvPool& p) { return *p.st_; }
    static KvPool make() { return KvPool(); }
};

namespace {

using detail::Access;
using detail::kNone;
using detail::PoolState;

// Look-ahead window handed to VmmDevice::premap when a pool grows: 256 pages
// (32 physical chunks of 8, 512 MiB) past the pool's mapped pages. That is
// ~64 decode steps of runway for a C1 pool (4 new pages per step), so the
// worker rides out the periods in which VMM calls stall: a 128-page window
// ran dry in one bench run whose cuMemSetAccess calls averaged ~6 ms (p99
// 70 ms) and the engine thread waited ~100 ms inside the timed region.
// Look-ahead only ever uses free budget (and at most kMaxCleanPages mapped
// ahead on a device).
// With more pools on the device the deeper window holds budget that other
// models then steal back (scheduler-driven C2 / C5 runs: 2-10x the
// engine-thread cost per page op at 256 pages vs 128), so the window is 256
// pages with at most two pools and 128 beyond; PRISM_PREMAP_PAGES fixes it.
std::uint64_t premap_pages(std::uint64_t pools) {
    static const std::uint64_t fixed = [] {
        const char* e = std::getenv("PRISM_PREMAP_PAGES");
        return e ? static_cast<std::uint64_t>(std::max(1, std::atoi(e))) : std::uint64_t{0};
    }();
    if (fixed) return fixed;
    return pools <= 2 ? 256 : 128;
}

// PRISM_PREMAP=0 turns the look-ahead off (A/B measurements).
bool premap_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PRISM_PREMAP");
        return !(e && e[0] == '0');
    }();
    return on;
}

inline bool is_candidate(const PoolState& s, std::uint32_t page) {
    return s.occ[page] > 0 && s.occ[page] < s.tpp;
}

// Refresh the search structures for one page after its occupancy changed.
void touch(PoolState& s, std::uint32_t page) {
    const bool cand = is_candidate(s, page);
    if (s.placement == PagePlacement::most_occupied_first) {
        s.partial.update(page, cand, s.occ.data());
    } else if (cand) {
        s.nonfull.set(page);
    } else {
        s.nonfull.clear(page);
    }
}

// reference pick_page (:158-186): best partially-filled mapped page, else the
// lowest-index unmapped page (needs_map).
std::uint32_t pick(const PoolState& s, bool& needs_map) {
    needs_map = false;
    const std::uint32_t p = s.placement == PagePlacement::most_occupied_first ? s.partial.best()
                                                                               : s.nonfull.find_first();
    if (p != kNone) return p;
    needs_map = true;
    return s.unmapped.find_first();
}

void check_usable(const PoolState& s, const PhysicalLedger& ledger, const char* what) {
    if (!s.alive) throw UsageError(std::string(what) + ": pool was freed");
    if (s.gpu != ledger.gpu_id()) throw UsageError(std::string(what) + ": pool belongs to another GPU");
}

void unmap_page(PoolState& s, PhysicalLedger& ledger, std::uint32_t page) {
    --s.mapped;
    s.unmapped.set(page);
    Access::pool_delta(ledger, s.id, -1);
    Access::note(ledger, s.model, AllocEventKind::unmap, 1);
    if (s.dev) s.dev->unmap(s.va + static_cast<std::uint64_t>(page) * s.dev->page_bytes());
}

// Clears one slot; throws UsageError for invalid handles exactly where the
// reference does (:244-253). Returns true when the page emptied.
bool release_slot(PoolState& s, PhysicalLedger& ledger, const TokenSlotHandle& h) {
    if (h.pool != s.id) throw UsageError("free_kv: handle belongs to another pool");
    if (h.page >= s.vpages) throw UsageError("free_kv: page index out of range");
    if (h.slot >= s.tpp || s.occ[h.page] == 0) throw UsageError("free_kv: stale handle");
    std::uint64_t& word = s.page_bits(h.page)[h.slot >> 6];
    const std::uint64_t bit = 1ull << (h.slot & 63);
    if (!(word & bit)) throw UsageError("free_kv: stale handle");
    word &= ~bit;
    --s.occupied;
    if (--s.occ[h.page] == 0) {
        unmap_page(s, ledger, h.page);
        return true;
    }
    return false;
}

void free_handles(PoolState& s, PhysicalLedger& ledger, const std::vector<TokenSlotHandle>& handles,
                  std::size_t& applied) {
    // Structure updates are batched per distinct page; the guard makes sure
    // they also happen for the prefix that was applied before a throw.
    std::vector<std::uint32_t> dirty;
    dirty.reserve(16);
    struct Flush {
        PoolState& s;
        std::vector<std::uint32_t>& d;
        ~Flush() {
            std::sort(d.begin(), d.end());
            d.erase(std::unique(d.begin(), d.end()), d.end());
            for (const std::uint32_t p : d) touch(s, p);
        }
    } flush{s, dirty};
    std::uint32_t last = kNone;
    for (const TokenSlotHandle& h : handles) {
        release_slot(s, ledger, h);
        ++applied;
        if (h.page != last) {
            dirty.push_back(h.page);
            last = h.page;
        }
    }
}

}  // namespace

KvPool alloc_kvcache(PhysicalLedger& ledger, const std::string& model_id, std::uint64_t token_bytes,
                     std::uint64_t virtual_capacity_pages, PagePlacement placement) {  // :108-128
    if (token_bytes == 0 || token_bytes > ledger.page_bytes()) {
        throw UsageError("alloc_kvcache: token size must be in (0, page_bytes]");
    }
    if (virtual_capacity_pages < 1) throw UsageError("alloc_kvcache: virtual capacity must be >= 1 page");
    if (virtual_capacity_pages >= kNone) throw UsageError("alloc_kvcache: virtual capacity too large");
    KvPool pool = Access::make();
    PoolState& s = Access::st(pool);
    s.id = Access::open_pool(ledger, model_id);
    s.gpu = ledger.gpu_id();
    s.model = model_id;
    s.token_bytes = token_bytes;
    s.tpp = ledger.page_bytes() / token_bytes;
    s.vpages = virtual_capacity_pages;
    s.placement = placement;
    s.words = static_cast<std::uint32_t>((s.tpp + 63) / 64);
    s.occ.assign(s.vpages, 0);
    s.bits.reset(static_cast<std::uint64_t*>(std::calloc(s.vpages * s.words, sizeof(std::uint64_t))));
    if (!s.bits) throw UsageError("alloc_kvcache: out of host memory for slot bitmaps");
    s.unmapped.reset_size(s.vpages, true);
    if (placement == PagePlacement::most_occupied_first) {
        s.partial.init(s.vpages);
    } else {
        s.nonfull.reset_size(s.vpages, false);
    }
    if (ledger.device()) {
        s.dev = ledger.device();
        s.dev_hold = s.dev->shared_from_this();  // the device outlives its pools
        s.va = s.dev->reserve(s.vpages);
    }
    s.alive = true;
    return pool;
}

void free_kvcache(PhysicalLedger& ledger, KvPool& pool) {  // :130-137
    PoolState& s = Access::st(pool);
    if (!s.alive) throw UsageError("free_kvcache: pool already freed");
    Access::close_pool(ledger, s.id, s.mapped);
    if (s.dev) {
        // The whole range goes back: its live and parked pages are unmapped
        // (after the stream drains) and their handles recycled.
        s.dev->release(s.va, s.vpages);
        s.va = 0;
        s.dev = nullptr;
        s.dev_hold.reset();
    }
    s.alive = false;
    s.mapped = 0;
    s.occupied = 0;
    s.occ.clear();
    s.occ.shrink_to_fit();
    s.bits.reset();
    s.partial = detail::Tournament();
    s.nonfull = detail::LevelBitset();
    s.unmapped = detail::LevelBitset();
    s.mirror.reset();
    s.ops.clear();
    s.freed_slots.clear();
}

AllocResult detail::alloc_kv_into(KvPool& pool, PhysicalLedger& ledger, std::uint64_t num_tokens,
                                  std::int64_t dest) {  // reference :188-244
    PoolState& s = Access::st(pool);
    check_usable(s, ledger, "alloc_kv");
    AllocResult res;
    if (num_tokens == 0) return res;

    const std::uint64_t partial_free = s.mapped * s.tpp - s.occupied;
    const std::uint64_t new_pages =
        num_tokens > partial_free ? (num_tokens - partial_free + s.tpp - 1) / s.tpp : 0;
    const std::uint64_t budget = new_page_budget(s, ledger);
    if (new_pages > budget) {  // all-or-nothing (:201-213)
        res.shortfall_pages = new_pages - budget;
        Access::note(ledger, s.model, AllocEventKind::alloc_fail, res.shortfall_pages);
        return res;
    }
    std::uint32_t next_unmapped = kNone;
    if (s.dev && new_pages > 0) {
        // Every partial slot is consumed before any new page, and each new
        // page is the lowest unmapped one at that moment, so the pages this
        // call maps are the new_pages lowest unmapped indices: map them in one
        // batch, BEFORE any ledger / buffer state is committed, so a device
        // failure (map_batch throws) leaves the ledger, the pool and the VMM
        // references exactly as they were.
        std::vector<std::uint64_t> vas;
        vas.reserve(new_pages);
        std::uint32_t p = s.unmapped.find_first();
        for (std::uint64_t k = 0; k < new_pages && p != kNone; ++k) {
            vas.push_back(s.va + static_cast<std::uint64_t>(p) * s.dev->page_bytes());
            p = s.unmapped.find_next(static_cast<std::uint64_t>(p) + 1);
        }
        next_unmapped = p;
        try {
            s.dev->map_batch(vas.data(), vas.size(), std::min<std::uint64_t>(new_pages, ledger.buffer_pages()));
        } catch (...) {
            // map_batch took a reference on every page before waiting
            for (const std::uint64_t va : vas) {
                try {
                    s.dev->unmap(va);
                } catch (...) {
                }
            }
            throw;
        }
    }
    res.buffer_hits = Access::take_buffer(ledger, new_pages);
    res.pages_mapped = new_pages - res.buffer_hits;
    if (res.buffer_hits) Access::note(ledger, s.model, AllocEventKind::buffer_hit, res.buffer_hits);
    if (res.pages_mapped) Access::note(ledger, s.model, AllocEventKind::map, res.pages_mapped);
    Access::pool_delta(ledger, s.id, static_cast<std::int64_t>(new_pages));

    res.handles.resize(num_tokens);
    TokenSlotHandle* out = res.handles.data();
    std::uint64_t remaining = num_tokens;
    const std::uint64_t last_word_bits = s.tpp - static_cast<std::uint64_t>(s.words - 1) * 64;
    if (s.dev && new_pages > 0) {
        std::vector<std::uint64_t> vas;
        std::uint32_t p = next_unmapped;
        // The pool is growing: its next maps will be the following lowest
        // unmapped pages. Hand them to the device's worker thread to map
        // (and make accessible) ahead of time, so those maps become revives.
        const std::uint64_t ahead = !premap_enabled() ? 0 : premap_pages(s.dev->pool_count());
        vas.clear();
        for (std::uint64_t k = 0; k < ahead && p != kNone; ++k) {
            vas.push_back(s.va + static_cast<std::uint64_t>(p) * s.dev->page_bytes());
            p = s.unmapped.find_next(static_cast<std::uint64_t>(p) + 1);
        }
        s.dev->premap(s.va, vas.data(), vas.size());
    }
    while (remaining > 0) {
        bool needs_map = false;
        const std::uint32_t page = pick(s, needs_map);
        if (page == kNone) throw UsageError("alloc_kv: internal page accounting error");
        if (needs_map) {
            ++s.mapped;
            s.unmapped.clear(page);
            s.hw = std::max<std::uint64_t>(s.hw, static_cast<std::uint64_t>(page) + 1);
        }
        // First free slots in ascending order (:225-241).
        std::uint64_t* words = s.page_bits(page);
        std::uint32_t taken = 0;
        for (std::uint32_t w = 0; w < s.words && remaining > 0; ++w) {
            const std::uint64_t valid = (w + 1 == s.words && last_word_bits < 64) ? (1ull << last_word_bits) - 1 : ~0ull;
            std::uint64_t freebits = ~words[w] & valid;
            while (freebits && remaining > 0) {
                const std::uint32_t b = static_cast<std::uint32_t>(__builtin_ctzll(freebits));
                freebits &= freebits - 1;
                words[w] |= 1ull << b;
                *out++ = TokenSlotHandle{s.id, page, w * 64 + b};
                ++taken;
                --remaining;
            }
        }
        s.occ[page] += taken;
        s.occupied += taken;
        touch(s, page);
    }
    if (s.mirror) s.ops.push_back(detail::DeviceOp{detail::DeviceOp::kAlloc, static_cast<std::uint32_t>(num_tokens), dest, 0});
    return res;
}

AllocResult alloc_kv(KvPool& pool, PhysicalLedger& ledger, std::uint64_t num_tokens) {
    return detail::alloc_kv_into(pool, ledger, num_tokens, -1);
}

void free_kv(KvPool& pool, PhysicalLedger& ledger, const std::vector<TokenSlotHandle>& handles) {  // :246-267
    PoolState& s = Access::st(pool);
    check_usable(s, ledger, "free_kv");
    const std::size_t before = s.freed_slots.size();
    if (s.mirror) {
        for (const TokenSlotHandle& h : handles) {
            s.freed_slots.push_back(static_cast<std::int32_t>(h.page * s.tpp + h.slot));
        }
    }
    std::size_t applied = 0;
    struct Record {
        PoolState& s;
        std::size_t before;
        std::size_t& applied;
        ~Record() {
            // Only the prefix that was applied (all of it unless a handle was
            // rejected) is replayed on the device mirror.
            if (!s.mirror) return;
            s.freed_slots.resize(before + applied);
            if (applied) {
                s.ops.push_back(detail::DeviceOp{detail::DeviceOp::kFreeList, static_cast<std::uint32_t>(applied), -1,
                                                 static_cast<std::int64_t>(before)});
            }
        }
    } record{s, before, applied};
    free_handles(s, ledger, handles, applied);
}

void detail::free_kv_row(KvPool& pool, PhysicalLedger& ledger, const std::vector<TokenSlotHandle>& handles,
                         std::int64_t row_first) {
    PoolState& s = Access::st(pool);
    check_usable(s, ledger, "free_kv");
    if (!s.mirror || row_first < 0) {
        free_kv(pool, ledger, handles);
        return;
    }
    std::size_t applied = 0;
    free_handles(s, ledger, handles, applied);  // engine-owned handles: never invalid
    if (!handles.empty()) {
        s.ops.push_back(detail::DeviceOp{detail::DeviceOp::kFreeRow, static_cast<std::uint32_t>(handles.size()), -1,
                                         row_first});
    }
}

std::uint64_t refill_buffer(PhysicalLedger& ledger, std::uint64_t target_pages) {
    return ledger.refill_buffer(target_pages);
}

}  // namespace msim::pagealloc
