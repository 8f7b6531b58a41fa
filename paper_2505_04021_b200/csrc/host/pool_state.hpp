// Private per-pool allocator state (prism-b200 host runtime).
//
// The reference keeps a vector<Page{mapped, occupied, vector<bool> slots}> and
// finds the next page with an O(V) scan (reference src/pagealloc.cpp:158-186).
// Here the same decision is answered in O(log V):
//   * Tournament  — segment tree whose root is the mapped, non-full page with
//                   the highest occupancy, ties to the lowest index (the exact
//                   order of the reference's strict '>' scan, :166).
//   * LevelBitset — 64-ary hierarchical bitset; find_first() gives the lowest
//                   set index in O(log64 V). Used for "lowest unmapped page"
//                   (:181-184) and for lowest_index_first's "lowest mapped
//                   non-full page" (:171-179).
// Invariant used throughout: a page is mapped <=> its occupancy is > 0 (the
// reference maps a page only to put a token in it and unmaps it when its last
// token leaves), so no separate mapped flag is stored.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "msim/pagealloc.hpp"

namespace prism {
class DevicePool;  // GPU-resident slot mirror (csrc/cuda/device_pool.cu)
void destroy_device_pool(DevicePool* p);
}  // namespace prism

namespace msim::pagealloc::detail {

constexpr std::uint32_t kNone = 0xFFFFFFFFu;

class LevelBitset {
public:
    LevelBitset() = default;
    explicit LevelBitset(std::uint64_t n, bool all_set) { reset_size(n, all_set); }

    void reset_size(std::uint64_t n, bool all_set) {
        n_ = n;
        levels_.clear();
        std::uint64_t count = n;
        do {
            const std::uint64_t words = (count + 63) / 64;
            levels_.emplace_back(words, 0ull);
            count = words;
        } while (count > 1);
        if (all_set) {
            // Fill bottom-up: a word at level k+1 has bit j set iff word j of level k is non-zero.
            std::uint64_t bits = n;
            for (auto& lvl : levels_) {
                for (std::uint64_t w = 0; w < lvl.size(); ++w) {
                    const std::uint64_t lo = w * 64;
                    const std::uint64_t take = bits - lo >= 64 ? 64 : bits - lo;
                    lvl[w] = take == 64 ? ~0ull : ((1ull << take) - 1);
                }
                bits = lvl.size();
            }
        }
    }

    bool test(std::uint64_t i) const { return (levels_[0][i >> 6] >> (i & 63)) & 1ull; }

    void set(std::uint64_t i) {
        for (auto& lvl : levels_) {
            std::uint64_t& w = lvl[i >> 6];
            const bool was_empty = w == 0;
            w |= 1ull << (i & 63);
            if (!was_empty) return;
            i >>= 6;
        }
    }

    void clear(std::uint64_t i) {
        for (auto& lvl : levels_) {
            std::uint64_t& w = lvl[i >> 6];
            w &= ~(1ull << (i & 63));
            if (w != 0) return;
            i >>= 6;
        }
    }

    // Lowest set index >= i, or kNone.
    std::uint32_t find_next(std::uint64_t i) const { return next_at(0, i); }

    // Lowest set index, or kNone.
    std::uint32_t find_first() const {
        if (levels_.empty() || levels_.back()[0] == 0) return kNone;
        std::uint64_t idx = 0;
        for (std::size_t k = levels_.size(); k-- > 0;) {
            const std::uint64_t w = levels_[k][idx];
            idx = idx * 64 + static_cast<std::uint64_t>(__builtin_ctzll(w));
        }
        return static_cast<std::uint32_t>(idx);
    }

private:
    // Lowest set bit index >= i in level k's bit space, or kNone. Bit j of
    // level k+1 is set iff word j of level k is non-zero, so an empty tail of
    // the current word continues at the next non-zero word found one level up.
    std::uint32_t next_at(std::size_t k, std::uint64_t i) const {
        const auto& lvl = levels_[k];
        if ((i >> 6) >= lvl.size()) return kNone;
        const std::uint64_t w = lvl[i >> 6] & (~0ull << (i & 63));
        if (w) return static_cast<std::uint32_t>((i >> 6) * 64 + static_cast<std::uint64_t>(__builtin_ctzll(w)));
        if (k + 1 == levels_.size()) return kNone;
        const std::uint32_t nw = next_at(k + 1, (i >> 6) + 1);
        if (nw == kNone) return kNone;
        return static_cast<std::uint32_t>(static_cast<std::uint64_t>(nw) * 64 +
                                          static_cast<std::uint64_t>(__builtin_ctzll(lvl[nw])));
    }

    std::uint64_t n_ = 0;
    std::vector<std::vector<std::uint64_t>> levels_;
};

// Argmax over leaves with key (occupancy desc, index asc); a leaf holds its
// page index when the page is mapped and not full, kNone otherwise.
class Tournament {
public:
    void init(std::uint64_t n) {
        leaves_ = 1;
        while (leaves_ < n) leaves_ <<= 1;
        win_.assign(2 * leaves_, kNone);
    }
    std::uint32_t best() const { return win_.empty() ? kNone : win_[1]; }

    // Re-evaluate leaf `page` after its occupancy / status changed.
    void update(std::uint32_t page, bool candidate, const std::uint32_t* occ) {
        std::uint64_t node = leaves_ + page;
        win_[node] = candidate ? page : kNone;
        for (node >>= 1; node >= 1; node >>= 1) {
            const std::uint32_t a = win_[2 * node];
            const std::uint32_t b = win_[2 * node + 1];
            std::uint32_t w;
            if (a == kNone) w = b;
            else if (b == kNone) w = a;
            else w = occ[b] > occ[a] ? b : a;  // left subtree holds the lower index
            // No early exit: an ancestor's winner can keep its index while its
            // occupancy (the key) changed, so always climb the log2(V) levels.
            win_[node] = w;
        }
    }

private:
    std::uint64_t leaves_ = 1;
    std::vector<std::uint32_t> win_;
};

// One allocator operation recorded for replay on the GPU-resident mirror by
// the batched device allocator (K1). `dest` is the element index in the
// engine's device block table where the op's slot ids go (-1: none), `row`
// is the block-table element range a FREE_ROW op releases.
struct DeviceOp {
    enum Kind : std::uint32_t { kAlloc = 1, kFreeList = 2, kFreeRow = 3 };
    Kind kind;
    std::uint32_t count;   // tokens allocated / handles freed
    std::int64_t dest;     // kAlloc: table element index of the first slot (or -1)
    std::int64_t first;    // kFreeList: index into freed_slots; kFreeRow: table element index
};

struct PoolState {
    PoolId id = 0;
    int gpu = 0;
    std::string model;
    std::uint64_t token_bytes = 0;
    std::uint64_t tpp = 0;       // tokens per page
    std::uint64_t vpages = 0;    // virtual capacity in pages
    std::uint64_t mapped = 0;
    std::uint64_t occupied = 0;
    std::uint64_t hw = 0;        // 1 + highest page index ever mapped (K1 scans [0, hw) only)
    std::uint32_t words = 0;     // 64-bit bitmap words per page
    PagePlacement placement = PagePlacement::most_occupied_first;
    std::optional<std::uint64_t> cap;
    bool alive = false;

    std::vector<std::uint32_t> occ;                         // per page
    std::unique_ptr<std::uint64_t[], void (*)(void*)> bits{nullptr, &std::free};  // vpages * words
    Tournament partial;      // most_occupied_first
    LevelBitset nonfull;     // lowest_index_first: mapped && occ < tpp
    LevelBitset unmapped;    // occ == 0

    // device side (only when the ledger has a VmmDevice)
    prism::VmmDevice* dev = nullptr;
    std::shared_ptr<prism::VmmDevice> dev_hold;
    std::uint64_t va = 0;    // base VA of page 0
    std::unique_ptr<prism::DevicePool, void (*)(prism::DevicePool*)> mirror{nullptr, &prism::destroy_device_pool};
    std::vector<DeviceOp> ops;           // pending replay for the mirror
    std::vector<std::int32_t> freed_slots;  // kFreeList payload (page * tpp + slot)

    std::uint64_t* page_bits(std::uint32_t page) { return bits.get() + static_cast<std::uint64_t>(page) * words; }
    const std::uint64_t* page_bits(std::uint32_t page) const {
        return bits.get() + static_cast<std::uint64_t>(page) * words;
    }
};

// Internal entry points used by the engine (csrc/host/engine.cpp) so the
// device op log knows where slot ids land in the device block table.
AllocResult alloc_kv_into(KvPool& pool, PhysicalLedger& ledger, std::uint64_t num_tokens, std::int64_t dest);
void free_kv_row(KvPool& pool, PhysicalLedger& ledger, const std::vector<TokenSlotHandle>& handles,
                 std::int64_t row_first);

}  // namespace msim::pagealloc::detail
