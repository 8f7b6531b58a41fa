// Shared CUDA helpers for the prism-b200 kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace prism {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    }
}
#define PRISM_CUDA(call) ::prism::cuda_check((call), #call)

// ---------------------------------------------------------------------------
// Paged KV layout inside one 2 MiB physical page (all layers of tpp tokens):
//   [layer][K=0 | V=1][kv_head][slot][head_dim]  bf16
// so one (layer, K|V, head) block holds tpp contiguous rows of head_dim, and a
// run of consecutive slots filled by one prefill chunk stays contiguous.
// Slot ids in block tables are page * tpp + slot.
struct KvGeom {
    std::uint64_t base;        // device VA of page 0
    std::uint64_t page_bytes;  // 2 MiB
    std::uint32_t tpp;         // tokens per page
    std::uint64_t magic;       // page = (sid * magic) >> 40 (see div_magic40)
    std::int32_t n_layers;
    std::int32_t n_kv;
    std::int32_t head_dim;
};

// floor(sid / tpp) as one 64-bit multiply + shift: magic = floor(2^40/tpp)+1
// is exact for sid * tpp < 2^40; slot ids are < 2^24 and tpp <= 1024 (the
// device path's limits), and sid * magic < 2^24 * 2^40 fits in 64 bits.
__host__ __device__ inline std::uint64_t div_magic40(std::uint32_t tpp) {
    return (std::uint64_t{1} << 40) / tpp + 1;
}

__device__ __forceinline__ std::uint32_t slot_page(std::uint32_t sid, std::uint64_t magic) {
    return static_cast<std::uint32_t>((static_cast<std::uint64_t>(sid) * magic) >> 40);
}

// Byte offset of row (sid, layer, kv, head) from the pool base.
__device__ __forceinline__ std::uint64_t row_offset(const KvGeom& g, std::uint32_t sid, int layer, int kv, int head) {
    const std::uint32_t page = slot_page(sid, g.magic);
    const std::uint32_t slot = sid - page * g.tpp;
    const std::uint64_t block = (static_cast<std::uint64_t>(layer) * 2 + kv) * g.n_kv + head;
    return static_cast<std::uint64_t>(page) * g.page_bytes +
           ((block * g.tpp + slot) * static_cast<std::uint64_t>(g.head_dim)) * 2;
}

// ---------------------------------------------------------------------------
// Deterministic synthetic K/V/Q content: bf16(2u - 1), u in [0,1)
// from a splitmix-style hash of (seed, model, request, position, layer, kind,
// head, dim). Depends only on logical coordinates, never on slots, so the CPU
// oracle (oracle/restate/prism_oracle.c, prism_synth_value) is layout-free.
// kind: 0 = K, 1 = V, 2 = Q.
__host__ __device__ inline std::uint64_t synth_mix(std::uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

__host__ __device__ inline float synth_value(std::uint64_t seed, std::uint64_t req, std::uint32_t pos, int layer,
                                             int kind, int head, int dim) {
    const std::uint64_t a = req * 0x9E3779B97F4A7C15ull ^ pos;
    const std::uint64_t b = (static_cast<std::uint64_t>(layer) << 40) | (static_cast<std::uint64_t>(kind) << 36) |
                            (static_cast<std::uint64_t>(head) << 20) | static_cast<std::uint64_t>(dim);
    const std::uint64_t u = synth_mix(seed ^ synth_mix(a) ^ (b * 0xD6E8FEB86659FD93ull));
    // 24 random bits -> [0,1) exactly representable; 2u-1 in [-1,1) with 24 bits,
    // then rounded to bf16 by the caller.
    return static_cast<float>(u >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
}

}  // namespace prism
