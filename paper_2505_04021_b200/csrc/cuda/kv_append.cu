// K2 — KV append / scatter: writes this step's new K/V rows into the slots
// K1 chose, for a range of layers. One thread moves one 16-byte chunk, so a
// (token, layer, K|V, head) row of head_dim bf16 (128 or 256 B) is written by
// 8 or 16 consecutive threads: coalesced source reads, full-sector stores.
// Also: the synthetic-content variants used by tests and the benchmark.
#include "cuda/device_impl.cuh"

namespace prism {

namespace {

struct AppendArgs {
    KvGeom g;
    const std::int32_t* slots;  // [n_tok]
    const TokenMeta* meta;      // [n_tok] (request == ~0: dead, skip)
    const uint4* k;             // [n_layer][n_tok][n_kv][D] (null: synthetic)
    const uint4* v;
    int layer_begin, n_layer, n_tok;
    std::uint64_t seed;
};

__device__ __forceinline__ std::uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const std::uint32_t*>(&p);
}

template <bool kSynthetic>
__global__ void __launch_bounds__(256) k2_append(AppendArgs a) {
    const int chunks_per_row = a.g.head_dim / 8;
    const std::uint64_t per_layer_kind = static_cast<std::uint64_t>(a.n_tok) * a.g.n_kv * chunks_per_row;
    const std::uint64_t total = per_layer_kind * 2 * a.n_layer;
    for (std::uint64_t c = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; c < total;
         c += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        // c = (((layer * 2 + kind) * n_tok + t) * n_kv + head) * cpr + chunk
        std::uint64_t r = c;
        const int chunk = static_cast<int>(r % chunks_per_row);
        r /= chunks_per_row;
        const int head = static_cast<int>(r % a.g.n_kv);
        r /= a.g.n_kv;
        const int t = static_cast<int>(r % a.n_tok);
        r /= a.n_tok;
        const int kind = static_cast<int>(r & 1);
        const int layer = static_cast<int>(r >> 1);
        const TokenMeta m = a.meta[t];
        if (m.request == ~0ull) continue;
        const std::uint32_t sid = static_cast<std::uint32_t>(a.slots[t]);
        uint4 val;
        if constexpr (kSynthetic) {
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                f[e] = synth_value(a.seed, m.request, m.pos, a.layer_begin + layer, kind, head, chunk * 8 + e);
            }
            val.x = pack_bf16x2(f[0], f[1]);
            val.y = pack_bf16x2(f[2], f[3]);
            val.z = pack_bf16x2(f[4], f[5]);
            val.w = pack_bf16x2(f[6], f[7]);
        } else {
            const std::uint64_t src = ((static_cast<std::uint64_t>(layer) * a.n_tok + t) * a.g.n_kv + head) *
                                          chunks_per_row + chunk;
            val = __ldg((kind ? a.v : a.k) + src);
        }
        char* dst = reinterpret_cast<char*>(a.g.base) + row_offset(a.g, sid, a.layer_begin + layer, kind, head) +
                    static_cast<std::uint64_t>(chunk) * 16;
        *reinterpret_cast<uint4*>(dst) = val;
    }
}

__global__ void __launch_bounds__(256) k_synth_q(const DecodeDesc* desc, int n_dec, int n_q, int head_dim, int layer,
                                                 std::uint64_t seed, float q_scale, __nv_bfloat16* q) {
    const std::uint64_t total = static_cast<std::uint64_t>(n_dec) * n_q * head_dim;
    for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
        const int d = static_cast<int>(i % head_dim);
        const int h = static_cast<int>((i / head_dim) % n_q);
        const int b = static_cast<int>(i / (static_cast<std::uint64_t>(head_dim) * n_q));
        const DecodeDesc dd = desc[b];
        const float x = synth_value(seed, dd.request, static_cast<std::uint32_t>(dd.ctx - 1), layer, 2, h, d);
        q[i] = __float2bfloat16_rn(x * q_scale);
    }
}

int grid_for(std::uint64_t work, int threads) {
    const std::uint64_t blocks = (work + threads - 1) / threads;
    return static_cast<int>(std::min<std::uint64_t>(blocks, 148ull * 16));
}

void launch_append(EngineDeviceImpl& d, int layer_begin, int layer_end, const void* k, const void* v, bool synth,
                   std::uint64_t seed) {
    if (layer_begin < 0 || layer_end > d.n_layers || layer_begin >= layer_end) {
        throw std::runtime_error("append_step_kv: bad layer range");
    }
    if (d.step_tokens == 0) return;
    d.k3_chain = d.k4_chain = false;
    AppendArgs a{d.geom,  d.step_slots, d.token_meta.dev, static_cast<const uint4*>(k), static_cast<const uint4*>(v),
                 layer_begin, layer_end - layer_begin, d.step_tokens, seed};
    const std::uint64_t work =
        static_cast<std::uint64_t>(d.step_tokens) * d.n_kv * (d.head_dim / 8) * 2 * (layer_end - layer_begin);
    if (synth) {
        k2_append<true><<<grid_for(work, 256), 256, 0, d.stream>>>(a);
    } else {
        if ((reinterpret_cast<std::uintptr_t>(k) | reinterpret_cast<std::uintptr_t>(v)) & 15) {
            throw std::runtime_error("append_step_kv: k/v must be 16-byte aligned");
        }
        k2_append<false><<<grid_for(work, 256), 256, 0, d.stream>>>(a);
    }
    PRISM_CUDA(cudaGetLastError());
}

}  // namespace

void append_step_kv(msim::engine::Engine& eng, int layer_begin, int layer_end, const void* k, const void* v) {
    launch_append(impl_of(eng), layer_begin, layer_end, k, v, false, 0);
}

void append_step_kv_synthetic(msim::engine::Engine& eng, int layer_begin, int layer_end, std::uint64_t seed) {
    launch_append(impl_of(eng), layer_begin, layer_end, nullptr, nullptr, true, seed);
}

void synth_decode_q(msim::engine::Engine& eng, int layer, std::uint64_t seed, float q_scale, void* q) {
    EngineDeviceImpl& d = impl_of(eng);
    if (d.step_decodes == 0) return;
    d.k3_chain = d.k4_chain = false;
    const std::uint64_t work = static_cast<std::uint64_t>(d.step_decodes) * d.n_q * d.head_dim;
    k_synth_q<<<grid_for(work, 256), 256, 0, d.stream>>>(d.decode_desc.dev, d.step_decodes, d.n_q, d.head_dim, layer,
                                                          seed, q_scale, static_cast<__nv_bfloat16*>(q));
    PRISM_CUDA(cudaGetLastError());
}

void PagedCtx::kv_append(int layer_begin, int layer_end, const std::int32_t* slots, int n_tok, const void* k,
                         const void* v) {
    if (layer_begin < 0 || layer_end > n_layers || layer_begin >= layer_end) {
        throw std::out_of_range("paged kv_append: bad layer range");
    }
    if (n_tok <= 0) return;
    if (!slots || !k || !v) throw std::invalid_argument("paged kv_append: null pointer");
    if ((reinterpret_cast<std::uintptr_t>(k) | reinterpret_cast<std::uintptr_t>(v)) & 15) {
        throw std::invalid_argument("paged kv_append: k/v must be 16-byte aligned");
    }
    PRISM_CUDA(cudaSetDevice(vmm->ordinal()));
    if (token_meta.cap < static_cast<std::size_t>(n_tok)) {
        token_meta.ensure(static_cast<std::size_t>(n_tok));
        for (std::size_t i = 0; i < token_meta.cap; ++i) token_meta.host[i] = TokenMeta{0, 0, 0};  // all live
        token_meta.upload(token_meta.cap, stream);
    }
    k3_chain = k4_chain = false;
    AppendArgs a{geom, slots, token_meta.dev, static_cast<const uint4*>(k), static_cast<const uint4*>(v),
                 layer_begin, layer_end - layer_begin, n_tok, 0};
    const std::uint64_t work = static_cast<std::uint64_t>(n_tok) * n_kv * (head_dim / 8) * 2 * (layer_end - layer_begin);
    k2_append<false><<<grid_for(work, 256), 256, 0, stream>>>(a);
    PRISM_CUDA(cudaGetLastError());
}

}  // namespace prism
