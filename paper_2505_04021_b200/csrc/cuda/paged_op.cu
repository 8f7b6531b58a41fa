// Pool-level K3 over caller-owned block tables (PagedCtx, device_impl.cuh):
// the decode-attention entry point SURVEY §8b suggests for engines that keep
// their own scheduler — decode_attn(pool, q, seq_slot_offsets[], slot_ids[],
// out) — on the same stream-K kernel the engine path launches. K2's
// pool-level append is in kv_append.cu (it shares that file's kernel).
#include <stdexcept>

#include "cuda/attn_common.cuh"
#include "cuda/device_impl.cuh"

namespace prism {

void launch_k3_streamk(PagedCtx& d, AttnArgs a, int n_dec);

PagedCtx::PagedCtx(const msim::pagealloc::KvPool& pool, int layers, int q_heads, int kv_heads, int d) {
    const msim::pagealloc::detail::PoolState* st = pool.state();
    if (!st || !st->alive) throw std::invalid_argument("paged op: pool is freed");
    if (!st->dev) throw std::invalid_argument("paged op: the pool's ledger has no VmmDevice attached");
    if (layers <= 0 || q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads) {
        throw std::invalid_argument("paged op: bad attention shape");
    }
    if (d != 64 && d != 128) throw std::invalid_argument("paged op: head_dim must be 64 or 128");
    if (q_heads / kv_heads > 8) throw std::invalid_argument("paged op: GQA group above 8 not supported");
    if (2ull * layers * kv_heads * d * 2 != st->token_bytes) {
        throw std::invalid_argument("paged op: pool token_bytes != 2 * layers * kv_heads * head_dim * 2");
    }
    vmm = st->dev;
    PRISM_CUDA(cudaSetDevice(vmm->ordinal()));
    stream = static_cast<cudaStream_t>(vmm->stream());
    n_layers = layers;
    n_q = q_heads;
    n_kv = kv_heads;
    head_dim = d;
    group = q_heads / kv_heads;
    geom.base = st->va;
    geom.page_bytes = vmm->page_bytes();
    geom.tpp = static_cast<std::uint32_t>(st->tpp);
    geom.magic = div_magic40(geom.tpp);
    geom.n_layers = layers;
    geom.n_kv = kv_heads;
    geom.head_dim = d;
}

PagedCtx::~PagedCtx() {
    cudaStreamSynchronize(stream);
    if (workspace) cudaFree(workspace);
    if (counters) cudaFree(counters);
}

float* PagedCtx::attn_workspace(std::size_t floats) {
    if (floats > workspace_floats) {
        k3_chain = k4_chain = false;
        if (workspace) {
            PRISM_CUDA(cudaStreamSynchronize(stream));
            PRISM_CUDA(cudaFree(workspace));
        }
        workspace_floats = std::max(floats, workspace_floats * 2);
        PRISM_CUDA(cudaMalloc(&workspace, workspace_floats * sizeof(float)));
    }
    return workspace;
}

int* PagedCtx::attn_counters(std::size_t n) {
    if (n > counters_n) {
        k3_chain = k4_chain = false;
        if (counters) {
            PRISM_CUDA(cudaStreamSynchronize(stream));
            PRISM_CUDA(cudaFree(counters));
        }
        counters_n = std::max(n, counters_n * 2);
        PRISM_CUDA(cudaMalloc(&counters, counters_n * sizeof(int)));
        PRISM_CUDA(cudaMemsetAsync(counters, 0, counters_n * sizeof(int), stream));
    }
    return counters;
}

void PagedCtx::decode_attention(int layer, const std::int32_t* offsets, int n_seqs, const std::int32_t* slot_ids,
                                const void* q, void* out, float scale) {
    if (layer < 0 || layer >= n_layers) throw std::out_of_range("paged decode_attention: bad layer");
    if (n_seqs <= 0) return;
    if (!offsets || !slot_ids || !q || !out) throw std::invalid_argument("paged decode_attention: null pointer");
    if (offsets[0] != 0) throw std::invalid_argument("paged decode_attention: offsets[0] must be 0");
    PRISM_CUDA(cudaSetDevice(vmm->ordinal()));
    // the previous call's descriptor upload must be done before the host copy is rewritten
    decode_desc.ensure(static_cast<std::size_t>(n_seqs));
    for (int b = 0; b < n_seqs; ++b) {
        const std::int32_t ctx = offsets[b + 1] - offsets[b];
        if (ctx <= 0) throw std::invalid_argument("paged decode_attention: every sequence needs >= 1 token");
        decode_desc.host[b] = DecodeDesc{offsets[b], ctx, 0, static_cast<std::uint64_t>(b)};
    }
    k3_chain = k4_chain = false;  // the descriptor upload precedes this launch
    decode_desc.upload(static_cast<std::size_t>(n_seqs), stream);
    ++step_serial;  // new block tables every call: rebuild the stream-K tile prefix
    AttnArgs a{};
    a.g = geom;
    a.layer = layer;
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.out = static_cast<__nv_bfloat16*>(out);
    a.table = slot_ids;
    a.desc = decode_desc.dev;
    a.scale_log2 = scale * 1.4426950408889634f;
    launch_k3_streamk(*this, a, n_seqs);
}

std::unique_ptr<PagedOp> make_paged_op(const msim::pagealloc::KvPool& pool, int n_layers, int n_q_heads,
                                       int n_kv_heads, int head_dim) {
    return std::make_unique<PagedCtx>(pool, n_layers, n_q_heads, n_kv_heads, head_dim);
}

}  // namespace prism
