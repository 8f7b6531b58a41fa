// prism-b200 — pool-level K2 / K3 over caller-owned block tables (the
// kv_append / decode_attn entry points SURVEY §8b suggests for an engine that
// keeps its own scheduler and slot tables). Implemented by PagedCtx
// (cuda/device_impl.cuh, cuda/paged_op.cu); everything runs on the pool's
// VMM device stream, so callers order their producers against it
// (prism_device_stream) exactly as for the engine entry points.
#pragma once
#include <cstdint>
#include <memory>

#include "msim/pagealloc.hpp"

namespace prism {

class PagedOp {
public:
    virtual ~PagedOp() = default;
    // offsets: HOST int32 [n_seqs + 1] (offsets[0] = 0, each sequence >= 1
    // token); slot_ids: DEVICE int32 (page * tpp + slot, token order); q / out:
    // device bf16 [n_seqs][n_q][head_dim]
    virtual void decode_attention(int layer, const std::int32_t* offsets, int n_seqs, const std::int32_t* slot_ids,
                                  const void* q, void* out, float scale) = 0;
    // K4, one request's prefill chunk: slot_ids DEVICE int32 = the request's
    // keys 0 .. first + n_tokens - 1 in token order (append the chunk's K/V
    // first); query i (position first + i) attends keys 0 .. first + i;
    // q / out: device bf16 [n_tokens][n_q][head_dim]
    virtual void prefill_attention(int layer, const std::int32_t* slot_ids, int first, int n_tokens, const void* q,
                                   void* out, float scale) = 0;
    // slots: DEVICE int32 [n_tok]; k / v: device bf16 [layer_end - layer_begin][n_tok][n_kv][head_dim]
    virtual void kv_append(int layer_begin, int layer_end, const std::int32_t* slots, int n_tok, const void* k,
                           const void* v) = 0;
};

std::unique_ptr<PagedOp> make_paged_op(const msim::pagealloc::KvPool& pool, int n_layers, int n_q_heads,
                                       int n_kv_heads, int head_dim);

}  // namespace prism
