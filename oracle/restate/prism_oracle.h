/* prism_oracle — CPU restatement of the Prism hot path. TEST INFRASTRUCTURE
 * ONLY: used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * arm as the checker; never linked into or called by the product.
 *
 * Parity status:
 *   allocator (po_*)    pinned: restates reference src/pagealloc.cpp and is
 *                       checked against golden vectors produced by the
 *                       compiled reference (tests/golden/, oracle/_ref);
 *   attention           UNPINNED by the reference (it has no attention
 *                       operator); restated from the standard
 *                       definition in fp64 with GQA mapping kv = q / (nq/nkv)
 *                       over the token order of EngineRequest::kv;
 *   synthetic content   defined by this repo, bit-identical to
 *                       csrc/cuda/common.cuh synth_value.
 */
#ifndef PRISM_ORACLE_H
#define PRISM_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* bf16 bit pattern of the synthetic value (kind 0 K, 1 V, 2 Q) times scale. */
uint16_t po_synth_bf16(uint64_t seed, uint64_t req, uint32_t pos, int layer, int kind, int head, int dim, float scale);
float po_bf16_to_float(uint16_t b);

/* fp64 decode attention over synthetic content for n_dec requests at one
 * layer: request r has context positions [0, ctx[r]); q at position ctx-1.
 * out: [n_dec][n_q][d] doubles. Uses OpenMP over (request, q head). */
void po_decode_attention_synth(uint64_t seed, int layer, size_t n_dec, const uint64_t* req_ids, const int32_t* ctx,
                               int n_q, int n_kv, int d, float q_scale, double scale, double* out);

/* fp64 decode attention over explicit bf16 tensors:
 * q [n_q][d], k/v [ctx][n_kv][d] for one request; out [n_q][d]. */
void po_decode_attention_dense(const uint16_t* q, const uint16_t* k, const uint16_t* v, int ctx, int n_q, int n_kv,
                               int d, double scale, double* out);

/* CPU paged decode attention over a HOST copy of the paged KV layout
 * ([layer][K|V][kv_head][slot][d] bf16 inside each page_bytes page; slot id =
 * page * tpp + slot), fp32 accumulation, n_threads pthreads. This is the
 * CPU-baseline "port" of the GPU kernel (the reference has no attention).
 * q: bf16 [n_dec][n_q][d]; table: slot ids; rows[b]: element offset of
 * request b's row; ctx[b]: its length. out: float [n_dec][n_q][d]. */
void po_paged_attention_cpu(const uint8_t* pool, uint64_t page_bytes, uint32_t tpp, int n_kv, int d, int layer,
                            const int32_t* table, const int64_t* rows, const int32_t* ctx, size_t n_dec,
                            const uint16_t* q, int n_q, float scale, float* out, int n_threads);

/* ---- allocator restatement (reference src/pagealloc.cpp:108-267) ---- */
typedef struct po_pool po_pool;
typedef struct {
    uint64_t capacity, kv_mapped, buffer, weights;
} po_ledger;

po_pool* po_pool_create(uint32_t pool_id, uint64_t tokens_per_page, uint64_t virtual_pages, int lowest_index_first);
void po_pool_destroy(po_pool* p);
/* alloc_kv: returns shortfall pages (0 = ok); out_page/out_slot hold n entries
 * on success; *buffer_hits / *direct set like AllocResult. */
uint64_t po_alloc(po_pool* p, po_ledger* l, uint64_t n, uint32_t* out_page, uint32_t* out_slot, uint64_t* buffer_hits,
                  uint64_t* direct);
/* free_kv: returns -1 on the first invalid handle (prefix applied), else the
 * number of pages unmapped. */
int64_t po_free(po_pool* p, po_ledger* l, uint32_t pool_id, const uint32_t* page, const uint32_t* slot, size_t n);
uint64_t po_mapped(const po_pool* p);
uint64_t po_occupied(const po_pool* p);
uint32_t po_page_occupied(const po_pool* p, uint32_t page);

#ifdef __cplusplus
}
#endif
#endif
