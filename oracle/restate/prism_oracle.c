/* prism_oracle.c — CPU restatement of the Prism hot path (test oracle only;
 * see prism_oracle.h for what is pinned and what is not). Plain C11. */
#define _GNU_SOURCE
#include "prism_oracle.h"

#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ synthetic content
 * Must stay bit-identical to csrc/cuda/common.cuh synth_value + RNE bf16. */
static uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

static float synth_float(uint64_t seed, uint64_t req, uint32_t pos, int layer, int kind, int head, int dim) {
    const uint64_t a = (req * 0x9E3779B97F4A7C15ull) ^ (uint64_t)pos;
    const uint64_t b = ((uint64_t)layer << 40) | ((uint64_t)kind << 36) | ((uint64_t)head << 20) | (uint64_t)dim;
    const uint64_t u = mix64(seed ^ mix64(a) ^ (b * 0xD6E8FEB86659FD93ull));
    return (float)(u >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
}

static uint16_t f32_to_bf16_rne(float f) {
    uint32_t x;
    memcpy(&x, &f, 4);
    if ((x & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((x >> 16) | 0x40); /* NaN */
    const uint32_t lsb = (x >> 16) & 1u;
    x += 0x7fffu + lsb;
    return (uint16_t)(x >> 16);
}

float po_bf16_to_float(uint16_t b) {
    const uint32_t x = (uint32_t)b << 16;
    float f;
    memcpy(&f, &x, 4);
    return f;
}

uint16_t po_synth_bf16(uint64_t seed, uint64_t req, uint32_t pos, int layer, int kind, int head, int dim, float scale) {
    return f32_to_bf16_rne(synth_float(seed, req, pos, layer, kind, head, dim) * scale);
}

/* ------------------------------------------------------------ attention */

static void attend(const double* q, int d, int ctx, const double* k, const double* v, size_t stride, double scale,
                   double* out, double* w) {
    double mx = -INFINITY;
    for (int t = 0; t < ctx; ++t) {
        double s = 0.0;
        for (int e = 0; e < d; ++e) s += q[e] * k[(size_t)t * stride + e];
        w[t] = s * scale;
        if (w[t] > mx) mx = w[t];
    }
    double sum = 0.0;
    for (int t = 0; t < ctx; ++t) {
        w[t] = exp(w[t] - mx);
        sum += w[t];
    }
    for (int e = 0; e < d; ++e) out[e] = 0.0;
    for (int t = 0; t < ctx; ++t) {
        const double p = w[t] / sum;
        for (int e = 0; e < d; ++e) out[e] += p * v[(size_t)t * stride + e];
    }
}

typedef struct {
    uint64_t seed;
    int layer;
    size_t n_dec;
    const uint64_t* req_ids;
    const int32_t* ctx;
    int n_q, n_kv, d;
    float q_scale;
    double scale;
    double* out;
    size_t next; /* work item counter (atomic) */
} synth_job;

static void synth_item(const synth_job* j, size_t b, int h) {
    const int group = j->n_q / j->n_kv, d = j->d, L = j->ctx[b];
    double* k = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1) * d);
    double* v = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1) * d);
    double* w = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1));
    double* q = (double*)malloc(sizeof(double) * (size_t)d);
    for (int t = 0; t < L; ++t) {
        for (int e = 0; e < d; ++e) {
            k[(size_t)t * d + e] = po_bf16_to_float(po_synth_bf16(j->seed, j->req_ids[b], (uint32_t)t, j->layer, 0, h, e, 1.0f));
            v[(size_t)t * d + e] = po_bf16_to_float(po_synth_bf16(j->seed, j->req_ids[b], (uint32_t)t, j->layer, 1, h, e, 1.0f));
        }
    }
    for (int g = 0; g < group; ++g) {
        const int qh = h * group + g;
        for (int e = 0; e < d; ++e) {
            q[e] = po_bf16_to_float(po_synth_bf16(j->seed, j->req_ids[b], (uint32_t)(L - 1), j->layer, 2, qh, e, j->q_scale));
        }
        attend(q, d, L, k, v, (size_t)d, j->scale, j->out + ((size_t)b * j->n_q + qh) * d, w);
    }
    free(k);
    free(v);
    free(w);
    free(q);
}

static void* synth_worker(void* arg) {
    synth_job* j = (synth_job*)arg;
    const size_t total = j->n_dec * (size_t)j->n_kv;
    for (;;) {
        const size_t i = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (i >= total) break;
        synth_item(j, i / (size_t)j->n_kv, (int)(i % (size_t)j->n_kv));
    }
    return NULL;
}

void po_decode_attention_synth(uint64_t seed, int layer, size_t n_dec, const uint64_t* req_ids, const int32_t* ctx,
                               int n_q, int n_kv, int d, float q_scale, double scale, double* out) {
    synth_job j = {seed, layer, n_dec, req_ids, ctx, n_q, n_kv, d, q_scale, scale, out, 0};
    long n_threads = sysconf(_SC_NPROCESSORS_ONLN);
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 64) n_threads = 64;
    pthread_t th[64];
    for (long t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, synth_worker, &j);
    for (long t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
}

void po_decode_attention_dense(const uint16_t* q, const uint16_t* k, const uint16_t* v, int ctx, int n_q, int n_kv,
                               int d, double scale, double* out) {
    const int group = n_q / n_kv;
    double* kd = (double*)malloc(sizeof(double) * (size_t)ctx * d);
    double* vd = (double*)malloc(sizeof(double) * (size_t)ctx * d);
    double* w = (double*)malloc(sizeof(double) * (size_t)(ctx > 0 ? ctx : 1));
    double* qd = (double*)malloc(sizeof(double) * (size_t)d);
    for (int h = 0; h < n_kv; ++h) {
        for (int t = 0; t < ctx; ++t) {
            for (int e = 0; e < d; ++e) {
                kd[(size_t)t * d + e] = po_bf16_to_float(k[((size_t)t * n_kv + h) * d + e]);
                vd[(size_t)t * d + e] = po_bf16_to_float(v[((size_t)t * n_kv + h) * d + e]);
            }
        }
        for (int g = 0; g < group; ++g) {
            const int qh = h * group + g;
            for (int e = 0; e < d; ++e) qd[e] = po_bf16_to_float(q[(size_t)qh * d + e]);
            attend(qd, d, ctx, kd, vd, (size_t)d, scale, out + (size_t)qh * d, w);
        }
    }
    free(kd);
    free(vd);
    free(w);
    free(qd);
}

/* ------------------------------------------------------------ CPU paged attention (baseline port) */
typedef struct {
    const uint8_t* pool;
    uint64_t page_bytes;
    uint32_t tpp;
    int n_kv, d, layer;
    const int32_t* table;
    const int64_t* rows;
    const int32_t* ctx;
    size_t n_dec;
    const uint16_t* q;
    int n_q;
    float scale;
    float* out;
    size_t next;
} paged_job;

static inline float bf(uint16_t b) {
    const uint32_t x = (uint32_t)b << 16;
    float f;
    memcpy(&f, &x, 4);
    return f;
}

static void paged_item(const paged_job* j, size_t b, int h) {
    const int g = j->n_q / j->n_kv, d = j->d, L = j->ctx[b];
    float qf[8][256];
    float acc[8][256];
    float m[8], l[8];
    for (int k = 0; k < g; ++k) {
        for (int e = 0; e < d; ++e) {
            qf[k][e] = bf(j->q[((size_t)b * j->n_q + (size_t)h * g + k) * d + e]) * j->scale;
            acc[k][e] = 0.f;
        }
        m[k] = -INFINITY;
        l[k] = 0.f;
    }
    const uint64_t row_bytes = (uint64_t)d * 2;
    const uint64_t kblock = ((uint64_t)(j->layer * 2 + 0) * j->n_kv + h) * j->tpp * row_bytes;
    const uint64_t vblock = ((uint64_t)(j->layer * 2 + 1) * j->n_kv + h) * j->tpp * row_bytes;
    for (int t = 0; t < L; ++t) {
        const uint32_t sid = (uint32_t)j->table[j->rows[b] + t];
        const uint32_t page = sid / j->tpp, slot = sid % j->tpp;
        const uint16_t* kr = (const uint16_t*)(j->pool + (uint64_t)page * j->page_bytes + kblock + slot * row_bytes);
        const uint16_t* vr = (const uint16_t*)(j->pool + (uint64_t)page * j->page_bytes + vblock + slot * row_bytes);
        float kf[256], vf[256];
        for (int e = 0; e < d; ++e) {
            kf[e] = bf(kr[e]);
            vf[e] = bf(vr[e]);
        }
        for (int k = 0; k < g; ++k) {
            /* 8 independent partial sums so the compiler vectorizes the dot
             * product without reassociation flags */
            float part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int e = 0; e < d; e += 8) {
                for (int u = 0; u < 8; ++u) part[u] += qf[k][e + u] * kf[e + u];
            }
            const float s = ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]));
            if (s > m[k]) { /* rescale only when the running max grows */
                const float a = expf(m[k] - s);
                l[k] *= a;
                for (int e = 0; e < d; ++e) acc[k][e] *= a;
                m[k] = s;
            }
            const float p = expf(s - m[k]);
            l[k] += p;
            for (int e = 0; e < d; ++e) acc[k][e] += p * vf[e];
        }
    }
    for (int k = 0; k < g; ++k) {
        float* o = j->out + ((size_t)b * j->n_q + (size_t)h * g + k) * d;
        for (int e = 0; e < d; ++e) o[e] = acc[k][e] / l[k];
    }
}

static void* paged_worker(void* arg) {
    paged_job* j = (paged_job*)arg;
    const size_t total = j->n_dec * (size_t)j->n_kv;
    for (;;) {
        const size_t i = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (i >= total) break;
        paged_item(j, i / (size_t)j->n_kv, (int)(i % (size_t)j->n_kv));
    }
    return NULL;
}

void po_paged_attention_cpu(const uint8_t* pool, uint64_t page_bytes, uint32_t tpp, int n_kv, int d, int layer,
                            const int32_t* table, const int64_t* rows, const int32_t* ctx, size_t n_dec,
                            const uint16_t* q, int n_q, float scale, float* out, int n_threads) {
    paged_job j = {pool, page_bytes, tpp, n_kv, d, layer, table, rows, ctx, n_dec, q, n_q, scale, out, 0};
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    pthread_t th[256];
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, paged_worker, &j);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------ allocator
 * Straight restatement of reference src/pagealloc.cpp: per-page
 * {mapped, occupied, slots[]} with the O(V) pick_page scan (:158-186), the
 * all-or-nothing budget check (:194-213), buffer-before-direct accounting
 * (:215-219), ascending first-free fill (:221-242) and unmap-on-empty
 * (:246-267). Deliberately naive: it is the checker, not the product. */
struct po_pool {
    uint32_t id;
    uint64_t tpp, vpages, mapped, occupied;
    int lowest_index_first;
    uint8_t* pmapped;  /* [vpages] */
    uint32_t* pocc;    /* [vpages] */
    uint8_t* slots;    /* [vpages * tpp] */
};

po_pool* po_pool_create(uint32_t pool_id, uint64_t tpp, uint64_t vpages, int lowest_index_first) {
    po_pool* p = (po_pool*)calloc(1, sizeof(po_pool));
    p->id = pool_id;
    p->tpp = tpp;
    p->vpages = vpages;
    p->lowest_index_first = lowest_index_first;
    p->pmapped = (uint8_t*)calloc(vpages, 1);
    p->pocc = (uint32_t*)calloc(vpages, sizeof(uint32_t));
    p->slots = (uint8_t*)calloc(vpages * tpp, 1);
    return p;
}

void po_pool_destroy(po_pool* p) {
    if (!p) return;
    free(p->pmapped);
    free(p->pocc);
    free(p->slots);
    free(p);
}

static int64_t pick_page(const po_pool* p, int* needs_map) {
    int64_t best = -1;
    *needs_map = 0;
    if (!p->lowest_index_first) {
        uint32_t best_occ = 0;
        for (uint64_t i = 0; i < p->vpages; ++i) {
            if (!p->pmapped[i] || p->pocc[i] >= p->tpp) continue;
            if (best < 0 || p->pocc[i] > best_occ) {
                best = (int64_t)i;
                best_occ = p->pocc[i];
            }
        }
    } else {
        for (uint64_t i = 0; i < p->vpages; ++i) {
            if (p->pmapped[i] && p->pocc[i] < p->tpp) {
                best = (int64_t)i;
                break;
            }
        }
    }
    if (best >= 0) return best;
    *needs_map = 1;
    for (uint64_t i = 0; i < p->vpages; ++i) {
        if (!p->pmapped[i]) return (int64_t)i;
    }
    return -1;
}

uint64_t po_alloc(po_pool* p, po_ledger* l, uint64_t n, uint32_t* out_page, uint32_t* out_slot, uint64_t* buffer_hits,
                  uint64_t* direct) {
    *buffer_hits = 0;
    *direct = 0;
    if (n == 0) return 0;
    const uint64_t partial_free = p->mapped * p->tpp - p->occupied;
    uint64_t new_pages = 0;
    if (n > partial_free) new_pages = (n - partial_free + p->tpp - 1) / p->tpp;
    const uint64_t free_pages = l->capacity - l->kv_mapped - l->buffer - l->weights;
    uint64_t budget = free_pages + l->buffer;
    if (budget > p->vpages - p->mapped) budget = p->vpages - p->mapped;
    if (new_pages > budget) return new_pages - budget;
    *buffer_hits = new_pages < l->buffer ? new_pages : l->buffer;
    l->buffer -= *buffer_hits;
    *direct = new_pages - *buffer_hits;
    l->kv_mapped += new_pages;
    uint64_t k = 0;
    while (k < n) {
        int needs_map = 0;
        const int64_t page = pick_page(p, &needs_map);
        if (page < 0) return ~0ull; /* accounting error */
        if (needs_map) {
            p->pmapped[page] = 1;
            p->pocc[page] = 0;
            memset(p->slots + (uint64_t)page * p->tpp, 0, p->tpp);
            ++p->mapped;
        }
        for (uint64_t s = 0; s < p->tpp && k < n; ++s) {
            uint8_t* bit = p->slots + (uint64_t)page * p->tpp + s;
            if (*bit) continue;
            *bit = 1;
            ++p->pocc[page];
            ++p->occupied;
            out_page[k] = (uint32_t)page;
            out_slot[k] = (uint32_t)s;
            ++k;
        }
    }
    return 0;
}

int64_t po_free(po_pool* p, po_ledger* l, uint32_t pool_id, const uint32_t* page, const uint32_t* slot, size_t n) {
    int64_t unmapped = 0;
    for (size_t i = 0; i < n; ++i) {
        if (pool_id != p->id || page[i] >= p->vpages) return -1;
        if (!p->pmapped[page[i]] || slot[i] >= p->tpp) return -1;
        uint8_t* bit = p->slots + (uint64_t)page[i] * p->tpp + slot[i];
        if (!*bit) return -1;
        *bit = 0;
        --p->pocc[page[i]];
        --p->occupied;
        if (p->pocc[page[i]] == 0) {
            p->pmapped[page[i]] = 0;
            --p->mapped;
            --l->kv_mapped;
            ++unmapped;
        }
    }
    return unmapped;
}

uint64_t po_mapped(const po_pool* p) { return p->mapped; }
uint64_t po_occupied(const po_pool* p) { return p->occupied; }
uint32_t po_page_occupied(const po_pool* p, uint32_t page) { return page < p->vpages ? p->pocc[page] : 0; }
