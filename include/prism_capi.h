/* prism-b200 C-ABI — the drop-in boundary for the elastic-KV + paged-decode
 * hot path of Prism (arXiv 2505.04021).
 *
 * Plain C: opaque handles, plain pointers and sizes, int status codes; no
 * exception ever crosses this boundary (C++ exceptions map to PRISM_E_*,
 * message in prism_last_error()). Every entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj).
 *
 * Two libraries export this ABI:
 *   paper_2505_04021_b200/libprism_b200.so   the product (host C++ runtime +
 *                                            CUDA VMM + sm_100a kernels);
 *   oracle/_ref/libmsim_ref.so               the reference compiled from its
 *                                            own sources + a thin wrapper
 *                                            (test oracle only; host subset,
 *                                            the GPU entry points are absent).
 * so parity tests drive both through identical calls.
 *
 * Threading: one ledger (with its pools / engines) is one serialization
 * domain (reference include/msim/pagealloc.hpp:42-44); different GPUs'
 * objects may be used from different threads concurrently.
 */
#ifndef PRISM_CAPI_H
#define PRISM_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRISM_ABI_VERSION 1

enum prism_status {
    PRISM_OK = 0,
    PRISM_E_USAGE = 1,     /* msim::UsageError: misuse, stale/foreign handle, bad size */
    PRISM_E_PARSE = 2,     /* msim::ParseError: bad trace input */
    PRISM_E_CONFIG = 3,    /* msim::ConfigError */
    PRISM_E_PLACEMENT = 4, /* msim::placement::PlacementError: a model fits on no GPU */
    PRISM_E_CUDA = 5,      /* CUDA / driver failure, or GPU entry point without a device */
    PRISM_E_ARG = 6,       /* null pointer / output buffer too small */
    PRISM_E_INTERNAL = 7
};

int prism_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* prism_last_error(void);
/* 1 when the library contains the CUDA data path (product), 0 for the oracle. */
int prism_has_device_path(void);

/* ------------------------------------------------------------------ types */

typedef struct prism_ledger prism_ledger; /* msim::pagealloc::PhysicalLedger */
typedef struct prism_pool prism_pool;     /* msim::pagealloc::KvPool */
typedef struct prism_gpu prism_gpu;       /* msim::engine::GpuState */
typedef struct prism_device prism_device; /* prism::VmmDevice (product only) */

/* msim::pagealloc::TokenSlotHandle (pagealloc.hpp:16-24) */
typedef struct {
    uint32_t pool;
    uint32_t page;
    uint32_t slot;
} prism_slot;

/* msim::pagealloc::AllocResult scalars (pagealloc.hpp:104-110) */
typedef struct {
    uint64_t shortfall_pages;
    uint64_t pages_mapped;
    uint64_t buffer_hits;
    uint64_t n_handles;
} prism_alloc_result;

/* msim::pagealloc::AllocEvent (pagealloc.hpp:34-40); kind: 0 map, 1 unmap,
 * 2 buffer_hit, 3 alloc_fail (AllocEventKind order). */
typedef struct {
    int64_t time_us;
    int32_t gpu_id;
    int32_t kind;
    uint64_t pages;
    char model_id[64];
} prism_event;

typedef struct {
    uint64_t capacity_pages, mapped_pages, buffer_pages, weight_pages, free_pages, page_bytes;
} prism_ledger_stats;

typedef struct {
    uint32_t id;
    int32_t alive;
    uint64_t token_bytes, tokens_per_page, virtual_capacity_pages, mapped_pages, occupied_slots;
    uint64_t device_base; /* product with a device attached: VA of page 0 */
} prism_pool_info;

/* msim::engine::ModelSpec (engine.hpp:16-25) + the prism-b200 attention shape */
typedef struct {
    const char* model_id;
    uint64_t weight_bytes;
    uint64_t token_kv_bytes;
    double prefill_tps;
    int32_t chunk_size;
    double ttft_slo_s;
    double tpot_slo_s;
    int32_t tp_degree;
    int32_t n_layers, n_q_heads, n_kv_heads, head_dim; /* 0: host-only model */
} prism_model_spec;

/* msim::engine::EngineParams (engine.hpp:27-34) */
typedef struct {
    double alpha_ms, beta_ms_per_token, map_latency_ms, engine_init_s, realign_s, reserve_frac;
} prism_engine_params;

/* msim::engine::ActivationOutcome (engine.hpp:129-135) */
typedef struct {
    int32_t engine_index;
    int64_t init_us, realign_us, load_us;
} prism_activation;

/* msim::engine::IterationOutcome scalars (engine.hpp:69-78); the id lists
 * are read with prism_engine_outcome_ids. */
typedef struct {
    int64_t duration_us;
    int32_t chunk_tokens;
    int32_t decode_tokens;
    uint64_t pages_mapped_direct;
    int32_t prefill_paused;
    uint32_t n_first_tokens, n_completions, n_preemptions;
} prism_outcome;

/* One request as EngineRequest exposes it (engine.hpp:57-67). */
typedef struct {
    uint64_t id;
    int32_t prompt_tokens, output_tokens, prompt_done, generated;
    uint64_t admit_seq;
    uint64_t n_slots; /* kv[0].size() */
    int64_t table_row;
} prism_request_info;

/* ------------------------------------------------------------------ defaults / params */

void prism_default_engine_params(prism_engine_params* out);
void prism_default_model_spec(prism_model_spec* out);

/* ------------------------------------------------------------------ ledger (pagealloc.hpp:45-102, src/pagealloc.cpp:17-106) */

int prism_ledger_create(int gpu_id, uint64_t capacity_pages, uint64_t page_bytes, prism_ledger** out);
void prism_ledger_destroy(prism_ledger* l);
int prism_ledger_get_stats(const prism_ledger* l, prism_ledger_stats* out);
int prism_ledger_pool_mapped_pages(const prism_ledger* l, uint32_t pool_id, uint64_t* out);
int prism_refill_buffer(prism_ledger* l, uint64_t target_pages, uint64_t* added); /* refill_buffer :193 */
int prism_ledger_reserve_weights(prism_ledger* l, const char* model_id, uint64_t pages, int* ok);
int prism_ledger_release_weights(prism_ledger* l, const char* model_id);
int prism_ledger_weight_pages_of(const prism_ledger* l, const char* model_id, uint64_t* out);
int prism_ledger_set_time(prism_ledger* l, int64_t now_us);
int prism_ledger_set_recording(prism_ledger* l, int on);
int prism_ledger_events(const prism_ledger* l, prism_event* out, size_t cap, size_t* n); /* n = total */
int prism_ledger_clear_events(prism_ledger* l);
int prism_ledger_check_invariants(const prism_ledger* l);

/* ------------------------------------------------------------------ pool (pagealloc.hpp:114-191) */

/* alloc_kvcache (pagealloc.hpp:176); placement: 0 most_occupied_first, 1 lowest_index_first */
int prism_kvcache_alloc(prism_ledger* l, const char* model_id, uint64_t token_bytes, uint64_t virtual_pages,
                        int placement, prism_pool** out);
/* free_kvcache (pagealloc.hpp:182); the handle stays valid (dead) until prism_pool_destroy */
int prism_kvcache_free(prism_ledger* l, prism_pool* p);
void prism_pool_destroy(prism_pool* p);
int prism_pool_info_get(const prism_pool* p, prism_pool_info* out);
/* alloc_kv (pagealloc.hpp:187). out must hold n slots; res.n_handles = n on success, 0 on shortfall. */
int prism_kv_alloc(prism_pool* p, prism_ledger* l, uint64_t n, prism_slot* out, prism_alloc_result* res);
/* free_kv (pagealloc.hpp:191); on PRISM_E_USAGE the prefix before the bad handle was applied, as in the reference. */
int prism_kv_free(prism_pool* p, prism_ledger* l, const prism_slot* handles, size_t n);
int prism_pool_allocatable_tokens(const prism_pool* p, const prism_ledger* l, uint64_t* out);
int prism_pool_page_occupied(const prism_pool* p, uint32_t page, uint64_t* out);
int prism_pool_page_mapped(const prism_pool* p, uint32_t page, int* out);
/* set_mapped_page_cap (pagealloc.hpp:131); cap < 0 clears it */
int prism_pool_set_cap(prism_pool* p, int64_t cap);

/* ------------------------------------------------------------------ engines (engine.hpp:82-147) */

int prism_gpu_create(int gpu_id, uint64_t capacity_pages, uint64_t page_bytes, prism_gpu** out);
void prism_gpu_destroy(prism_gpu* g);
/* Borrowed view of GpuState::ledger (do not destroy). */
prism_ledger* prism_gpu_ledger(prism_gpu* g);
int prism_gpu_engine_count(const prism_gpu* g, int* out);
/* activate (engine.hpp:140); method 0 naive, 1 parallel; *ok = 0 when the weights do not fit. */
int prism_gpu_activate(prism_gpu* g, const prism_model_spec* spec, int method, const prism_engine_params* params,
                       prism_activation* out, int* ok);
int prism_gpu_finish_activation(prism_gpu* g, int engine_index); /* engine.hpp:143 */
int prism_gpu_deactivate(prism_gpu* g, int engine_index);        /* engine.hpp:147 */
int prism_engine_status(const prism_gpu* g, int engine_index, int* status); /* EngineStatus order */
int prism_engine_push(prism_gpu* g, int engine_index, uint64_t id, int prompt_tokens, int output_tokens);
/* step (engine.hpp:113) for a single-part engine on this GPU's ledger. */
int prism_engine_step(prism_gpu* g, int engine_index, const prism_engine_params* params, int64_t now_us,
                      prism_outcome* out);
/* Id lists of the last step's outcome: which 0 first_tokens, 1 completions, 2 preemptions. */
int prism_engine_outcome_ids(const prism_gpu* g, int engine_index, int which, uint64_t* out, size_t cap, size_t* n);
int prism_engine_counts(const prism_gpu* g, int engine_index, size_t* batch, size_t* queue);
/* where 0 batch, 1 local_queue; index in that container's order */
int prism_engine_request(const prism_gpu* g, int engine_index, int where, size_t index, prism_request_info* out);
/* kv[0] handles of a batch request, token order */
int prism_engine_request_kv(const prism_gpu* g, int engine_index, uint64_t request_id, prism_slot* out, size_t cap,
                            size_t* n);
int prism_engine_mapped_pages(const prism_gpu* g, int engine_index, uint64_t* out);
int prism_engine_next_chunk_need(const prism_gpu* g, int engine_index, uint64_t* out);
int prism_engine_has_runnable_work(const prism_gpu* g, int engine_index, int* out);
int prism_engine_reserved_pages(const prism_gpu* g, int engine_index, double reserve_frac, uint64_t* out);
/* throughput_of (engine.hpp:162) */
int prism_throughput_of(uint64_t kv_budget_bytes, const prism_model_spec* spec, int prompt_tokens, int output_tokens,
                        const prism_engine_params* params, uint64_t page_bytes, double warmup_s, double window_s,
                        double* tokens_per_s, int* max_batch);

/* ------------------------------------------------------------------ global scheduler (placement.hpp:20-109) */

typedef struct {
    prism_model_spec spec;
    double rate;
    const int32_t* current_gpus; /* n_current entries, one per TP part */
    int32_t n_current;
} prism_model_demand;

typedef struct {
    const char* model_id;
    double idle_s, ttft_slo_s;
    uint64_t weight_bytes, weight_pages;
} prism_resident;

typedef struct {
    int32_t gpu_id;
    uint64_t capacity_bytes, weight_bytes;
    double w_req_rate;
    uint64_t capacity_pages, free_pages, page_bytes;
    const prism_resident* residents;
    int32_t n_residents;
} prism_gpu_view;

typedef struct {
    int32_t model_index; /* into the models array */
    int32_t part_index, from_gpu, to_gpu;
} prism_migration;

typedef struct {
    double max_kvpr_after;
    int32_t critical_gpu;
    double critical_shared_before_bytes, critical_last_weight_bytes;
    uint32_t n_migrations;
} prism_plan_info;

/* kvpr (placement.hpp:45) */
int prism_kvpr(double w_req_rate, double shared_kv_bytes, double* out);
/* place_models (placement.hpp:88). assignment: for model i its tp_degree GPUs at
 * offset sum_{j<i} tp_j (cap = sum tp); kvpr_before/after: n_gpus each. */
int prism_place_models(const prism_model_demand* models, size_t n_models, const prism_gpu_view* gpus, size_t n_gpus,
                       double tau_per_gb, int32_t* assignment, size_t assignment_cap, double* kvpr_before,
                       double* kvpr_after, prism_migration* migrations, size_t migrations_cap, prism_plan_info* info);
/* eviction_tick (placement.hpp:100) with the common predicate "free_pages <
 * min_free_pages" (the reference takes a std::function). out: (gpu index,
 * resident index) pairs in eviction order. */
int prism_eviction_tick(const prism_gpu_view* gpus, size_t n_gpus, double idle_threshold_s, uint64_t min_free_pages,
                        int32_t* out_pairs, size_t cap, size_t* n);
/* activate_on_arrival[_tp] (placement.hpp:104-109); *found = 0 -> nullopt */
int prism_activate_on_arrival(const prism_model_spec* spec, const prism_gpu_view* gpus, size_t n_gpus, int32_t* gpu,
                              int* found);
int prism_activate_on_arrival_tp(const prism_model_spec* spec, const prism_gpu_view* gpus, size_t n_gpus,
                                 int32_t* out, size_t cap, int* found);

/* ------------------------------------------------------------------ local scheduler (admission.hpp:14-48) */

typedef struct {
    uint64_t id;
    const char* model_id;
    double arrival_s;
    int32_t prompt_tokens;
    double ttft_slo_s, exec_estimate_s;
} prism_queued_request;

/* moore_hodgson (admission.hpp:30): admit / deferred as indices into queue, in decision order. */
int prism_moore_hodgson(const prism_queued_request* queue, size_t n, double now_s, int32_t* admit, size_t* n_admit,
                        int32_t* deferred, size_t* n_deferred);
/* dispatch (admission.hpp:44) over an admit list (indices into reqs); gate returns DispatchStatus (0 dispatched). */
typedef int (*prism_dispatch_gate)(void* ctx, const prism_queued_request* r);
int prism_dispatch(const prism_queued_request* reqs, const int32_t* admit, size_t n_admit, prism_dispatch_gate gate,
                   void* ctx, uint64_t* dispatched, size_t* n_dispatched);
/* requeue_deferred (admission.hpp:47): out = indices into the concatenation [queue..., deferred...]. */
int prism_requeue_deferred(const prism_queued_request* deferred, size_t n_deferred, const prism_queued_request* queue,
                           size_t n_queue, int32_t* out, size_t* n_out);

/* ------------------------------------------------------------------ workload (workload.hpp:14-78) */

typedef struct {
    double arrival_s;
    char model_id[64];
    int32_t prompt_tokens, output_tokens;
} prism_trace_event;

typedef struct {
    double start_s, end_s, rate_per_s;
} prism_rate_segment;

typedef struct {
    const char* model_id;
    const prism_rate_segment* segments;
    int32_t n_segments;
    double prompt_median, prompt_sigma, output_median, output_sigma;
} prism_model_profile;

/* synth_trace (workload.hpp:78): n = total events (call with cap 0 to size). */
int prism_synth_trace(const prism_model_profile* profiles, size_t n_profiles, uint64_t seed, prism_trace_event* out,
                      size_t cap, size_t* n);
/* scale_trace (workload.hpp:29) */
int prism_scale_trace(const prism_trace_event* in, size_t n_in, int factor, uint64_t seed, double jitter_window_s,
                      prism_trace_event* out, size_t cap, size_t* n);
/* parse_trace_lines (workload.hpp:24) */
int prism_parse_trace_text(const char* text, const char* origin, prism_trace_event* out, size_t cap, size_t* n);

/* ------------------------------------------------------------------ simcore (msim/simcore.hpp)
 * The deterministic discrete-event driver the reference specifies
 * (SimMetrics / run / attainment) but does not implement:
 * place_models at t=0, arrivals -> engine queues (activate_on_arrival for
 * models without an engine), one engine::step at a time per GPU, eviction_tick
 * every tick_s. Host-only; built into both the product and the reference
 * oracle library (identical results are a parity test). */
typedef struct prism_sim prism_sim;

typedef struct {
    int32_t policy; /* 0 prism, 1 mux_flexible, 2 static_partition, 3 qlm_timeshare */
    int32_t n_gpus;
    uint64_t capacity_pages, page_bytes; /* per GPU */
    prism_engine_params params;
    int32_t method; /* 0 naive, 1 parallel activation */
    double tau_per_gb, tick_s, idle_evict_s, pressure_free_frac;
    uint64_t buffer_target_pages;
    int32_t initial_placement;
    uint64_t max_events;
    /* measured weight-load bandwidths (GB/s; 0 = the reference's modelled
     * curves, engine.hpp ActivationParams) and fixed cost (s) per load:
     * load_latency = fixed + weight_bytes / bandwidth (prism_wloader_*). */
    double parallel_load_gbs, naive_load_gbs, load_fixed_s;
    /* local scheduler of the prism policy: 0 Algorithm 2
     * (moore_hodgson + dispatch gate + requeue_deferred over one queue per
     * GPU), 1 per-model FIFO into the engine queues */
    int32_t local_scheduler;
} prism_sim_config;

typedef struct {
    int64_t end_us;
    uint64_t events, iterations, activations, evictions, preemptions, output_tokens, n_requests, completed;
    int32_t truncated;
    uint64_t dispatches, schedule_rounds; /* Algorithm 2 */
} prism_sim_summary;

typedef struct {
    uint64_t id; /* 1-based trace index */
    int64_t arrival_us, first_token_us, completion_us; /* -1: never */
    int32_t prompt_tokens, output_tokens, preemptions, gpu;
} prism_sim_request;

void prism_default_sim_config(prism_sim_config* out);
/* rates[i]: demand of model i for the initial placement (may be NULL = 0). */
int prism_sim_run(const prism_sim_config* cfg, const prism_model_spec* specs, const double* rates, size_t n_models,
                  const prism_trace_event* trace, size_t n_trace, prism_sim** out);
int prism_sim_summary_get(const prism_sim* s, prism_sim_summary* out);
int prism_sim_requests(const prism_sim* s, prism_sim_request* out, size_t cap, size_t* n);
int prism_sim_gpu_busy(const prism_sim* s, int64_t* out, size_t cap, size_t* n);
/* TTFT / TPOT / both attainment at slo_scale for model_id (NULL or "" = all). */
int prism_sim_attainment(const prism_sim* s, const char* model_id, double slo_scale, double* ttft, double* tpot,
                         double* both, uint64_t* n);
void prism_sim_free(prism_sim* s);

/* The two-level scheduler driving the GPU data path (product only; north
 * star (4)): prism_sim_run's event loop — place_models / eviction_tick /
 * activate_on_arrival globally, Algorithm 2 per GPU, engine::step — with
 * every simulated GPU in `owned` backed by a VmmDevice on a physical device
 * (ordinals[g % n_ordinals]): pools reserve VA and map 2 MiB pages on
 * demand, activation attaches each engine's GPU half, eviction frees the
 * pool's VA and returns its chunks for reuse, and every iteration runs K1
 * (inside engine::step), K2, K4 (prefill chunk) and K3 (decodes) for all
 * layers. measured = 0: iterations are charged their modelled duration (the
 * records equal prism_sim_run's); 1: the GPU time of the iteration's kernels
 * (CUDA events on the engine stream; attention path only — there are no
 * model weights / GEMMs). */
typedef struct {
    int32_t measured;
    uint64_t seed;                 /* synthetic K/V content */
    const int32_t* ordinals;       /* physical CUDA devices (NULL: device 0) */
    size_t n_ordinals;
    const int32_t* owned;          /* simulated GPUs run on a device (NULL / 0: all) */
    size_t n_owned;
    int32_t max_decode_batch;      /* per engine step (0: 512) */
    uint64_t chunk_pages;          /* VMM chunk (0: default) */
} prism_serving_options;
typedef struct {
    uint64_t iterations, attached, detached, k2_launches, k3_launches, k4_launches, decode_tokens, prefill_tokens;
    uint64_t gpu_us, modelled_us; /* measured mode: charged GPU time and the cost model's for the same iterations */
    uint64_t vmm_maps, vmm_unmaps, vmm_revived, vmm_creates, vmm_driver_unmaps, vmm_steals, vmm_urgent;
    double vmm_caller_ns, vmm_worker_ns, wall_s;
} prism_serving_stats;
int prism_sim_run_device(const prism_sim_config* cfg, const prism_model_spec* specs, const double* rates,
                         size_t n_models, const prism_trace_event* trace, size_t n_trace,
                         const prism_serving_options* opts, prism_sim** out);
/* PRISM_E_USAGE for a run without the device path */
int prism_sim_serving_get(const prism_sim* s, prism_serving_stats* out);

/* ------------------------------------------------------------------ GPU data path (product only; no reference counterpart) */

/* prism::VmmDevice on CUDA device `ordinal` (2 MiB pages). Physical memory
 * is managed in chunks of `chunk_pages` logical pages (one VMM handle each;
 * 0 = PRISM_CHUNK_PAGES or 8); prism_device_open uses the default. */
int prism_device_open(int ordinal, uint64_t page_bytes, prism_device** out);
int prism_device_open_chunked(int ordinal, uint64_t page_bytes, uint64_t chunk_pages, prism_device** out);
int prism_device_chunk_pages(const prism_device* d, uint64_t* out);
void prism_device_close(prism_device* d);
/* Ledger capacity in pages after leaving reserve_bytes of free HBM. */
int prism_device_capacity_pages(const prism_device* d, uint64_t reserve_bytes, uint64_t* out);
/* Startup reservation of physical memory: create handles for `pages` logical
 * pages (bounded by the ledger's physical budget) on the VMM worker and keep
 * that many ready, so maps while serving never wait on cuMemCreate. Pair with
 * prism_device_quiesce to wait for it. */
int prism_device_reserve(prism_device* d, uint64_t pages);
typedef struct {
    uint64_t maps, revived, creates, unmaps, driver_unmaps;
    double map_ns_total, unmap_ns_total;
    double map_ns_p50, map_ns_p99, unmap_ns_p50, unmap_ns_p99;
    uint64_t buffered, cached, pending;
    double create_ns_total, map_call_ns_total, access_ns_total; /* per driver call kind */
    uint64_t access_calls;
    uint64_t steals; /* parked pages moved to another VA (cross-model memory movement) */
    double steal_ns_total; /* cuMemUnmap time of steals (worker thread) */
    double background_ns_total; /* worker-thread driver time (all per-page driver calls run there) */
    uint64_t premaps;           /* chunks the worker mapped ahead of need */
    uint64_t premapped_hits;    /* logical maps that revived a chunk mapped ahead */
    uint64_t over_budget;       /* urgent maps that found no safe idle chunk and created past the budget */
    uint64_t caller_steals_clean; /* steals that took a pre-mapped page */
    double wait_ns_total;       /* caller time waiting for the worker's queued maps (inside map_ns_total) */
    uint64_t urgent;            /* chunks the worker mapped on demand (not anticipated by the look-ahead) */
    uint64_t total_chunks;      /* physical chunks held (mapped, cached, in flight) */
    uint64_t chunk_pages;       /* logical pages per chunk */
    /* raw driver-call latency per physical chunk (worker thread, bounded sample):
     * cuMemMap + cuMemSetAccess, cuMemCreate, cuMemUnmap of a steal */
    double drv_map_ns_p50, drv_map_ns_p99, drv_create_ns_p50, drv_create_ns_p99, drv_unmap_ns_p50, drv_unmap_ns_p99;
    uint64_t reserve_steals;    /* background steals into the handle reserve (PRISM_VMM_RESERVE_CHUNKS) */
} prism_device_stats;
int prism_device_stats_get(const prism_device* d, prism_device_stats* out);
int prism_device_reset_stats(prism_device* d);
int prism_device_reclaim(prism_device* d, int wait);
/* Block until the device's background worker is idle (tests, benchmarks). */
int prism_device_quiesce(prism_device* d);
/* Record a fence on the device stream: pages unmapped before it become
 * reclaimable (cuMemUnmap'ed by prism_device_reclaim(d, 0)) once it passes. */
int prism_device_fence(prism_device* d);
int prism_device_synchronize(prism_device* d);
void* prism_device_stream(const prism_device* d); /* cudaStream_t of the GPU's work stream */
/* PhysicalLedger::attach_device; before any pool is created on the ledger. */
int prism_ledger_attach_device(prism_ledger* l, prism_device* d);

/* Pool-level GPU slot mirror (K1 without an engine): replays the pool's
 * pending alloc/free log on the device; out receives the slot ids
 * (page * tokens_per_page + slot) of every logged allocation, in order. */
int prism_pool_attach_mirror(prism_pool* p);
int prism_pool_sync_mirror(prism_pool* p, int32_t* out, size_t cap, size_t* n);
int prism_pool_read_mirror(prism_pool* p, uint32_t* occ, size_t occ_cap, uint32_t* bits, size_t bits_cap);

typedef struct {
    int64_t table_capacity;
    int32_t max_decode_batch;
    int32_t max_step_tokens;
} prism_engine_device_options;

/* prism::attach_engine_device (msim/kvcache_device.hpp). */
int prism_engine_attach_device(prism_gpu* g, int engine_index, const prism_engine_device_options* opts);
/* Last step: slots allocated (prefill chunk first, then decodes) and decoded requests. */
int prism_engine_step_info(const prism_gpu* g, int engine_index, int32_t* n_step_tokens, int32_t* n_decodes);
int prism_engine_step_decode_ids(const prism_gpu* g, int engine_index, uint64_t* out, size_t cap, size_t* n);
/* Device copy of the last step's slot ids (synchronous; verifies the device allocator agreed with the host). */
int prism_engine_step_slots(const prism_gpu* g, int engine_index, int32_t* out, size_t cap, size_t* n);
int prism_engine_table_row(const prism_gpu* g, int engine_index, int64_t row, int32_t len, int32_t* out);
/* K2: k, v device bf16 [layer_end-layer_begin][n_step_tokens][n_kv][head_dim] */
int prism_engine_append_kv(prism_gpu* g, int engine_index, int layer_begin, int layer_end, const void* k,
                           const void* v);
int prism_engine_append_kv_synthetic(prism_gpu* g, int engine_index, int layer_begin, int layer_end, uint64_t seed);
/* K3: q, out device bf16 [n_decodes][n_q_heads][head_dim]; chunk <= 0 picks the split size. */
int prism_engine_decode_attention(prism_gpu* g, int engine_index, int layer, const void* q, void* out, float scale,
                                  int32_t chunk);
/* K3 implementation: 3 tensor-core stream-K persistent, equal KV-tile ranges
 * per CTA (default); 0 tensor-core mma.sync, 2-stage cp.async ring, 3 CTAs/SM,
 * split-K; 1 CUDA-core SIMT; 2 tensor-core, 3-stage ring, 2 CTAs/SM.
 * A positive `chunk` in prism_engine_decode_attention selects the split-K
 * kernels (0 when variant 3 is set). */
int prism_set_attention_variant(int variant);
/* K4, chunked-prefill attention of the last step's prefill chunk (no reference
 * counterpart: the reference allocates the chunk, engine.cpp:182-210, but
 * computes no attention). q, out: device bf16
 * [n_tokens][n_q_heads][head_dim]; query i at position first + i attends keys
 * 0..first+i of its request (causal), K/V from the pages (append them first). */
int prism_engine_prefill_info(const prism_gpu* g, int engine_index, int32_t* n_tokens, int32_t* first,
                              uint64_t* request);
int prism_engine_prefill_attention(prism_gpu* g, int engine_index, int layer, const void* q, void* out, float scale);
/* Diagnostics: progress words of the last K4 launch (PRISM_K4_DEBUG=1), readable while it runs. */
int prism_debug_k4_progress(uint32_t* out, int32_t n, int32_t* got);
/* Diagnostics: timeline of the last K4 launch's CTA (0,0) (PRISM_K4_TRACE=1): [5][1024] globaltimer ns
 * (loader tile issued, S issued, P·V issued, softmax has S, softmax posted P). */
int prism_debug_k4_trace(uint64_t* out, int32_t n, int32_t* got);
/* Diagnostics: per-CTA stamps of the last K3 launch (PRISM_K3_TRACE=1): [grid][8] globaltimer ns
 * (running, prologue issued, after the PDL wait, first tile, last tile, done, tiles). */
int prism_debug_k3_trace(uint64_t* out, int32_t n, int32_t* got);
int prism_engine_synth_q(prism_gpu* g, int engine_index, int layer, uint64_t seed, float q_scale, void* q);
/* End-to-end: the same attention with HOST buffers (pinned or pageable);
 * copies q in, runs K2 for new_k/new_v (host, may be null) over all layers
 * and K3 for every layer, copies out back; synchronous. q/out: [n_layers][n_decodes][n_q][d]. */
int prism_engine_decode_host(prism_gpu* g, int engine_index, const void* new_k, const void* new_v, const void* q,
                             void* out, float scale);
/* Same, enqueued only (copies on a per-engine copy stream overlapping the
 * kernels); host buffers must stay valid until prism_engine_wait_host. */
int prism_engine_decode_host_async(prism_gpu* g, int engine_index, const void* new_k, const void* new_v,
                                   const void* q, void* out, float scale);
int prism_engine_wait_host(prism_gpu* g, int engine_index);
int prism_engine_synchronize(prism_gpu* g, int engine_index);

/* ---- pool-level K2 / K3 over caller-owned block tables ----
 * For an engine that keeps its own scheduler and slot tables (SURVEY §8b's
 * suggested kv_append / decode_attn; the reference has no attention,
 * SPEC.md:278): slot ids are page * tpp + slot of handles from prism_kv_alloc
 * (pagealloc.hpp:188) in token order. Runs on the pool's device stream
 * (prism_device_stream); the pool must outlive the handle. */
typedef struct prism_paged prism_paged;
int prism_paged_create(const prism_pool* p, int n_layers, int n_q_heads, int n_kv_heads, int head_dim,
                       prism_paged** out);
int prism_paged_destroy(prism_paged* pa);
/* K2: slots device int32 [n_tokens]; k, v device bf16 [layer_end-layer_begin][n_tokens][n_kv][head_dim] */
int prism_paged_kv_append(prism_paged* pa, int layer_begin, int layer_end, const int32_t* slots, int32_t n_tokens,
                          const void* k, const void* v);
/* K4: one request's prefill chunk; slot_ids device int32 = its keys 0..first+n_tokens-1 (append the chunk first);
 * query i attends keys 0..first+i; q, out device bf16 [n_tokens][n_q][head_dim] */
int prism_paged_prefill_attention(prism_paged* pa, int layer, const int32_t* slot_ids, int32_t first, int32_t n_tokens,
                                  const void* q, void* out, float scale);
/* K3: seq_offsets HOST int32 [n_seqs+1] into slot_ids (device int32); q, out device bf16 [n_seqs][n_q][head_dim] */
int prism_paged_decode_attention(prism_paged* pa, int layer, const int32_t* seq_offsets, int32_t n_seqs,
                                 const int32_t* slot_ids, const void* q, void* out, float scale);

/* ---- model weight loading for activation ----
 * Replaces the modelled weight-load latency of activation
 * (ActivationParams::load_latency_s, reference engine.hpp:46-48,
 * src/engine.cpp:44-51) with the paper's data path:
 * chunked multi-stream loads, and the per-helper half of a staged fan-in into
 * another GPU (peer or IPC pointer). Enqueue-only; prism_wloader_wait
 * synchronises and reports device milliseconds. Host memory must be pinned. */
typedef struct prism_wloader prism_wloader;
int prism_wloader_create(int device, int n_streams, uint64_t chunk_bytes, prism_wloader** out);
int prism_wloader_destroy(prism_wloader* w);
/* host -> dst (this loader's GPU), chunks round-robin over the streams */
int prism_wloader_load(prism_wloader* w, const void* host, void* dst, uint64_t bytes);
/* baseline: one cudaMemcpyAsync */
int prism_wloader_load_naive(prism_wloader* w, const void* host, void* dst, uint64_t bytes);
/* fan-in helper: chunks i % n_parts == part, host -> this GPU's staging -> dst (any GPU) */
int prism_wloader_load_part(prism_wloader* w, const void* host, void* dst, uint64_t bytes, int part, int n_parts);
int prism_wloader_wait(prism_wloader* w, double* ms);
/* cudaHostRegister / Unregister (pin an existing host buffer) */
int prism_host_register(void* host, uint64_t bytes);
int prism_host_unregister(void* host);
/* CUDA IPC for fan-in across processes: 64-byte handle of a cudaMalloc'ed pointer */
int prism_ipc_handle(const void* dptr, void* handle64);
int prism_ipc_open(int device, const void* handle64, void** dptr);
int prism_ipc_close(int device, void* dptr);

#ifdef __cplusplus
}
#endif

#endif /* PRISM_CAPI_H */
