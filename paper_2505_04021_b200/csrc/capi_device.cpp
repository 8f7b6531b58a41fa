// C-ABI (include/prism_capi.h), GPU data-path subset — product only.
// VMM device, pool mirror (K1), engine device (K1/K2/K3) and the host-buffer
// end-to-end entry point.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include <cuda_runtime.h>

#include "host/pool_state.hpp"
#include "host/vmm.hpp"
#include "host/weight_load.hpp"
#include "host/paged_op.hpp"
#include "host/serving.hpp"
#include "msim/kvcache_device.hpp"
#include "prism_capi.h"
#include "capi_handles.hpp"

namespace pa = msim::pagealloc;
namespace me = msim::engine;

struct prism_device {
    std::shared_ptr<prism::VmmDevice> dev;  // ledgers / pools hold further references
};

namespace {

template <class F>
int dguard(F&& f) {
    try {
        f();
        return PRISM_OK;
    } catch (const msim::UsageError& e) {
        prism_capi_detail::set_error(e.what());
        return PRISM_E_USAGE;
    } catch (const std::invalid_argument& e) {
        prism_capi_detail::set_error(e.what());
        return PRISM_E_ARG;
    } catch (const std::out_of_range& e) {
        prism_capi_detail::set_error(e.what());
        return PRISM_E_ARG;
    } catch (const std::exception& e) {
        prism_capi_detail::set_error(e.what());
        return PRISM_E_CUDA;
    } catch (...) {
        prism_capi_detail::set_error("unknown exception");
        return PRISM_E_INTERNAL;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}

me::Engine& engine_at(prism_gpu* g, int i) {
    need(g, "gpu");
    if (i < 0 || static_cast<std::size_t>(i) >= g->g.engines.size()) throw std::out_of_range("engine index");
    return g->g.engines[static_cast<std::size_t>(i)];
}
const me::Engine& engine_at(const prism_gpu* g, int i) { return engine_at(const_cast<prism_gpu*>(g), i); }

double percentile(std::vector<float> v, double q) {
    if (v.empty()) return 0.0;
    const std::size_t k = static_cast<std::size_t>(q * static_cast<double>(v.size() - 1) + 0.5);
    std::nth_element(v.begin(), v.begin() + static_cast<std::ptrdiff_t>(k), v.end());
    return v[k];
}

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

extern "C" {

int prism_has_device_path(void) { return 1; }

int prism_device_open(int ordinal, uint64_t page_bytes, prism_device** out) {
    return prism_device_open_chunked(ordinal, page_bytes, 0, out);
}

int prism_device_open_chunked(int ordinal, uint64_t page_bytes, uint64_t chunk_pages, prism_device** out) {
    return dguard([&] {
        need(out, "out");
        auto* d = new prism_device();
        try {
            d->dev = prism::VmmDevice::open(ordinal, page_bytes, chunk_pages);
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

void prism_device_close(prism_device* d) { delete d; }

int prism_device_capacity_pages(const prism_device* d, uint64_t reserve_bytes, uint64_t* out) {
    return dguard([&] {
        need(d, "device");
        need(out, "out");
        *out = d->dev->capacity_pages(reserve_bytes);
    });
}

int prism_device_stats_get(const prism_device* d, prism_device_stats* out) {
    return dguard([&] {
        need(d, "device");
        need(out, "out");
        const prism::VmmStats s = d->dev->stats();
        out->maps = s.maps;
        out->revived = s.revived;
        out->creates = s.creates;
        out->unmaps = s.unmaps;
        out->driver_unmaps = s.driver_unmaps;
        out->map_ns_total = s.map_ns_total;
        out->unmap_ns_total = s.unmap_ns_total;
        out->map_ns_p50 = percentile(s.map_ns, 0.5);
        out->map_ns_p99 = percentile(s.map_ns, 0.99);
        out->unmap_ns_p50 = percentile(s.unmap_ns, 0.5);
        out->unmap_ns_p99 = percentile(s.unmap_ns, 0.99);
        out->buffered = d->dev->buffered_handles();
        out->cached = d->dev->cached_handles();
        out->pending = d->dev->pending_unmaps();
        out->create_ns_total = s.create_ns_total;
        out->map_call_ns_total = s.map_call_ns_total;
        out->access_ns_total = s.access_ns_total;
        out->access_calls = s.access_calls;
        out->steals = s.steals;
        out->steal_ns_total = s.steal_ns_total;
        out->background_ns_total = s.background_ns_total;
        out->premaps = s.premaps;
        out->premapped_hits = s.premapped_hits;
        out->over_budget = s.over_budget;
        out->caller_steals_clean = s.caller_steals_clean;
        out->wait_ns_total = s.wait_ns_total;
        out->urgent = s.urgent;
        out->total_chunks = d->dev->total_handles();
        out->chunk_pages = d->dev->chunk_pages();
        out->drv_map_ns_p50 = percentile(s.drv_map_ns, 0.5);
        out->drv_map_ns_p99 = percentile(s.drv_map_ns, 0.99);
        out->drv_create_ns_p50 = percentile(s.drv_create_ns, 0.5);
        out->drv_create_ns_p99 = percentile(s.drv_create_ns, 0.99);
        out->drv_unmap_ns_p50 = percentile(s.drv_unmap_ns, 0.5);
        out->drv_unmap_ns_p99 = percentile(s.drv_unmap_ns, 0.99);
        out->reserve_steals = s.reserve_steals;
    });
}

int prism_device_reset_stats(prism_device* d) {
    return dguard([&] {
        need(d, "device");
        d->dev->reset_stats();
    });
}

int prism_device_reclaim(prism_device* d, int wait) {
    return dguard([&] {
        need(d, "device");
        d->dev->reclaim(wait != 0);
    });
}

int prism_device_chunk_pages(const prism_device* d, uint64_t* out) {
    return dguard([&] {
        need(d, "device");
        need(out, "out");
        *out = d->dev->chunk_pages();
    });
}

int prism_device_reserve(prism_device* d, uint64_t pages) {
    return dguard([&] {
        need(d, "device");
        d->dev->reserve_physical(pages);
    });
}

int prism_device_quiesce(prism_device* d) {
    return dguard([&] {
        need(d, "device");
        d->dev->quiesce();
    });
}

int prism_device_fence(prism_device* d) {
    return dguard([&] {
        need(d, "device");
        d->dev->fence();
    });
}

int prism_device_synchronize(prism_device* d) {
    return dguard([&] {
        need(d, "device");
        check(cudaStreamSynchronize(static_cast<cudaStream_t>(d->dev->stream())), "cudaStreamSynchronize");
    });
}

void* prism_device_stream(const prism_device* d) { return d ? d->dev->stream() : nullptr; }

int prism_ledger_attach_device(prism_ledger* l, prism_device* d) {
    return dguard([&] {
        need(l, "ledger");
        l->l->attach_device(d ? d->dev.get() : nullptr);
    });
}

int prism_pool_attach_mirror(prism_pool* p) {
    return dguard([&] {
        need(p, "pool");
        prism::attach_pool_mirror(p->pool);
    });
}

int prism_pool_sync_mirror(prism_pool* p, int32_t* out, size_t cap, size_t* n) {
    return dguard([&] {
        need(p, "pool");
        const auto v = prism::sync_pool_mirror(p->pool);
        if (n) *n = v.size();
        if (out) {
            if (v.size() > cap) throw std::invalid_argument("output buffer too small");
            std::copy(v.begin(), v.end(), out);
        }
    });
}

int prism_pool_read_mirror(prism_pool* p, uint32_t* occ, size_t occ_cap, uint32_t* bits, size_t bits_cap) {
    return dguard([&] {
        need(p, "pool");
        std::vector<std::uint32_t> o, b;
        prism::read_pool_mirror(p->pool, o, b);
        if (occ) {
            if (o.size() > occ_cap) throw std::invalid_argument("occ buffer too small");
            std::copy(o.begin(), o.end(), occ);
        }
        if (bits) {
            if (b.size() > bits_cap) throw std::invalid_argument("bits buffer too small");
            std::copy(b.begin(), b.end(), bits);
        }
    });
}

int prism_engine_attach_device(prism_gpu* g, int engine_index, const prism_engine_device_options* opts) {
    return dguard([&] {
        me::Engine& e = engine_at(g, engine_index);
        prism::EngineDeviceOptions o;
        if (opts) {
            if (opts->table_capacity > 0) o.table_capacity = opts->table_capacity;
            if (opts->max_decode_batch > 0) o.max_decode_batch = opts->max_decode_batch;
            if (opts->max_step_tokens > 0) o.max_step_tokens = opts->max_step_tokens;
        }
        prism::attach_engine_device(e, g->g.ledger, o);
    });
}

int prism_engine_step_info(const prism_gpu* g, int engine_index, int32_t* n_step_tokens, int32_t* n_decodes) {
    return dguard([&] {
        const me::Engine& e = engine_at(g, engine_index);
        if (n_step_tokens) *n_step_tokens = prism::last_step_tokens(e);
        if (n_decodes) *n_decodes = prism::last_step_decodes(e);
    });
}

int prism_engine_step_decode_ids(const prism_gpu* g, int engine_index, uint64_t* out, size_t cap, size_t* n) {
    return dguard([&] {
        const auto& ids = prism::last_step_decode_ids(engine_at(g, engine_index));
        if (n) *n = ids.size();
        if (out) {
            if (ids.size() > cap) throw std::invalid_argument("output buffer too small");
            std::copy(ids.begin(), ids.end(), out);
        }
    });
}

int prism_engine_step_slots(const prism_gpu* g, int engine_index, int32_t* out, size_t cap, size_t* n) {
    return dguard([&] {
        const auto v = prism::last_step_slots(engine_at(g, engine_index));
        if (n) *n = v.size();
        if (out) {
            if (v.size() > cap) throw std::invalid_argument("output buffer too small");
            std::copy(v.begin(), v.end(), out);
        }
    });
}

int prism_engine_table_row(const prism_gpu* g, int engine_index, int64_t row, int32_t len, int32_t* out) {
    return dguard([&] {
        need(out, "out");
        const auto v = prism::read_table_row(engine_at(g, engine_index), row, len);
        std::copy(v.begin(), v.end(), out);
    });
}

int prism_engine_append_kv(prism_gpu* g, int engine_index, int layer_begin, int layer_end, const void* k,
                           const void* v) {
    return dguard([&] {
        need(k, "k");
        need(v, "v");
        prism::append_step_kv(engine_at(g, engine_index), layer_begin, layer_end, k, v);
    });
}

int prism_engine_append_kv_synthetic(prism_gpu* g, int engine_index, int layer_begin, int layer_end, uint64_t seed) {
    return dguard([&] { prism::append_step_kv_synthetic(engine_at(g, engine_index), layer_begin, layer_end, seed); });
}

}  // extern "C"

namespace prism {
void launch_decode_attention(class EngineDeviceImpl& d, int layer, const void* q, void* out, float scale, int chunk);
int k4_debug_read(unsigned* out, int n);
int k4_trace_read(unsigned long long* out, int n);
int k3_trace_read(unsigned long long* out, int n);
EngineDeviceImpl& impl_of(const msim::engine::Engine& eng);
void set_attention_variant(int v);
}  // namespace prism

extern "C" {

int prism_engine_decode_attention(prism_gpu* g, int engine_index, int layer, const void* q, void* out, float scale,
                                  int32_t chunk) {
    return dguard([&] {
        need(q, "q");
        need(out, "out");
        prism::launch_decode_attention(prism::impl_of(engine_at(g, engine_index)), layer, q, out, scale, chunk);
    });
}

int prism_engine_prefill_info(const prism_gpu* g, int engine_index, int32_t* n_tokens, int32_t* first,
                              uint64_t* request) {
    return dguard([&] {
        const me::Engine& e = engine_at(g, engine_index);
        if (n_tokens) *n_tokens = prism::last_step_prefill_tokens(e);
        if (first) *first = prism::last_step_prefill_first(e);
        if (request) *request = prism::last_step_prefill_request(e);
    });
}

int prism_engine_prefill_attention(prism_gpu* g, int engine_index, int layer, const void* q, void* out, float scale) {
    return dguard([&] {
        need(q, "q");
        need(out, "out");
        prism::prefill_attention(engine_at(g, engine_index), layer, q, out, scale);
    });
}

int prism_debug_k4_progress(uint32_t* out, int32_t n, int32_t* got) {
    return dguard([&] {
        need(out, "out");
        const int m = prism::k4_debug_read(out, n);
        if (got) *got = m;
    });
}

int prism_debug_k3_trace(uint64_t* out, int32_t n, int32_t* got) {
    return dguard([&] {
        need(out, "out");
        const int m = prism::k3_trace_read(reinterpret_cast<unsigned long long*>(out), n);
        if (got) *got = m;
    });
}

int prism_debug_k4_trace(uint64_t* out, int32_t n, int32_t* got) {
    return dguard([&] {
        need(out, "out");
        const int m = prism::k4_trace_read(reinterpret_cast<unsigned long long*>(out), n);
        if (got) *got = m;
    });
}

int prism_set_attention_variant(int variant) {
    return dguard([&] {
        if (variant < 0 || variant > 3) throw std::invalid_argument("attention variant must be 0..3");
        prism::set_attention_variant(variant);
    });
}

int prism_engine_synth_q(prism_gpu* g, int engine_index, int layer, uint64_t seed, float q_scale, void* q) {
    return dguard([&] {
        need(q, "q");
        prism::synth_decode_q(engine_at(g, engine_index), layer, seed, q_scale, q);
    });
}

int prism_engine_decode_host(prism_gpu* g, int engine_index, const void* new_k, const void* new_v, const void* q,
                             void* out, float scale) {
    return dguard([&] {
        need(q, "q");
        need(out, "out");
        prism::decode_host(engine_at(g, engine_index), new_k, new_v, q, out, scale, /*wait=*/true);
    });
}

int prism_engine_decode_host_async(prism_gpu* g, int engine_index, const void* new_k, const void* new_v,
                                   const void* q, void* out, float scale) {
    return dguard([&] {
        need(q, "q");
        need(out, "out");
        prism::decode_host(engine_at(g, engine_index), new_k, new_v, q, out, scale, /*wait=*/false);
    });
}

int prism_engine_wait_host(prism_gpu* g, int engine_index) {
    return dguard([&] { prism::wait_host(engine_at(g, engine_index)); });
}

int prism_engine_synchronize(prism_gpu* g, int engine_index) {
    return dguard([&] {
        auto stream = static_cast<cudaStream_t>(prism::engine_stream(engine_at(g, engine_index)));
        check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
    });
}

}  // extern "C"

// ---------------------------------------------------------------- weight loading (§8f-2)

struct prism_wloader {
    std::unique_ptr<prism::WeightLoader> w;
};

namespace {
struct DevSet {
    int prev = 0;
    explicit DevSet(int d) {
        if (cudaGetDevice(&prev) != cudaSuccess) throw std::runtime_error("cudaGetDevice failed");
        if (cudaSetDevice(d) != cudaSuccess) throw std::runtime_error("cudaSetDevice failed");
    }
    ~DevSet() { cudaSetDevice(prev); }
};
void rt_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

int prism_wloader_create(int device, int n_streams, uint64_t chunk_bytes, prism_wloader** out) {
    return dguard([&] {
        need(out, "out");
        auto h = std::make_unique<prism_wloader>();
        h->w = std::make_unique<prism::WeightLoader>(device, n_streams, static_cast<std::size_t>(chunk_bytes));
        *out = h.release();
    });
}

int prism_wloader_destroy(prism_wloader* w) {
    return dguard([&] { delete w; });
}

int prism_wloader_load(prism_wloader* w, const void* host, void* dst, uint64_t bytes) {
    return dguard([&] {
        need(w, "loader");
        w->w->load(host, dst, static_cast<std::size_t>(bytes));
    });
}

int prism_wloader_load_naive(prism_wloader* w, const void* host, void* dst, uint64_t bytes) {
    return dguard([&] {
        need(w, "loader");
        w->w->load_naive(host, dst, static_cast<std::size_t>(bytes));
    });
}

int prism_wloader_load_part(prism_wloader* w, const void* host, void* dst, uint64_t bytes, int part, int n_parts) {
    return dguard([&] {
        need(w, "loader");
        w->w->load_part(host, dst, static_cast<std::size_t>(bytes), part, n_parts);
    });
}

int prism_wloader_wait(prism_wloader* w, double* ms) {
    return dguard([&] {
        need(w, "loader");
        const double t = w->w->wait();
        if (ms) *ms = t;
    });
}

int prism_host_register(void* host, uint64_t bytes) {
    return dguard([&] {
        need(host, "host");
        rt_check(cudaHostRegister(host, static_cast<std::size_t>(bytes), cudaHostRegisterDefault), "cudaHostRegister");
    });
}

int prism_host_unregister(void* host) {
    return dguard([&] {
        need(host, "host");
        rt_check(cudaHostUnregister(host), "cudaHostUnregister");
    });
}

int prism_ipc_handle(const void* dptr, void* handle64) {
    return dguard([&] {
        need(dptr, "dptr");
        need(handle64, "handle");
        cudaIpcMemHandle_t h;
        rt_check(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)), "cudaIpcGetMemHandle");
        static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
        std::memcpy(handle64, &h, sizeof(h));
    });
}

int prism_ipc_open(int device, const void* handle64, void** dptr) {
    return dguard([&] {
        need(handle64, "handle");
        need(dptr, "dptr");
        DevSet g(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        rt_check(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

int prism_ipc_close(int device, void* dptr) {
    return dguard([&] {
        need(dptr, "dptr");
        DevSet g(device);
        rt_check(cudaIpcCloseMemHandle(dptr), "cudaIpcCloseMemHandle");
    });
}

}  // extern "C"

// ---------------------------------------------------------------- pool-level K2 / K3

struct prism_paged {
    std::unique_ptr<prism::PagedOp> op;
};

extern "C" {

int prism_paged_create(const prism_pool* p, int n_layers, int n_q_heads, int n_kv_heads, int head_dim,
                       prism_paged** out) {
    return dguard([&] {
        need(p, "pool");
        need(out, "out");
        auto h = std::make_unique<prism_paged>();
        h->op = prism::make_paged_op(p->pool, n_layers, n_q_heads, n_kv_heads, head_dim);
        *out = h.release();
    });
}

int prism_paged_destroy(prism_paged* pa) {
    return dguard([&] { delete pa; });
}

int prism_paged_kv_append(prism_paged* pa, int layer_begin, int layer_end, const int32_t* slots, int32_t n_tokens,
                          const void* k, const void* v) {
    return dguard([&] {
        need(pa, "paged");
        pa->op->kv_append(layer_begin, layer_end, slots, n_tokens, k, v);
    });
}

int prism_paged_prefill_attention(prism_paged* pa, int layer, const int32_t* slot_ids, int32_t first, int32_t n_tokens,
                                  const void* q, void* out, float scale) {
    return dguard([&] {
        need(pa, "paged");
        pa->op->prefill_attention(layer, slot_ids, first, n_tokens, q, out, scale);
    });
}

int prism_paged_decode_attention(prism_paged* pa, int layer, const int32_t* seq_offsets, int32_t n_seqs,
                                 const int32_t* slot_ids, const void* q, void* out, float scale) {
    return dguard([&] {
        need(pa, "paged");
        pa->op->decode_attention(layer, seq_offsets, n_seqs, slot_ids, q, out, scale);
    });
}

int prism_sim_run_device(const prism_sim_config* cfg, const prism_model_spec* specs, const double* rates,
                         size_t n_models, const prism_trace_event* trace, size_t n_trace,
                         const prism_serving_options* opts, prism_sim** out) {
    return dguard([&] {
        need(out, "out");
        prism::ServingOptions o;
        std::vector<int> ordinals{0};
        if (opts) {
            o.measured = opts->measured != 0;
            if (opts->seed) o.seed = opts->seed;
            if (opts->ordinals && opts->n_ordinals) ordinals.assign(opts->ordinals, opts->ordinals + opts->n_ordinals);
            if (opts->owned && opts->n_owned) o.owned.assign(opts->owned, opts->owned + opts->n_owned);
            if (opts->max_decode_batch > 0) o.max_decode_batch = opts->max_decode_batch;
            o.chunk_pages = opts->chunk_pages;
        }
        auto sim = std::make_unique<prism_sim>();
        const auto t0 = std::chrono::steady_clock::now();
        prism::DeviceExecutor ex(ordinals, o);
        prism_capi_detail::sim_run(cfg, specs, rates, n_models, trace, n_trace, &ex, sim.get());
        ex.synchronize();
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const prism::ServingStats& st = ex.stats();
        const prism::VmmStats v = ex.vmm_stats();
        sim->device = true;
        sim->serving = prism_serving_stats{st.iterations, st.attached, st.detached, st.k2_launches, st.k3_launches,
                                           st.k4_launches, st.decode_tokens, st.prefill_tokens, st.gpu_us,
                                           st.modelled_us, v.maps, v.unmaps, v.revived, v.creates,
                                           v.driver_unmaps, v.steals, v.urgent,
                                           v.map_ns_total + v.unmap_ns_total, v.background_ns_total, wall};
        *out = sim.release();
    });
}

}  // extern "C"
