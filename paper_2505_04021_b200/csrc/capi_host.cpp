// C-ABI (include/prism_capi.h), host subset: ledger, pools, engines,
// schedulers, traces.
//
// Written purely against the public msim:: C++ API of the reference
// (proj/include/msim/*.hpp), so the SAME file is compiled twice:
//   * against this repo's drop-in headers + runtime -> libprism_b200.so
//     (PRISM_PRODUCT defined; adds the fields only the product has);
//   * against the reference's own headers + sources -> oracle/_ref/
//     libmsim_ref.so (the test oracle, built by oracle/Makefile).
// Parity tests therefore drive both libraries through identical calls.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "msim/admission.hpp"
#include "msim/engine.hpp"
#include "msim/errors.hpp"
#include "msim/pagealloc.hpp"
#include "msim/placement.hpp"
#include "msim/simcore.hpp"
#include "msim/workload.hpp"
#include "prism_capi.h"
#include "capi_handles.hpp"

namespace pa = msim::pagealloc;
namespace me = msim::engine;
namespace pl = msim::placement;
namespace ad = msim::admission;
namespace wl = msim::workload;
namespace sc = msim::simcore;

namespace prism_capi_detail {

thread_local std::string g_error;

void set_error(const char* what) { g_error = what ? what : ""; }

template <class F>
int guard(F&& f) {
    try {
        f();
        return PRISM_OK;
    } catch (const pl::PlacementError& e) {
        set_error(e.what());
        return PRISM_E_PLACEMENT;
    } catch (const msim::ParseError& e) {
        set_error(e.what());
        return PRISM_E_PARSE;
    } catch (const msim::ConfigError& e) {
        set_error(e.what());
        return PRISM_E_CONFIG;
    } catch (const msim::UsageError& e) {
        set_error(e.what());
        return PRISM_E_USAGE;
    } catch (const std::invalid_argument& e) {
        set_error(e.what());
        return PRISM_E_ARG;
    } catch (const std::out_of_range& e) {
        set_error(e.what());
        return PRISM_E_ARG;
    } catch (const std::runtime_error& e) {
        set_error(e.what());
        return PRISM_E_CUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return PRISM_E_INTERNAL;
    } catch (...) {
        set_error("unknown exception");
        return PRISM_E_INTERNAL;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}

void room(std::size_t have, std::size_t cap, const char* what) {
    if (have > cap) throw std::invalid_argument(std::string("output buffer too small: ") + what);
}

me::ModelSpec to_spec(const prism_model_spec& s) {
    me::ModelSpec m;
    m.model_id = s.model_id ? s.model_id : "";
    m.weight_bytes = s.weight_bytes;
    m.token_kv_bytes = s.token_kv_bytes;
    m.prefill_tps = s.prefill_tps;
    m.chunk_size = s.chunk_size;
    m.ttft_slo_s = s.ttft_slo_s;
    m.tpot_slo_s = s.tpot_slo_s;
    m.tp_degree = s.tp_degree;
#ifdef PRISM_PRODUCT
    m.n_layers = s.n_layers;
    m.n_q_heads = s.n_q_heads;
    m.n_kv_heads = s.n_kv_heads;
    m.head_dim = s.head_dim;
#endif
    return m;
}

me::EngineParams to_params(const prism_engine_params* p) {
    me::EngineParams e;
    if (!p) return e;
    e.alpha_ms = p->alpha_ms;
    e.beta_ms_per_token = p->beta_ms_per_token;
    e.map_latency_ms = p->map_latency_ms;
    e.engine_init_s = p->engine_init_s;
    e.realign_s = p->realign_s;
    e.reserve_frac = p->reserve_frac;
    return e;
}

me::Engine& engine_at(prism_gpu* g, int i) {
    need(g, "gpu");
    if (i < 0 || static_cast<std::size_t>(i) >= g->g.engines.size()) throw std::out_of_range("engine index");
    return g->g.engines[static_cast<std::size_t>(i)];
}
const me::Engine& engine_at(const prism_gpu* g, int i) { return engine_at(const_cast<prism_gpu*>(g), i); }

pl::GpuView to_view(const prism_gpu_view& v) {
    pl::GpuView g;
    g.gpu_id = v.gpu_id;
    g.capacity_bytes = v.capacity_bytes;
    g.weight_bytes = v.weight_bytes;
    g.w_req_rate = v.w_req_rate;
    g.capacity_pages = v.capacity_pages;
    g.free_pages = v.free_pages;
    g.page_bytes = v.page_bytes;
    for (int32_t i = 0; i < v.n_residents; ++i) {
        const prism_resident& r = v.residents[i];
        pl::ResidentModel m;
        m.idle_s = r.idle_s;
        m.ttft_slo_s = r.ttft_slo_s;
        m.weight_bytes = r.weight_bytes;
        m.weight_pages = r.weight_pages;
        g.residents[r.model_id] = m;
    }
    return g;
}

std::vector<pl::GpuView> to_views(const prism_gpu_view* v, std::size_t n) {
    std::vector<pl::GpuView> out;
    out.reserve(n);
    for (std::size_t i = 0; i < n; ++i) out.push_back(to_view(v[i]));
    return out;
}

ad::QueuedRequest to_req(const prism_queued_request& q) {
    ad::QueuedRequest r;
    r.id = q.id;
    r.model_id = q.model_id ? q.model_id : "";
    r.arrival_s = q.arrival_s;
    r.prompt_tokens = q.prompt_tokens;
    r.ttft_slo_s = q.ttft_slo_s;
    r.exec_estimate_s = q.exec_estimate_s;
    return r;
}

void to_event(const wl::TraceEvent& e, prism_trace_event& o) {
    o.arrival_s = e.arrival_s;
    std::memset(o.model_id, 0, sizeof(o.model_id));
    std::strncpy(o.model_id, e.model_id.c_str(), sizeof(o.model_id) - 1);
    o.prompt_tokens = e.prompt_tokens;
    o.output_tokens = e.output_tokens;
}

void emit_trace(const std::vector<wl::TraceEvent>& t, prism_trace_event* out, std::size_t cap, std::size_t* n) {
    need(n, "n");
    *n = t.size();
    if (!out) return;
    room(t.size(), cap, "trace");
    for (std::size_t i = 0; i < t.size(); ++i) to_event(t[i], out[i]);
}

}  // namespace prism_capi_detail

using namespace prism_capi_detail;

extern "C" {

int prism_abi_version(void) { return PRISM_ABI_VERSION; }
const char* prism_last_error(void) { return g_error.c_str(); }

void prism_default_engine_params(prism_engine_params* out) {
    if (!out) return;
    const me::EngineParams e;
    *out = prism_engine_params{e.alpha_ms, e.beta_ms_per_token, e.map_latency_ms, e.engine_init_s, e.realign_s,
                               e.reserve_frac};
}

void prism_default_model_spec(prism_model_spec* out) {
    if (!out) return;
    const me::ModelSpec s;
    std::memset(out, 0, sizeof(*out));
    out->model_id = "";
    out->prefill_tps = s.prefill_tps;
    out->chunk_size = s.chunk_size;
    out->ttft_slo_s = s.ttft_slo_s;
    out->tpot_slo_s = s.tpot_slo_s;
    out->tp_degree = s.tp_degree;
}

// ---------------------------------------------------------------- ledger

int prism_ledger_create(int gpu_id, uint64_t capacity_pages, uint64_t page_bytes, prism_ledger** out) {
    return guard([&] {
        need(out, "out");
        auto* h = new prism_ledger();
        try {
            h->owned = std::make_unique<pa::PhysicalLedger>(gpu_id, capacity_pages, page_bytes);
        } catch (...) {
            delete h;
            throw;
        }
        h->l = h->owned.get();
        *out = h;
    });
}

void prism_ledger_destroy(prism_ledger* l) {
    if (l && l->owned) delete l;
}

int prism_ledger_get_stats(const prism_ledger* l, prism_ledger_stats* out) {
    return guard([&] {
        need(l, "ledger");
        need(out, "out");
        const pa::PhysicalLedger& x = *l->l;
        *out = prism_ledger_stats{x.capacity_pages(), x.mapped_pages(), x.buffer_pages(), x.weight_pages(),
                                  x.free_pages(), x.page_bytes()};
    });
}

int prism_ledger_pool_mapped_pages(const prism_ledger* l, uint32_t pool_id, uint64_t* out) {
    return guard([&] {
        need(l, "ledger");
        need(out, "out");
        *out = l->l->pool_mapped_pages(pool_id);
    });
}

int prism_refill_buffer(prism_ledger* l, uint64_t target_pages, uint64_t* added) {
    return guard([&] {
        need(l, "ledger");
        const uint64_t a = pa::refill_buffer(*l->l, target_pages);
        if (added) *added = a;
    });
}

int prism_ledger_reserve_weights(prism_ledger* l, const char* model_id, uint64_t pages, int* ok) {
    return guard([&] {
        need(l, "ledger");
        need(model_id, "model_id");
        const bool r = l->l->reserve_weight_pages(model_id, pages);
        if (ok) *ok = r ? 1 : 0;
    });
}

int prism_ledger_release_weights(prism_ledger* l, const char* model_id) {
    return guard([&] {
        need(l, "ledger");
        need(model_id, "model_id");
        l->l->release_weight_pages(model_id);
    });
}

int prism_ledger_weight_pages_of(const prism_ledger* l, const char* model_id, uint64_t* out) {
    return guard([&] {
        need(l, "ledger");
        need(model_id, "model_id");
        need(out, "out");
        *out = l->l->weight_pages_of(model_id);
    });
}

int prism_ledger_set_time(prism_ledger* l, int64_t now_us) {
    return guard([&] {
        need(l, "ledger");
        l->l->set_time(now_us);
    });
}

int prism_ledger_set_recording(prism_ledger* l, int on) {
    return guard([&] {
        need(l, "ledger");
        l->l->set_recording(on != 0);
    });
}

int prism_ledger_events(const prism_ledger* l, prism_event* out, size_t cap, size_t* n) {
    return guard([&] {
        need(l, "ledger");
        need(n, "n");
        const auto& ev = l->l->events();
        *n = ev.size();
        if (!out) return;
        room(ev.size(), cap, "events");
        for (std::size_t i = 0; i < ev.size(); ++i) {
            prism_event& o = out[i];
            o.time_us = ev[i].time_us;
            o.gpu_id = ev[i].gpu_id;
            o.kind = static_cast<int32_t>(ev[i].kind);
            o.pages = ev[i].pages;
            std::memset(o.model_id, 0, sizeof(o.model_id));
            std::strncpy(o.model_id, ev[i].model_id.c_str(), sizeof(o.model_id) - 1);
        }
    });
}

int prism_ledger_clear_events(prism_ledger* l) {
    return guard([&] {
        need(l, "ledger");
        l->l->clear_events();
    });
}

int prism_ledger_check_invariants(const prism_ledger* l) {
    return guard([&] {
        need(l, "ledger");
        l->l->check_invariants();
    });
}

// ---------------------------------------------------------------- pools

int prism_kvcache_alloc(prism_ledger* l, const char* model_id, uint64_t token_bytes, uint64_t virtual_pages,
                        int placement, prism_pool** out) {
    return guard([&] {
        need(l, "ledger");
        need(model_id, "model_id");
        need(out, "out");
        const auto pp = placement == 1 ? pa::PagePlacement::lowest_index_first : pa::PagePlacement::most_occupied_first;
        *out = new prism_pool(pa::alloc_kvcache(*l->l, model_id, token_bytes, virtual_pages, pp));
    });
}

int prism_kvcache_free(prism_ledger* l, prism_pool* p) {
    return guard([&] {
        need(l, "ledger");
        need(p, "pool");
        pa::free_kvcache(*l->l, p->pool);
    });
}

void prism_pool_destroy(prism_pool* p) { delete p; }

int prism_pool_info_get(const prism_pool* p, prism_pool_info* out) {
    return guard([&] {
        need(p, "pool");
        need(out, "out");
        const pa::KvPool& k = p->pool;
        out->id = k.id();
        out->alive = k.alive() ? 1 : 0;
        out->token_bytes = k.token_bytes();
        out->tokens_per_page = k.tokens_per_page();
        out->virtual_capacity_pages = k.virtual_capacity_pages();
        out->mapped_pages = k.mapped_pages();
        out->occupied_slots = k.occupied_slots();
#ifdef PRISM_PRODUCT
        out->device_base = k.device_base();
#else
        out->device_base = 0;
#endif
    });
}

int prism_kv_alloc(prism_pool* p, prism_ledger* l, uint64_t n, prism_slot* out, prism_alloc_result* res) {
    return guard([&] {
        need(p, "pool");
        need(l, "ledger");
        pa::AllocResult r = pa::alloc_kv(p->pool, *l->l, n);
        if (res) *res = prism_alloc_result{r.shortfall_pages, r.pages_mapped, r.buffer_hits, r.handles.size()};
        if (!r.handles.empty()) {
            need(out, "out");
            for (std::size_t i = 0; i < r.handles.size(); ++i) {
                out[i] = prism_slot{r.handles[i].pool, r.handles[i].page, r.handles[i].slot};
            }
        }
    });
}

int prism_kv_free(prism_pool* p, prism_ledger* l, const prism_slot* handles, size_t n) {
    return guard([&] {
        need(p, "pool");
        need(l, "ledger");
        if (n) need(handles, "handles");
        std::vector<pa::TokenSlotHandle> hs(n);
        for (std::size_t i = 0; i < n; ++i) hs[i] = pa::TokenSlotHandle{handles[i].pool, handles[i].page, handles[i].slot};
        pa::free_kv(p->pool, *l->l, hs);
    });
}

int prism_pool_allocatable_tokens(const prism_pool* p, const prism_ledger* l, uint64_t* out) {
    return guard([&] {
        need(p, "pool");
        need(l, "ledger");
        need(out, "out");
        *out = p->pool.allocatable_tokens(*l->l);
    });
}

int prism_pool_page_occupied(const prism_pool* p, uint32_t page, uint64_t* out) {
    return guard([&] {
        need(p, "pool");
        need(out, "out");
        *out = p->pool.page_occupied(page);
    });
}

int prism_pool_page_mapped(const prism_pool* p, uint32_t page, int* out) {
    return guard([&] {
        need(p, "pool");
        need(out, "out");
        *out = p->pool.page_mapped(page) ? 1 : 0;
    });
}

int prism_pool_set_cap(prism_pool* p, int64_t cap) {
    return guard([&] {
        need(p, "pool");
        if (cap < 0) {
            p->pool.set_mapped_page_cap(std::nullopt);
        } else {
            p->pool.set_mapped_page_cap(static_cast<std::uint64_t>(cap));
        }
    });
}

// ---------------------------------------------------------------- engines

int prism_gpu_create(int gpu_id, uint64_t capacity_pages, uint64_t page_bytes, prism_gpu** out) {
    return guard([&] {
        need(out, "out");
        *out = new prism_gpu(gpu_id, capacity_pages, page_bytes);
    });
}

void prism_gpu_destroy(prism_gpu* g) { delete g; }

prism_ledger* prism_gpu_ledger(prism_gpu* g) { return g ? &g->view : nullptr; }

int prism_gpu_engine_count(const prism_gpu* g, int* out) {
    return guard([&] {
        need(g, "gpu");
        need(out, "out");
        *out = static_cast<int>(g->g.engines.size());
    });
}

int prism_gpu_activate(prism_gpu* g, const prism_model_spec* spec, int method, const prism_engine_params* params,
                       prism_activation* out, int* ok) {
    return guard([&] {
        need(g, "gpu");
        need(spec, "spec");
        const me::ActivationParams act;
        const auto m = method == 0 ? me::ActivationMethod::naive : me::ActivationMethod::parallel;
        const auto r = me::activate(g->g, to_spec(*spec), m, act, to_params(params));
        if (ok) *ok = r.has_value() ? 1 : 0;
        if (r && out) *out = prism_activation{r->engine_index, r->init_us, r->realign_us, r->load_us};
        if (g->last.size() < g->g.engines.size()) g->last.resize(g->g.engines.size());
    });
}

int prism_gpu_finish_activation(prism_gpu* g, int engine_index) {
    return guard([&] {
        need(g, "gpu");
        me::finish_activation(g->g, engine_index);
    });
}

int prism_gpu_deactivate(prism_gpu* g, int engine_index) {
    return guard([&] {
        need(g, "gpu");
        me::deactivate(g->g, engine_index);
    });
}

int prism_engine_status(const prism_gpu* g, int engine_index, int* status) {
    return guard([&] {
        need(status, "status");
        *status = static_cast<int>(engine_at(g, engine_index).status);
    });
}

int prism_engine_push(prism_gpu* g, int engine_index, uint64_t id, int prompt_tokens, int output_tokens) {
    return guard([&] {
        me::EngineRequest r;
        r.id = id;
        r.prompt_tokens = prompt_tokens;
        r.output_tokens = output_tokens;
        engine_at(g, engine_index).local_queue.push_back(std::move(r));
    });
}

int prism_engine_step(prism_gpu* g, int engine_index, const prism_engine_params* params, int64_t now_us,
                      prism_outcome* out) {
    return guard([&] {
        me::Engine& e = engine_at(g, engine_index);
        std::vector<pa::PhysicalLedger*> ledgers(e.pools.size(), &g->g.ledger);
        me::IterationOutcome o = me::step(e, ledgers, to_params(params), now_us);
        if (out) {
            *out = prism_outcome{o.duration_us,
                                 o.chunk_tokens,
                                 o.decode_tokens,
                                 o.pages_mapped_direct,
                                 o.prefill_paused ? 1 : 0,
                                 static_cast<uint32_t>(o.first_tokens.size()),
                                 static_cast<uint32_t>(o.completions.size()),
                                 static_cast<uint32_t>(o.preemptions.size())};
        }
        if (g->last.size() < g->g.engines.size()) g->last.resize(g->g.engines.size());
        g->last[static_cast<std::size_t>(engine_index)] = std::move(o);
    });
}

int prism_engine_outcome_ids(const prism_gpu* g, int engine_index, int which, uint64_t* out, size_t cap, size_t* n) {
    return guard([&] {
        engine_at(g, engine_index);
        need(n, "n");
        if (static_cast<std::size_t>(engine_index) >= g->last.size()) throw std::out_of_range("no step yet");
        const me::IterationOutcome& o = g->last[static_cast<std::size_t>(engine_index)];
        const std::vector<std::uint64_t>& v = which == 0 ? o.first_tokens : which == 1 ? o.completions : o.preemptions;
        *n = v.size();
        if (!out) return;
        room(v.size(), cap, "ids");
        std::copy(v.begin(), v.end(), out);
    });
}

int prism_engine_counts(const prism_gpu* g, int engine_index, size_t* batch, size_t* queue) {
    return guard([&] {
        const me::Engine& e = engine_at(g, engine_index);
        if (batch) *batch = e.batch.size();
        if (queue) *queue = e.local_queue.size();
    });
}

int prism_engine_request(const prism_gpu* g, int engine_index, int where, size_t index, prism_request_info* out) {
    return guard([&] {
        need(out, "out");
        const me::Engine& e = engine_at(g, engine_index);
        const me::EngineRequest* r = nullptr;
        if (where == 0) {
            if (index >= e.batch.size()) throw std::out_of_range("batch index");
            r = &e.batch[index];
        } else {
            if (index >= e.local_queue.size()) throw std::out_of_range("queue index");
            r = &e.local_queue[index];
        }
        out->id = r->id;
        out->prompt_tokens = r->prompt_tokens;
        out->output_tokens = r->output_tokens;
        out->prompt_done = r->prompt_done;
        out->generated = r->generated;
        out->admit_seq = r->admit_seq;
        out->n_slots = r->kv.empty() ? 0 : r->kv[0].size();
#ifdef PRISM_PRODUCT
        out->table_row = r->table_row;
#else
        out->table_row = -1;
#endif
    });
}

int prism_engine_request_kv(const prism_gpu* g, int engine_index, uint64_t request_id, prism_slot* out, size_t cap,
                            size_t* n) {
    return guard([&] {
        need(n, "n");
        const me::Engine& e = engine_at(g, engine_index);
        const auto it = std::find_if(e.batch.begin(), e.batch.end(),
                                     [&](const me::EngineRequest& r) { return r.id == request_id; });
        if (it == e.batch.end()) throw std::out_of_range("request not in batch");
        const auto& kv = it->kv.empty() ? std::vector<pa::TokenSlotHandle>{} : it->kv[0];
        *n = kv.size();
        if (!out) return;
        room(kv.size(), cap, "kv");
        for (std::size_t i = 0; i < kv.size(); ++i) out[i] = prism_slot{kv[i].pool, kv[i].page, kv[i].slot};
    });
}

int prism_engine_mapped_pages(const prism_gpu* g, int engine_index, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = engine_at(g, engine_index).mapped_pages();
    });
}

int prism_engine_next_chunk_need(const prism_gpu* g, int engine_index, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = engine_at(g, engine_index).next_chunk_need();
    });
}

int prism_engine_has_runnable_work(const prism_gpu* g, int engine_index, int* out) {
    return guard([&] {
        need(out, "out");
        const me::Engine& e = engine_at(g, engine_index);
        std::vector<pa::PhysicalLedger*> ledgers(e.pools.size(), const_cast<pa::PhysicalLedger*>(&g->g.ledger));
        *out = e.has_runnable_work(ledgers) ? 1 : 0;
    });
}

int prism_engine_reserved_pages(const prism_gpu* g, int engine_index, double reserve_frac, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = engine_at(g, engine_index).reserved_pages(reserve_frac);
    });
}

int prism_throughput_of(uint64_t kv_budget_bytes, const prism_model_spec* spec, int prompt_tokens, int output_tokens,
                        const prism_engine_params* params, uint64_t page_bytes, double warmup_s, double window_s,
                        double* tokens_per_s, int* max_batch) {
    return guard([&] {
        need(spec, "spec");
        me::ThroughputMix mix;
        mix.prompt_tokens = prompt_tokens;
        mix.output_tokens = output_tokens;
        const me::ThroughputResult r =
            me::throughput_of(kv_budget_bytes, to_spec(*spec), mix, to_params(params), page_bytes, warmup_s, window_s);
        if (tokens_per_s) *tokens_per_s = r.tokens_per_s;
        if (max_batch) *max_batch = r.max_batch;
    });
}

// ---------------------------------------------------------------- placement

int prism_kvpr(double w_req_rate, double shared_kv_bytes, double* out) {
    return guard([&] {
        need(out, "out");
        *out = pl::kvpr(w_req_rate, shared_kv_bytes);
    });
}

int prism_place_models(const prism_model_demand* models, size_t n_models, const prism_gpu_view* gpus, size_t n_gpus,
                       double tau_per_gb, int32_t* assignment, size_t assignment_cap, double* kvpr_before,
                       double* kvpr_after, prism_migration* migrations, size_t migrations_cap, prism_plan_info* info) {
    return guard([&] {
        if (n_models) need(models, "models");
        if (n_gpus) need(gpus, "gpus");
        std::vector<pl::ModelDemand> ms;
        for (std::size_t i = 0; i < n_models; ++i) {
            pl::ModelDemand d;
            d.spec = to_spec(models[i].spec);
            d.rate = models[i].rate;
            for (int32_t k = 0; k < models[i].n_current; ++k) d.current_gpus.push_back(models[i].current_gpus[k]);
            ms.push_back(std::move(d));
        }
        const pl::PlacementPlan plan = pl::place_models(ms, to_views(gpus, n_gpus), tau_per_gb);
        std::size_t off = 0;
        for (std::size_t i = 0; i < ms.size(); ++i) {
            const auto it = plan.assignment.find(ms[i].spec.model_id);
            const std::size_t tp = static_cast<std::size_t>(std::max(1, ms[i].spec.tp_degree));
            for (std::size_t k = 0; k < tp; ++k) {
                if (assignment) {
                    room(off + 1, assignment_cap, "assignment");
                    assignment[off] = it != plan.assignment.end() && k < it->second.size() ? it->second[k] : -1;
                }
                ++off;
            }
        }
        for (std::size_t gi = 0; gi < n_gpus; ++gi) {
            if (kvpr_before) kvpr_before[gi] = plan.kvpr_before[gi];
            if (kvpr_after) kvpr_after[gi] = plan.kvpr_after[gi];
        }
        if (migrations) {
            room(plan.migrations.size(), migrations_cap, "migrations");
            for (std::size_t k = 0; k < plan.migrations.size(); ++k) {
                const pl::Migration& mg = plan.migrations[k];
                int32_t idx = -1;
                for (std::size_t i = 0; i < ms.size(); ++i) {
                    if (ms[i].spec.model_id == mg.model_id) {
                        idx = static_cast<int32_t>(i);
                        break;
                    }
                }
                migrations[k] = prism_migration{idx, mg.part_index, mg.from_gpu, mg.to_gpu};
            }
        }
        if (info) {
            *info = prism_plan_info{plan.max_kvpr_after, plan.critical_gpu, plan.critical_shared_before_bytes,
                                    plan.critical_last_weight_bytes, static_cast<uint32_t>(plan.migrations.size())};
        }
    });
}

int prism_eviction_tick(const prism_gpu_view* gpus, size_t n_gpus, double idle_threshold_s, uint64_t min_free_pages,
                        int32_t* out_pairs, size_t cap, size_t* n) {
    return guard([&] {
        need(n, "n");
        const auto views = to_views(gpus, n_gpus);
        const auto ev = pl::eviction_tick(views, idle_threshold_s,
                                          [&](const pl::GpuView& g) { return g.free_pages < min_free_pages; });
        *n = ev.size();
        if (!out_pairs) return;
        room(ev.size() * 2, cap, "evictions");
        for (std::size_t k = 0; k < ev.size(); ++k) {
            int32_t gi = -1, ri = -1;
            for (std::size_t i = 0; i < n_gpus; ++i) {
                if (gpus[i].gpu_id != ev[k].gpu_id) continue;
                gi = static_cast<int32_t>(i);
                for (int32_t r = 0; r < gpus[i].n_residents; ++r) {
                    if (ev[k].model_id == gpus[i].residents[r].model_id) ri = r;
                }
                break;
            }
            out_pairs[2 * k] = gi;
            out_pairs[2 * k + 1] = ri;
        }
    });
}

int prism_activate_on_arrival(const prism_model_spec* spec, const prism_gpu_view* gpus, size_t n_gpus, int32_t* gpu,
                              int* found) {
    return guard([&] {
        need(spec, "spec");
        const auto r = pl::activate_on_arrival(to_spec(*spec), to_views(gpus, n_gpus));
        if (found) *found = r ? 1 : 0;
        if (gpu) *gpu = r ? *r : -1;
    });
}

int prism_activate_on_arrival_tp(const prism_model_spec* spec, const prism_gpu_view* gpus, size_t n_gpus,
                                 int32_t* out, size_t cap, int* found) {
    return guard([&] {
        need(spec, "spec");
        const auto r = pl::activate_on_arrival_tp(to_spec(*spec), to_views(gpus, n_gpus));
        if (found) *found = r ? 1 : 0;
        if (r && out) {
            room(r->size(), cap, "gpus");
            std::copy(r->begin(), r->end(), out);
        }
    });
}

// ---------------------------------------------------------------- admission

int prism_moore_hodgson(const prism_queued_request* queue, size_t n, double now_s, int32_t* admit, size_t* n_admit,
                        int32_t* deferred, size_t* n_deferred) {
    return guard([&] {
        if (n) need(queue, "queue");
        std::vector<ad::QueuedRequest> q;
        for (std::size_t i = 0; i < n; ++i) q.push_back(to_req(queue[i]));
        const ad::ScheduleDecision d = ad::moore_hodgson(q, now_s);
        // Report positions in the input; ids are unique per queue.
        auto index_of = [&](const ad::QueuedRequest& r) {
            for (std::size_t i = 0; i < n; ++i) {
                if (queue[i].id == r.id) return static_cast<int32_t>(i);
            }
            return int32_t{-1};
        };
        if (n_admit) *n_admit = d.admit.size();
        if (n_deferred) *n_deferred = d.deferred.size();
        if (admit) {
            for (std::size_t i = 0; i < d.admit.size(); ++i) admit[i] = index_of(d.admit[i]);
        }
        if (deferred) {
            for (std::size_t i = 0; i < d.deferred.size(); ++i) deferred[i] = index_of(d.deferred[i]);
        }
    });
}

int prism_dispatch(const prism_queued_request* reqs, const int32_t* admit, size_t n_admit, prism_dispatch_gate gate,
                   void* ctx, uint64_t* dispatched, size_t* n_dispatched) {
    return guard([&] {
        if (!gate) throw std::invalid_argument("null argument: gate");
        ad::ScheduleDecision d;
        std::vector<const prism_queued_request*> src;
        for (std::size_t i = 0; i < n_admit; ++i) {
            d.admit.push_back(to_req(reqs[admit[i]]));
            src.push_back(&reqs[admit[i]]);
        }
        const auto ids = ad::dispatch(d, [&](const ad::QueuedRequest& r) {
            for (const prism_queued_request* p : src) {
                if (p->id == r.id) return static_cast<ad::DispatchStatus>(gate(ctx, p));
            }
            return ad::DispatchStatus::model_unavailable;
        });
        if (n_dispatched) *n_dispatched = ids.size();
        if (dispatched) std::copy(ids.begin(), ids.end(), dispatched);
    });
}

int prism_requeue_deferred(const prism_queued_request* deferred, size_t n_deferred, const prism_queued_request* queue,
                           size_t n_queue, int32_t* out, size_t* n_out) {
    return guard([&] {
        std::vector<ad::QueuedRequest> d, q;
        for (std::size_t i = 0; i < n_deferred; ++i) d.push_back(to_req(deferred[i]));
        for (std::size_t i = 0; i < n_queue; ++i) q.push_back(to_req(queue[i]));
        const auto merged = ad::requeue_deferred(d, q);
        if (n_out) *n_out = merged.size();
        if (!out) return;
        for (std::size_t k = 0; k < merged.size(); ++k) {
            int32_t idx = -1;
            for (std::size_t i = 0; i < n_queue && idx < 0; ++i) {
                if (queue[i].id == merged[k].id) idx = static_cast<int32_t>(i);
            }
            for (std::size_t i = 0; i < n_deferred && idx < 0; ++i) {
                if (deferred[i].id == merged[k].id) idx = static_cast<int32_t>(n_queue + i);
            }
            out[k] = idx;
        }
    });
}

// ---------------------------------------------------------------- workload

int prism_synth_trace(const prism_model_profile* profiles, size_t n_profiles, uint64_t seed, prism_trace_event* out,
                      size_t cap, size_t* n) {
    return guard([&] {
        wl::SynthSpec spec;
        for (std::size_t i = 0; i < n_profiles; ++i) {
            wl::ModelProfile p;
            p.model_id = profiles[i].model_id ? profiles[i].model_id : "";
            for (int32_t k = 0; k < profiles[i].n_segments; ++k) {
                const prism_rate_segment& s = profiles[i].segments[k];
                p.segments.push_back(wl::RateSegment{s.start_s, s.end_s, s.rate_per_s});
            }
            p.prompt_median = profiles[i].prompt_median;
            p.prompt_sigma = profiles[i].prompt_sigma;
            p.output_median = profiles[i].output_median;
            p.output_sigma = profiles[i].output_sigma;
            spec.models.push_back(std::move(p));
        }
        emit_trace(wl::synth_trace(spec, seed), out, cap, n);
    });
}

int prism_scale_trace(const prism_trace_event* in, size_t n_in, int factor, uint64_t seed, double jitter_window_s,
                      prism_trace_event* out, size_t cap, size_t* n) {
    return guard([&] {
        std::vector<wl::TraceEvent> t;
        for (std::size_t i = 0; i < n_in; ++i) {
            t.push_back(wl::TraceEvent{in[i].arrival_s, in[i].model_id, in[i].prompt_tokens, in[i].output_tokens});
        }
        emit_trace(wl::scale_trace(t, factor, seed, jitter_window_s), out, cap, n);
    });
}

int prism_parse_trace_text(const char* text, const char* origin, prism_trace_event* out, size_t cap, size_t* n) {
    return guard([&] {
        need(text, "text");
        emit_trace(wl::parse_trace_lines(text, origin ? origin : "<mem>"), out, cap, n);
    });
}

}  // extern "C"

namespace prism_capi_detail {

void sim_run(const prism_sim_config* cfg, const prism_model_spec* specs, const double* rates, size_t n_models,
             const prism_trace_event* trace, size_t n_trace, sc::IterationExecutor* executor, prism_sim* sim) {
    need(cfg, "cfg");
    if (n_models) need(specs, "specs");
    if (n_trace) need(trace, "trace");
    sc::SimConfig c;
    if (cfg->policy < 0 || cfg->policy > 3) throw std::invalid_argument("prism_sim_run: unknown policy");
    c.policy = static_cast<sc::Policy>(cfg->policy);
    c.n_gpus = cfg->n_gpus;
    c.capacity_pages = cfg->capacity_pages;
    c.page_bytes = cfg->page_bytes;
    c.params = to_params(&cfg->params);
    c.method = cfg->method ? me::ActivationMethod::parallel : me::ActivationMethod::naive;
    const auto curve = [&](double gbs) {
        std::vector<std::pair<double, double>> c2;
        for (double b : {16e9, 28e9}) c2.emplace_back(b, cfg->load_fixed_s + b / (gbs * 1e9));
        return c2;
    };
    if (cfg->parallel_load_gbs > 0.0) c.activation.parallel_curve = curve(cfg->parallel_load_gbs);
    if (cfg->naive_load_gbs > 0.0) c.activation.naive_curve = curve(cfg->naive_load_gbs);
    c.tau_per_gb = cfg->tau_per_gb;
    c.tick_s = cfg->tick_s;
    c.idle_evict_s = cfg->idle_evict_s;
    c.pressure_free_frac = cfg->pressure_free_frac;
    c.buffer_target_pages = cfg->buffer_target_pages;
    c.initial_placement = cfg->initial_placement != 0;
    c.max_events = cfg->max_events;
    if (cfg->local_scheduler < 0 || cfg->local_scheduler > 1) {
        throw std::invalid_argument("prism_sim_run: unknown local scheduler");
    }
    c.local = static_cast<sc::LocalScheduler>(cfg->local_scheduler);
    c.executor = executor;
    for (std::size_t i = 0; i < n_models; ++i) {
        sc::ModelEntry m;
        m.spec = to_spec(specs[i]);
        m.rate = rates ? rates[i] : 0.0;
        sim->models.push_back(std::move(m));
    }
    std::vector<wl::TraceEvent> t;
    t.reserve(n_trace);
    for (std::size_t i = 0; i < n_trace; ++i) {
        t.push_back(wl::TraceEvent{trace[i].arrival_s, trace[i].model_id, trace[i].prompt_tokens,
                                   trace[i].output_tokens});
    }
    sim->metrics = sc::run(c, sim->models, t);
}

}  // namespace prism_capi_detail

extern "C" {

/* ------------------------------------------------------------------ simcore */

void prism_default_sim_config(prism_sim_config* out) {
    if (!out) return;
    const sc::SimConfig d;
    *out = prism_sim_config{};
    out->policy = static_cast<int32_t>(d.policy);
    out->n_gpus = d.n_gpus;
    out->capacity_pages = d.capacity_pages;
    out->page_bytes = d.page_bytes;
    prism_default_engine_params(&out->params);
    out->method = d.method == me::ActivationMethod::parallel ? 1 : 0;
    out->tau_per_gb = d.tau_per_gb;
    out->tick_s = d.tick_s;
    out->idle_evict_s = d.idle_evict_s;
    out->pressure_free_frac = d.pressure_free_frac;
    out->buffer_target_pages = d.buffer_target_pages;
    out->initial_placement = d.initial_placement ? 1 : 0;
    out->max_events = d.max_events;
    out->local_scheduler = static_cast<int32_t>(d.local);
}

int prism_sim_run(const prism_sim_config* cfg, const prism_model_spec* specs, const double* rates, size_t n_models,
                  const prism_trace_event* trace, size_t n_trace, prism_sim** out) {
    return guard([&] {
        need(out, "out");
        auto sim = std::make_unique<prism_sim>();
        prism_capi_detail::sim_run(cfg, specs, rates, n_models, trace, n_trace, nullptr, sim.get());
        *out = sim.release();
    });
}

int prism_sim_summary_get(const prism_sim* s, prism_sim_summary* out) {
    return guard([&] {
        need(s, "sim");
        need(out, "out");
        const sc::SimMetrics& m = s->metrics;
        *out = prism_sim_summary{};
        out->end_us = m.end_us;
        out->events = m.events;
        out->iterations = m.iterations;
        out->activations = m.activations;
        out->evictions = m.evictions;
        out->preemptions = m.preemptions;
        out->output_tokens = m.output_tokens;
        out->n_requests = m.requests.size();
        for (const auto& r : m.requests) out->completed += r.completion_us >= 0;
        out->truncated = m.truncated ? 1 : 0;
        out->dispatches = m.dispatches;
        out->schedule_rounds = m.schedule_rounds;
    });
}

int prism_sim_requests(const prism_sim* s, prism_sim_request* out, size_t cap, size_t* n) {
    return guard([&] {
        need(s, "sim");
        const auto& rs = s->metrics.requests;
        if (n) *n = rs.size();
        if (!out) return;
        room(rs.size(), cap, "requests");
        for (std::size_t i = 0; i < rs.size(); ++i) {
            out[i] = prism_sim_request{rs[i].id, rs[i].arrival_us, rs[i].first_token_us, rs[i].completion_us,
                                       rs[i].prompt_tokens, rs[i].output_tokens, rs[i].preemptions, rs[i].gpu};
        }
    });
}

int prism_sim_gpu_busy(const prism_sim* s, int64_t* out, size_t cap, size_t* n) {
    return guard([&] {
        need(s, "sim");
        const auto& b = s->metrics.gpu_busy_us;
        if (n) *n = b.size();
        if (!out) return;
        room(b.size(), cap, "gpu_busy");
        for (std::size_t i = 0; i < b.size(); ++i) out[i] = b[i];
    });
}

int prism_sim_attainment(const prism_sim* s, const char* model_id, double slo_scale, double* ttft, double* tpot,
                         double* both, uint64_t* n) {
    return guard([&] {
        need(s, "sim");
        const auto a = sc::attainment(s->metrics, s->models, slo_scale);
        const auto it = a.find(model_id ? model_id : "");
        if (it == a.end()) throw std::invalid_argument("prism_sim_attainment: no requests for that model");
        if (ttft) *ttft = it->second.ttft;
        if (tpot) *tpot = it->second.tpot;
        if (both) *both = it->second.both;
        if (n) *n = it->second.n;
    });
}

int prism_sim_serving_get(const prism_sim* s, prism_serving_stats* out) {
    return guard([&] {
        need(s, "sim");
        need(out, "out");
        if (!s->device) throw msim::UsageError("prism_sim_serving_get: the run did not drive the GPU data path");
        *out = s->serving;
    });
}

void prism_sim_free(prism_sim* s) { delete s; }

}  // extern "C"
