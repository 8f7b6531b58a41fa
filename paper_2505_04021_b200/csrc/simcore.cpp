// prism-b200 — simcore (include/msim/simcore.hpp): the deterministic
// discrete-event composition of engine::step, placement and the allocator
// that the reference specifies but does not implement.
// Only the public msim:: API is used, so this file also compiles against the
// reference's headers and sources (oracle/Makefile): both builds must yield
// identical metrics.
#include "msim/simcore.hpp"

#include <algorithm>
#include <array>
#include <deque>
#include <map>
#include <queue>
#include <string>
#include <tuple>
#include <vector>

#include "msim/admission.hpp"
#include "msim/defaults.hpp"
#include "msim/errors.hpp"
#include "msim/placement.hpp"

namespace msim::simcore {

namespace {

namespace me = msim::engine;
namespace pl = msim::placement;
namespace ad = msim::admission;

enum Kind : int { kArrival = 0, kIterationDone = 1, kActivationDone = 2, kSchedulerTick = 3 };

struct Event {
    SimTime t;
    int kind;
    std::uint64_t seq;
    std::int64_t a;  // arrival: trace index; iteration_done: gpu; activation_done: model index
    bool operator>(const Event& o) const { return std::tie(t, kind, seq) > std::tie(o.t, o.kind, o.seq); }
};

struct ModelState {
    int gpu = -1;       // GPU holding its engine (serving or loading), -1: none
    int engine = -1;
    bool loading = false;
    std::deque<std::size_t> waiting;  // trace indices not yet in the engine queue
    std::uint64_t outstanding = 0;    // arrived, not completed
    SimTime idle_since = 0;           // last time outstanding dropped to 0
};

struct Gpu {
    me::GpuState gs;
    bool busy = false;
    std::size_t rr = 0;  // next engine index the round robin looks at
    std::vector<ad::QueuedRequest> queue;  // Algorithm 2: the GPU's shared request queue (arrival order)
    Gpu(int id, std::uint64_t cap, std::uint64_t page) : gs(id, cap, page) {}
};

class Sim {
public:
    Sim(const SimConfig& cfg, const std::vector<ModelEntry>& models, const std::vector<workload::TraceEvent>& trace)
        : cfg_(cfg), models_(models), trace_(trace) {
        if (cfg.n_gpus < 1) throw UsageError("simcore: n_gpus must be >= 1");
        if (cfg.capacity_pages == 0 || cfg.page_bytes == 0) throw UsageError("simcore: empty GPU");
        for (std::size_t i = 0; i < models.size(); ++i) {
            const auto& s = models[i].spec;
            if (s.tp_degree != 1) throw UsageError("simcore: tp_degree != 1 is not supported: " + s.model_id);
            const std::uint64_t wp = (s.weight_bytes + cfg.page_bytes - 1) / cfg.page_bytes;
            if (wp >= cfg.capacity_pages) throw UsageError("simcore: model fits no GPU: " + s.model_id);
            if (!index_.emplace(s.model_id, i).second) throw UsageError("simcore: duplicate model " + s.model_id);
        }
        for (const auto& ev : trace) {
            if (!index_.count(ev.model_id)) throw UsageError("simcore: trace names an unknown model: " + ev.model_id);
        }
        for (int g = 0; g < cfg.n_gpus; ++g) gpus_.emplace_back(g, cfg.capacity_pages, cfg.page_bytes);
        if (cfg.executor) {
            for (Gpu& g : gpus_) cfg.executor->gpu_created(g.gs.gpu_id, g.gs);
        }
        state_.resize(models.size());
        cap_pages_.assign(models.size(), 0);
        m_.requests.resize(trace.size());
        m_.gpu_busy_us.assign(static_cast<std::size_t>(cfg.n_gpus), 0);
        for (std::size_t i = 0; i < trace.size(); ++i) {
            RequestRecord& r = m_.requests[i];
            r.id = i + 1;
            r.model_id = trace[i].model_id;
            r.arrival_us = seconds_to_us(trace[i].arrival_s);
            r.prompt_tokens = trace[i].prompt_tokens;
            r.output_tokens = trace[i].output_tokens;
            push(r.arrival_us, kArrival, static_cast<std::int64_t>(i));
        }
    }

    SimMetrics run() {
        if (cfg_.initial_placement && !models_.empty() && cfg_.policy != Policy::qlm_timeshare) place_all();
        if (!trace_.empty()) push(seconds_to_us(cfg_.tick_s), kSchedulerTick, 0);
        while (!q_.empty()) {
            if (m_.events >= cfg_.max_events) {
                m_.truncated = true;
                break;
            }
            const Event ev = q_.top();
            q_.pop();
            ++m_.events;
            now_ = ev.t;
            m_.end_us = now_;
            switch (ev.kind) {
                case kArrival: on_arrival(static_cast<std::size_t>(ev.a)); break;
                case kIterationDone: on_iteration_done(static_cast<int>(ev.a)); break;
                case kActivationDone: on_activation_done(static_cast<std::size_t>(ev.a)); break;
                case kSchedulerTick: on_tick(); break;
            }
        }
        return std::move(m_);
    }

private:
    void push(SimTime t, int kind, std::int64_t a) { q_.push(Event{t, kind, seq_++, a}); }

    // ------------------------------------------------------------ views
    std::vector<pl::GpuView> views() const {
        std::vector<pl::GpuView> out;
        for (const Gpu& g : gpus_) {
            pl::GpuView v;
            v.gpu_id = g.gs.gpu_id;
            v.capacity_pages = g.gs.ledger.capacity_pages();
            v.capacity_bytes = v.capacity_pages * cfg_.page_bytes;
            v.free_pages = g.gs.ledger.free_pages();
            v.page_bytes = cfg_.page_bytes;
            for (std::size_t i = 0; i < models_.size(); ++i) {
                const ModelState& s = state_[i];
                if (s.gpu != v.gpu_id) continue;
                const auto& spec = models_[i].spec;
                pl::ResidentModel r;
                r.idle_s = (s.outstanding == 0 && !s.loading) ? us_to_seconds(now_ - s.idle_since) : 0.0;
                r.ttft_slo_s = spec.ttft_slo_s;
                r.weight_bytes = spec.weight_bytes;
                r.weight_pages = (spec.weight_bytes + cfg_.page_bytes - 1) / cfg_.page_bytes;
                v.weight_bytes += spec.weight_bytes;
                v.w_req_rate += models_[i].rate / spec.ttft_slo_s;
                v.residents.emplace(spec.model_id, r);
            }
            out.push_back(std::move(v));
        }
        return out;
    }

    // ------------------------------------------------------------ activation
    bool start_activation(std::size_t mi, int gpu) {
        Gpu& g = gpus_[static_cast<std::size_t>(gpu)];
        const auto act = me::activate(g.gs, models_[mi].spec, cfg_.method, cfg_.activation, cfg_.params);
        if (!act) return false;
        ModelState& s = state_[mi];
        s.gpu = gpu;
        s.engine = act->engine_index;
        s.loading = true;
        ++m_.activations;
        push(now_ + act->total_us(), kActivationDone, static_cast<std::int64_t>(mi));
        return true;
    }

    void place_all() {
        std::vector<pl::ModelDemand> demand;
        for (const ModelEntry& m : models_) {
            pl::ModelDemand d;
            d.spec = m.spec;
            d.rate = m.rate;
            demand.push_back(d);
        }
        pl::PlacementPlan plan;
        try {
            plan = pl::place_models(demand, views(), cfg_.tau_per_gb);
        } catch (const pl::PlacementError& e) {
            // prism: not everything fits at once, models activate on arrival;
            // the frozen-colocation baselines need every model placed
            if (frozen()) throw UsageError(std::string("simcore: policy needs all models placed: ") + e.what());
            return;
        }
        for (std::size_t i = 0; i < models_.size(); ++i) {
            const auto it = plan.assignment.find(models_[i].spec.model_id);
            if (it == plan.assignment.end() || it->second.empty()) continue;
            if (!start_activation(i, it->second.front()) && frozen()) {
                throw UsageError("simcore: policy could not activate " + models_[i].spec.model_id);
            }
        }
        if (cfg_.policy == Policy::static_partition) {
            // equal share of each GPU's KV pages (capacity - weights - buffer)
            for (Gpu& g : gpus_) {
                std::uint64_t weights = 0, n = 0;
                for (std::size_t i = 0; i < models_.size(); ++i) {
                    if (state_[i].gpu != g.gs.gpu_id) continue;
                    weights += (models_[i].spec.weight_bytes + cfg_.page_bytes - 1) / cfg_.page_bytes;
                    ++n;
                }
                const std::uint64_t cap = g.gs.ledger.capacity_pages();
                const std::uint64_t kv = cap > weights + cfg_.buffer_target_pages
                                             ? cap - weights - cfg_.buffer_target_pages
                                             : 0;
                for (std::size_t i = 0; i < models_.size(); ++i) {
                    if (state_[i].gpu == g.gs.gpu_id) cap_pages_[i] = n ? kv / n : 0;
                }
            }
        }
    }

    bool frozen() const { return cfg_.policy != Policy::prism; }

    bool try_activate(std::size_t mi) {
        if (frozen()) return false;  // frozen colocation: no arrival-triggered activation
        const auto gpu = pl::activate_on_arrival(models_[mi].spec, views());
        return gpu && start_activation(mi, *gpu);
    }

    void on_activation_done(std::size_t mi) {
        ModelState& s = state_[mi];
        Gpu& g = gpus_[static_cast<std::size_t>(s.gpu)];
        me::finish_activation(g.gs, s.engine);
        if (cfg_.executor) cfg_.executor->attached(s.gpu, g.gs, s.engine);
        s.loading = false;
        me::Engine& e = g.gs.engines[static_cast<std::size_t>(s.engine)];
        if (cfg_.policy == Policy::static_partition) e.pools.front().set_mapped_page_cap(cap_pages_[mi]);
        while (!s.waiting.empty()) {
            admit(e, s.waiting.front(), s.gpu);
            s.waiting.pop_front();
        }
        schedule(s.gpu);
        wake(s.gpu);
    }

    // ------------------------------------------------------------ requests
    void enqueue(me::Engine& e, std::size_t ti, int gpu) {
        me::EngineRequest r;
        r.id = ti + 1;
        r.prompt_tokens = trace_[ti].prompt_tokens;
        r.output_tokens = trace_[ti].output_tokens;
        e.local_queue.push_back(std::move(r));
        m_.requests[ti].gpu = gpu;
    }

    bool algorithm2() const { return cfg_.policy == Policy::prism && cfg_.local == LocalScheduler::moore_hodgson; }

    // A request for a resident, serving model: Algorithm 2 queues it on its
    // GPU (dispatched by schedule()); FIFO hands it to the engine at once.
    void admit(me::Engine& e, std::size_t ti, int gpu) {
        if (!algorithm2()) {
            enqueue(e, ti, gpu);
            return;
        }
        const me::ModelSpec& spec = models_[index_.at(trace_[ti].model_id)].spec;
        ad::QueuedRequest q;
        q.id = ti + 1;
        q.model_id = spec.model_id;
        q.arrival_s = trace_[ti].arrival_s;
        q.prompt_tokens = trace_[ti].prompt_tokens;
        q.ttft_slo_s = spec.ttft_slo_s;
        q.exec_estimate_s = static_cast<double>(q.prompt_tokens) / me::effective_prefill_tps(spec, cfg_.params);
        gpus_[static_cast<std::size_t>(gpu)].queue.push_back(std::move(q));
        m_.requests[ti].gpu = gpu;
    }

    // Algorithm 2 on one GPU: Moore-Hodgson over the GPU's
    // queue, dispatch in deadline order through the immediately-runnable gate,
    // deferred requests merged back (never dropped).
    void schedule(int gpu) {
        if (!algorithm2()) return;
        Gpu& g = gpus_[static_cast<std::size_t>(gpu)];
        if (g.queue.empty()) return;
        ++m_.schedule_rounds;
        ad::ScheduleDecision d = ad::moore_hodgson(g.queue, us_to_seconds(now_));
        const std::vector<pagealloc::PhysicalLedger*> ledgers{&g.gs.ledger};
        const auto gate = [&](const ad::QueuedRequest& r) {
            const ModelState& s = state_[index_.at(r.model_id)];
            if (s.gpu != gpu || s.loading) return ad::DispatchStatus::model_unavailable;
            me::Engine& e = g.gs.engines[static_cast<std::size_t>(s.engine)];
            if (!e.serving()) return ad::DispatchStatus::model_unavailable;
            // no engine-local queuing: the engine's prefill pipeline must be empty
            if (!e.local_queue.empty()) return ad::DispatchStatus::engine_busy;
            for (const auto& b : e.batch) {
                if (b.prompt_done < b.prompt_tokens) return ad::DispatchStatus::engine_busy;
            }
            // KV headroom: the first chunk (next_chunk_need, reference
            // src/engine.cpp:63-78) plus the engine's reserved pages
            const int chunk = std::min(e.model->chunk_size, r.prompt_tokens);
            const std::uint64_t need = static_cast<std::uint64_t>(chunk) + (chunk == r.prompt_tokens ? 1 : 0);
            const pagealloc::KvPool& pool = e.pools.front();
            const std::uint64_t reserve = e.reserved_pages(cfg_.params.reserve_frac) * pool.tokens_per_page();
            if (pool.allocatable_tokens(*ledgers.front()) < need + reserve) return ad::DispatchStatus::no_memory;
            enqueue(e, static_cast<std::size_t>(r.id - 1), gpu);
            return ad::DispatchStatus::dispatched;
        };
        // No starvation: the admit list (every request in
        // it meets its deadline) goes first; the deferred ones — late under
        // any schedule that keeps the admitted on time — stay eligible and
        // follow in deadline order, so spare capacity still serves them.
        ad::ScheduleDecision all;
        all.now_s = d.now_s;
        all.admit = d.admit;
        std::vector<ad::QueuedRequest> late = d.deferred;
        std::sort(late.begin(), late.end(), [](const ad::QueuedRequest& a, const ad::QueuedRequest& b) {
            if (a.deadline_s() != b.deadline_s()) return a.deadline_s() < b.deadline_s();
            if (a.arrival_s != b.arrival_s) return a.arrival_s < b.arrival_s;
            return a.id < b.id;
        });
        all.admit.insert(all.admit.end(), late.begin(), late.end());
        const std::vector<std::uint64_t> sent = ad::dispatch(all, gate);
        m_.dispatches += sent.size();
        if (sent.empty()) return;
        std::vector<ad::QueuedRequest> rest;
        rest.reserve(d.admit.size());
        for (const ad::QueuedRequest& r : d.admit) {
            if (std::find(sent.begin(), sent.end(), r.id) == sent.end()) rest.push_back(r);
        }
        std::vector<ad::QueuedRequest> deferred;
        for (const ad::QueuedRequest& r : d.deferred) {
            if (std::find(sent.begin(), sent.end(), r.id) == sent.end()) deferred.push_back(r);
        }
        g.queue = ad::requeue_deferred(deferred, std::move(rest));
    }

    void on_arrival(std::size_t ti) {
        const std::size_t mi = index_.at(trace_[ti].model_id);
        ModelState& s = state_[mi];
        ++s.outstanding;
        if (s.gpu >= 0 && !s.loading) {
            admit(gpus_[static_cast<std::size_t>(s.gpu)].gs.engines[static_cast<std::size_t>(s.engine)], ti, s.gpu);
            schedule(s.gpu);
            wake(s.gpu);
            return;
        }
        s.waiting.push_back(ti);
        if (s.gpu < 0) {
            if (cfg_.policy == Policy::qlm_timeshare) {
                qlm_swap();
            } else {
                try_activate(mi);
            }
        }
    }

    // QLM time sharing: a GPU whose resident model has drained (or that has
    // none) takes the model of the oldest waiting request, paying engine init
    // + the naive weight load.
    void qlm_swap() {
        for (Gpu& g : gpus_) {
            int res = -1;
            for (std::size_t i = 0; i < models_.size(); ++i) {
                if (state_[i].gpu == g.gs.gpu_id) res = static_cast<int>(i);
            }
            if (res >= 0 && (state_[res].loading || state_[res].outstanding > 0)) continue;
            std::size_t best = models_.size(), oldest = 0;
            for (std::size_t i = 0; i < models_.size(); ++i) {
                const ModelState& c = state_[i];
                if (c.gpu >= 0 || c.waiting.empty()) continue;
                if (best == models_.size() || c.waiting.front() < oldest) {
                    best = i;
                    oldest = c.waiting.front();
                }
            }
            if (best == models_.size()) return;
            if (res >= 0) {
                ModelState& r = state_[res];
                if (cfg_.executor) cfg_.executor->detaching(g.gs.gpu_id, g.gs, r.engine);
                me::deactivate(g.gs, r.engine);
                r.gpu = -1;
                r.engine = -1;
                ++m_.evictions;
            }
            const auto act = me::activate(g.gs, models_[best].spec, me::ActivationMethod::naive, cfg_.activation,
                                          cfg_.params);
            if (!act) continue;
            ModelState& s = state_[best];
            s.gpu = g.gs.gpu_id;
            s.engine = act->engine_index;
            s.loading = true;
            ++m_.activations;
            const SimTime cost = seconds_to_us(cfg_.params.engine_init_s) + act->realign_us + act->load_us;
            push(now_ + cost, kActivationDone, static_cast<std::int64_t>(best));
        }
    }

    // ------------------------------------------------------------ iterations
    void wake(int gpu) {
        if (!gpus_[static_cast<std::size_t>(gpu)].busy) step_next(gpu);
    }

    void step_next(int gpu) {
        Gpu& g = gpus_[static_cast<std::size_t>(gpu)];
        const std::vector<pagealloc::PhysicalLedger*> ledgers{&g.gs.ledger};
        const std::size_t n = g.gs.engines.size();
        for (std::size_t k = 0; k < n; ++k) {
            const std::size_t ei = (g.rr + k) % n;
            me::Engine& e = g.gs.engines[ei];
            if (!e.serving() || !e.has_runnable_work(ledgers)) continue;
            if (cfg_.executor) cfg_.executor->before_step(gpu, g.gs, static_cast<int>(ei));
            const me::IterationOutcome o = me::step(e, ledgers, cfg_.params, now_);
            SimTime dur = std::max<SimTime>(o.duration_us, 1);
            if (cfg_.executor) {
                dur = std::max<SimTime>(cfg_.executor->iteration(gpu, g.gs, static_cast<int>(ei), o, dur), 1);
            }
            const SimTime end = now_ + dur;
            for (std::uint64_t id : o.first_tokens) m_.requests[id - 1].first_token_us = end;
            for (std::uint64_t id : o.preemptions) {
                RequestRecord& r = m_.requests[id - 1];
                r.first_token_us = -1;  // restarts from scratch
                ++r.preemptions;
                ++m_.preemptions;
            }
            for (std::uint64_t id : o.completions) {
                RequestRecord& r = m_.requests[id - 1];
                r.completion_us = end;
                m_.output_tokens += static_cast<std::uint64_t>(r.output_tokens);
                ModelState& s = state_[index_.at(r.model_id)];
                if (--s.outstanding == 0) s.idle_since = end;
            }
            pagealloc::refill_buffer(g.gs.ledger, cfg_.buffer_target_pages);
            ++m_.iterations;
            m_.gpu_busy_us[static_cast<std::size_t>(gpu)] += dur;
            g.rr = (ei + 1) % n;
            g.busy = true;
            push(end, kIterationDone, gpu);
            return;
        }
        g.busy = false;
    }

    void on_iteration_done(int gpu) {
        gpus_[static_cast<std::size_t>(gpu)].busy = false;
        schedule(gpu);
        step_next(gpu);
        if (cfg_.policy == Policy::qlm_timeshare) qlm_swap();
    }

    // ------------------------------------------------------------ global tick
    bool any_waiting() const {
        for (const ModelState& s : state_) {
            if (s.gpu < 0 && !s.waiting.empty()) return true;
        }
        return false;
    }

    void on_tick() {
        if (frozen()) {  // no eviction, no activation: only keep ticking while work is open
            bool open = false;
            for (const ModelState& s : state_) open = open || s.outstanding > 0;
            if (open) push(now_ + seconds_to_us(cfg_.tick_s), kSchedulerTick, 0);
            return;
        }
        const bool demand = any_waiting();
        const double frac = cfg_.pressure_free_frac;
        const auto pressured = [demand, frac](const pl::GpuView& v) {
            return demand || static_cast<double>(v.free_pages) < frac * static_cast<double>(v.capacity_pages);
        };
        for (const pl::Eviction& ev : pl::eviction_tick(views(), cfg_.idle_evict_s, pressured)) {
            const std::size_t mi = index_.at(ev.model_id);
            ModelState& s = state_[mi];
            Gpu& g = gpus_[static_cast<std::size_t>(s.gpu)];
            me::Engine& e = g.gs.engines[static_cast<std::size_t>(s.engine)];
            if (s.loading || !e.drained()) continue;
            if (cfg_.executor) cfg_.executor->detaching(s.gpu, g.gs, s.engine);
            me::deactivate(g.gs, s.engine);
            s.gpu = -1;
            s.engine = -1;
            ++m_.evictions;
        }
        for (std::size_t mi = 0; mi < models_.size(); ++mi) {
            if (state_[mi].gpu < 0 && !state_[mi].waiting.empty()) try_activate(mi);
        }
        // Evictions return weight pages to the GPU's free budget: an idle GPU
        // whose work was blocked on memory (a paused prefill, a request the
        // dispatch gate refused) may run again.
        for (Gpu& g : gpus_) {
            if (g.busy) continue;
            schedule(g.gs.gpu_id);
            wake(g.gs.gpu_id);
        }
        // keep ticking while requests are outstanding
        bool open = false;
        for (const ModelState& s : state_) open = open || s.outstanding > 0;
        if (open || q_.size() > 0) push(now_ + seconds_to_us(cfg_.tick_s), kSchedulerTick, 0);
    }

    const SimConfig& cfg_;
    const std::vector<ModelEntry>& models_;
    const std::vector<workload::TraceEvent>& trace_;
    std::map<std::string, std::size_t> index_;
    std::vector<Gpu> gpus_;
    std::vector<ModelState> state_;
    std::vector<std::uint64_t> cap_pages_;  // static_partition: per-model mapped-page cap
    std::priority_queue<Event, std::vector<Event>, std::greater<Event>> q_;
    std::uint64_t seq_ = 0;
    SimTime now_ = 0;
    SimMetrics m_;
};

}  // namespace

SimMetrics run(const SimConfig& cfg, const std::vector<ModelEntry>& models,
               const std::vector<workload::TraceEvent>& trace) {
    Sim sim(cfg, models, trace);
    return sim.run();
}

std::map<std::string, Attainment> attainment(const SimMetrics& m, const std::vector<ModelEntry>& models,
                                             double slo_scale) {
    std::map<std::string, const engine::ModelSpec*> spec;
    for (const ModelEntry& e : models) spec[e.spec.model_id] = &e.spec;
    std::map<std::string, std::array<std::uint64_t, 4>> acc;  // n, ttft ok, tpot ok, both ok
    for (const RequestRecord& r : m.requests) {
        const engine::ModelSpec* s = spec.at(r.model_id);
        bool ttft_ok = false, tpot_ok = false;
        if (r.first_token_us >= 0 && r.completion_us >= 0) {
            ttft_ok = us_to_seconds(r.first_token_us - r.arrival_us) <= slo_scale * s->ttft_slo_s;
            const double tpot = r.output_tokens > 1
                                    ? us_to_seconds(r.completion_us - r.first_token_us) / (r.output_tokens - 1)
                                    : 0.0;
            tpot_ok = tpot <= slo_scale * s->tpot_slo_s;
        }
        for (const std::string& key : {r.model_id, std::string()}) {
            auto& a = acc[key];
            a[0] += 1;
            a[1] += ttft_ok;
            a[2] += tpot_ok;
            a[3] += ttft_ok && tpot_ok;
        }
    }
    std::map<std::string, Attainment> out;
    for (const auto& [k, a] : acc) {
        const double n = static_cast<double>(a[0]);
        out[k] = Attainment{a[0], a[1] / n, a[2] / n, a[3] / n};
    }
    return out;
}

}  // namespace msim::simcore
