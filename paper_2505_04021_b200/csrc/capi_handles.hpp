// Layouts of the C-ABI's opaque handles (include/prism_capi.h), shared by
// csrc/capi_host.cpp (compiled for both the product and the reference
// oracle) and csrc/capi_device.cpp (product only). Uses only the public
// msim:: API.
#pragma once
#include <cstdint>
#include <memory>
#include <vector>

#include "msim/engine.hpp"
#include "msim/pagealloc.hpp"
#include "msim/simcore.hpp"
#include "prism_capi.h"

struct prism_ledger {
    std::unique_ptr<msim::pagealloc::PhysicalLedger> owned;
    msim::pagealloc::PhysicalLedger* l = nullptr;
};

struct prism_pool {
    explicit prism_pool(msim::pagealloc::KvPool&& p) : pool(std::move(p)) {}
    msim::pagealloc::KvPool pool;
};

struct prism_gpu {
    prism_gpu(int id, std::uint64_t cap, std::uint64_t page) : g(id, cap, page) { view.l = &g.ledger; }
    msim::engine::GpuState g;
    prism_ledger view;
    std::vector<msim::engine::IterationOutcome> last;  // last step outcome per engine
};

// prism_sim: a finished simcore run (metrics + the models it ran, for SLOs;
// serving counters when the GPU data path executed it, product only)
struct prism_sim {
    msim::simcore::SimMetrics metrics;
    std::vector<msim::simcore::ModelEntry> models;
    bool device = false;
    prism_serving_stats serving{};
};

namespace prism_capi_detail {
void set_error(const char* what);
// prism_sim_run with an optional executor (prism_sim_run_device)
void sim_run(const prism_sim_config* cfg, const prism_model_spec* specs, const double* rates, size_t n_models,
             const prism_trace_event* trace, size_t n_trace, msim::simcore::IterationExecutor* executor,
             prism_sim* out);
}
