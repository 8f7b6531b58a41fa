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

namespace prism_capi_detail {
void set_error(const char* what);
}
