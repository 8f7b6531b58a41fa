// EngineDeviceImpl: block-table arena, per-step descriptors, and the public
// prism:: device API entry points (msim/kvcache_device.hpp) that do not
// launch the append / attention kernels.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "cuda/device_impl.cuh"

namespace prism {

namespace pa = msim::pagealloc;
namespace me = msim::engine;

constexpr std::uint64_t kCacheTarget = 32;  // ready physical handles kept per GPU

EngineDeviceImpl& impl_of(const me::Engine& eng) {
    auto* p = dynamic_cast<EngineDeviceImpl*>(eng.device.get());
    if (!p) throw std::runtime_error("engine has no GPU device attached (prism::attach_engine_device)");
    return *p;
}

EngineDeviceImpl::EngineDeviceImpl(me::Engine& eng, pa::PhysicalLedger& ledger, const EngineDeviceOptions& o)
    : opts(o) {
    if (!eng.model) throw std::runtime_error("attach_engine_device: engine has no model");
    const me::ModelSpec& m = *eng.model;
    if (eng.pools.size() != 1) throw std::runtime_error("attach_engine_device: device path needs exactly one TP part");
    vmm = ledger.device();
    if (!vmm) throw std::runtime_error("attach_engine_device: ledger has no VmmDevice attached");
    if (m.n_layers <= 0 || m.n_q_heads <= 0 || m.n_kv_heads <= 0 || m.head_dim <= 0) {
        throw std::runtime_error("attach_engine_device: ModelSpec lacks the attention shape");
    }
    if (m.n_q_heads % m.n_kv_heads) throw std::runtime_error("attach_engine_device: n_q_heads % n_kv_heads != 0");
    const std::uint64_t tb = 2ull * m.n_layers * m.n_kv_heads * m.head_dim * 2;
    if (tb != m.token_kv_bytes) throw std::runtime_error("attach_engine_device: token_kv_bytes != 2*L*n_kv*d*2");
    if (m.head_dim != 64 && m.head_dim != 128) throw std::runtime_error("attach_engine_device: head_dim must be 64 or 128");
    group = m.n_q_heads / m.n_kv_heads;
    if (group > 8) throw std::runtime_error("attach_engine_device: GQA group above 8 not supported");
    n_q = m.n_q_heads;
    n_kv = m.n_kv_heads;
    head_dim = m.head_dim;
    n_layers = m.n_layers;
    PRISM_CUDA(cudaSetDevice(vmm->ordinal()));
    stream = static_cast<cudaStream_t>(vmm->stream());

    pool = eng.pools[0].state();
    if (!pool->dev) throw std::runtime_error("attach_engine_device: pool was created before the device was attached");
    if (!pool->mirror) pool->mirror.reset(new DevicePool(*pool, vmm->ordinal()));
    geom.base = pool->va;
    geom.page_bytes = vmm->page_bytes();
    geom.tpp = static_cast<std::uint32_t>(pool->tpp);
    geom.magic = div_magic40(geom.tpp);
    geom.n_layers = n_layers;
    geom.n_kv = n_kv;
    geom.head_dim = head_dim;

    table_cap = std::max<std::int64_t>(opts.table_capacity, 1024);
    PRISM_CUDA(cudaMalloc(&table, sizeof(std::int32_t) * table_cap));
    free_ranges[0] = table_cap;
    PRISM_CUDA(cudaMalloc(&step_slots, sizeof(std::int32_t) * std::max(opts.max_step_tokens, 1)));
}

EngineDeviceImpl::~EngineDeviceImpl() {
    cudaStreamSynchronize(stream);
    if (copy_stream) {
        cudaStreamSynchronize(copy_stream);
        cudaStreamDestroy(copy_stream);
    }
    for (cudaEvent_t ev : host_events) cudaEventDestroy(ev);
    if (host_done) cudaEventDestroy(host_done);
    for (cudaEvent_t e : stage_free) {
        if (e) cudaEventDestroy(e);
    }
    if (host_stage) cudaFree(host_stage);
    if (table) cudaFree(table);
    if (step_slots) cudaFree(step_slots);
    if (workspace) cudaFree(workspace);
    if (counters) cudaFree(counters);
}

std::int64_t EngineDeviceImpl::acquire_row(std::int64_t capacity) {
    capacity = std::max<std::int64_t>(capacity, 1);
    for (auto it = free_ranges.begin(); it != free_ranges.end(); ++it) {
        if (it->second < capacity) continue;
        const std::int64_t off = it->first;
        const std::int64_t left = it->second - capacity;
        free_ranges.erase(it);
        if (left) free_ranges[off + capacity] = left;
        row_len[off] = capacity;
        return off;
    }
    grow_table(table_cap + capacity);
    return acquire_row(capacity);
}

void EngineDeviceImpl::release_row(std::int64_t row) {
    const auto it = row_len.find(row);
    if (it == row_len.end()) throw std::runtime_error("release_row: unknown row");
    std::int64_t off = row, len = it->second;
    row_len.erase(it);
    auto next = free_ranges.lower_bound(off);
    if (next != free_ranges.end() && next->first == off + len) {
        len += next->second;
        next = free_ranges.erase(next);
    }
    if (next != free_ranges.begin()) {
        auto prev = std::prev(next);
        if (prev->first + prev->second == off) {
            prev->second += len;
            return;
        }
    }
    free_ranges[off] = len;
}

void EngineDeviceImpl::grow_table(std::int64_t need) {
    std::int64_t cap = table_cap;
    while (cap < need) cap *= 2;
    std::int32_t* bigger = nullptr;
    PRISM_CUDA(cudaMalloc(&bigger, sizeof(std::int32_t) * cap));
    PRISM_CUDA(cudaMemcpyAsync(bigger, table, sizeof(std::int32_t) * table_cap, cudaMemcpyDeviceToDevice, stream));
    PRISM_CUDA(cudaStreamSynchronize(stream));
    PRISM_CUDA(cudaFree(table));
    // extend (and merge with) the trailing free range
    std::int64_t off = table_cap, len = cap - table_cap;
    if (!free_ranges.empty()) {
        auto last = std::prev(free_ranges.end());
        if (last->first + last->second == table_cap) {
            off = last->first;
            len += last->second;
            free_ranges.erase(last);
        }
    }
    free_ranges[off] = len;
    table = bigger;
    table_cap = cap;
}

void EngineDeviceImpl::begin_step(me::Engine&) {
    k3_chain = k4_chain = false;
    // Pages unmapped during earlier steps become reclaimable once the fence
    // recorded here (after every kernel the caller issued for those steps)
    // has passed; see VmmDevice.
    vmm->fence();
    vmm->defer_access(true);  // this step's fresh pages share cuMemSetAccess calls
}

void EngineDeviceImpl::end_step(me::Engine&, const me::IterationOutcome& out, const std::vector<StepDecode>& decodes,
                                std::uint64_t prefill_id, std::int64_t prefill_row, std::int32_t prefill_first,
                                std::int32_t prefill_tokens) {
    vmm->defer_access(false);  // pages must be accessible before K2/K3 run
    ++step_serial;
    k3_chain = k4_chain = false;
    // K1: replay this step's allocations / frees on the device slot state.
    const std::int64_t n = pool->mirror->replay(*pool, table, step_slots, opts.max_step_tokens, stream);
    step_tokens = static_cast<int>(n);
    step_decodes = static_cast<int>(decodes.size());
    if (step_decodes > opts.max_decode_batch) throw std::runtime_error("step decoded more requests than max_decode_batch");
    // Token metadata in allocation order: prefill chunk first, then decodes.
    const auto dead = [&](std::uint64_t id) {
        return std::find(out.preemptions.begin(), out.preemptions.end(), id) != out.preemptions.end();
    };
    token_meta.ensure(static_cast<std::size_t>(std::max<std::int64_t>(n, 1)));
    std::int64_t k = 0;
    this->prefill_row = -1;
    this->prefill_chunk = 0;
    if (prefill_row >= 0 && !dead(prefill_id)) {
        this->prefill_row = prefill_row;
        this->prefill_first = prefill_first;
        this->prefill_chunk = out.chunk_tokens;
        this->prefill_request = prefill_id;
    }
    if (prefill_row >= 0) {
        const bool is_dead = dead(prefill_id);
        for (std::int32_t t = 0; t < prefill_tokens; ++t, ++k) {
            token_meta.host[k] = TokenMeta{is_dead ? ~0ull : prefill_id, static_cast<std::uint32_t>(prefill_first + t), 0};
        }
    }
    for (const StepDecode& d : decodes) {
        token_meta.host[k++] = TokenMeta{d.request_id, static_cast<std::uint32_t>(d.ctx_len - 1), 0};
    }
    if (k != n) throw std::runtime_error("end_step: slot count mismatch between host and device op log");
    token_meta.upload(static_cast<std::size_t>(n), stream);
    decode_desc.ensure(std::max<std::size_t>(decodes.size(), 1));
    decode_ids.clear();
    for (std::size_t i = 0; i < decodes.size(); ++i) {
        decode_desc.host[i] = DecodeDesc{decodes[i].row, decodes[i].ctx_len, 0, decodes[i].request_id};
        decode_ids.push_back(decodes[i].request_id);
    }
    decode_desc.upload(decodes.size(), stream);
    // The GPU is busy with this step now: create the physical handles the
    // next steps' fresh pages will need (cuMemCreate off the map path).
    vmm->prefill_cache(kCacheTarget);
}

float* EngineDeviceImpl::attn_workspace(std::size_t floats) {
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

int* EngineDeviceImpl::attn_counters(std::size_t n) {
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

// ---------------------------------------------------------------- host-buffer path

void launch_decode_attention(EngineDeviceImpl& d, int layer, const void* q, void* out, float scale, int chunk);

void decode_host(me::Engine& eng, const void* new_k, const void* new_v, const void* q, void* out, float scale,
                 bool wait) {
    EngineDeviceImpl& d = impl_of(eng);
    const int n_tok = d.step_tokens, n_dec = d.step_decodes, L = d.n_layers;
    const std::size_t kv_bytes = static_cast<std::size_t>(L) * n_tok * d.n_kv * d.head_dim * 2;
    const std::size_t q_layer = static_cast<std::size_t>(n_dec) * d.n_q * d.head_dim * 2;
    const std::size_t need = 2 * kv_bytes + 2 * q_layer * L + 256;
    if (!d.copy_stream) {
        PRISM_CUDA(cudaStreamCreateWithFlags(&d.copy_stream, cudaStreamNonBlocking));
        PRISM_CUDA(cudaEventCreateWithFlags(&d.host_done, cudaEventDisableTiming));
    }
    while (d.host_events.size() < 2 * static_cast<std::size_t>(L) + 1) {
        cudaEvent_t ev;
        PRISM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        d.host_events.push_back(ev);
    }
    // Two staging sets, alternating per call: the copies of this call only
    // wait for the compute work of the call before the previous one (the last
    // reader of this set), so the next step's inputs stream in while the
    // current step's kernels run.
    const std::size_t set_bytes = (need + 255) / 256 * 256;
    if (2 * set_bytes > d.host_stage_bytes) {
        PRISM_CUDA(cudaStreamSynchronize(d.copy_stream));
        PRISM_CUDA(cudaStreamSynchronize(d.stream));
        if (d.host_stage) PRISM_CUDA(cudaFree(d.host_stage));
        PRISM_CUDA(cudaMalloc(&d.host_stage, 2 * set_bytes));
        d.host_stage_bytes = 2 * set_bytes;
        d.stage_used[0] = d.stage_used[1] = false;
    }
    for (cudaEvent_t& e : d.stage_free) {
        if (!e) PRISM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int set = d.stage_parity;
    d.stage_parity ^= 1;
    char* dk = static_cast<char*>(d.host_stage) + set * (d.host_stage_bytes / 2);
    char* dv = dk + kv_bytes;
    char* dq = dv + kv_bytes;
    char* dout = dq + q_layer * L;
    cudaStream_t cs = d.copy_stream;
    std::vector<cudaEvent_t>& ev = d.host_events;
    if (d.stage_used[set]) PRISM_CUDA(cudaStreamWaitEvent(cs, d.stage_free[set], 0));
    // All inputs (new K/V rows, q of every layer) go in one burst and gate
    // the compute stream once; outputs go back in groups of kOutGroup layers
    // while the following layers' K3 run. Few cross-stream edges keep the K3
    // launches back to back (programmatic-dependent chain).
    static const int kOutGroup = [] {  // layers per output copy (PRISM_E2E_OUT_GROUP, default 4)
        const char* e = std::getenv("PRISM_E2E_OUT_GROUP");
        const int v = e ? std::atoi(e) : 4;
        return v > 0 ? v : 4;
    }();
    const bool with_kv = new_k && new_v && n_tok;
    if (with_kv) {
        PRISM_CUDA(cudaMemcpyAsync(dk, new_k, kv_bytes, cudaMemcpyHostToDevice, cs));
        PRISM_CUDA(cudaMemcpyAsync(dv, new_v, kv_bytes, cudaMemcpyHostToDevice, cs));
    }
    if (n_dec) PRISM_CUDA(cudaMemcpyAsync(dq, q, q_layer * L, cudaMemcpyHostToDevice, cs));
    PRISM_CUDA(cudaEventRecord(ev[1], cs));
    PRISM_CUDA(cudaStreamWaitEvent(d.stream, ev[1], 0));
    if (with_kv) append_step_kv(eng, 0, L, dk, dv);
    if (n_dec) {
        for (int l = 0; l < L; ++l) {
            launch_decode_attention(d, l, dq + q_layer * l, dout + q_layer * l, scale, 0);
            if ((l + 1) % kOutGroup == 0 || l + 1 == L) {
                const int first = l / kOutGroup * kOutGroup;
                cudaEvent_t e = ev[2 + l / kOutGroup];
                PRISM_CUDA(cudaEventRecord(e, d.stream));
                PRISM_CUDA(cudaStreamWaitEvent(cs, e, 0));
                PRISM_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + q_layer * first, dout + q_layer * first,
                                           q_layer * (l + 1 - first), cudaMemcpyDeviceToHost, cs));
            }
        }
    }
    PRISM_CUDA(cudaEventRecord(d.stage_free[set], d.stream));
    d.stage_used[set] = true;
    PRISM_CUDA(cudaEventRecord(d.host_done, cs));
    if (wait) wait_host(eng);
}

void wait_host(const me::Engine& eng) {
    EngineDeviceImpl& d = impl_of(eng);
    if (d.host_done) PRISM_CUDA(cudaEventSynchronize(d.host_done));
}

// ---------------------------------------------------------------- public API

void attach_engine_device(me::Engine& eng, pa::PhysicalLedger& ledger, const EngineDeviceOptions& opts) {
    eng.device = std::make_shared<EngineDeviceImpl>(eng, ledger, opts);
}

int last_step_tokens(const me::Engine& eng) { return impl_of(eng).step_tokens; }
int last_step_decodes(const me::Engine& eng) { return impl_of(eng).step_decodes; }
const std::vector<std::uint64_t>& last_step_decode_ids(const me::Engine& eng) { return impl_of(eng).decode_ids; }
void* engine_stream(const me::Engine& eng) { return impl_of(eng).stream; }

std::vector<std::int32_t> last_step_slots(const me::Engine& eng) {
    EngineDeviceImpl& d = impl_of(eng);
    std::vector<std::int32_t> h(static_cast<std::size_t>(d.step_tokens));
    if (!h.empty()) {
        PRISM_CUDA(cudaMemcpyAsync(h.data(), d.step_slots, h.size() * sizeof(std::int32_t), cudaMemcpyDeviceToHost,
                                   d.stream));
    }
    PRISM_CUDA(cudaStreamSynchronize(d.stream));
    if (d.pool->mirror->status(d.stream) != 0) throw std::runtime_error("device slot allocator diverged from host");
    return h;
}

std::vector<std::int32_t> read_table_row(const me::Engine& eng, std::int64_t row, int len) {
    EngineDeviceImpl& d = impl_of(eng);
    std::vector<std::int32_t> h(static_cast<std::size_t>(len));
    if (len) {
        PRISM_CUDA(cudaMemcpyAsync(h.data(), d.table + row, h.size() * sizeof(std::int32_t), cudaMemcpyDeviceToHost,
                                   d.stream));
    }
    PRISM_CUDA(cudaStreamSynchronize(d.stream));
    return h;
}

void attach_pool_mirror(pa::KvPool& pool) {
    pa::detail::PoolState* s = pool.state();
    if (!s->dev) throw std::runtime_error("attach_pool_mirror: pool has no device");
    if (!s->mirror) s->mirror.reset(new DevicePool(*s, s->dev->ordinal()));
}

std::vector<std::int32_t> sync_pool_mirror(pa::KvPool& pool) {
    pa::detail::PoolState* s = pool.state();
    if (!s->mirror) throw std::runtime_error("sync_pool_mirror: no mirror attached");
    auto stream = static_cast<cudaStream_t>(s->dev->stream());
    std::int64_t total = 0;
    for (const auto& op : s->ops) {
        if (op.kind == pa::detail::DeviceOp::kAlloc) total += op.count;
    }
    std::int32_t* out = nullptr;
    if (total) PRISM_CUDA(cudaMallocAsync(&out, sizeof(std::int32_t) * total, stream));
    s->mirror->replay(*s, nullptr, out, total, stream);
    std::vector<std::int32_t> h(static_cast<std::size_t>(total));
    if (total) {
        PRISM_CUDA(cudaMemcpyAsync(h.data(), out, sizeof(std::int32_t) * total, cudaMemcpyDeviceToHost, stream));
        PRISM_CUDA(cudaFreeAsync(out, stream));
    }
    PRISM_CUDA(cudaStreamSynchronize(stream));
    if (s->mirror->status(stream) != 0) throw std::runtime_error("device slot allocator diverged from host");
    return h;
}

void read_pool_mirror(pa::KvPool& pool, std::vector<std::uint32_t>& occ, std::vector<std::uint32_t>& bits) {
    pa::detail::PoolState* s = pool.state();
    if (!s->mirror) throw std::runtime_error("read_pool_mirror: no mirror attached");
    auto stream = static_cast<cudaStream_t>(s->dev->stream());
    DevicePool& m = *s->mirror;
    occ.resize(m.vpages);
    bits.resize(static_cast<std::size_t>(m.vpages) * m.words);
    PRISM_CUDA(cudaMemcpyAsync(occ.data(), m.occ, occ.size() * 4, cudaMemcpyDeviceToHost, stream));
    PRISM_CUDA(cudaMemcpyAsync(bits.data(), m.bits, bits.size() * 4, cudaMemcpyDeviceToHost, stream));
    PRISM_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace prism
