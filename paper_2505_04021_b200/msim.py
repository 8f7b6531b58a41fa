"""Python mirror of the reference's msim interface over the C-ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(proj/include/msim/pagealloc.hpp, engine.hpp, placement.hpp, admission.hpp,
workload.hpp), so parity tests read like the reference's own tests. Every
object is bound to one library (`capi.product()` by default, or the
reference oracle library for parity runs), so the same test drives both.

Errors: UsageError / ParseError / PlacementError (capi.py) mirror
msim::UsageError / ParseError / placement::PlacementError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

from . import capi
from .capi import Slot

MOST_OCCUPIED_FIRST = 0
LOWEST_INDEX_FIRST = 1
EVENT_KINDS = ("map", "unmap", "buffer_hit", "alloc_fail")
ENGINE_STATUS = ("pooled", "aligning", "loading", "serving", "draining")
PAGE_BYTES = 2 << 20


def _lib(lib):
    return lib if lib is not None else capi.product()


@dataclass(frozen=True)
class TokenSlotHandle:
    pool: int
    page: int
    slot: int


@dataclass
class AllocResult:
    handles: list
    shortfall_pages: int = 0
    pages_mapped: int = 0
    buffer_hits: int = 0

    def ok(self) -> bool:
        return self.shortfall_pages == 0


@dataclass(frozen=True)
class AllocEvent:
    time_us: int
    gpu_id: int
    model_id: str
    kind: str
    pages: int


class PhysicalLedger:
    """msim::pagealloc::PhysicalLedger (pagealloc.hpp:45-102)."""

    def __init__(self, gpu_id: int, capacity_pages: int, page_bytes: int = PAGE_BYTES, lib=None, _borrow=None):
        self.lib = _lib(lib)
        self._own = _borrow is None
        if _borrow is not None:
            self.h = C.c_void_p(_borrow)
        else:
            self.h = C.c_void_p()
            self.lib.call("prism_ledger_create", gpu_id, capacity_pages, page_bytes, C.byref(self.h))

    def __del__(self):
        if getattr(self, "_own", False) and getattr(self, "h", None) and self.h.value:
            self.lib.prism_ledger_destroy(self.h)
            self.h = None

    def _stats(self) -> capi.LedgerStats:
        s = capi.LedgerStats()
        self.lib.call("prism_ledger_get_stats", self.h, C.byref(s))
        return s

    def capacity_pages(self) -> int:
        return self._stats().capacity_pages

    def mapped_pages(self) -> int:
        return self._stats().mapped_pages

    def buffer_pages(self) -> int:
        return self._stats().buffer_pages

    def weight_pages(self) -> int:
        return self._stats().weight_pages

    def free_pages(self) -> int:
        return self._stats().free_pages

    def page_bytes(self) -> int:
        return self._stats().page_bytes

    def pool_mapped_pages(self, pool_id: int) -> int:
        v = C.c_uint64()
        self.lib.call("prism_ledger_pool_mapped_pages", self.h, pool_id, C.byref(v))
        return v.value

    def refill_buffer(self, target_pages: int) -> int:
        v = C.c_uint64()
        self.lib.call("prism_refill_buffer", self.h, target_pages, C.byref(v))
        return v.value

    def reserve_weight_pages(self, model_id: str, pages: int) -> bool:
        ok = C.c_int()
        self.lib.call("prism_ledger_reserve_weights", self.h, model_id.encode(), pages, C.byref(ok))
        return bool(ok.value)

    def release_weight_pages(self, model_id: str) -> None:
        self.lib.call("prism_ledger_release_weights", self.h, model_id.encode())

    def weight_pages_of(self, model_id: str) -> int:
        v = C.c_uint64()
        self.lib.call("prism_ledger_weight_pages_of", self.h, model_id.encode(), C.byref(v))
        return v.value

    def set_time(self, now_us: int) -> None:
        self.lib.call("prism_ledger_set_time", self.h, now_us)

    def set_recording(self, on: bool) -> None:
        self.lib.call("prism_ledger_set_recording", self.h, 1 if on else 0)

    def events(self) -> list:
        n = C.c_size_t()
        self.lib.call("prism_ledger_events", self.h, None, 0, C.byref(n))
        buf = (capi.Event * max(n.value, 1))()
        self.lib.call("prism_ledger_events", self.h, buf, n.value, C.byref(n))
        return [AllocEvent(e.time_us, e.gpu_id, e.model_id.decode(), EVENT_KINDS[e.kind], e.pages)
                for e in buf[:n.value]]

    def clear_events(self) -> None:
        self.lib.call("prism_ledger_clear_events", self.h)

    def check_invariants(self) -> None:
        self.lib.call("prism_ledger_check_invariants", self.h)

    def attach_device(self, device: "Device") -> None:
        self.lib.call("prism_ledger_attach_device", self.h, device.h)


class KvPool:
    """msim::pagealloc::KvPool (pagealloc.hpp:114-172); created by alloc_kvcache."""

    def __init__(self, lib, handle):
        self.lib = lib
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.lib.prism_pool_destroy(self.h)
            self.h = None

    def _info(self) -> capi.PoolInfo:
        s = capi.PoolInfo()
        self.lib.call("prism_pool_info_get", self.h, C.byref(s))
        return s

    def id(self) -> int:
        return self._info().id

    def alive(self) -> bool:
        return bool(self._info().alive)

    def token_bytes(self) -> int:
        return self._info().token_bytes

    def tokens_per_page(self) -> int:
        return self._info().tokens_per_page

    def virtual_capacity_pages(self) -> int:
        return self._info().virtual_capacity_pages

    def mapped_pages(self) -> int:
        return self._info().mapped_pages

    def occupied_slots(self) -> int:
        return self._info().occupied_slots

    def free_slots_in_mapped(self) -> int:
        i = self._info()
        return i.mapped_pages * i.tokens_per_page - i.occupied_slots

    def device_base(self) -> int:
        return self._info().device_base

    def allocatable_tokens(self, ledger: PhysicalLedger) -> int:
        v = C.c_uint64()
        self.lib.call("prism_pool_allocatable_tokens", self.h, ledger.h, C.byref(v))
        return v.value

    def can_alloc(self, ledger: PhysicalLedger, n: int) -> bool:
        return n <= self.allocatable_tokens(ledger)

    def page_occupied(self, page: int) -> int:
        v = C.c_uint64()
        self.lib.call("prism_pool_page_occupied", self.h, page, C.byref(v))
        return v.value

    def page_mapped(self, page: int) -> bool:
        v = C.c_int()
        self.lib.call("prism_pool_page_mapped", self.h, page, C.byref(v))
        return bool(v.value)

    def set_mapped_page_cap(self, cap: Optional[int]) -> None:
        self.lib.call("prism_pool_set_cap", self.h, -1 if cap is None else cap)

    # --- GPU slot mirror (product only) ---
    def attach_mirror(self) -> None:
        self.lib.call("prism_pool_attach_mirror", self.h)

    def sync_mirror(self) -> list:
        n = C.c_size_t()
        cap = 1 << 20
        buf = (C.c_int32 * cap)()
        self.lib.call("prism_pool_sync_mirror", self.h, buf, cap, C.byref(n))
        return list(buf[:n.value])


def alloc_kvcache(ledger: PhysicalLedger, model_id: str, token_bytes: int, virtual_capacity_pages: int,
                  placement: int = MOST_OCCUPIED_FIRST) -> KvPool:
    h = C.c_void_p()
    ledger.lib.call("prism_kvcache_alloc", ledger.h, model_id.encode(), token_bytes, virtual_capacity_pages,
                    placement, C.byref(h))
    return KvPool(ledger.lib, h)


def free_kvcache(ledger: PhysicalLedger, pool: KvPool) -> None:
    ledger.lib.call("prism_kvcache_free", ledger.h, pool.h)


def alloc_kv_raw(pool: KvPool, ledger: PhysicalLedger, n: int):
    """alloc_kv returning the raw ctypes slot array (fast path for fuzzing)."""
    buf = (Slot * max(n, 1))()
    res = capi.AllocResult()
    pool.lib.call("prism_kv_alloc", pool.h, ledger.h, n, buf, C.byref(res))
    return buf, res


def alloc_kv(pool: KvPool, ledger: PhysicalLedger, n: int) -> AllocResult:
    buf, res = alloc_kv_raw(pool, ledger, n)
    handles = [TokenSlotHandle(s.pool, s.page, s.slot) for s in buf[:res.n_handles]]
    return AllocResult(handles, res.shortfall_pages, res.pages_mapped, res.buffer_hits)


def free_kv(pool: KvPool, ledger: PhysicalLedger, handles: Sequence[TokenSlotHandle]) -> None:
    arr = (Slot * max(len(handles), 1))(*[Slot(h.pool, h.page, h.slot) for h in handles])
    pool.lib.call("prism_kv_free", pool.h, ledger.h, arr, len(handles))


def refill_buffer(ledger: PhysicalLedger, target_pages: int) -> int:
    return ledger.refill_buffer(target_pages)


# ---------------------------------------------------------------- engine


@dataclass
class ModelSpec:
    """msim::engine::ModelSpec (engine.hpp:16-25) + the attention shape."""

    model_id: str
    weight_bytes: int = 0
    token_kv_bytes: int = 0
    prefill_tps: float = 0.0
    chunk_size: int = 512
    ttft_slo_s: float = 1.0
    tpot_slo_s: float = 0.05
    tp_degree: int = 1
    n_layers: int = 0
    n_q_heads: int = 0
    n_kv_heads: int = 0
    head_dim: int = 0

    def to_c(self) -> capi.ModelSpec:
        s = capi.ModelSpec()
        self._keep = self.model_id.encode()
        s.model_id = self._keep
        for f in ("weight_bytes", "token_kv_bytes", "prefill_tps", "chunk_size", "ttft_slo_s", "tpot_slo_s",
                  "tp_degree", "n_layers", "n_q_heads", "n_kv_heads", "head_dim"):
            setattr(s, f, getattr(self, f))
        return s

    @staticmethod
    def llm(model_id: str, n_layers: int, n_q: int, n_kv: int, d: int, weight_bytes: int = 0, **kw) -> "ModelSpec":
        return ModelSpec(model_id, weight_bytes, 2 * n_layers * n_kv * d * 2, n_layers=n_layers, n_q_heads=n_q,
                         n_kv_heads=n_kv, head_dim=d, **kw)


@dataclass
class EngineParams:
    alpha_ms: float = 6.0
    beta_ms_per_token: float = 0.025
    map_latency_ms: float = 0.2
    engine_init_s: float = 5.0
    realign_s: float = 0.05
    reserve_frac: float = 0.05

    def to_c(self) -> capi.EngineParams:
        return capi.EngineParams(self.alpha_ms, self.beta_ms_per_token, self.map_latency_ms, self.engine_init_s,
                                 self.realign_s, self.reserve_frac)


@dataclass
class IterationOutcome:
    duration_us: int
    chunk_tokens: int
    decode_tokens: int
    first_tokens: list
    completions: list
    preemptions: list
    pages_mapped_direct: int
    prefill_paused: bool


@dataclass
class RequestInfo:
    id: int
    prompt_tokens: int
    output_tokens: int
    prompt_done: int
    generated: int
    admit_seq: int
    n_slots: int
    table_row: int

    def live_slots(self) -> int:
        return self.prompt_done + self.generated


class GpuState:
    """msim::engine::GpuState (engine.hpp:116-127) plus its engines."""

    def __init__(self, gpu_id: int, capacity_pages: int, page_bytes: int = PAGE_BYTES, lib=None):
        self.lib = _lib(lib)
        self.h = C.c_void_p()
        self.lib.call("prism_gpu_create", gpu_id, capacity_pages, page_bytes, C.byref(self.h))
        self.ledger = PhysicalLedger(gpu_id, 0, lib=self.lib, _borrow=self.lib.prism_gpu_ledger(self.h))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.ledger = None
            self.lib.prism_gpu_destroy(self.h)
            self.h = None

    def activate(self, spec: ModelSpec, method: int = 1, params: Optional[EngineParams] = None):
        out, ok = capi.Activation(), C.c_int()
        cs = spec.to_c()
        self.lib.call("prism_gpu_activate", self.h, C.byref(cs), method, C.byref((params or EngineParams()).to_c()),
                      C.byref(out), C.byref(ok))
        return out if ok.value else None

    def finish_activation(self, engine_index: int) -> None:
        self.lib.call("prism_gpu_finish_activation", self.h, engine_index)

    def deactivate(self, engine_index: int) -> None:
        self.lib.call("prism_gpu_deactivate", self.h, engine_index)

    def engine(self, index: int) -> "Engine":
        return Engine(self, index)


class Engine:
    """One msim::engine::Engine inside a GpuState."""

    def __init__(self, gpu: GpuState, index: int):
        self.gpu, self.index, self.lib = gpu, index, gpu.lib

    def status(self) -> str:
        v = C.c_int()
        self.lib.call("prism_engine_status", self.gpu.h, self.index, C.byref(v))
        return ENGINE_STATUS[v.value]

    def push(self, request_id: int, prompt_tokens: int, output_tokens: int) -> None:
        self.lib.call("prism_engine_push", self.gpu.h, self.index, request_id, prompt_tokens, output_tokens)

    def _ids(self, which: int) -> list:
        n = C.c_size_t()
        self.lib.call("prism_engine_outcome_ids", self.gpu.h, self.index, which, None, 0, C.byref(n))
        buf = (C.c_uint64 * max(n.value, 1))()
        self.lib.call("prism_engine_outcome_ids", self.gpu.h, self.index, which, buf, n.value, C.byref(n))
        return list(buf[:n.value])

    def step(self, params: Optional[EngineParams] = None, now_us: int = 0) -> IterationOutcome:
        o = capi.Outcome()
        self.lib.call("prism_engine_step", self.gpu.h, self.index, C.byref((params or EngineParams()).to_c()),
                      now_us, C.byref(o))
        return IterationOutcome(o.duration_us, o.chunk_tokens, o.decode_tokens, self._ids(0), self._ids(1),
                                self._ids(2), o.pages_mapped_direct, bool(o.prefill_paused))

    def counts(self):
        b, q = C.c_size_t(), C.c_size_t()
        self.lib.call("prism_engine_counts", self.gpu.h, self.index, C.byref(b), C.byref(q))
        return b.value, q.value

    def _request(self, where: int, i: int) -> RequestInfo:
        r = capi.RequestInfo()
        self.lib.call("prism_engine_request", self.gpu.h, self.index, where, i, C.byref(r))
        return RequestInfo(r.id, r.prompt_tokens, r.output_tokens, r.prompt_done, r.generated, r.admit_seq,
                           r.n_slots, r.table_row)

    def batch(self) -> list:
        return [self._request(0, i) for i in range(self.counts()[0])]

    def local_queue(self) -> list:
        return [self._request(1, i) for i in range(self.counts()[1])]

    def request_kv_raw(self, request_id: int):
        n = C.c_size_t()
        self.lib.call("prism_engine_request_kv", self.gpu.h, self.index, request_id, None, 0, C.byref(n))
        buf = (Slot * max(n.value, 1))()
        self.lib.call("prism_engine_request_kv", self.gpu.h, self.index, request_id, buf, n.value, C.byref(n))
        return buf, n.value

    def request_kv(self, request_id: int) -> list:
        buf, n = self.request_kv_raw(request_id)
        return [TokenSlotHandle(s.pool, s.page, s.slot) for s in buf[:n]]

    def mapped_pages(self) -> int:
        v = C.c_uint64()
        self.lib.call("prism_engine_mapped_pages", self.gpu.h, self.index, C.byref(v))
        return v.value

    def next_chunk_need(self) -> int:
        v = C.c_uint64()
        self.lib.call("prism_engine_next_chunk_need", self.gpu.h, self.index, C.byref(v))
        return v.value

    def has_runnable_work(self) -> bool:
        v = C.c_int()
        self.lib.call("prism_engine_has_runnable_work", self.gpu.h, self.index, C.byref(v))
        return bool(v.value)

    def reserved_pages(self, reserve_frac: float) -> int:
        v = C.c_uint64()
        self.lib.call("prism_engine_reserved_pages", self.gpu.h, self.index, reserve_frac, C.byref(v))
        return v.value

    # ---- GPU data path (product only) ----
    def attach_device(self, table_capacity: int = 0, max_decode_batch: int = 0, max_step_tokens: int = 0) -> None:
        o = capi.EngineDeviceOptions(table_capacity, max_decode_batch, max_step_tokens)
        self.lib.call("prism_engine_attach_device", self.gpu.h, self.index, C.byref(o))

    def step_info(self):
        t, d = C.c_int32(), C.c_int32()
        self.lib.call("prism_engine_step_info", self.gpu.h, self.index, C.byref(t), C.byref(d))
        return t.value, d.value

    def step_decode_ids(self) -> list:
        n = C.c_size_t()
        buf = (C.c_uint64 * 65536)()
        self.lib.call("prism_engine_step_decode_ids", self.gpu.h, self.index, buf, 65536, C.byref(n))
        return list(buf[:n.value])

    def step_slots(self) -> list:
        n = C.c_size_t()
        cap = 1 << 20
        buf = (C.c_int32 * cap)()
        self.lib.call("prism_engine_step_slots", self.gpu.h, self.index, buf, cap, C.byref(n))
        return list(buf[:n.value])

    def table_row(self, row: int, length: int) -> list:
        buf = (C.c_int32 * max(length, 1))()
        self.lib.call("prism_engine_table_row", self.gpu.h, self.index, row, length, buf)
        return list(buf[:length])

    def append_kv(self, layer_begin: int, layer_end: int, k_ptr: int, v_ptr: int) -> None:
        self.lib.call("prism_engine_append_kv", self.gpu.h, self.index, layer_begin, layer_end, C.c_void_p(k_ptr),
                      C.c_void_p(v_ptr))

    def append_kv_synthetic(self, layer_begin: int, layer_end: int, seed: int) -> None:
        self.lib.call("prism_engine_append_kv_synthetic", self.gpu.h, self.index, layer_begin, layer_end, seed)

    def decode_attention(self, layer: int, q_ptr: int, out_ptr: int, scale: float, chunk: int = 0) -> None:
        self.lib.call("prism_engine_decode_attention", self.gpu.h, self.index, layer, C.c_void_p(q_ptr),
                      C.c_void_p(out_ptr), scale, chunk)

    def prefill_info(self):
        """(query tokens, first position, request id) of the last step's
        prefill chunk; tokens == 0 when there is none."""
        n, first, rid = C.c_int32(), C.c_int32(), C.c_uint64()
        self.lib.call("prism_engine_prefill_info", self.gpu.h, self.index, C.byref(n), C.byref(first), C.byref(rid))
        return n.value, first.value, rid.value

    def prefill_attention(self, layer: int, q_ptr: int, out_ptr: int, scale: float) -> None:
        self.lib.call("prism_engine_prefill_attention", self.gpu.h, self.index, layer, C.c_void_p(q_ptr),
                      C.c_void_p(out_ptr), scale)

    def synth_q(self, layer: int, seed: int, q_scale: float, q_ptr: int) -> None:
        self.lib.call("prism_engine_synth_q", self.gpu.h, self.index, layer, seed, q_scale, C.c_void_p(q_ptr))

    def decode_host(self, new_k_ptr, new_v_ptr, q_ptr, out_ptr, scale: float) -> None:
        self.lib.call("prism_engine_decode_host", self.gpu.h, self.index, C.c_void_p(new_k_ptr),
                      C.c_void_p(new_v_ptr), C.c_void_p(q_ptr), C.c_void_p(out_ptr), scale)

    def decode_host_async(self, new_k_ptr, new_v_ptr, q_ptr, out_ptr, scale: float) -> None:
        self.lib.call("prism_engine_decode_host_async", self.gpu.h, self.index, C.c_void_p(new_k_ptr),
                      C.c_void_p(new_v_ptr), C.c_void_p(q_ptr), C.c_void_p(out_ptr), scale)

    def wait_host(self) -> None:
        self.lib.call("prism_engine_wait_host", self.gpu.h, self.index)

    def synchronize(self) -> None:
        self.lib.call("prism_engine_synchronize", self.gpu.h, self.index)


def throughput_of(kv_budget_bytes: int, spec: ModelSpec, prompt_tokens: int = 2048, output_tokens: int = 2048,
                  params: Optional[EngineParams] = None, page_bytes: int = PAGE_BYTES, warmup_s: float = 20.0,
                  window_s: float = 60.0, lib=None):
    lib = _lib(lib)
    tps, mb = C.c_double(), C.c_int()
    cs = spec.to_c()
    lib.call("prism_throughput_of", kv_budget_bytes, C.byref(cs), prompt_tokens, output_tokens,
             C.byref((params or EngineParams()).to_c()), page_bytes, warmup_s, window_s, C.byref(tps), C.byref(mb))
    return tps.value, mb.value


class Device:
    """prism::VmmDevice — CUDA VMM backend of one GPU (product only)."""

    def __init__(self, ordinal: int = 0, page_bytes: int = PAGE_BYTES, lib=None, chunk_pages: int = 0):
        """chunk_pages: logical pages per physical VMM handle (0: default 8)."""
        self.lib = _lib(lib)
        if not self.lib.has_device:
            raise capi.CudaError(5, f"{self.lib.path} has no GPU data path")
        self.h = C.c_void_p()
        self.lib.call("prism_device_open_chunked", ordinal, page_bytes, chunk_pages, C.byref(self.h))

    def chunk_pages(self) -> int:
        v = C.c_uint64()
        self.lib.call("prism_device_chunk_pages", self.h, C.byref(v))
        return v.value

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.lib.prism_device_close(self.h)
            self.h = None

    def capacity_pages(self, reserve_bytes: int) -> int:
        v = C.c_uint64()
        self.lib.call("prism_device_capacity_pages", self.h, reserve_bytes, C.byref(v))
        return v.value

    def stats(self) -> dict:
        s = capi.DeviceStats()
        self.lib.call("prism_device_stats_get", self.h, C.byref(s))
        return {f: getattr(s, f) for f, _ in capi.DeviceStats._fields_}

    def reset_stats(self) -> None:
        self.lib.call("prism_device_reset_stats", self.h)

    def reserve(self, pages: int) -> None:
        """Create physical handles for `pages` pages up front (startup
        reservation; bounded by the ledger budget)."""
        self.lib.call("prism_device_reserve", self.h, pages)

    def quiesce(self) -> None:
        """Wait until the background VMM worker has no queued work."""
        self.lib.call("prism_device_quiesce", self.h)

    def reclaim(self, wait: bool) -> None:
        self.lib.call("prism_device_reclaim", self.h, 1 if wait else 0)

    def fence(self) -> None:
        self.lib.call("prism_device_fence", self.h)

    def synchronize(self) -> None:
        self.lib.call("prism_device_synchronize", self.h)

    def stream(self) -> int:
        return self.lib.prism_device_stream(self.h) or 0


class PagedOp:
    """Pool-level K2 / K3 over caller-owned block tables (C-ABI prism_paged_*;
    SURVEY §8b's suggested kv_append / decode_attn): for an engine with its
    own scheduler. Slot ids are page * tokens_per_page + slot of handles from
    alloc_kv. Pointers are integers (``tensor.data_ptr()``); everything runs on
    the pool's device stream (``Device.stream()``)."""

    def __init__(self, pool: KvPool, n_layers: int, n_q_heads: int, n_kv_heads: int, head_dim: int):
        self.lib, self.pool = pool.lib, pool  # the pool outlives this op
        self.h = C.c_void_p()
        self.lib.call("prism_paged_create", pool.h, n_layers, n_q_heads, n_kv_heads, head_dim, C.byref(self.h))

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.lib.prism_paged_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def kv_append(self, layer_begin: int, layer_end: int, slots: int, n_tokens: int, k: int, v: int) -> None:
        """K2: slots device int32 [n_tokens]; k / v device bf16 [layers][n_tokens][n_kv][head_dim]."""
        self.lib.call("prism_paged_kv_append", self.h, layer_begin, layer_end, C.c_void_p(slots), n_tokens,
                      C.c_void_p(k), C.c_void_p(v))

    def prefill_attention(self, layer: int, slot_ids: int, first: int, n_tokens: int, q: int, out: int,
                          scale: float) -> None:
        """K4: one request's chunk; slot_ids = its keys 0 .. first + n_tokens - 1 (device int32)."""
        self.lib.call("prism_paged_prefill_attention", self.h, layer, C.c_void_p(slot_ids), first, n_tokens,
                      C.c_void_p(q), C.c_void_p(out), scale)

    def decode_attention(self, layer: int, seq_offsets: Sequence[int], slot_ids: int, q: int, out: int,
                         scale: float) -> None:
        """K3: seq_offsets (host) [n_seqs + 1] into the device slot-id array."""
        n = len(seq_offsets) - 1
        offs = (C.c_int32 * len(seq_offsets))(*seq_offsets)
        self.lib.call("prism_paged_decode_attention", self.h, layer, offs, n, C.c_void_p(slot_ids), C.c_void_p(q),
                      C.c_void_p(out), scale)


# ---------------------------------------------------------------- weight loading


class WeightLoader:
    """prism::WeightLoader — model weight loading for activation (SURVEY
    §8f-2; replaces the modelled
    ActivationParams::load_latency_s, reference engine.hpp:46-48 /
    src/engine.cpp:44-51). Pointers are plain integers (device or pinned
    host addresses, e.g. ``tensor.data_ptr()``); every load is enqueued on the
    loader's own streams and ``wait()`` returns its device milliseconds."""

    def __init__(self, device: int = 0, n_streams: int = 4, chunk_bytes: int = 8 << 20, lib=None):
        self.lib = _lib(lib)
        if not self.lib.has_device:
            raise capi.CudaError(5, f"{self.lib.path} has no GPU data path")
        self.device = device
        self.h = C.c_void_p()
        self.lib.call("prism_wloader_create", device, n_streams, chunk_bytes, C.byref(self.h))

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.lib.prism_wloader_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, host: int, dst: int, nbytes: int) -> None:
        """Chunked load, chunks round-robin over the loader's streams."""
        self.lib.call("prism_wloader_load", self.h, C.c_void_p(host), C.c_void_p(dst), nbytes)

    def load_naive(self, host: int, dst: int, nbytes: int) -> None:
        """Baseline: one cudaMemcpyAsync."""
        self.lib.call("prism_wloader_load_naive", self.h, C.c_void_p(host), C.c_void_p(dst), nbytes)

    def load_part(self, host: int, dst: int, nbytes: int, part: int, n_parts: int) -> None:
        """Fan-in helper: chunks i % n_parts == part through this GPU's staging into dst (any GPU)."""
        self.lib.call("prism_wloader_load_part", self.h, C.c_void_p(host), C.c_void_p(dst), nbytes, part, n_parts)

    def wait(self) -> float:
        ms = C.c_double()
        self.lib.call("prism_wloader_wait", self.h, C.byref(ms))
        return ms.value


def ipc_handle(dptr: int, lib=None) -> bytes:
    """64-byte CUDA IPC handle of a cudaMalloc'ed device pointer."""
    lib = _lib(lib)
    buf = (C.c_ubyte * 64)()
    lib.call("prism_ipc_handle", C.c_void_p(dptr), buf)
    return bytes(buf)


def ipc_open(device: int, handle: bytes, lib=None) -> int:
    lib = _lib(lib)
    buf = (C.c_ubyte * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    lib.call("prism_ipc_open", device, buf, C.byref(p))
    return p.value


def ipc_close(device: int, dptr: int, lib=None) -> None:
    _lib(lib).call("prism_ipc_close", device, C.c_void_p(dptr))


def fanin_parts(n_bytes: int, chunk_bytes: int, n_parts: int) -> list:
    """Which byte ranges each helper of an n_parts fan-in copies (chunk i goes
    to part i % n_parts) — the plan WeightLoader.load_part executes; every
    byte is covered exactly once."""
    parts = [[] for _ in range(n_parts)]
    for i, off in enumerate(range(0, n_bytes, chunk_bytes)):
        parts[i % n_parts].append((off, min(chunk_bytes, n_bytes - off)))
    return parts


def measured_activation_curve(gbs: float, fixed_s: float = 0.0, sizes=(16e9, 28e9)) -> list:
    """ActivationParams.parallel_curve points (weight bytes, seconds) from a
    measured load bandwidth: seconds = fixed_s + bytes / (gbs * 1e9); the
    reference interpolates linearly between such anchors
    (src/engine.cpp:44-51)."""
    return [(float(b), fixed_s + float(b) / (gbs * 1e9)) for b in sizes]


# ---------------------------------------------------------------- schedulers


@dataclass
class ResidentModel:
    idle_s: float = 0.0
    ttft_slo_s: float = 0.0
    weight_bytes: int = 0
    weight_pages: int = 0


@dataclass
class GpuViewPy:
    gpu_id: int = 0
    capacity_bytes: int = 0
    weight_bytes: int = 0
    w_req_rate: float = 0.0
    capacity_pages: int = 0
    free_pages: int = 0
    page_bytes: int = PAGE_BYTES
    residents: dict = field(default_factory=dict)


@dataclass
class ModelDemandPy:
    spec: ModelSpec
    rate: float = 0.0
    current_gpus: list = field(default_factory=list)


@dataclass
class PlacementPlan:
    assignment: dict
    migrations: list
    kvpr_before: list
    kvpr_after: list
    max_kvpr_after: float
    critical_gpu: int
    critical_shared_before_bytes: float
    critical_last_weight_bytes: float


def _views(gpus: Sequence[GpuViewPy]):
    keep = []
    arr = (capi.GpuView * max(len(gpus), 1))()
    for i, g in enumerate(gpus):
        res = (capi.Resident * max(len(g.residents), 1))()
        for j, (mid, r) in enumerate(sorted(g.residents.items())):
            b = mid.encode()
            keep.append(b)
            res[j] = capi.Resident(b, r.idle_s, r.ttft_slo_s, r.weight_bytes, r.weight_pages)
        keep.append(res)
        arr[i] = capi.GpuView(g.gpu_id, g.capacity_bytes, g.weight_bytes, g.w_req_rate, g.capacity_pages,
                              g.free_pages, g.page_bytes, res, len(g.residents))
    return arr, keep


def kvpr(w_req_rate: float, shared_kv_bytes: float, lib=None) -> float:
    v = C.c_double()
    _lib(lib).call("prism_kvpr", w_req_rate, shared_kv_bytes, C.byref(v))
    return v.value


def place_models(models: Sequence[ModelDemandPy], gpus: Sequence[GpuViewPy], tau_per_gb: float,
                 lib=None) -> PlacementPlan:
    lib = _lib(lib)
    keep = []
    marr = (capi.ModelDemand * max(len(models), 1))()
    total_parts = 0
    for i, m in enumerate(models):
        cur = (C.c_int32 * max(len(m.current_gpus), 1))(*m.current_gpus)
        keep.append(cur)
        cs = m.spec.to_c()
        keep.append(m.spec)
        marr[i] = capi.ModelDemand(cs, m.rate, cur, len(m.current_gpus))
        total_parts += max(1, m.spec.tp_degree)
    garr, gkeep = _views(gpus)
    n = len(gpus)
    assign = (C.c_int32 * max(total_parts, 1))()
    before = (C.c_double * max(n, 1))()
    after = (C.c_double * max(n, 1))()
    migs = (capi.Migration * max(total_parts, 1))()
    info = capi.PlanInfo()
    lib.call("prism_place_models", marr, len(models), garr, n, tau_per_gb, assign, total_parts, before, after, migs,
             total_parts, C.byref(info))
    out, off = {}, 0
    for m in models:
        tp = max(1, m.spec.tp_degree)
        out[m.spec.model_id] = list(assign[off:off + tp])
        off += tp
    migrations = [(models[x.model_index].spec.model_id, x.part_index, x.from_gpu, x.to_gpu)
                  for x in migs[:info.n_migrations]]
    return PlacementPlan(out, migrations, list(before[:n]), list(after[:n]), info.max_kvpr_after, info.critical_gpu,
                         info.critical_shared_before_bytes, info.critical_last_weight_bytes)


def eviction_tick(gpus: Sequence[GpuViewPy], idle_threshold_s: float, min_free_pages: int, lib=None) -> list:
    lib = _lib(lib)
    garr, keep = _views(gpus)
    n = C.c_size_t()
    cap = 2 * sum(len(g.residents) for g in gpus) + 2
    out = (C.c_int32 * cap)()
    lib.call("prism_eviction_tick", garr, len(gpus), idle_threshold_s, min_free_pages, out, cap, C.byref(n))
    res = []
    for k in range(n.value):
        g = gpus[out[2 * k]]
        res.append((g.gpu_id, sorted(g.residents)[out[2 * k + 1]]))
    return res


def activate_on_arrival(spec: ModelSpec, gpus: Sequence[GpuViewPy], lib=None):
    lib = _lib(lib)
    garr, keep = _views(gpus)
    g, found = C.c_int32(), C.c_int()
    cs = spec.to_c()
    lib.call("prism_activate_on_arrival", C.byref(cs), garr, len(gpus), C.byref(g), C.byref(found))
    return g.value if found.value else None


def activate_on_arrival_tp(spec: ModelSpec, gpus: Sequence[GpuViewPy], lib=None):
    lib = _lib(lib)
    garr, keep = _views(gpus)
    out = (C.c_int32 * max(spec.tp_degree, 1))()
    found = C.c_int()
    cs = spec.to_c()
    lib.call("prism_activate_on_arrival_tp", C.byref(cs), garr, len(gpus), out, max(spec.tp_degree, 1),
             C.byref(found))
    return list(out[:max(spec.tp_degree, 1)]) if found.value else None


@dataclass
class QueuedRequest:
    id: int
    model_id: str = "m"
    arrival_s: float = 0.0
    prompt_tokens: int = 0
    ttft_slo_s: float = 0.0
    exec_estimate_s: float = 0.0

    def deadline_s(self) -> float:
        return self.arrival_s + self.ttft_slo_s


def _qarr(reqs: Sequence[QueuedRequest]):
    keep = [r.model_id.encode() for r in reqs]
    arr = (capi.QueuedRequest * max(len(reqs), 1))()
    for i, r in enumerate(reqs):
        arr[i] = capi.QueuedRequest(r.id, keep[i], r.arrival_s, r.prompt_tokens, r.ttft_slo_s, r.exec_estimate_s)
    return arr, keep


def moore_hodgson(queue: Sequence[QueuedRequest], now_s: float, lib=None):
    """Returns (admit, deferred) lists of QueuedRequest (admission.hpp:30)."""
    lib = _lib(lib)
    arr, keep = _qarr(queue)
    n = len(queue)
    a = (C.c_int32 * max(n, 1))()
    d = (C.c_int32 * max(n, 1))()
    na, nd = C.c_size_t(), C.c_size_t()
    lib.call("prism_moore_hodgson", arr, n, now_s, a, C.byref(na), d, C.byref(nd))
    return [queue[i] for i in a[:na.value]], [queue[i] for i in d[:nd.value]]


def dispatch(admit: Sequence[QueuedRequest], gate, lib=None) -> list:
    lib = _lib(lib)
    arr, keep = _qarr(admit)
    idx = (C.c_int32 * max(len(admit), 1))(*range(len(admit)))

    def _gate(_ctx, rp):
        r = rp.contents
        return int(gate(QueuedRequest(r.id, r.model_id.decode(), r.arrival_s, r.prompt_tokens, r.ttft_slo_s,
                                      r.exec_estimate_s)))

    cb = capi.GATE(_gate)
    out = (C.c_uint64 * max(len(admit), 1))()
    n = C.c_size_t()
    lib.call("prism_dispatch", arr, idx, len(admit), cb, None, out, C.byref(n))
    return list(out[:n.value])


def requeue_deferred(deferred: Sequence[QueuedRequest], queue: Sequence[QueuedRequest], lib=None) -> list:
    lib = _lib(lib)
    darr, k1 = _qarr(deferred)
    qarr, k2 = _qarr(queue)
    out = (C.c_int32 * max(len(deferred) + len(queue), 1))()
    n = C.c_size_t()
    lib.call("prism_requeue_deferred", darr, len(deferred), qarr, len(queue), out, C.byref(n))
    both = list(queue) + list(deferred)
    return [both[i] for i in out[:n.value]]


# ---------------------------------------------------------------- workload


@dataclass(frozen=True)
class TraceEvent:
    arrival_s: float
    model_id: str
    prompt_tokens: int
    output_tokens: int


@dataclass
class ModelProfile:
    model_id: str
    segments: list  # (start_s, end_s, rate_per_s)
    prompt_median: float = 512.0
    prompt_sigma: float = 0.4
    output_median: float = 128.0
    output_sigma: float = 0.4


def _events(buf, n) -> list:
    return [TraceEvent(e.arrival_s, e.model_id.decode(), e.prompt_tokens, e.output_tokens) for e in buf[:n]]


def synth_trace(profiles: Sequence[ModelProfile], seed: int, lib=None) -> list:
    lib = _lib(lib)
    keep = []
    parr = (capi.ModelProfile * max(len(profiles), 1))()
    for i, p in enumerate(profiles):
        segs = (capi.RateSegment * max(len(p.segments), 1))(*[capi.RateSegment(*s) for s in p.segments])
        mid = p.model_id.encode()
        keep += [segs, mid]
        parr[i] = capi.ModelProfile(mid, segs, len(p.segments), p.prompt_median, p.prompt_sigma, p.output_median,
                                    p.output_sigma)
    n = C.c_size_t()
    lib.call("prism_synth_trace", parr, len(profiles), seed, None, 0, C.byref(n))
    buf = (capi.TraceEvent * max(n.value, 1))()
    lib.call("prism_synth_trace", parr, len(profiles), seed, buf, n.value, C.byref(n))
    return _events(buf, n.value)


def scale_trace(trace: Sequence[TraceEvent], factor: int, seed: int, jitter_window_s: float = 1.0, lib=None) -> list:
    lib = _lib(lib)
    arr = (capi.TraceEvent * max(len(trace), 1))()
    for i, e in enumerate(trace):
        arr[i] = capi.TraceEvent(e.arrival_s, e.model_id.encode(), e.prompt_tokens, e.output_tokens)
    cap = max(len(trace) * max(factor, 1), 1)
    out = (capi.TraceEvent * cap)()
    n = C.c_size_t()
    lib.call("prism_scale_trace", arr, len(trace), factor, seed, jitter_window_s, out, cap, C.byref(n))
    return _events(out, n.value)


def parse_trace_lines(text: str, origin: str = "mem", lib=None) -> list:
    lib = _lib(lib)
    n = C.c_size_t()
    lib.call("prism_parse_trace_text", text.encode(), origin.encode(), None, 0, C.byref(n))
    buf = (capi.TraceEvent * max(n.value, 1))()
    lib.call("prism_parse_trace_text", text.encode(), origin.encode(), buf, n.value, C.byref(n))
    return _events(buf, n.value)


# ---------------------------------------------------------------- simcore


@dataclass
class SimConfig:
    """msim::simcore::SimConfig (include/msim/simcore.hpp); defaults = the
    reference's defaults.hpp (tick 10 s, idle eviction 10 s, pressure 10%,
    tau 0.05, buffer 8 pages)."""

    n_gpus: int = 1
    capacity_pages: int = 0
    page_bytes: int = 2 << 20
    policy: str = "prism"  # | "mux_flexible" | "static_partition" | "qlm_timeshare"
    params: EngineParams = field(default_factory=EngineParams)
    parallel_activation: bool = True
    tau_per_gb: float = 0.05
    tick_s: float = 10.0
    idle_evict_s: float = 10.0
    pressure_free_frac: float = 0.10
    buffer_target_pages: int = 8
    initial_placement: bool = True
    max_events: int = 200_000_000
    # measured weight-load bandwidth (GB/s) replacing the modelled activation
    # curves (WeightLoader; 0 = the reference's curves) + fixed s per load
    parallel_load_gbs: float = 0.0
    naive_load_gbs: float = 0.0
    load_fixed_s: float = 0.0
    local_scheduler: str = "moore_hodgson"  # Algorithm 2, or "fifo" (per-model FIFO into engine queues)


class SimResult:
    """A finished simcore run: summary, per-request records, attainment."""

    def __init__(self, lib, h):
        self.lib, self.h = lib, h
        s = capi.SimSummary()
        lib.call("prism_sim_summary_get", h, C.byref(s))
        self.summary = {f: getattr(s, f) for f, _ in capi.SimSummary._fields_}
        n = C.c_size_t()
        lib.call("prism_sim_requests", h, None, 0, C.byref(n))
        buf = (capi.SimRequest * max(n.value, 1))()
        lib.call("prism_sim_requests", h, buf, n.value, C.byref(n))
        self.requests = [{f: getattr(r, f) for f, _ in capi.SimRequest._fields_} for r in buf[:n.value]]
        lib.call("prism_sim_gpu_busy", h, None, 0, C.byref(n))
        busy = (C.c_int64 * max(n.value, 1))()
        lib.call("prism_sim_gpu_busy", h, busy, n.value, C.byref(n))
        self.gpu_busy_us = list(busy[:n.value])

    def attainment(self, slo_scale: float = 1.0, model_id: str = "") -> dict:
        t, p, b, n = C.c_double(), C.c_double(), C.c_double(), C.c_uint64()
        self.lib.call("prism_sim_attainment", self.h, model_id.encode(), slo_scale, C.byref(t), C.byref(p),
                      C.byref(b), C.byref(n))
        return {"ttft": t.value, "tpot": p.value, "both": b.value, "n": n.value}

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.dll.prism_sim_free(self.h)
            self.h = None


def simulate(cfg: SimConfig, models: Sequence, trace: Sequence[TraceEvent], lib=None, serving=None) -> SimResult:
    """msim::simcore::run. models: (ModelSpec, rate) pairs; rate = demand
    for the initial placement. serving: a ServingConfig to drive the GPU data
    path with the same event loop (prism_sim_run_device, product only)."""
    lib = _lib(lib)
    c = capi.SimConfig()
    lib.dll.prism_default_sim_config(C.byref(c))
    c.policy = {"prism": 0, "mux_flexible": 1, "static_partition": 2, "qlm_timeshare": 3}[cfg.policy]
    c.n_gpus, c.capacity_pages, c.page_bytes = cfg.n_gpus, cfg.capacity_pages, cfg.page_bytes
    c.params = cfg.params.to_c()
    c.method = 1 if cfg.parallel_activation else 0
    c.tau_per_gb, c.tick_s, c.idle_evict_s = cfg.tau_per_gb, cfg.tick_s, cfg.idle_evict_s
    c.pressure_free_frac, c.buffer_target_pages = cfg.pressure_free_frac, cfg.buffer_target_pages
    c.initial_placement, c.max_events = int(cfg.initial_placement), cfg.max_events
    c.parallel_load_gbs, c.naive_load_gbs, c.load_fixed_s = cfg.parallel_load_gbs, cfg.naive_load_gbs, cfg.load_fixed_s
    c.local_scheduler = {"moore_hodgson": 0, "fifo": 1}[cfg.local_scheduler]
    specs = (capi.ModelSpec * max(len(models), 1))(*[m[0].to_c() for m in models])
    rates = (C.c_double * max(len(models), 1))(*[m[1] for m in models])
    arr = (capi.TraceEvent * max(len(trace), 1))()
    for i, e in enumerate(trace):
        arr[i] = capi.TraceEvent(e.arrival_s, e.model_id.encode(), e.prompt_tokens, e.output_tokens)
    h = C.c_void_p()
    if serving is None:
        lib.call("prism_sim_run", C.byref(c), specs, rates, len(models), arr, len(trace), C.byref(h))
        return SimResult(lib, h)
    o = capi.ServingOptions()
    o.measured = int(serving.measured)
    o.seed = serving.seed
    ords = (C.c_int32 * max(len(serving.ordinals), 1))(*serving.ordinals)
    owned = (C.c_int32 * max(len(serving.owned), 1))(*serving.owned)
    o.ordinals, o.n_ordinals = ords, len(serving.ordinals)
    o.owned, o.n_owned = owned, len(serving.owned)
    o.max_decode_batch, o.chunk_pages = serving.max_decode_batch, serving.chunk_pages
    lib.call("prism_sim_run_device", C.byref(c), specs, rates, len(models), arr, len(trace), C.byref(o), C.byref(h))
    res = SimResult(lib, h)
    st = capi.ServingStats()
    lib.call("prism_sim_serving_get", h, C.byref(st))
    res.serving = {f: getattr(st, f) for f, _ in capi.ServingStats._fields_}
    return res


@dataclass
class ServingConfig:
    """prism_serving_options: simcore's event loop driving the GPU data path
    (every iteration runs K1 / K2 / K4 / K3 on the device). measured=False:
    iterations are charged their modelled duration (records equal the
    host-only run); True: the measured GPU time of the iteration's kernels."""
    measured: bool = False
    seed: int = 20251017
    ordinals: list = field(default_factory=lambda: [0])
    owned: list = field(default_factory=list)  # simulated GPUs executed on a device (empty: all)
    max_decode_batch: int = 512
    chunk_pages: int = 0
