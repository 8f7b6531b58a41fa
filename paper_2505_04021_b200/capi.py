"""ctypes binding of the prism-b200 C-ABI (include/prism_capi.h).

The same declarations bind two libraries that export the ABI:

* ``paper_2505_04021_b200/libprism_b200.so`` — the product (host C++ runtime,
  CUDA VMM, sm_100a kernels);
* ``oracle/_ref/libmsim_ref.so`` — the reference compiled from its own
  sources behind the same ABI (test oracle; host subset only).

This is also the reference-side binding a maintainer would add (see
INTEGRATION.md): the reference has no Python; the C-ABI is the boundary.
"""
from __future__ import annotations

import ctypes as C
import os
from ctypes import POINTER, byref, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_uint32
from ctypes import c_uint64, c_void_p

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
PRODUCT_LIB = os.path.join(PKG_DIR, "libprism_b200.so")
# A/B timing of two builds on one box (tools only): PRISM_PRODUCT_LIB names
# another build of the same sources; unset, the in-tree product is loaded.
PRODUCT_LIB = os.environ.get("PRISM_PRODUCT_LIB", PRODUCT_LIB)

PRISM_OK = 0
STATUS_NAMES = {0: "OK", 1: "USAGE", 2: "PARSE", 3: "CONFIG", 4: "PLACEMENT", 5: "CUDA", 6: "ARG", 7: "INTERNAL"}


class PrismError(RuntimeError):
    """A C-ABI call returned a non-zero status; ``status`` names the class."""

    def __init__(self, code: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {message}")
        self.code = code
        self.status = STATUS_NAMES.get(code, str(code))
        self.message = message


class UsageError(PrismError):
    pass


class ParseError(PrismError):
    pass


class PlacementError(PrismError):
    pass


class CudaError(PrismError):
    pass


_ERR_CLASS = {1: UsageError, 2: ParseError, 4: PlacementError, 5: CudaError}


class Slot(C.Structure):
    _fields_ = [("pool", c_uint32), ("page", c_uint32), ("slot", c_uint32)]


class AllocResult(C.Structure):
    _fields_ = [("shortfall_pages", c_uint64), ("pages_mapped", c_uint64), ("buffer_hits", c_uint64),
                ("n_handles", c_uint64)]


class Event(C.Structure):
    _fields_ = [("time_us", c_int64), ("gpu_id", c_int32), ("kind", c_int32), ("pages", c_uint64),
                ("model_id", C.c_char * 64)]


class LedgerStats(C.Structure):
    _fields_ = [(n, c_uint64) for n in ("capacity_pages", "mapped_pages", "buffer_pages", "weight_pages",
                                        "free_pages", "page_bytes")]


class PoolInfo(C.Structure):
    _fields_ = [("id", c_uint32), ("alive", c_int32)] + [
        (n, c_uint64) for n in ("token_bytes", "tokens_per_page", "virtual_capacity_pages", "mapped_pages",
                                "occupied_slots", "device_base")]


class ModelSpec(C.Structure):
    _fields_ = [("model_id", c_char_p), ("weight_bytes", c_uint64), ("token_kv_bytes", c_uint64),
                ("prefill_tps", c_double), ("chunk_size", c_int32), ("ttft_slo_s", c_double),
                ("tpot_slo_s", c_double), ("tp_degree", c_int32), ("n_layers", c_int32), ("n_q_heads", c_int32),
                ("n_kv_heads", c_int32), ("head_dim", c_int32)]


class EngineParams(C.Structure):
    _fields_ = [(n, c_double) for n in ("alpha_ms", "beta_ms_per_token", "map_latency_ms", "engine_init_s",
                                        "realign_s", "reserve_frac")]


class Activation(C.Structure):
    _fields_ = [("engine_index", c_int32), ("init_us", c_int64), ("realign_us", c_int64), ("load_us", c_int64)]


class Outcome(C.Structure):
    _fields_ = [("duration_us", c_int64), ("chunk_tokens", c_int32), ("decode_tokens", c_int32),
                ("pages_mapped_direct", c_uint64), ("prefill_paused", c_int32), ("n_first_tokens", c_uint32),
                ("n_completions", c_uint32), ("n_preemptions", c_uint32)]


class RequestInfo(C.Structure):
    _fields_ = [("id", c_uint64), ("prompt_tokens", c_int32), ("output_tokens", c_int32),
                ("prompt_done", c_int32), ("generated", c_int32), ("admit_seq", c_uint64), ("n_slots", c_uint64),
                ("table_row", c_int64)]


class ModelDemand(C.Structure):
    _fields_ = [("spec", ModelSpec), ("rate", c_double), ("current_gpus", POINTER(c_int32)),
                ("n_current", c_int32)]


class Resident(C.Structure):
    _fields_ = [("model_id", c_char_p), ("idle_s", c_double), ("ttft_slo_s", c_double),
                ("weight_bytes", c_uint64), ("weight_pages", c_uint64)]


class GpuView(C.Structure):
    _fields_ = [("gpu_id", c_int32), ("capacity_bytes", c_uint64), ("weight_bytes", c_uint64),
                ("w_req_rate", c_double), ("capacity_pages", c_uint64), ("free_pages", c_uint64),
                ("page_bytes", c_uint64), ("residents", POINTER(Resident)), ("n_residents", c_int32)]


class Migration(C.Structure):
    _fields_ = [("model_index", c_int32), ("part_index", c_int32), ("from_gpu", c_int32), ("to_gpu", c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("max_kvpr_after", c_double), ("critical_gpu", c_int32),
                ("critical_shared_before_bytes", c_double), ("critical_last_weight_bytes", c_double),
                ("n_migrations", c_uint32)]


class QueuedRequest(C.Structure):
    _fields_ = [("id", c_uint64), ("model_id", c_char_p), ("arrival_s", c_double), ("prompt_tokens", c_int32),
                ("ttft_slo_s", c_double), ("exec_estimate_s", c_double)]


class TraceEvent(C.Structure):
    _fields_ = [("arrival_s", c_double), ("model_id", C.c_char * 64), ("prompt_tokens", c_int32),
                ("output_tokens", c_int32)]


class SimConfig(C.Structure):
    _fields_ = [("policy", c_int32), ("n_gpus", c_int32), ("capacity_pages", c_uint64), ("page_bytes", c_uint64),
                ("params", EngineParams), ("method", c_int32), ("tau_per_gb", c_double), ("tick_s", c_double),
                ("idle_evict_s", c_double), ("pressure_free_frac", c_double), ("buffer_target_pages", c_uint64),
                ("initial_placement", c_int32), ("max_events", c_uint64), ("parallel_load_gbs", c_double),
                ("naive_load_gbs", c_double), ("load_fixed_s", c_double), ("local_scheduler", c_int32)]


class SimSummary(C.Structure):
    _fields_ = [("end_us", c_int64)] + [(n, c_uint64) for n in (
        "events", "iterations", "activations", "evictions", "preemptions", "output_tokens", "n_requests",
        "completed")] + [("truncated", c_int32), ("dispatches", c_uint64), ("schedule_rounds", c_uint64)]


class SimRequest(C.Structure):
    _fields_ = [("id", c_uint64), ("arrival_us", c_int64), ("first_token_us", c_int64),
                ("completion_us", c_int64), ("prompt_tokens", c_int32), ("output_tokens", c_int32),
                ("preemptions", c_int32), ("gpu", c_int32)]


class ServingOptions(C.Structure):
    _fields_ = [("measured", c_int32), ("seed", c_uint64), ("ordinals", C.POINTER(c_int32)), ("n_ordinals", c_size_t),
                ("owned", C.POINTER(c_int32)), ("n_owned", c_size_t), ("max_decode_batch", c_int32),
                ("chunk_pages", c_uint64)]


class ServingStats(C.Structure):
    _fields_ = [(n, c_uint64) for n in (
        "iterations", "attached", "detached", "k2_launches", "k3_launches", "k4_launches", "decode_tokens",
        "prefill_tokens", "gpu_us", "modelled_us", "vmm_maps", "vmm_unmaps", "vmm_revived", "vmm_creates",
        "vmm_driver_unmaps", "vmm_steals", "vmm_urgent")] + [(n, c_double) for n in (
        "vmm_caller_ns", "vmm_worker_ns", "wall_s")]


class RateSegment(C.Structure):
    _fields_ = [("start_s", c_double), ("end_s", c_double), ("rate_per_s", c_double)]


class ModelProfile(C.Structure):
    _fields_ = [("model_id", c_char_p), ("segments", POINTER(RateSegment)), ("n_segments", c_int32),
                ("prompt_median", c_double), ("prompt_sigma", c_double), ("output_median", c_double),
                ("output_sigma", c_double)]


class DeviceStats(C.Structure):
    _fields_ = [(n, c_uint64) for n in ("maps", "revived", "creates", "unmaps", "driver_unmaps")] + [
        (n, c_double) for n in ("map_ns_total", "unmap_ns_total", "map_ns_p50", "map_ns_p99", "unmap_ns_p50",
                                "unmap_ns_p99")] + [(n, c_uint64) for n in ("buffered", "cached", "pending")] + [
        (n, c_double) for n in ("create_ns_total", "map_call_ns_total", "access_ns_total")] + [
        ("access_calls", c_uint64), ("steals", c_uint64), ("steal_ns_total", c_double),
        ("background_ns_total", c_double)] + [(n, c_uint64) for n in ("premaps", "premapped_hits", "over_budget",
                                                                 "caller_steals_clean")] + [
        ("wait_ns_total", c_double), ("urgent", c_uint64), ("total_chunks", c_uint64), ("chunk_pages", c_uint64)] + [
        (n, c_double) for n in ("drv_map_ns_p50", "drv_map_ns_p99", "drv_create_ns_p50", "drv_create_ns_p99",
                                "drv_unmap_ns_p50", "drv_unmap_ns_p99")] + [("reserve_steals", c_uint64)]


class EngineDeviceOptions(C.Structure):
    _fields_ = [("table_capacity", c_int64), ("max_decode_batch", c_int32), ("max_step_tokens", c_int32)]


GATE = C.CFUNCTYPE(c_int, c_void_p, POINTER(QueuedRequest))

P = POINTER
_HOST_DECLS = {
    "prism_abi_version": (c_int, []),
    "prism_last_error": (c_char_p, []),
    "prism_has_device_path": (c_int, []),
    "prism_default_engine_params": (None, [P(EngineParams)]),
    "prism_default_model_spec": (None, [P(ModelSpec)]),
    "prism_ledger_create": (c_int, [c_int, c_uint64, c_uint64, P(c_void_p)]),
    "prism_ledger_destroy": (None, [c_void_p]),
    "prism_ledger_get_stats": (c_int, [c_void_p, P(LedgerStats)]),
    "prism_ledger_pool_mapped_pages": (c_int, [c_void_p, c_uint32, P(c_uint64)]),
    "prism_refill_buffer": (c_int, [c_void_p, c_uint64, P(c_uint64)]),
    "prism_ledger_reserve_weights": (c_int, [c_void_p, c_char_p, c_uint64, P(c_int)]),
    "prism_ledger_release_weights": (c_int, [c_void_p, c_char_p]),
    "prism_ledger_weight_pages_of": (c_int, [c_void_p, c_char_p, P(c_uint64)]),
    "prism_ledger_set_time": (c_int, [c_void_p, c_int64]),
    "prism_ledger_set_recording": (c_int, [c_void_p, c_int]),
    "prism_ledger_events": (c_int, [c_void_p, P(Event), c_size_t, P(c_size_t)]),
    "prism_ledger_clear_events": (c_int, [c_void_p]),
    "prism_ledger_check_invariants": (c_int, [c_void_p]),
    "prism_kvcache_alloc": (c_int, [c_void_p, c_char_p, c_uint64, c_uint64, c_int, P(c_void_p)]),
    "prism_kvcache_free": (c_int, [c_void_p, c_void_p]),
    "prism_pool_destroy": (None, [c_void_p]),
    "prism_pool_info_get": (c_int, [c_void_p, P(PoolInfo)]),
    "prism_kv_alloc": (c_int, [c_void_p, c_void_p, c_uint64, P(Slot), P(AllocResult)]),
    "prism_kv_free": (c_int, [c_void_p, c_void_p, P(Slot), c_size_t]),
    "prism_pool_allocatable_tokens": (c_int, [c_void_p, c_void_p, P(c_uint64)]),
    "prism_pool_page_occupied": (c_int, [c_void_p, c_uint32, P(c_uint64)]),
    "prism_pool_page_mapped": (c_int, [c_void_p, c_uint32, P(c_int)]),
    "prism_pool_set_cap": (c_int, [c_void_p, c_int64]),
    "prism_gpu_create": (c_int, [c_int, c_uint64, c_uint64, P(c_void_p)]),
    "prism_gpu_destroy": (None, [c_void_p]),
    "prism_gpu_ledger": (c_void_p, [c_void_p]),
    "prism_gpu_engine_count": (c_int, [c_void_p, P(c_int)]),
    "prism_gpu_activate": (c_int, [c_void_p, P(ModelSpec), c_int, P(EngineParams), P(Activation), P(c_int)]),
    "prism_gpu_finish_activation": (c_int, [c_void_p, c_int]),
    "prism_gpu_deactivate": (c_int, [c_void_p, c_int]),
    "prism_engine_status": (c_int, [c_void_p, c_int, P(c_int)]),
    "prism_engine_push": (c_int, [c_void_p, c_int, c_uint64, c_int, c_int]),
    "prism_engine_step": (c_int, [c_void_p, c_int, P(EngineParams), c_int64, P(Outcome)]),
    "prism_engine_outcome_ids": (c_int, [c_void_p, c_int, c_int, P(c_uint64), c_size_t, P(c_size_t)]),
    "prism_engine_counts": (c_int, [c_void_p, c_int, P(c_size_t), P(c_size_t)]),
    "prism_engine_request": (c_int, [c_void_p, c_int, c_int, c_size_t, P(RequestInfo)]),
    "prism_engine_request_kv": (c_int, [c_void_p, c_int, c_uint64, P(Slot), c_size_t, P(c_size_t)]),
    "prism_engine_mapped_pages": (c_int, [c_void_p, c_int, P(c_uint64)]),
    "prism_engine_next_chunk_need": (c_int, [c_void_p, c_int, P(c_uint64)]),
    "prism_engine_has_runnable_work": (c_int, [c_void_p, c_int, P(c_int)]),
    "prism_engine_reserved_pages": (c_int, [c_void_p, c_int, c_double, P(c_uint64)]),
    "prism_throughput_of": (c_int, [c_uint64, P(ModelSpec), c_int, c_int, P(EngineParams), c_uint64, c_double,
                                    c_double, P(c_double), P(c_int)]),
    "prism_kvpr": (c_int, [c_double, c_double, P(c_double)]),
    "prism_place_models": (c_int, [P(ModelDemand), c_size_t, P(GpuView), c_size_t, c_double, P(c_int32),
                                   c_size_t, P(c_double), P(c_double), P(Migration), c_size_t, P(PlanInfo)]),
    "prism_eviction_tick": (c_int, [P(GpuView), c_size_t, c_double, c_uint64, P(c_int32), c_size_t,
                                    P(c_size_t)]),
    "prism_activate_on_arrival": (c_int, [P(ModelSpec), P(GpuView), c_size_t, P(c_int32), P(c_int)]),
    "prism_activate_on_arrival_tp": (c_int, [P(ModelSpec), P(GpuView), c_size_t, P(c_int32), c_size_t,
                                             P(c_int)]),
    "prism_moore_hodgson": (c_int, [P(QueuedRequest), c_size_t, c_double, P(c_int32), P(c_size_t), P(c_int32),
                                    P(c_size_t)]),
    "prism_dispatch": (c_int, [P(QueuedRequest), P(c_int32), c_size_t, GATE, c_void_p, P(c_uint64),
                               P(c_size_t)]),
    "prism_requeue_deferred": (c_int, [P(QueuedRequest), c_size_t, P(QueuedRequest), c_size_t, P(c_int32),
                                       P(c_size_t)]),
    "prism_synth_trace": (c_int, [P(ModelProfile), c_size_t, c_uint64, P(TraceEvent), c_size_t, P(c_size_t)]),
    "prism_scale_trace": (c_int, [P(TraceEvent), c_size_t, c_int, c_uint64, c_double, P(TraceEvent), c_size_t,
                                  P(c_size_t)]),
    "prism_parse_trace_text": (c_int, [c_char_p, c_char_p, P(TraceEvent), c_size_t, P(c_size_t)]),
    "prism_default_sim_config": (None, [P(SimConfig)]),
    "prism_sim_run": (c_int, [P(SimConfig), P(ModelSpec), P(c_double), c_size_t, P(TraceEvent), c_size_t,
                              P(c_void_p)]),
    "prism_sim_summary_get": (c_int, [c_void_p, P(SimSummary)]),
    "prism_sim_requests": (c_int, [c_void_p, P(SimRequest), c_size_t, P(c_size_t)]),
    "prism_sim_gpu_busy": (c_int, [c_void_p, P(c_int64), c_size_t, P(c_size_t)]),
    "prism_sim_attainment": (c_int, [c_void_p, c_char_p, c_double, P(c_double), P(c_double), P(c_double),
                                     P(c_uint64)]),
    "prism_sim_free": (None, [c_void_p]),
    "prism_sim_serving_get": (c_int, [c_void_p, P(ServingStats)]),
}

_DEVICE_DECLS = {
    "prism_device_open": (c_int, [c_int, c_uint64, P(c_void_p)]),
    "prism_device_open_chunked": (c_int, [c_int, c_uint64, c_uint64, P(c_void_p)]),
    "prism_device_chunk_pages": (c_int, [c_void_p, P(c_uint64)]),
    "prism_device_close": (None, [c_void_p]),
    "prism_sim_run_device": (c_int, [P(SimConfig), P(ModelSpec), P(c_double), c_size_t, P(TraceEvent), c_size_t,
                                     P(ServingOptions), P(c_void_p)]),
    "prism_device_capacity_pages": (c_int, [c_void_p, c_uint64, P(c_uint64)]),
    "prism_device_stats_get": (c_int, [c_void_p, P(DeviceStats)]),
    "prism_device_reset_stats": (c_int, [c_void_p]),
    "prism_device_reclaim": (c_int, [c_void_p, c_int]),
    "prism_device_quiesce": (c_int, [c_void_p]),
    "prism_device_reserve": (c_int, [c_void_p, c_uint64]),
    "prism_device_fence": (c_int, [c_void_p]),
    "prism_device_synchronize": (c_int, [c_void_p]),
    "prism_device_stream": (c_void_p, [c_void_p]),
    "prism_ledger_attach_device": (c_int, [c_void_p, c_void_p]),
    "prism_pool_attach_mirror": (c_int, [c_void_p]),
    "prism_pool_sync_mirror": (c_int, [c_void_p, P(c_int32), c_size_t, P(c_size_t)]),
    "prism_pool_read_mirror": (c_int, [c_void_p, P(c_uint32), c_size_t, P(c_uint32), c_size_t]),
    "prism_engine_attach_device": (c_int, [c_void_p, c_int, P(EngineDeviceOptions)]),
    "prism_engine_step_info": (c_int, [c_void_p, c_int, P(c_int32), P(c_int32)]),
    "prism_engine_step_decode_ids": (c_int, [c_void_p, c_int, P(c_uint64), c_size_t, P(c_size_t)]),
    "prism_engine_step_slots": (c_int, [c_void_p, c_int, P(c_int32), c_size_t, P(c_size_t)]),
    "prism_engine_table_row": (c_int, [c_void_p, c_int, c_int64, c_int32, P(c_int32)]),
    "prism_engine_append_kv": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p]),
    "prism_engine_append_kv_synthetic": (c_int, [c_void_p, c_int, c_int, c_int, c_uint64]),
    "prism_engine_decode_attention": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_float, c_int32]),
    "prism_engine_prefill_info": (c_int, [c_void_p, c_int, P(c_int32), P(c_int32), P(c_uint64)]),
    "prism_engine_prefill_attention": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_float]),
    "prism_debug_k4_progress": (c_int, [P(c_uint32), c_int32, P(c_int32)]),
    "prism_debug_k4_trace": (c_int, [P(c_uint64), c_int32, P(c_int32)]),
    "prism_debug_k3_trace": (c_int, [P(c_uint64), c_int32, P(c_int32)]),
    "prism_engine_synth_q": (c_int, [c_void_p, c_int, c_int, c_uint64, c_float, c_void_p]),
    "prism_set_attention_variant": (c_int, [c_int]),
    "prism_engine_decode_host": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_float]),
    "prism_engine_synchronize": (c_int, [c_void_p, c_int]),
    "prism_engine_decode_host_async": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_float]),
    "prism_engine_wait_host": (c_int, [c_void_p, c_int]),
    "prism_paged_create": (c_int, [c_void_p, c_int, c_int, c_int, c_int, P(c_void_p)]),
    "prism_paged_destroy": (c_int, [c_void_p]),
    "prism_paged_kv_append": (c_int, [c_void_p, c_int, c_int, c_void_p, c_int32, c_void_p, c_void_p]),
    "prism_paged_prefill_attention": (c_int, [c_void_p, c_int, c_void_p, c_int32, c_int32, c_void_p, c_void_p,
                                              c_float]),
    "prism_paged_decode_attention": (c_int, [c_void_p, c_int, P(c_int32), c_int32, c_void_p, c_void_p, c_void_p,
                                             c_float]),
    "prism_wloader_create": (c_int, [c_int, c_int, c_uint64, P(c_void_p)]),
    "prism_wloader_destroy": (c_int, [c_void_p]),
    "prism_wloader_load": (c_int, [c_void_p, c_void_p, c_void_p, c_uint64]),
    "prism_wloader_load_naive": (c_int, [c_void_p, c_void_p, c_void_p, c_uint64]),
    "prism_wloader_load_part": (c_int, [c_void_p, c_void_p, c_void_p, c_uint64, c_int, c_int]),
    "prism_wloader_wait": (c_int, [c_void_p, P(c_double)]),
    "prism_host_register": (c_int, [c_void_p, c_uint64]),
    "prism_host_unregister": (c_int, [c_void_p]),
    "prism_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "prism_ipc_open": (c_int, [c_int, c_void_p, P(c_void_p)]),
    "prism_ipc_close": (c_int, [c_int, c_void_p]),
}

HOST_SYMBOLS = sorted(_HOST_DECLS)
DEVICE_SYMBOLS = sorted(_DEVICE_DECLS)


class Lib:
    """A loaded C-ABI library with checked calls: ``lib.call("prism_x", ...)``
    raises the PrismError subclass of a non-zero status."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} is missing — build it first (python -c 'import __graft_entry__ as g; g.build()' or make)")
        self.path = path
        self.dll = C.CDLL(path, mode=os.RTLD_LOCAL | os.RTLD_NOW)
        self.has_device = False
        for name, (res, args) in _HOST_DECLS.items():
            fn = getattr(self.dll, name)
            fn.restype = res
            fn.argtypes = args
        if int(self.dll.prism_has_device_path()):
            self.has_device = True
            for name, (res, args) in _DEVICE_DECLS.items():
                fn = getattr(self.dll, name)
                fn.restype = res
                fn.argtypes = args

    def __getattr__(self, name):
        return getattr(self.dll, name)

    def call(self, name: str, *args):
        rc = getattr(self.dll, name)(*args)
        if rc != PRISM_OK:
            msg = (self.dll.prism_last_error() or b"").decode(errors="replace")
            raise _ERR_CLASS.get(rc, PrismError)(rc, msg)
        return rc


_PRODUCT: Lib | None = None


def product() -> Lib:
    """The product library; raises if it has not been built (no fallback)."""
    global _PRODUCT
    if _PRODUCT is None:
        _PRODUCT = Lib(PRODUCT_LIB)
    return _PRODUCT


def load(path: str) -> Lib:
    return Lib(path)


__all__ = [n for n in dir() if not n.startswith("_")] + ["byref"]
