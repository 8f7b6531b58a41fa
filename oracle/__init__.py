"""Oracle loaders — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the timed CPU
baseline: the product (paper_2505_04021_b200) never imports it.

* ``reference()``   oracle/_ref/libmsim_ref.so — the reference's own C++
                    sources compiled behind the prism C-ABI (host subset).
* ``restate()``     oracle/_ref/libprism_oracle.so — the C restatement
                    (synthetic content, fp64 attention, naive allocator).
Both are built by ``make -C oracle`` (the reference half only where
/root/reference exists; the built .so files travel to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REFERENCE_LIB = os.path.join(REF_DIR, "libmsim_ref.so")
RESTATE_LIB = os.path.join(REF_DIR, "libprism_oracle.so")
REF_UNIT_REFERENCE = os.path.join(REF_DIR, "ref_unit_reference")
REF_UNIT_PRODUCT = os.path.join(REF_DIR, "ref_unit_product")

_restate = None
_reference = None


def have_reference() -> bool:
    return os.path.exists(REFERENCE_LIB)


def reference():
    """capi.Lib bound to the compiled reference (raises if not built)."""
    global _reference
    if _reference is None:
        from paper_2505_04021_b200 import capi

        _reference = capi.load(REFERENCE_LIB)
    return _reference


def restate():
    global _restate
    if _restate is None:
        if not os.path.exists(RESTATE_LIB):
            raise FileNotFoundError(f"{RESTATE_LIB} missing: run make -C oracle restate")
        lib = C.CDLL(RESTATE_LIB)
        lib.po_synth_bf16.restype = C.c_uint16
        lib.po_synth_bf16.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float]
        lib.po_bf16_to_float.restype = C.c_float
        lib.po_bf16_to_float.argtypes = [C.c_uint16]
        lib.po_decode_attention_synth.restype = None
        lib.po_decode_attention_synth.argtypes = [C.c_uint64, C.c_int, C.c_size_t, C.POINTER(C.c_uint64),
                                                  C.POINTER(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_float,
                                                  C.c_double, C.POINTER(C.c_double)]
        lib.po_decode_attention_dense.restype = None
        lib.po_decode_attention_dense.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                  C.c_int, C.c_double, C.POINTER(C.c_double)]
        lib.po_paged_attention_cpu.restype = None
        lib.po_paged_attention_cpu.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int,
                                               C.c_float, C.c_void_p, C.c_int]
        lib.po_pool_create.restype = C.c_void_p
        lib.po_pool_create.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_int]
        lib.po_pool_destroy.argtypes = [C.c_void_p]
        lib.po_alloc.restype = C.c_uint64
        lib.po_alloc.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        lib.po_free.restype = C.c_int64
        lib.po_free.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                C.c_size_t]
        lib.po_mapped.restype = C.c_uint64
        lib.po_mapped.argtypes = [C.c_void_p]
        lib.po_occupied.restype = C.c_uint64
        lib.po_occupied.argtypes = [C.c_void_p]
        lib.po_page_occupied.restype = C.c_uint32
        lib.po_page_occupied.argtypes = [C.c_void_p, C.c_uint32]
        _restate = lib
    return _restate


def synth_attention(seed: int, layer: int, req_ids, ctx_lens, n_q: int, n_kv: int, d: int, q_scale: float,
                    scale: float) -> np.ndarray:
    """fp64 oracle output [n_dec, n_q, d] for synthetic K/V/Q content."""
    lib = restate()
    req = np.ascontiguousarray(req_ids, dtype=np.uint64)
    ctx = np.ascontiguousarray(ctx_lens, dtype=np.int32)
    out = np.zeros((len(req), n_q, d), dtype=np.float64)
    lib.po_decode_attention_synth(seed, layer, len(req), req.ctypes.data_as(C.POINTER(C.c_uint64)),
                                  ctx.ctypes.data_as(C.POINTER(C.c_int32)), n_q, n_kv, d, q_scale, scale,
                                  out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def dense_attention(q_bf16: np.ndarray, k_bf16: np.ndarray, v_bf16: np.ndarray, scale: float) -> np.ndarray:
    """fp64 oracle for one request from explicit bf16 bit patterns (uint16):
    q [n_q, d], k/v [ctx, n_kv, d] -> out [n_q, d]."""
    lib = restate()
    q = np.ascontiguousarray(q_bf16, dtype=np.uint16)
    k = np.ascontiguousarray(k_bf16, dtype=np.uint16)
    v = np.ascontiguousarray(v_bf16, dtype=np.uint16)
    n_q, d = q.shape
    ctx, n_kv, _ = k.shape
    out = np.zeros((n_q, d), dtype=np.float64)
    lib.po_decode_attention_dense(q.ctypes.data, k.ctypes.data, v.ctypes.data, ctx, n_q, n_kv, d, scale,
                                  out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def synth_bf16(seed: int, req: int, pos: int, layer: int, kind: int, head: int, dim: int, scale: float = 1.0) -> int:
    return int(restate().po_synth_bf16(seed, req, pos, layer, kind, head, dim, scale))
