"""The C-ABI boundary: the product library loads without a GPU, exports every
entry point include/prism_capi.h declares, and fails loudly (status, not a
crash or a silent fallback) when a GPU entry point is used without CUDA."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2505_04021_b200 import capi, msim

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "prism_capi.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(prism_[a-z0-9_]+)\s*\(", text))
    names.discard("prism_dispatch_gate")  # typedef
    return sorted(names)


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_product_exports_every_declared_symbol(product):
    missing = [s for s in declared_symbols() if s not in exported(product.path)]
    assert not missing, f"declared in prism_capi.h but not exported: {missing}"


def test_binding_covers_header(product):
    bound = set(capi.HOST_SYMBOLS) | set(capi.DEVICE_SYMBOLS)
    assert set(declared_symbols()) == bound


def test_product_has_device_path_and_abi_version(product):
    assert product.prism_abi_version() == 1
    assert product.has_device


def test_reference_oracle_exports_host_subset(reference):
    syms = exported(reference.path)
    assert all(s in syms for s in capi.HOST_SYMBOLS)
    assert not any(s in syms for s in capi.DEVICE_SYMBOLS)
    assert not reference.has_device
    # only the C-ABI leaks out of the oracle library
    assert all(s.startswith("prism_") for s in syms if not s.startswith("_"))


def test_errors_map_to_status_codes(product):
    led = msim.PhysicalLedger(0, 4, lib=product)
    pool = msim.alloc_kvcache(led, "m", 16 << 10, 10)
    with pytest.raises(capi.UsageError):
        msim.alloc_kvcache(led, "m", 16 << 10, 10)
    with pytest.raises(capi.UsageError, match="stale"):
        msim.free_kv(pool, led, [msim.TokenSlotHandle(pool.id(), 0, 0)])
    with pytest.raises(capi.PrismError) as e:
        product.call("prism_ledger_create", 0, 1, 2 << 20, None)
    assert e.value.status == "ARG"
    with pytest.raises(capi.ParseError, match="mem:1"):
        msim.parse_trace_lines("{t: nope}", "mem", lib=product)


def test_gpu_entry_points_fail_loudly_without_cuda(product):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    rc = product.prism_device_open(0, 2 << 20, C.byref(h))
    assert rc == 5, rc  # PRISM_E_CUDA
    assert product.prism_last_error()


def test_package_fails_loudly_when_library_missing(tmp_path):
    with pytest.raises(FileNotFoundError):
        capi.load(str(tmp_path / "nope.so"))
