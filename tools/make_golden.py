"""Generate tests/golden/*.json from the compiled REFERENCE (oracle/_ref/
libmsim_ref.so, built by `make -C oracle` from /root/reference/proj/src).

The GPU box has no /root/reference, so parity there is anchored on these
committed fixtures. Every scenario is driven through the same C-ABI calls the
product exposes (paper_2505_04021_b200.msim with lib=reference). Large
streams are stored as sha256 digests plus a short prefix.

Run: python tools/make_golden.py   (requires oracle/_ref/libmsim_ref.so)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2505_04021_b200 import msim  # noqa: E402
from tests import scenarios  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def digest(values) -> str:
    h = hashlib.sha256()
    h.update(json.dumps(values, separators=(",", ":")).encode())
    return h.hexdigest()


def main() -> None:
    if not oracle.have_reference():
        raise SystemExit("oracle/_ref/libmsim_ref.so missing: run make -C oracle first")
    ref = oracle.reference()
    os.makedirs(OUT, exist_ok=True)
    golden = {
        "generator": "tools/make_golden.py",
        "reference": "/root/reference/proj/src (compiled by oracle/Makefile)",
        "allocator": [scenarios.allocator_fuzz(ref, **c) for c in scenarios.ALLOC_CASES],
        "allocator_known": scenarios.allocator_known_answers(ref),
        "engine": [scenarios.engine_trace(ref, **c) for c in scenarios.ENGINE_CASES],
        "placement": [scenarios.placement_case(ref, **c) for c in scenarios.PLACEMENT_CASES],
        "eviction": scenarios.eviction_cases(ref),
        "admission": [scenarios.admission_case(ref, **c) for c in scenarios.ADMISSION_CASES],
        "traces": [scenarios.trace_case(ref, **c) for c in scenarios.TRACE_CASES],
        "c1_full_ledger": {k: v for k, v in scenarios.c1_full_ledger(ref, **scenarios.C1_FULL).items()
                           if k not in ("engines", "gpu")},
    }
    path = os.path.join(OUT, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(golden, f, indent=1, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
