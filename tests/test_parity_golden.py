"""Bit-exact parity of the product's host path (allocator, engine step,
placement, eviction, admission, traces) with the reference, anchored on the
committed golden vectors produced by the compiled reference
(tools/make_golden.py). Runs on CPU and on the GPU box (no /root/reference
needed)."""
import json

import pytest

from tests import scenarios as S


def _norm(x):
    return json.loads(json.dumps(x))


@pytest.mark.parametrize("i", range(len(S.ALLOC_CASES)))
def test_allocator_streams(product, golden, i):
    assert _norm(S.allocator_fuzz(product, **S.ALLOC_CASES[i])) == golden["allocator"][i]


def test_allocator_known_answers(product, golden):
    got = _norm(S.allocator_known_answers(product))
    assert got == golden["allocator_known"]
    # The reference floors tokens_per_page (48 KiB -> 42), against its own test's 43.
    assert got["tpp_48k"] == 42 and got["tpp_16k"] == 128
    assert got["most_occupied_pages"] == [0]
    assert got["shortfall"] == [2, 0, 0]
    assert got["buffer_hits"] == [3, 0, 5, 2, 0]


@pytest.mark.parametrize("i", range(len(S.ENGINE_CASES)))
def test_engine_traces(product, golden, i):
    got = _norm(S.engine_trace(product, **S.ENGINE_CASES[i]))
    assert got == golden["engine"][i]


def test_engine_pressure_case_exercises_preemption(golden):
    summary = {e["name"]: e["summary"] for e in golden["engine"]}
    assert summary["c1-pressure"]["preemptions"] > 0
    assert summary["c1-pressure"]["paused"] > 0


@pytest.mark.parametrize("i", range(len(S.PLACEMENT_CASES)))
def test_placement_plans(product, golden, i):
    assert _norm(S.placement_case(product, **S.PLACEMENT_CASES[i])) == golden["placement"][i]


def test_eviction_and_arrival(product, golden):
    assert _norm(S.eviction_cases(product)) == golden["eviction"]


@pytest.mark.parametrize("i", range(len(S.ADMISSION_CASES)))
def test_admission(product, golden, i):
    assert _norm(S.admission_case(product, **S.ADMISSION_CASES[i])) == golden["admission"][i]


@pytest.mark.parametrize("i", range(len(S.TRACE_CASES)))
def test_traces(product, golden, i):
    assert _norm(S.trace_case(product, **S.TRACE_CASES[i])) == golden["traces"][i]


def test_c1_full_b200_ledger(product, golden):
    """C1 exactly as bench.py times it, on the 85,830-page B200 ledger (every
    pool's V = 85,830): outcomes, per-step handle stream, events and block
    tables equal the compiled reference's."""
    got = S.c1_full_ledger(product, **S.C1_FULL)
    ref = golden["c1_full_ledger"]
    for k, v in ref.items():
        assert _norm(got[k]) == v, k
    assert ref["steps"] >= 2 * (64 + 50)
