"""simcore (include/msim/simcore.hpp): the deterministic discrete-event driver
the reference specifies but does not implement.

Parity: simcore.cpp uses only the public msim:: API and is compiled into both
the product library and the oracle library built from the reference's own
sources (oracle/Makefile); the same configuration must give identical
per-request records and counters on both. Properties from SPEC's simcore
module: determinism, conservation (every request completes), causality
(arrival <= first token <= completion, TTFT >= one prefill chunk), attainment
in [0, 1], non-decreasing in the SLO scale and 1.0 as it grows without bound,
and (on the config-5 shape) non-decreasing in the GPU count.
"""
import pytest

from paper_2505_04021_b200 import msim
from tests import scenarios as S

from paper_2505_04021_b200.configs import B200_LEDGER_PAGES as LEDGER_PAGES, c5_case, slo_models as _models
from paper_2505_04021_b200.configs import slo_of as _slo


def _run(lib, n_gpus, models, trace, capacity=LEDGER_PAGES, **kw):
    cfg = msim.SimConfig(n_gpus=n_gpus, capacity_pages=capacity, **kw)
    return msim.simulate(cfg, models, trace, lib=lib)


def _c1(lib):
    specs = _models(1, ["llama3.1-8b"])
    a, b = specs[0], S.shape_spec("llama3.1-8b", "llama3.1-8b#1", chunk=512, ttft=_slo("llama3.1-8b")[0])
    b.tpot_slo_s = a.tpot_slo_s
    prof = [msim.ModelProfile(s.model_id, [(0.0, 30.0, 6.0)], 1024.0, 0.3, 128.0, 0.4) for s in (a, b)]
    return [(a, 6.0), (b, 6.0)], msim.synth_trace(prof, 42, lib=lib)


def _c2(lib):
    specs = _models(1)
    prof = []
    for i, s in enumerate(specs):
        segs = [(t, t + 10.0, 3.0) for t in range(10 * (i % 2), 80, 20)]
        prof.append(msim.ModelProfile(s.model_id, segs, 256.0, 0.6, 64.0, 0.6))
    return [(s, 1.5) for s in specs], msim.synth_trace(prof, 42, lib=lib)


def _c5(lib, copies=2, horizon=180.0):
    models, prof = c5_case(copies=copies, horizon=horizon)
    return models, msim.synth_trace(prof, 42, lib=lib)


def _check_invariants(res, trace):
    s = res.summary
    assert not s["truncated"]
    assert s["n_requests"] == len(trace) == s["completed"]
    for r in res.requests:
        assert r["arrival_us"] <= r["first_token_us"] <= r["completion_us"]
        assert r["gpu"] >= 0
    prev = None
    for scale in (0.1, 0.5, 1.0, 2.0, 10.0, 1e9):
        a = res.attainment(scale)
        assert 0.0 <= a["both"] <= min(a["ttft"], a["tpot"]) <= 1.0
        if prev:
            assert a["ttft"] >= prev["ttft"] and a["tpot"] >= prev["tpot"] and a["both"] >= prev["both"]
        prev = a
    assert prev["both"] == 1.0


@pytest.mark.parametrize("local", ["moore_hodgson", "fifo"])
@pytest.mark.parametrize("case", ["c1", "c2", "c5x2"])
def test_product_matches_reference_build(product, reference, case, local):
    """Same simcore source over the reference's engine / placement /
    allocator / admission vs over the product's: identical records and
    counters, with Algorithm 2 (moore_hodgson -> dispatch gate ->
    requeue_deferred) and with per-model FIFO admission."""
    if case == "c1":
        models, trace = _c1(product)
        runs = [_run(lib, 1, models, trace, capacity=18_000, local_scheduler=local) for lib in (product, reference)]
    elif case == "c2":
        models, trace = _c2(product)
        runs = [_run(lib, 1, models, trace, capacity=37_000, local_scheduler=local) for lib in (product, reference)]
    else:
        models, trace = _c5(product, copies=2, horizon=120.0)
        runs = [_run(lib, 2, models, trace, capacity=24_000, local_scheduler=local) for lib in (product, reference)]
    if local == "moore_hodgson":
        assert runs[0].summary["dispatches"] == len(trace) and runs[0].summary["schedule_rounds"] > 0
    else:
        assert runs[0].summary["dispatches"] == 0
    a, b = runs
    assert a.summary == b.summary
    assert a.requests == b.requests
    assert a.gpu_busy_us == b.gpu_busy_us
    for scale in (0.5, 1.0, 4.0):
        assert a.attainment(scale) == b.attainment(scale)
    _check_invariants(a, trace)


def test_deterministic_and_conserving(product):
    models, trace = _c2(product)
    a = _run(product, 1, models, trace, capacity=37_000)
    b = _run(product, 1, models, trace, capacity=37_000)
    assert a.summary == b.summary and a.requests == b.requests
    _check_invariants(a, trace)
    # TTFT is at least one prefill chunk's modelled time (SPEC: TTFT >= p / c)
    p = msim.EngineParams()
    for r in a.requests:
        first_chunk = min(r["prompt_tokens"], 512)
        assert r["first_token_us"] - r["arrival_us"] >= int(p.alpha_ms * 1e3 + p.beta_ms_per_token * 1e3 * first_chunk) - 1


def test_pressure_forces_eviction_and_reactivation(product):
    """Config 5 on one GPU: the 16 models' weights exceed the ledger, so idle
    models are evicted and re-activated on arrival; all requests still
    complete."""
    models, trace = _c5(product, copies=2, horizon=180.0)
    weight_pages = sum((m.weight_bytes + (2 << 20) - 1) // (2 << 20) for m, _ in models)
    cap = weight_pages // 2
    res = _run(product, 1, models, trace, capacity=cap, idle_evict_s=5.0, tick_s=2.0)
    _check_invariants(res, trace)
    assert res.summary["evictions"] > 0
    assert res.summary["activations"] > len({m.model_id for m, _ in models}) // 2


def test_attainment_non_decreasing_in_gpu_count(product):
    """SPEC sweep(gpu_count): prism's attainment is non-decreasing in the GPU
    count (config-5 shape, 1 / 2 / 4 / 8 GPUs at the B200 ledger size)."""
    models, trace = _c5(product, copies=6, horizon=120.0)
    att = []
    for n in (1, 2, 4, 8):
        res = _run(product, n, models, trace)
        _check_invariants(res, trace)
        att.append(res.attainment(1.0)["both"])
    assert all(b >= a - 1e-12 for a, b in zip(att, att[1:])), att


def test_infeasible_config_raises(product):
    big = S.shape_spec("llama3.1-8b", "huge", chunk=512)
    big.weight_bytes = 400 << 30
    with pytest.raises(msim.capi.UsageError):
        _run(product, 1, [(big, 1.0)], [msim.TraceEvent(0.0, "huge", 10, 2)])
    spec = S.shape_spec("llama3.1-8b", "m", chunk=512)
    with pytest.raises(msim.capi.UsageError):
        _run(product, 1, [(spec, 1.0)], [msim.TraceEvent(0.0, "unknown", 10, 2)])


@pytest.mark.parametrize("policy", ["mux_flexible", "static_partition"])
def test_baseline_policies_match_reference_build(product, reference, policy):
    """SPEC policies module: the baselines run in the same harness; the
    reference-source build agrees record for record."""
    models, trace = _c2(product)
    a, b = (_run(lib, 1, models, trace, capacity=37_000, policy=policy) for lib in (product, reference))
    assert a.summary == b.summary and a.requests == b.requests
    _check_invariants(a, trace)
    assert a.summary["evictions"] == 0
    assert a.summary["activations"] == len(models)  # frozen colocation: placed once


def test_static_partition_cannot_borrow_idle_memory(product):
    """SPEC §3.2 behaviour: two llama-8B-shaped models on one GPU, A idle,
    B overloaded. static_partition caps B at half the KV pages (no borrowing)
    -> more preemptions than mux_flexible (shares on demand); prism also
    evicts the idle A under pressure and hands its weight pages to B."""
    specs = _models(2, ["llama3.1-8b"])
    a, b = specs
    prof = [msim.ModelProfile(b.model_id, [(0.0, 40.0, 8.0)], 1500.0, 0.3, 200.0, 0.3)]
    trace = msim.synth_trace(prof, 7, lib=product)
    models = [(a, 1.0), (b, 8.0)]
    runs = {p: _run(product, 1, models, trace, capacity=20_000, policy=p, tick_s=2.0, idle_evict_s=2.0)
            for p in ("prism", "mux_flexible", "static_partition")}
    for r in runs.values():
        _check_invariants(r, trace)
    assert runs["static_partition"].summary["preemptions"] > runs["mux_flexible"].summary["preemptions"]
    assert runs["prism"].summary["evictions"] >= 1
    for scale in (1.0, 4.0, 16.0):
        att = {p: r.attainment(scale)["both"] for p, r in runs.items()}
        assert att["prism"] > att["mux_flexible"] > att["static_partition"], (scale, att)


def test_frozen_policy_needs_everything_placed(product):
    models, trace = _c5(product, copies=6, horizon=60.0)
    with pytest.raises(msim.capi.UsageError):
        _run(product, 1, models, trace, policy="mux_flexible")


def test_qlm_timeshare_swaps(product, reference):
    """SPEC qlm_timeshare: alternating arrivals for two models on one GPU pay
    a swap on every alternation; a single-model workload pays none beyond
    the first load; the reference-source build agrees."""
    specs = _models(1, ["llama3.1-8b", "qwen2.5-7b"])
    alt = [msim.TraceEvent(2.0 + 30.0 * i, specs[i % 2].model_id, 200, 20) for i in range(6)]
    models = [(s, 1.0) for s in specs]
    a, b = (_run(lib, 1, models, alt, capacity=30_000, policy="qlm_timeshare") for lib in (product, reference))
    assert a.summary == b.summary and a.requests == b.requests
    _check_invariants(a, alt)
    assert a.summary["activations"] == 6 and a.summary["evictions"] == 5
    p = msim.EngineParams()
    for r in a.requests:  # every request waits for a stop-and-restart activation
        assert r["first_token_us"] - r["arrival_us"] >= int(p.engine_init_s * 1e6)
    one = [msim.TraceEvent(2.0 + 30.0 * i, specs[0].model_id, 200, 20) for i in range(6)]
    c = _run(product, 1, models, one, capacity=30_000, policy="qlm_timeshare")
    assert c.summary["activations"] == 1 and c.summary["evictions"] == 0
    # more GPUs with the same load: swaps do not decrease (SPEC, directional)
    two = _run(product, 2, models, alt, capacity=30_000, policy="qlm_timeshare")
    assert two.summary["activations"] >= 2


def test_measured_load_bandwidth_replaces_modelled_curve(product, reference):
    """a measured weight-load bandwidth (WeightLoader) replaces
    the modelled activation curve. Config 1's two models are activated at
    t = 0 (initial placement, parallel load), so the first request's TTFT
    moves by exactly the load-time difference between two bandwidths; the
    reference-source build agrees record for record."""
    models, trace = _c1(product)
    # FIFO admission isolates the load time (Algorithm 2 may reorder requests
    # whose deadlines passed during the load)
    kw = dict(capacity=18_000, local_scheduler="fifo")
    slow = _run(product, 1, models, trace, parallel_load_gbs=10.0, **kw)
    fast = _run(product, 1, models, trace, parallel_load_gbs=100.0, **kw)
    ref = _run(reference, 1, models, trace, parallel_load_gbs=10.0, **kw)
    assert slow.requests == ref.requests and slow.summary == ref.summary
    _check_invariants(slow, trace)
    _check_invariants(fast, trace)
    w = models[0][0].weight_bytes
    first = min(range(len(trace)), key=lambda i: trace[i].arrival_s)
    d = slow.requests[first]["first_token_us"] - fast.requests[first]["first_token_us"]
    assert d > 0
    assert abs(d - (w / 10e9 - w / 100e9) * 1e6) < 0.02 * (w / 10e9) * 1e6 + 10
    # the default (0) keeps the reference's modelled curve
    dflt = _run(product, 1, models, trace, capacity=18_000)
    base = _run(reference, 1, models, trace, capacity=18_000)
    assert dflt.requests == base.requests


def _priority_case(lib, seed):
    """SPEC.md:715 (acceptance 10): two colocated llama3.2-3b-shaped models
    on one GPU under memory pressure (300 KV pages beside the weights): a
    strict-SLO short-prompt model (TTFT 0.1 s, 128-token prompts, 25 req/s)
    and a loose-SLO long-prompt model (TTFT 5 s, 3,000-token prompts, 3
    req/s)."""
    strict = S.shape_spec("llama3.2-3b", "strict", chunk=512, ttft=0.1)
    loose = S.shape_spec("llama3.2-3b", "loose", chunk=512, ttft=5.0)
    strict.tpot_slo_s = loose.tpot_slo_s = 1.0
    prof = [msim.ModelProfile("strict", [(0.0, 60.0, 25.0)], 128.0, 0.3, 64.0, 0.4),
            msim.ModelProfile("loose", [(0.0, 60.0, 3.0)], 3000.0, 0.3, 256.0, 0.4)]
    trace = msim.synth_trace(prof, seed, lib=lib)
    return [(strict, 25.0), (loose, 3.0)], trace


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_local_scheduler_priority_effect(product, seed):
    """SPEC acceptance 10: enabling Algorithm 2 admission improves the
    strict-SLO model's TTFT attainment by >= 0.20 absolute versus per-model
    FIFO dispatch, without reducing the loose model's below FIFO - 0.05."""
    models, trace = _priority_case(product, seed)
    cap = 2 * 3067 + 300
    mh = _run(product, 1, models, trace, capacity=cap, local_scheduler="moore_hodgson")
    ff = _run(product, 1, models, trace, capacity=cap, local_scheduler="fifo")
    _check_invariants(mh, trace)
    _check_invariants(ff, trace)
    gain = mh.attainment(1.0, "strict")["ttft"] - ff.attainment(1.0, "strict")["ttft"]
    assert gain >= 0.20, gain
    assert mh.attainment(1.0, "loose")["ttft"] >= ff.attainment(1.0, "loose")["ttft"] - 0.05


def test_local_scheduler_priority_case_matches_reference_build(product, reference):
    models, trace = _priority_case(product, 3)
    a, b = (_run(lib, 1, models, trace, capacity=2 * 3067 + 300) for lib in (product, reference))
    assert a.summary == b.summary and a.requests == b.requests
