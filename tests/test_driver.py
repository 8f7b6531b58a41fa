"""TraceDriver (the composition loop the reference lacks) and its SLO metrics
(SPEC.md:523-526): TTFT = first token - arrival, TPOT = (completion - first
token) / (output - 1); attainment is monotone in the SLO scale."""
from paper_2505_04021_b200 import msim
from paper_2505_04021_b200.driver import TraceDriver
from tests import scenarios as S


def _run(capacity, rate):
    gpu = msim.GpuState(0, capacity)
    engines = {}
    for shape in ("llama3.1-8b", "qwen2.5-0.5b"):
        spec = S.shape_spec(shape, shape, chunk=256, weight_scale=0.0)
        act = gpu.activate(spec)
        gpu.finish_activation(act.engine_index)
        engines[shape] = gpu.engine(act.engine_index)
    trace = msim.synth_trace([msim.ModelProfile(s, [(0.0, 20.0, rate)], 700, 0.5, 80, 0.5) for s in engines], 7)
    drv = TraceDriver(engines, trace)
    drv.run(20000)
    return drv, trace


def test_all_requests_complete_and_metrics_are_consistent():
    drv, trace = _run(3000, 4.0)
    assert drv.next == len(trace)
    done = [r for r in drv.requests.values() if r[4] is not None]
    assert len(done) == len(trace)
    for mid, arr, n_out, first, comp in done:
        assert arr <= first <= comp
    slo = {m: 0.2 for m in drv.engines}
    tpot = {m: 0.02 for m in drv.engines}
    prev = None
    for scale in (0.25, 0.5, 1.0, 2.0, 8.0, 1e6):
        att = drv.slo_attainment(slo, tpot, scale)
        for m, v in att.items():
            assert 0.0 <= v["ttft"] <= 1.0 and 0.0 <= v["tpot"] <= 1.0
            if prev:
                assert v["ttft"] >= prev[m]["ttft"] and v["tpot"] >= prev[m]["tpot"]
        prev = att
    assert all(v["ttft"] == 1.0 and v["tpot"] == 1.0 for v in prev.values())


def test_pressure_causes_queueing_delay():
    light, _ = _run(3000, 1.0)
    heavy, _ = _run(260, 12.0)  # small ledger, high rate: pauses / preemptions
    slo = {m: 0.5 for m in light.engines}
    tpot = {m: 0.05 for m in light.engines}
    a = light.slo_attainment(slo, tpot)
    b = heavy.slo_attainment(slo, tpot)
    assert sum(v["ttft"] for v in b.values()) < sum(v["ttft"] for v in a.values())
    assert sum(len(o.preemptions) + int(o.prefill_paused) for _, o in heavy.outcomes) > 0
