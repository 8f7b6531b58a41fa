"""The golden engine traces (C1, C1 under memory pressure with preemption,
C2 bursty 8 shapes, C3 long prompts) re-run with the GPU data path
attached: real VMM pages, K1 device slot allocation every step, K2 appends.
The host outcomes/events/tables must still equal the reference's golden
vectors, and the device's slot ids must equal the host handles every step."""
import json

import pytest

from paper_2505_04021_b200 import msim
from paper_2505_04021_b200.driver import TraceDriver
from tests import scenarios as S

pytestmark = pytest.mark.gpu
SEED = 99


def _run_with_device(product, device, name, seed, capacity, models, rate, horizon, prompt, output, chunk, steps,
                     weight_scale, bursty=False):
    gpu = msim.GpuState(0, capacity, lib=product)
    gpu.ledger.attach_device(device)
    gpu.ledger.set_recording(True)
    engines, layers, tpps = {}, {}, {}
    for shape, mid in models:
        spec = S.shape_spec(shape, mid, chunk=chunk, weight_scale=weight_scale)
        tpps[mid] = (2 << 20) // spec.token_kv_bytes
        act = gpu.activate(spec)
        gpu.finish_activation(act.engine_index)
        e = gpu.engine(act.engine_index)
        e.attach_device(max_step_tokens=chunk + 1 + 512)
        engines[mid] = e
        layers[mid] = spec.n_layers
    profiles = []
    for k, (shape, mid) in enumerate(models):
        if bursty:
            segs = [(t, t + 5.0, rate if (int(t // 5) + k) % 2 == 0 else 0.0) for t in range(0, int(horizon), 5)]
        else:
            segs = [(0.0, horizon, rate)]
        profiles.append(msim.ModelProfile(mid, segs, prompt[0], prompt[1], output[0], output[1]))
    trace = msim.synth_trace(profiles, seed, lib=product)
    checked = [0]

    def on_step(mid, e, o):
        e.append_kv_synthetic(0, layers[mid], SEED)
        slots = e.step_slots()  # raises if the device allocator diverged
        n_tok, _ = e.step_info()
        assert len(slots) == n_tok
        checked[0] += 1

    drv = TraceDriver(engines, trace, on_step=on_step)
    drv.run(steps)
    outcomes = [[mid, o.duration_us, o.chunk_tokens, o.decode_tokens, o.first_tokens, o.completions, o.preemptions,
                 o.pages_mapped_direct, o.prefill_paused] for mid, o in drv.outcomes]
    tables = {}
    for mid, e in engines.items():
        tpp = tpps[mid]
        for r in e.batch():
            buf, n = e.request_kv_raw(r.id)
            handles = [(s.page, s.slot) for s in buf[:n]]
            tables[str(r.id)] = S.digest(handles)
            assert e.table_row(r.table_row, n) == [p * tpp + s for p, s in handles]
    events = [[ev.time_us, ev.model_id, ev.kind, ev.pages] for ev in gpu.ledger.events()]
    return dict(outcome_digest=S.digest(outcomes), event_digest=S.digest(events),
                table_digest=S.digest(sorted(tables.items())), steps=checked[0])


@pytest.mark.parametrize("i", range(len(S.ENGINE_CASES)))
def test_golden_engine_trace_with_device(product, device, golden, i):
    case = S.ENGINE_CASES[i]
    got = _run_with_device(product, device, **case)
    ref = golden["engine"][i]
    assert got["outcome_digest"] == ref["outcome_digest"]
    assert got["event_digest"] == ref["event_digest"]
    assert got["table_digest"] == ref["table_digest"]
    assert got["steps"] == ref["summary"]["steps"]
    st = device.stats()
    assert st["maps"] >= st["unmaps"]
    json.dumps(st)
