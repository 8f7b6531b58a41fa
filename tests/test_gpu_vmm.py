"""Elastic KV memory on real CUDA VMM: pages map on demand into each model's
reserved VA range, park when the ledger unmaps them (revived in place if the
same page is mapped again), and are stolen across models when the physical
budget (ledger capacity minus weights) is exhausted. Data written before a
park must survive a revive; pages moved between models must carry the new
owner's data — checked through K2 (append) and K3 (attention) against the
oracle."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2505_04021_b200 import msim
from tests import scenarios as S

pytestmark = pytest.mark.gpu
SEED = 4242


def _attn_ok(eng, spec):
    ids = eng.step_decode_ids()
    live = {r.id: r.live_slots() for r in eng.batch()}
    keep = [i for i, rid in enumerate(ids) if rid in live]
    if not keep:
        return
    q = torch.empty((len(ids), spec.n_q_heads, spec.head_dim), dtype=torch.bfloat16, device="cuda")
    o = torch.empty_like(q)
    scale = 1 / math.sqrt(spec.head_dim)
    eng.synth_q(1, SEED, 4.0, q.data_ptr())
    eng.decode_attention(1, q.data_ptr(), o.data_ptr(), scale)
    eng.synchronize()
    ref = oracle.synth_attention(SEED, 1, [ids[i] for i in keep], [live[ids[i]] for i in keep], spec.n_q_heads,
                                 spec.n_kv_heads, spec.head_dim, 4.0, scale)
    err = np.abs(o.float().cpu().numpy()[keep] - ref)
    assert (err <= 2e-3 + 1e-2 * np.abs(ref)).all(), err.max()


def test_map_park_revive_and_steal_across_models(product, device):
    cap = 24  # pages: two llama-8B-shaped models must trade physical pages
    gpu = msim.GpuState(0, cap, lib=product)
    gpu.ledger.attach_device(device)
    device.reset_stats()
    engines = []
    for mid in ("a", "b"):
        spec = S.shape_spec("llama3.1-8b", mid, chunk=128, weight_scale=0.0)
        act = gpu.activate(spec)
        gpu.finish_activation(act.engine_index)
        e = gpu.engine(act.engine_index)
        e.attach_device()
        engines.append((e, spec))
    rid = 0
    for rnd in range(6):
        # model (rnd % 2) runs a burst that needs most of the GPU, then drains
        e, spec = engines[rnd % 2]
        for _ in range(3):
            rid += 1
            e.push(rid, 90 + 7 * rnd, 12)
        steps = 0
        while sum(e.counts()) and steps < 400:
            e.step()
            e.append_kv_synthetic(0, spec.n_layers, SEED)
            steps += 1
            if steps % 5 == 0:
                _attn_ok(e, spec)
        assert sum(e.counts()) == 0
        assert gpu.ledger.mapped_pages() == 0
    st = device.stats()
    assert st["maps"] > 0 and st["unmaps"] == st["maps"]
    assert st["revived"] > 0, st          # same-model reuse needed no driver call
    assert st["steals"] > 0, st           # memory moved between the two models
    # never more physical pages than the budget allows
    assert st["creates"] <= cap, st


def test_weights_shrink_the_physical_budget(product, device):
    gpu = msim.GpuState(0, 40, lib=product)
    gpu.ledger.attach_device(device)
    spec = S.shape_spec("llama3.1-8b", "w1", chunk=512, weight_scale=0.0)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    e = gpu.engine(act.engine_index)
    e.attach_device()
    e.push(1, 500, 2)
    while sum(e.counts()):
        e.step()
    assert gpu.ledger.mapped_pages() == 0
    # 32 more weight pages: parked pages beyond the new budget are released
    assert gpu.ledger.reserve_weight_pages("big", 32)
    gpu.ledger.release_weight_pages("big")
