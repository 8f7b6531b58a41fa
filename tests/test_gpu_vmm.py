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


def test_worker_premaps_the_next_pages(product, device):
    """A growing pool hands its next lowest unmapped pages to the device's
    worker thread, which maps their physical chunks ahead of need: the
    pool's next maps need no driver call."""
    K = device.chunk_pages()
    gpu = msim.GpuState(0, 400, lib=product)
    gpu.ledger.attach_device(device)
    pool = msim.alloc_kvcache(gpu.ledger, "pm", 131072, 400)  # 16 tokens per page
    device.reset_stats()
    first = msim.alloc_kv(pool, gpu.ledger, 16)  # maps page 0 (urgent chunk), hints the next pages
    device.quiesce()
    st = device.stats()
    # the look-ahead window: 256 pages with at most two pools on the device,
    # 128 with more (pools of earlier tests may still be alive on it)
    windows = [len({p // K for p in range(1, w + 1)} - {0}) for w in (256, 128)]
    assert st["maps"] == 1 and st["urgent"] == 1 and st["premaps"] in windows, st
    grow = msim.alloc_kv(pool, gpu.ledger, 8 * 16)  # pages 1..8
    st = device.stats()
    assert st["revived"] == 8 and st["urgent"] == 1, st  # no page needed a driver call
    assert st["premapped_hits"] == len({p // K for p in range(1, 9)} - {0}), st
    assert sorted({h.page for h in grow.handles}) == list(range(1, 9))
    msim.free_kv(pool, gpu.ledger, first.handles + grow.handles)
    device.quiesce()
    device.reclaim(True)
    assert device.stats()["pending"] == 0
    msim.free_kvcache(gpu.ledger, pool)


def test_worker_stays_within_the_physical_budget(product, device):
    cap = 12
    K = device.chunk_pages()
    gpu = msim.GpuState(0, cap, lib=product)
    gpu.ledger.attach_device(device)
    device.reclaim(True)
    pool = msim.alloc_kvcache(gpu.ledger, "tight", 131072, 400)
    device.reset_stats()
    held = msim.alloc_kv(pool, gpu.ledger, 10 * 16).handles  # 10 pages; the hint asks for more
    device.quiesce()
    # physical budget: ceil(cap / K) chunks + one partial chunk per pool
    budget_chunks = -(-cap // K) + 1
    assert device.stats()["total_chunks"] <= budget_chunks
    more = msim.alloc_kv(pool, gpu.ledger, 2 * 16)  # the rest of the ledger still maps
    assert more.shortfall_pages == 0
    assert msim.alloc_kv(pool, gpu.ledger, 1).shortfall_pages == 1
    assert device.stats()["total_chunks"] <= budget_chunks
    msim.free_kv(pool, gpu.ledger, held + more.handles)
    device.quiesce()
    device.reclaim(True)
    msim.free_kvcache(gpu.ledger, pool)


def test_concurrent_pools_with_worker_keep_data(product, device):
    """Two models alternate bursts on a tight ledger while the worker
    pre-maps and moves pages between them; attention stays exact."""
    gpu = msim.GpuState(0, 20, lib=product)
    gpu.ledger.attach_device(device)
    engines = []
    for mid in ("x", "y"):
        spec = S.shape_spec("llama3.1-8b", mid, chunk=64, weight_scale=0.0)
        act = gpu.activate(spec)
        gpu.finish_activation(act.engine_index)
        e = gpu.engine(act.engine_index)
        e.attach_device()
        engines.append((e, spec))
    rid = 0
    for rnd in range(4):
        for e, spec in engines:
            rid += 1
            e.push(rid, 40 + 9 * rnd, 30)
        steps = 0
        while any(sum(e.counts()) for e, _ in engines) and steps < 600:
            for e, spec in engines:
                if sum(e.counts()):
                    e.step()
                    e.append_kv_synthetic(0, spec.n_layers, SEED)
                    if steps % 7 == 0:
                        _attn_ok(e, spec)
            steps += 1
        assert gpu.ledger.mapped_pages() == 0
    device.quiesce()


def test_startup_reservation_backs_later_maps(product):
    """prism_device_reserve: physical handles for the requested pages are
    created up front, once (later maps consume them; no standing refill),
    bounded by the ledger's physical budget; the data path is unchanged."""
    dev = msim.Device(0, lib=product)
    try:
        gpu = msim.GpuState(0, 600, lib=product)
        gpu.ledger.attach_device(dev)
        spec = S.shape_spec("llama3.2-1b", "resv", chunk=256, weight_scale=0.0)
        act = gpu.activate(spec)
        gpu.finish_activation(act.engine_index)
        eng = gpu.engine(act.engine_index)
        eng.attach_device()
        dev.reserve(400)
        dev.quiesce()
        st = dev.stats()
        assert st["cached"] * st["chunk_pages"] >= 400 and st["creates"] * st["chunk_pages"] >= 400
        for i, p in enumerate([300, 500, 120]):
            eng.push(i + 1, p, 8)
        while sum(eng.counts()):
            eng.step()
            eng.append_kv_synthetic(0, spec.n_layers, SEED)
            _attn_ok(eng, spec)
        st = dev.stats()
        assert st["total_chunks"] * st["chunk_pages"] <= 600  # never past the physical budget
    finally:
        dev.close()


_SAME_STEP_FREE = r"""
import math, sys
import torch
from paper_2505_04021_b200 import msim
from tests import scenarios as S
dev = msim.Device(0, chunk_pages=1)          # one page per physical handle
gpu = msim.GpuState(0, 64)
gpu.ledger.attach_device(dev)
spec = S.shape_spec("llama3.1-8b", "m", chunk=64, weight_scale=0.0)   # 16 tokens per page
act = gpu.activate(spec)
gpu.finish_activation(act.engine_index)
eng = gpu.engine(act.engine_index)
eng.attach_device()
eng.push(1, 15, 2)    # prefill 15 (+1 first token) fills page 0 exactly
eng.push(2, 47, 2)    # pages 1-3
for step in range(10):
    if not sum(eng.counts()):
        break
    eng.step()        # decode steps: each lands on a FRESH page and completes -> freed in the same step
    eng.append_kv_synthetic(0, spec.n_layers, 7)
    if eng.step_decode_ids():
        q = torch.zeros((len(eng.step_decode_ids()), 32, 128), dtype=torch.bfloat16, device="cuda")
        o = torch.empty_like(q)
        for layer in range(spec.n_layers):
            eng.decode_attention(layer, q.data_ptr(), o.data_ptr(), 1 / math.sqrt(128))
    eng.synchronize()
    torch.cuda.synchronize()
assert sum(eng.counts()) == 0 and gpu.ledger.mapped_pages() == 0
print("ok")
"""


def test_page_freed_in_its_allocating_step_is_still_mapped_for_the_kernels():
    """A decode token that lands on a fresh page of a request completing in
    the same step: the page is mapped and freed within one step (completion
    frees run before the step's K2 / K3, reference engine.cpp:250-262), but
    K2 still writes its K/V row and K3 reads it. With the look-ahead off
    (PRISM_PREMAP=0) the chunk is still queued when the free arrives; it must
    be mapped before the kernels run all the same (found by the scheduler-
    driven C5 run: an illegal address in K2)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PRISM_PREMAP="0", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", _SAME_STEP_FREE], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_released_pool_hands_its_memory_to_the_next_pool(product):
    """free_kvcache of a pool with mapped chunks (a model's eviction): its
    chunks go back as cached handles and its VA range is freed. A pool
    created right after, on a ledger too tight for both, maps all its pages
    without creating handles past the physical budget; when it is released
    too, every handle is cached and nothing stays mapped."""
    cap = 32
    dev = msim.Device(0, lib=product)
    try:
        K = dev.chunk_pages()
        gpu = msim.GpuState(0, cap, lib=product)
        gpu.ledger.attach_device(dev)
        a = msim.alloc_kvcache(gpu.ledger, "old", 131072, 400)  # 16 tokens per page
        held = msim.alloc_kv(a, gpu.ledger, cap * 16).handles
        assert len({h.page for h in held}) == cap
        dev.quiesce()
        mapped_before = dev.stats()["total_chunks"] - dev.stats()["cached"]
        assert mapped_before >= cap // K
        msim.free_kv(a, gpu.ledger, held)
        dev.reset_stats()
        msim.free_kvcache(gpu.ledger, a)
        b = msim.alloc_kvcache(gpu.ledger, "new", 131072, 400)
        got = msim.alloc_kv(b, gpu.ledger, cap * 16)
        assert got.shortfall_pages == 0
        dev.quiesce()
        st = dev.stats()
        assert st["total_chunks"] * K <= cap + K, st      # nothing created past the budget
        msim.free_kv(b, gpu.ledger, got.handles)
        msim.free_kvcache(gpu.ledger, b)
        dev.quiesce()  # waits for the retired ranges too
        st = dev.stats()
        assert st["pending"] == 0 and st["cached"] == st["total_chunks"], st
    finally:
        dev.close()


def test_background_reserve_steals_keep_data_and_budget(product, device):
    """Once an urgent map had to steal (budget spent), the worker keeps up to
    PRISM_VMM_RESERVE_CHUNKS (default 8) unmapped handles ready by stealing
    safe idle chunks in the background; the next urgent maps take those
    handles. Attention stays exact and the physical budget holds."""
    cap = 96
    K = device.chunk_pages()
    gpu = msim.GpuState(0, cap, lib=product)
    gpu.ledger.attach_device(device)
    device.reclaim(True)
    device.reset_stats()
    engines = []
    for mid in ("r0", "r1", "r2"):
        spec = S.shape_spec("llama3.1-8b", mid, chunk=256, weight_scale=0.0)
        act = gpu.activate(spec)
        gpu.finish_activation(act.engine_index)
        e = gpu.engine(act.engine_index)
        e.attach_device()
        engines.append((e, spec))
    rid = 0
    budget_chunks = -(-cap // K) + len(engines)
    for rnd in range(9):
        e, spec = engines[rnd % 3]
        for _ in range(4):
            rid += 1
            e.push(rid, 300 + 11 * rnd, 16)
        steps = 0
        while sum(e.counts()) and steps < 600:
            e.step()
            e.append_kv_synthetic(0, spec.n_layers, SEED)
            steps += 1
            if steps % 6 == 0:
                _attn_ok(e, spec)
        assert sum(e.counts()) == 0
        assert gpu.ledger.mapped_pages() == 0
        assert device.stats()["total_chunks"] <= budget_chunks
    device.quiesce()
    st = device.stats()
    assert st["steals"] > 0, st
    assert st["reserve_steals"] > 0, st
    assert st["over_budget"] == 0, st
