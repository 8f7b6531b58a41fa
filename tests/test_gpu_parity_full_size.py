"""Parity at the sizes bench.py times (VERDICT r01 "parity at the sizes you
time"), on the GPU through the C-ABI:

* C1 on the 85,830-page B200 ledger with the device attached (VMM pages,
  K1, K2 every step): outcomes, handle stream, events and tables equal the
  compiled reference's golden digests; the device slot ids of every step are
  the host's new handles; every block-table row equals the host handles at
  the end; K3 over the final contexts vs the fp64 oracle (sampled).
* C3 decode: 16 x 32,768 contexts grown by 8K chunks (bench decode_c3's
  configuration), K3 vs the fp64 oracle on sampled requests and layers.
* C3 prefill: one request prefilled to 32,768 keys in 512-token chunks
  (bench prefill_c3's configuration); K4 at the last chunks vs the fp64
  oracle on sampled query tokens (keys 0..pos).
Tolerance (BASELINE north star): |gpu - oracle| <= 2e-3 + 1e-2 |oracle|.
"""
import math
import random

import numpy as np
import pytest
import torch

import oracle
from paper_2505_04021_b200 import msim
from tests import scenarios as S
from tests.test_gpu_attention import _close

pytestmark = pytest.mark.gpu
SEED = 20251017


def test_c1_full_b200_ledger_with_device(product, device, golden):
    tpp = 16
    seen = [0]

    def on_step(mid, e, new):
        e.append_kv_synthetic(0, 32, SEED)  # K2 into the slots K1 wrote
        host = sorted(p * tpp + s for _, hs in new for p, s in hs)
        assert sorted(e.step_slots()) == host  # raises if K1 diverged from the host allocator
        seen[0] += 1

    got = S.c1_full_ledger(product, device=device, on_step=on_step, **S.C1_FULL)
    ref = golden["c1_full_ledger"]
    for k in ("steps", "outcome_digest", "handle_stream_digest", "event_digest", "events", "table_digest",
              "mapped", "free"):
        assert got[k] == ref[k], k
    assert seen[0] == ref["steps"]
    scale = 1 / math.sqrt(128)
    rng = random.Random(7)
    for mid, e in got["engines"]:
        for r in e.batch():
            buf, n = e.request_kv_raw(r.id)
            assert e.table_row(r.table_row, n) == [s.page * tpp + s.slot for s in buf[:n]]
        ids = e.step_decode_ids()
        live = {r.id: r.live_slots() for r in e.batch()}
        q = torch.empty((len(ids), 32, 128), dtype=torch.bfloat16, device="cuda")
        o = torch.empty_like(q)
        pick = sorted(rng.sample(range(len(ids)), 4))
        for layer in (0, 31):
            e.synth_q(layer, SEED, 4.0, q.data_ptr())
            e.decode_attention(layer, q.data_ptr(), o.data_ptr(), scale)
            e.synchronize()
            ref_o = oracle.synth_attention(SEED, layer, [ids[i] for i in pick], [live[ids[i]] for i in pick],
                                           32, 8, 128, 4.0, scale)
            _close(o.float().cpu().numpy()[pick], ref_o)


def test_k3_c3_full_size(product, device):
    """16 x 32,768 (bench decode_c3): split over many stream-K CTAs; sampled
    requests x layers against the fp64 oracle over all 32K keys."""
    batch, ctx = 16, 32768
    gpu = msim.GpuState(0, batch * (ctx + 600) // 16 + 200, lib=product)
    gpu.ledger.attach_device(device)
    spec = msim.ModelSpec.llm("c3-decode", 32, 32, 8, 128, chunk_size=8192)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device(max_step_tokens=8192 + batch + 8)
    for i in range(batch):
        eng.push(i + 1, ctx - 1, 1_000_000)
    while eng.counts()[1] or any(r.prompt_done < r.prompt_tokens for r in eng.batch()):
        eng.step()
        eng.append_kv_synthetic(0, 32, SEED)
    eng.step()
    eng.append_kv_synthetic(0, 32, SEED)
    ids = eng.step_decode_ids()
    live = {r.id: r.live_slots() for r in eng.batch()}
    assert len(ids) == batch and all(live[i] >= ctx for i in ids)  # prompt 32,767 + first token + decodes
    q = torch.empty((batch, 32, 128), dtype=torch.bfloat16, device="cuda")
    o = torch.empty_like(q)
    scale = 1 / math.sqrt(128)
    pick = [0, 7, 15]
    for layer in (0, 13, 31):
        eng.synth_q(layer, SEED, 4.0, q.data_ptr())
        eng.decode_attention(layer, q.data_ptr(), o.data_ptr(), scale)
        eng.synchronize()
        ref = oracle.synth_attention(SEED, layer, [ids[i] for i in pick], [live[ids[i]] for i in pick], 32, 8, 128,
                                     4.0, scale)
        _close(o.float().cpu().numpy()[pick], ref)


def _synth_q_rows(req, positions, layer, n_q, d, q_scale):
    lib = oracle.restate()
    out = np.zeros((len(positions), n_q, d), dtype=np.uint16)
    for i, p in enumerate(positions):
        for h in range(n_q):
            for e in range(d):
                out[i, h, e] = lib.po_synth_bf16(SEED, req, p, layer, 2, h, e, q_scale)
    return out


def test_k4_c3_32k_prefix(product, device):
    """One request prefilled to 32,768 keys in 512-token chunks (bench
    prefill_c3): K4 at chunks ending at 16K and 32K keys, sampled query
    tokens against the fp64 oracle over keys 0..pos (synthetic K/V content,
    q of the sampled tokens = the oracle's synthetic q at that position)."""
    ctx, chunk, layer, q_scale = 32768, 512, 5, 4.0
    gpu = msim.GpuState(0, ctx // 16 + 64, lib=product)
    gpu.ledger.attach_device(device)
    spec = msim.ModelSpec.llm("c3-prefill", 32, 32, 8, 128, chunk_size=chunk)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device(max_step_tokens=chunk + 8)
    eng.push(1, ctx, 2)
    scale = 1 / math.sqrt(128)
    rng = random.Random(3)
    checked = 0
    while True:
        eng.step()
        eng.append_kv_synthetic(0, 32, SEED)
        n, first, rid = eng.prefill_info()
        if n == 0:
            break
        if first + n in (ctx // 2, ctx):
            picks = sorted({0, n - 1, *[rng.randrange(n) for _ in range(4)]})
            qh = np.random.default_rng(first).integers(0x3c00, 0x3f80, size=(n, 32, 128), dtype=np.uint16)
            qh[picks] = _synth_q_rows(rid, [first + i for i in picks], layer, 32, 128, q_scale)
            q = torch.from_numpy(qh.view(np.int16)).view(torch.bfloat16).cuda()
            o = torch.full_like(q, float("nan"))
            torch.cuda.current_stream().synchronize()
            eng.prefill_attention(layer, q.data_ptr(), o.data_ptr(), scale)
            eng.synchronize()
            oc = o.float().cpu().numpy()
            assert not np.isnan(oc).any()
            ref = oracle.synth_attention(SEED, layer, [rid] * len(picks), [first + i + 1 for i in picks], 32, 8, 128,
                                         q_scale, scale)
            _close(oc[picks], ref)
            checked += len(picks)
        if first + n >= ctx:
            break
    assert checked >= 8


@pytest.mark.parametrize("n_q,n_kv,chunk", [(14, 2, 1024), (32, 8, 384)])
def test_k4_head_dim_64_long_prefix(product, device, n_q, n_kv, chunk):
    """K4 on the head_dim-64 path (16-half K/V ring, two Q buffers) at long
    prefixes: qwen2.5-0.5b (GQA 7, padded Q-tile rows) and llama3.2-1b
    (GQA 4) shapes prefilled to 8K keys; at the chunks ending at 4K and 8K
    keys, sampled query tokens against the fp64 oracle (cut units, partials
    and merges all exercised: the grid spreads each launch over the SMs)."""
    ctx, layer, q_scale, d = 8192, 3, 4.0, 64
    gpu = msim.GpuState(0, ctx // 64 + 64, lib=product)
    gpu.ledger.attach_device(device)
    spec = msim.ModelSpec.llm("k4-d64", 16, n_q, n_kv, d, chunk_size=chunk)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device(max_step_tokens=chunk + 8)
    eng.push(1, ctx, 2)
    scale = 1 / math.sqrt(d)
    rng = random.Random(n_q)
    checked = 0
    while True:
        eng.step()
        eng.append_kv_synthetic(0, 16, SEED)
        n, first, rid = eng.prefill_info()
        if n == 0:
            break
        if first < ctx // 2 <= first + n or first + n >= ctx:
            picks = sorted({0, n - 1, *[rng.randrange(n) for _ in range(5)]})
            qh = np.random.default_rng(first).integers(0x3c00, 0x3f80, size=(n, n_q, d), dtype=np.uint16)
            qh[picks] = _synth_q_rows(rid, [first + i for i in picks], layer, n_q, d, q_scale)
            q = torch.from_numpy(qh.view(np.int16)).view(torch.bfloat16).cuda()
            o = torch.full_like(q, float("nan"))
            torch.cuda.current_stream().synchronize()
            eng.prefill_attention(layer, q.data_ptr(), o.data_ptr(), scale)
            eng.synchronize()
            oc = o.float().cpu().numpy()
            assert not np.isnan(oc).any()
            ref = oracle.synth_attention(SEED, layer, [rid] * len(picks), [first + i + 1 for i in picks], n_q, n_kv, d,
                                         q_scale, scale)
            _close(oc[picks], ref)
            checked += len(picks)
        if first + n >= ctx:
            break
    assert checked >= 8
