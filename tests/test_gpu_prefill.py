"""K4 (chunked-prefill paged attention, tcgen05/TMEM) parity on the GPU
through the C-ABI, against the fp64 CPU oracle (oracle/restate,
dense_attention) on the same bf16 bits.

For every step that allocated a prefill chunk, the chunk's K/V rows are
appended (K2, explicit random content) and K4 runs for one layer; sampled
query tokens i of the chunk (position first + i) are compared with the oracle
over that request's keys 0..first+i in token order. Tolerance as for K3
(BASELINE north star "max-abs 2e-3 / rel 1e-2"), elementwise:
    |gpu - oracle| <= 2e-3 + 1e-2 * |oracle|
"""
import math
import random

import numpy as np
import pytest
import torch

import oracle
from tests import scenarios as S
from tests.test_gpu_attention import _close, _engine

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def _run_prefills(product, device, shape, prompts, chunk, q_scale=2.0, layer=1, samples=12, seed=0):
    gpu, spec, eng = _engine(product, device, shape, chunk=chunk)
    L, nkv, nq, d = spec.n_layers, spec.n_kv_heads, spec.n_q_heads, spec.head_dim
    for i, p in enumerate(prompts):
        eng.push(i + 1, p, 3)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    rng = random.Random(seed)
    scale = 1 / math.sqrt(d)
    store = {}  # request -> [ (k [L][nkv][d], v) per token ] (CPU bf16)
    checked = 0
    while sum(eng.counts()):
        pre = {r.id: r.n_slots for r in eng.batch()}
        out = eng.step()
        n_tok, n_dec = eng.step_info()
        if n_tok == 0:
            continue
        k = (torch.rand((L, n_tok, nkv, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
        v = (torch.rand((L, n_tok, nkv, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
        eng.append_kv(0, L, k.data_ptr(), v.data_ptr())
        after = {r.id: r for r in eng.batch()}
        order = []
        if out.chunk_tokens:
            rid = next(r.id for r in after.values() if r.n_slots - pre.get(r.id, 0) > 1 or r.id not in pre)
            order += [rid] * (after[rid].n_slots - pre.get(rid, 0))
        order += eng.step_decode_ids()
        kc, vc = k[layer].cpu(), v[layer].cpu()
        for t, rid in enumerate(order):
            store.setdefault(rid, []).append((kc[t], vc[t]))
        n_pf, first, prid = eng.prefill_info()
        if n_pf:
            assert n_pf == out.chunk_tokens and prid == order[0]
            q = ((torch.rand((n_pf, nq, d), generator=gen, device="cuda") * 2 - 1) * q_scale).to(torch.bfloat16)
            o = torch.full_like(q, float("nan"))
            eng.prefill_attention(layer, q.data_ptr(), o.data_ptr(), scale)
            eng.synchronize()
            oc, qc = o.float().cpu().numpy(), q.cpu()
            assert not np.isnan(oc).any(), "K4 left output rows unwritten"
            kk = torch.stack([t[0] for t in store[prid]])  # [ctx][nkv][d]
            vv = torch.stack([t[1] for t in store[prid]])
            picks = sorted({0, n_pf - 1, *[rng.randrange(n_pf) for _ in range(samples)]})
            for i in picks:
                p = first + i
                ref = oracle.dense_attention(_bits(qc[i]), _bits(kk[:p + 1]), _bits(vv[:p + 1]), scale)
                _close(oc[i], ref)
                checked += 1
        for rid in out.completions:
            store.pop(rid, None)
    return checked


@pytest.mark.parametrize("shape", list(S.SHAPES))
def test_prefill_all_config_shapes(product, device, shape):
    """The 8 model shapes (head_dim 64/128, GQA groups 3..8 packed into the
    128-row MMA tile): ragged prompts incl. 1 token, chunks not a multiple of
    the query tile, multi-chunk prompts (prefix > 0) spanning several
    128-key tiles."""
    n = _run_prefills(product, device, shape, [1, 37, 128, 300, 611], chunk=160, seed=hash(shape) & 0xff)
    assert n > 20


def test_prefill_long_prefix_rescale(product, device):
    """C3-like: 512-token chunks over a growing prefix (up to ~2.6K keys, 21
    key tiles); large q makes the running max jump across tiles, exercising
    the lazy O rescale in TMEM."""
    n = _run_prefills(product, device, "llama3.1-8b", [2600], chunk=512, q_scale=8.0, layer=30, samples=24)
    assert n > 50


@pytest.mark.parametrize("shape", ["qwen2.5-1.5b", "llama3.1-8b"])
def test_prefill_chained_layers_write_in_order(product, device, shape):
    """Consecutive K4 launches of an engine form a programmatic-dependent
    chain: a launch's CTAs start on the SMs its predecessor frees and read
    q / K / V at once; only their writes (out, partials, tickets — shared by
    the chain) wait. Back-to-back launches with no synchronisation: (a) every
    layer into its own out buffer, each equal to its layer's oracle; (b)
    every layer into ONE shared buffer, repeated, which must end with the
    last layer's result (write-after-write order across the chain)."""
    gpu, spec, eng = _engine(product, device, shape, chunk=512)
    L, nkv, nq, d = spec.n_layers, spec.n_kv_heads, spec.n_q_heads, spec.head_dim
    eng.push(1, 1400, 2)
    gen = torch.Generator(device="cuda").manual_seed(7)
    rng = random.Random(7)
    scale = 1 / math.sqrt(d)
    ks, vs = [], []  # per step: [L][tok][nkv][d] (CPU bf16), request 1 only
    tested = 0
    while sum(eng.counts()) and tested < 2:
        eng.step()
        n_tok, _ = eng.step_info()
        if n_tok == 0:
            continue
        k = (torch.rand((L, n_tok, nkv, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
        v = (torch.rand((L, n_tok, nkv, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
        eng.append_kv(0, L, k.data_ptr(), v.data_ptr())
        n_pf, first, _ = eng.prefill_info()
        if not n_pf:
            continue
        # one request: the step's rows are its chunk (+ its first output
        # token's slot on the last chunk), in token order
        ks.append(k.cpu())
        vs.append(v.cpu())
        if first == 0:
            continue  # test chunks with a prefix (several key tiles, cut units)
        q = ((torch.rand((L, n_pf, nq, d), generator=gen, device="cuda") * 2 - 1) * 2.0).to(torch.bfloat16)
        outs = torch.full_like(q, float("nan"))
        shared = torch.full_like(q[0], float("nan"))
        for layer in range(L):  # (a)
            eng.prefill_attention(layer, q[layer].data_ptr(), outs[layer].data_ptr(), scale)
        for _ in range(3):  # (b)
            for layer in range(L):
                eng.prefill_attention(layer, q[layer].data_ptr(), shared.data_ptr(), scale)
        eng.synchronize()
        assert not torch.isnan(outs.float()).any(), "a chained K4 left output rows unwritten"
        kk, vv = torch.cat(ks, dim=1), torch.cat(vs, dim=1)  # [L][ctx][nkv][d]
        qc, oc, sc = q.cpu(), outs.float().cpu().numpy(), shared.float().cpu().numpy()
        for layer in (0, L // 2, L - 1):
            for i in sorted({0, n_pf - 1, *[rng.randrange(n_pf) for _ in range(6)]}):
                p = first + i
                ref = oracle.dense_attention(_bits(qc[layer, i]), _bits(kk[layer, :p + 1]), _bits(vv[layer, :p + 1]),
                                             scale)
                _close(oc[layer, i], ref)
                if layer == L - 1:
                    _close(sc[i], ref)
        tested += 1
    assert tested == 2
