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
