"""Two engines on two devices' streams (two VmmDevice instances on one GPU,
each with its own stream) running stream-K K3 concurrently, interleaved
launch by launch: each grid is sized for the whole GPU, so each runs while
the other holds SMs (partial residency). The stream-K merge must neither
deadlock (its CTA ranges are drawn in reverse dispatch order, so a merging
CTA only waits on CTAs already resident) nor mix the two launches' partials;
both outputs match the fp64 oracle."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2505_04021_b200 import msim
from tests.test_gpu_attention import _close

pytestmark = pytest.mark.gpu
SEED = 20251017


def _engine(product, dev, name, prompts):
    gpu = msim.GpuState(0, 4000, lib=product)
    gpu.ledger.attach_device(dev)
    spec = msim.ModelSpec.llm(name, 32, 28, 4, 128, chunk_size=4096)  # qwen2.5-7b shape (G = 7)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device()
    for i, p in enumerate(prompts):
        eng.push(i + 1, p, 1000)
    while eng.counts()[1] or any(r.prompt_done < r.prompt_tokens for r in eng.batch()):
        eng.step()
        eng.append_kv_synthetic(0, 32, SEED)
    eng.step()
    eng.append_kv_synthetic(0, 32, SEED)
    return gpu, eng


def test_two_streams_concurrent_streamk(product):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    product.call("prism_set_attention_variant", 3)
    d1, d2 = msim.Device(0, lib=product), msim.Device(0, lib=product)
    try:
        g1, e1 = _engine(product, d1, "m1", [3000, 2100, 700, 4096] * 4)
        g2, e2 = _engine(product, d2, "m2", [1500, 5000, 333] * 5)
        scale = 1 / math.sqrt(128)
        bufs = []
        for e, dev in ((e1, d1), (e2, d2)):
            n = len(e.step_decode_ids())
            with torch.cuda.stream(torch.cuda.ExternalStream(dev.stream())):
                q = torch.empty((32, n, 28, 128), dtype=torch.bfloat16, device="cuda")
                o = torch.empty_like(q)
            for layer in range(32):
                e.synth_q(layer, SEED, 4.0, q[layer].data_ptr())
            bufs.append((q, o))
        d1.synchronize()
        d2.synchronize()
        for rep in range(5):
            for layer in range(32):  # interleaved: the two chains overlap on the GPU
                e1.decode_attention(layer, bufs[0][0][layer].data_ptr(), bufs[0][1][layer].data_ptr(), scale)
                e2.decode_attention(layer, bufs[1][0][layer].data_ptr(), bufs[1][1][layer].data_ptr(), scale)
        d1.synchronize()
        d2.synchronize()
        for e, (q, o) in ((e1, bufs[0]), (e2, bufs[1])):
            ids = e.step_decode_ids()
            live = {r.id: r.live_slots() for r in e.batch()}
            for layer in (0, 31):
                ref = oracle.synth_attention(SEED, layer, ids, [live[i] for i in ids], 28, 4, 128, 4.0, scale)
                _close(o[layer].float().cpu().numpy(), ref)
        del e1, e2, g1, g2
    finally:
        d1.close()
        d2.close()


def _bits(t):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def test_two_streams_concurrent_prefill_chains(product):
    """K4 programmatic-dependent chains on two streams at once (two
    VmmDevice instances on one GPU), interleaved launch by launch: each
    launch is sized for the whole GPU and its CTAs start on SMs as they free
    up, waiting for their own stream's previous launch only at their first
    global write. Sampled query tokens of both chains match the fp64
    oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d1, d2 = msim.Device(0, lib=product), msim.Device(0, lib=product)
    L, nq, nkv, d = 32, 28, 4, 128
    check = (1, L - 1)
    try:
        runs = []
        for dev, name, prompt, seed in ((d1, "p1", 1700, 11), (d2, "p2", 1300, 12)):
            gpu = msim.GpuState(0, 4000, lib=product)
            gpu.ledger.attach_device(dev)
            spec = msim.ModelSpec.llm(name, L, nq, nkv, d, chunk_size=512)
            act = gpu.activate(spec)
            gpu.finish_activation(act.engine_index)
            eng = gpu.engine(act.engine_index)
            eng.attach_device()
            eng.push(1, prompt, 2)
            gen = torch.Generator(device="cuda").manual_seed(seed)
            ks, vs = [], []
            with torch.cuda.stream(torch.cuda.ExternalStream(dev.stream())):
                while True:  # prefill up to the last chunk (a prefix of 1-3 chunks)
                    eng.step()
                    n_tok, _ = eng.step_info()
                    k = (torch.rand((L, n_tok, nkv, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
                    v = (torch.rand((L, n_tok, nkv, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
                    eng.append_kv(0, L, k.data_ptr(), v.data_ptr())
                    ks.append(k[list(check)].cpu())
                    vs.append(v[list(check)].cpu())
                    n_pf, first, _ = eng.prefill_info()
                    if first + n_pf >= prompt:
                        break
                q = ((torch.rand((L, n_pf, nq, d), generator=gen, device="cuda") * 2 - 1) * 2.0).to(torch.bfloat16)
                o = torch.full_like(q, float("nan"))
            dev.synchronize()
            runs.append((gpu, eng, q, o, first, n_pf, torch.cat(ks, dim=1), torch.cat(vs, dim=1)))
        scale = 1 / math.sqrt(d)
        for rep in range(3):
            for layer in range(L):  # interleaved: the two chains overlap on the GPU
                for _, eng, q, o, *_ in runs:
                    eng.prefill_attention(layer, q[layer].data_ptr(), o[layer].data_ptr(), scale)
        d1.synchronize()
        d2.synchronize()
        for _, eng, q, o, first, n_pf, kk, vv in runs:
            assert not torch.isnan(o.float()).any()
            qc, oc = q.cpu(), o.float().cpu().numpy()
            for ci, layer in enumerate(check):
                for i in (0, 7, n_pf // 2, n_pf - 1):
                    p = first + i
                    ref = oracle.dense_attention(_bits(qc[layer, i]), _bits(kk[ci, :p + 1]), _bits(vv[ci, :p + 1]), scale)
                    _close(oc[layer, i], ref)
        del runs
    finally:
        d1.close()
        d2.close()
