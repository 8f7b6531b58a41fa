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
