"""K3 (default stream-K kernel) GB/s for every SURVEY §8d model shape at
64 decodes x 2K context: one engine per shape, 32 (or L) back-to-back
launches timed with CUDA events, algorithmic bytes as in bench.py."""
import json
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402
from paper_2505_04021_b200.configs import SHAPES, shape_spec  # noqa: E402

B, CTX = int(os.environ.get("B", 64)), int(os.environ.get("CTX", 2048))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = msim.Device(0)
torch.cuda.set_stream(torch.cuda.ExternalStream(dev.stream()))
ONLY = os.environ.get("SHAPES")
for name, (L, nq, nkv, d, _) in SHAPES.items():
    if ONLY and name not in ONLY.split(","):
        continue
    spec = shape_spec(name, name, chunk=8192, weight_scale=0.0)
    tpp = (2 << 20) // spec.token_kv_bytes
    gpu = msim.GpuState(0, B * (CTX + 64) // tpp + 400)
    gpu.ledger.attach_device(dev)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device(max_step_tokens=8192 + B + 8)
    for i in range(B):
        eng.push(i + 1, CTX - 1, 1_000_000)
    while eng.counts()[1] or any(r.prompt_done < r.prompt_tokens for r in eng.batch()):
        eng.step()
        eng.append_kv_synthetic(0, L, 1)
    eng.step()
    eng.append_kv_synthetic(0, L, 1)
    q = torch.randn((L, B, nq, d), device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    sc = 1 / math.sqrt(d)
    for layer in range(L):
        eng.decode_attention(layer, q[layer].data_ptr(), o[layer].data_ptr(), sc)
    dev.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.perf_counter()
    for _ in range(3):
        for layer in range(L):
            eng.decode_attention(layer, q[layer].data_ptr(), o[layer].data_ptr(), sc)
    host_us = (time.perf_counter() - t0) * 1e6 / (3 * L)  # host submission time per launch
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / (3 * L)
    ctx = sum(r.live_slots() for r in eng.batch())
    nbytes = ctx * nkv * d * 4 + 2 * B * nq * d * 2
    print(json.dumps({"shape": name, "G": nq // nkv, "d": d, "n_kv": nkv, "ms": round(ms, 4),
                      "GBps": round(nbytes / ms / 1e6, 1), "frac": round(nbytes / ms / 1e6 / peak, 4),
                      "host_submit_us_per_launch": round(host_us, 2)}), flush=True)
    del eng, gpu
