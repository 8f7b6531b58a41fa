"""K3 tuning sweep on a B200: attention-only GB/s for each kernel variant and
split size, on the C1 shape (64 x 2K, llama-8B KV) and the C3 shape
(16 x 32K). Prints one JSON line per (config, variant, chunk)."""
import json
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402

L, NQ, NKV, D = 32, 32, 8, 128
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
VARIANTS = {0: "mma-2stage", 1: "simt", 2: "mma-3stage", 3: "streamk", 4: "bulk"}


def build(dev, B, ctx):
    tpp = 16
    gpu = msim.GpuState(0, B * (ctx + 600) // tpp + 200)
    gpu.ledger.attach_device(dev)
    spec = msim.ModelSpec.llm(f"m{B}x{ctx}", L, NQ, NKV, D, chunk_size=8192)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device(max_step_tokens=8192 + B + 8)
    for i in range(B):
        eng.push(i + 1, ctx - 1, 1_000_000)
    while eng.counts()[1] or any(r.prompt_done < r.prompt_tokens for r in eng.batch()):
        eng.step()
        eng.append_kv_synthetic(0, L, 1)
    eng.step()
    eng.append_kv_synthetic(0, L, 1)
    return gpu, eng


def time_k3(dev, eng, B, chunk, reps):
    q = torch.empty((L, B, NQ, D), dtype=torch.bfloat16, device="cuda")
    o = torch.empty_like(q)
    for layer in range(L):
        eng.synth_q(layer, 1, 1.0, q[layer].data_ptr())
    scale = 1 / math.sqrt(D)
    stream = torch.cuda.ExternalStream(dev.stream())
    for layer in range(L):
        eng.decode_attention(layer, q[layer].data_ptr(), o[layer].data_ptr(), scale, chunk)
    dev.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(reps):
        for layer in range(L):
            eng.decode_attention(layer, q[layer].data_ptr(), o[layer].data_ptr(), scale, chunk)
    e.record(stream)
    e.synchronize()
    ms = s.elapsed_time(e) / (reps * L)
    ctx = sum(r.live_slots() for r in eng.batch())
    nbytes = ctx * NKV * D * 4 + 2 * B * NQ * D * 2
    return ms, nbytes / ms / 1e6


def main():
    dev = msim.Device(0)
    lib = msim.capi.product()
    for name, B, ctx, chunks, reps in (("C1", 64, 2048, (0, 256, 512, 1024, 2048), 10),
                                       ("C3", 16, 32768, (0, 512, 1024, 2048, 4096), 3)):
        gpu, eng = build(dev, B, ctx)
        for v in [int(x) for x in os.environ.get("K3_VARIANTS", "3,0,2,1").split(",")]:
            lib.call("prism_set_attention_variant", v)
            for chunk in (chunks if v < 3 else (0,)):
                ms, gbs = time_k3(dev, eng, B, chunk, reps)
                print(json.dumps({"config": name, "variant": VARIANTS[v], "chunk": chunk, "ms_per_launch": round(ms, 4),
                                  "GBps": round(gbs, 1), "frac_of_peak": round(gbs / PEAK, 4)}), flush=True)
        del eng, gpu
    lib.call("prism_set_attention_variant", 3)


if __name__ == "__main__":
    main()
