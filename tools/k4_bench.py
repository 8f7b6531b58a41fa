"""K4 (chunked-prefill attention) throughput on a B200: one llama3.1-8b-shaped
request prefilled in chunks of CHUNK tokens up to CTX; at each chunk, K4 is
timed (CUDA events on the engine stream, REPS x LAYERS launches) and its
useful FLOPs counted causally: 4 * n_q * d * sum_i (first + i + 1).
Prints one JSON line per chunk and a summary against MEASURED_PEAKS.json."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402
from tests import scenarios as S  # noqa: E402

CHUNK = int(os.environ.get("CHUNK", 512))
CTX = int(os.environ.get("CTX", 32768))
REPS, LAYERS = int(os.environ.get("REPS", 3)), 8
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))
dev = msim.Device(0)
torch.cuda.set_stream(torch.cuda.ExternalStream(dev.stream()))  # producers on the engine stream
spec = S.shape_spec("llama3.1-8b", "k4", chunk=CHUNK, weight_scale=0.0)
gpu = msim.GpuState(0, CTX // 16 + 64)
gpu.ledger.attach_device(dev)
act = gpu.activate(spec)
gpu.finish_activation(act.engine_index)
eng = gpu.engine(act.engine_index)
eng.attach_device(max_step_tokens=CHUNK + 8)
eng.push(1, CTX, 2)
L, nkv, nq, d = spec.n_layers, spec.n_kv_heads, spec.n_q_heads, spec.head_dim
stream = torch.cuda.ExternalStream(dev.stream())
q = torch.randn((CHUNK, nq, d), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
scale = 1 / math.sqrt(d)
rows = []
while True:
    eng.step()
    eng.append_kv_synthetic(0, L, 1)
    n, first, _ = eng.prefill_info()
    if n == 0:
        break
    for layer in range(2):  # warm
        eng.prefill_attention(layer, q.data_ptr(), o.data_ptr(), scale)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(REPS):
        for layer in range(LAYERS):
            eng.prefill_attention(layer, q.data_ptr(), o.data_ptr(), scale)
    e.record(stream)
    e.synchronize()
    ms = s.elapsed_time(e) / (REPS * LAYERS)
    flops = 4.0 * nq * d * sum(first + i + 1 for i in range(n))
    rows.append((first, n, ms, flops / ms / 1e9))
    if first % 4096 == 0 or first + n >= CTX:
        print(json.dumps({"first": first, "tokens": n, "ms": round(ms, 4), "TFLOPs": round(flops / ms / 1e9, 1)}),
              flush=True)
    if first + n >= CTX:
        break
tot_flops = sum(4.0 * nq * d * sum(f + i + 1 for i in range(n)) for f, n, _, _ in rows)
tot_ms = sum(ms for _, _, ms, _ in rows)
print(json.dumps({"summary": f"K4 llama3.1-8b chunk {CHUNK} up to {CTX}", "mean_TFLOPs": round(tot_flops / tot_ms / 1e9, 1),
                  "peak_bf16_TFLOPs": peaks.get("bf16_tflops"), "frac": round(tot_flops / tot_ms / 1e9 / peaks["bf16_tflops"], 4)}))
