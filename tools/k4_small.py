"""K4 latency on the short prefill chunks a serving run issues (the C2
serving launch list has K4 as ~65% of GPU time at ~37 us per launch):
one request of PROMPT tokens prefilled in one chunk (first = 0) for each
SURVEY shape in SHAPES; mean K4 time over 100 back-to-back launches (CUDA
events on the engine stream) and the causal TFLOP/s it reaches."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402
from paper_2505_04021_b200.configs import SHAPES, shape_spec  # noqa: E402

dev = msim.Device(0)
stream = torch.cuda.ExternalStream(dev.stream())
torch.cuda.set_stream(stream)
for name in os.environ.get("SHAPES", "llama3.1-8b,qwen2.5-0.5b").split(","):
    L, nq, nkv, d, _ = SHAPES[name]
    for prompt in [int(x) for x in os.environ.get("PROMPTS", "64,256,512,1024,2048").split(",")]:
        spec = shape_spec(name, "s", chunk=prompt, weight_scale=0.0)
        tpp = (2 << 20) // spec.token_kv_bytes
        gpu = msim.GpuState(0, prompt // tpp + 64)
        gpu.ledger.attach_device(dev)
        act = gpu.activate(spec)
        gpu.finish_activation(act.engine_index)
        eng = gpu.engine(act.engine_index)
        eng.attach_device(max_step_tokens=prompt + 8)
        eng.push(1, prompt, 4)
        eng.step()
        eng.append_kv_synthetic(0, L, 1)
        n, first, _ = eng.prefill_info()
        q = torch.randn((n, nq, d), device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        sc = 1 / math.sqrt(d)
        for _ in range(5):
            eng.prefill_attention(0, q.data_ptr(), o.data_ptr(), sc)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for i in range(100):
            eng.prefill_attention(i % L, q.data_ptr(), o.data_ptr(), sc)
        e.record(stream)
        e.synchronize()
        us = s.elapsed_time(e) * 1e3 / 100
        flops = 4.0 * nq * d * sum(first + i + 1 for i in range(n))
        print(json.dumps({"shape": name, "prompt": prompt, "chunk": n, "us_per_launch": round(us, 2),
                          "TFLOPs": round(flops / us / 1e6, 1)}), flush=True)
        del eng, gpu
