"""K4 per-CTA launch timeline (PRISM_K4_CTA_TRACE): prefill one
llama3.1-8b request to the chunk starting at FIRST (CHUNK tokens), then run
K4 over 5 consecutive layers (a PDL chain) after 5 warm-up launches and print,
per launch, when its CTAs started, returned from the
first-write PDL wait and ended (us from the first CTA start of the first
traced launch), plus the per-CTA busy time spread."""
import ctypes as C
import math
import os
import statistics
import sys

os.environ["PRISM_K4_CTA_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_04021_b200 import msim  # noqa: E402
from paper_2505_04021_b200.configs import shape_spec  # noqa: E402

CHUNK = int(os.environ.get("CHUNK", 512))
FIRST = int(os.environ.get("FIRST", 3584))
dev = msim.Device(0)
torch.cuda.set_stream(torch.cuda.ExternalStream(dev.stream()))
lib = msim.capi.product()
spec = shape_spec("llama3.1-8b", "t", chunk=CHUNK, weight_scale=0.0)
ctx = FIRST + CHUNK
gpu = msim.GpuState(0, ctx // 16 + 64)
gpu.ledger.attach_device(dev)
act = gpu.activate(spec)
gpu.finish_activation(act.engine_index)
eng = gpu.engine(act.engine_index)
eng.attach_device(max_step_tokens=CHUNK + 8)
eng.push(1, ctx, 2)
q = torch.randn((CHUNK, 32, 128), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
while True:
    eng.step()
    eng.append_kv_synthetic(0, 32, 1)
    n, first, _ = eng.prefill_info()
    if first + n >= ctx:
        break
SAME = os.environ.get("SAME_LAYER") == "1"  # every launch on layer 0: its K/V stays in L2
for layer in range(10):  # 5 warm-up + 5 traced, one chain
    eng.prefill_attention(0 if SAME else layer % 32, q.data_ptr(), o.data_ptr(), 1 / math.sqrt(128))
eng.synchronize()
buf = (C.c_uint64 * (16 * 1024))()
got = C.c_int32()
lib.call("prism_debug_k4_trace", buf, 16 * 1024, C.byref(got))
base = 13 * 1024
launches = []
for li in range(5):
    rows = []
    for c in range(148):
        r = [buf[base + (li * 148 + c) * 4 + k] for k in range(4)]
        if r[0]:
            rows.append(r)
    launches.append(rows)
t0 = min(r[0] for r in launches[0])
us = lambda x: (x - t0) / 1e3
flops = 4.0 * 32 * 128 * sum(first + i + 1 for i in range(n))
print(f"chunk {n} tokens at first={first}: {flops / 1e9:.1f} GFLOP per launch")
prev_end = None
for li, rows in enumerate(launches):
    st = sorted(us(r[0]) for r in rows)
    wt = sorted(us(r[2]) for r in rows if r[2])
    en = sorted(us(r[3]) for r in rows)
    busy = [(r[3] - r[0]) / 1e3 for r in rows]
    print(f"launch {li}: {len(rows)} CTAs | start {st[0]:8.2f} .. {st[-1]:8.2f} "
          f"| wait returned {wt[0] if wt else float('nan'):8.2f} .. {wt[-1] if wt else float('nan'):8.2f} ({len(wt)} CTAs) "
          f"| end {en[0]:8.2f} .. {en[-1]:8.2f} (median {statistics.median(en):8.2f}) "
          f"| CTA busy min/med/max {min(busy):6.2f} / {statistics.median(busy):6.2f} / {max(busy):6.2f}"
          + (f" | period {en[-1] - prev_end:6.2f}" if prev_end is not None else ""))
    prev_end = en[-1]

# per CTA of the last launch: SM id and busy time, in blockIdx order
rows = launches[-1]
print("last launch, per CTA (blockIdx: sm busy_us):")
print(" ".join(f"{c}:{r[1]}:{(r[3] - r[0]) / 1e3:.1f}" for c, r in enumerate(rows)))
