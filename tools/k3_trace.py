"""Per-CTA timeline of one K3 launch inside a back-to-back chain (C1 shape by
default: 64 decodes x 2K, llama3.1-8b KV). PRISM_K3_TRACE=1 stamps, per CTA:
running, prologue copies issued, after the PDL wait, first tile, last tile,
done. Prints where a launch's time goes relative to its streaming work."""
import ctypes as C
import math
import os
import statistics as st
import sys

os.environ["PRISM_K3_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_04021_b200 import msim  # noqa: E402
from paper_2505_04021_b200.configs import SHAPES, shape_spec  # noqa: E402

SHAPE = os.environ.get("SHAPE", "llama3.1-8b")
B, CTX = int(os.environ.get("B", 64)), int(os.environ.get("CTX", 2048))
L, nq, nkv, d, _ = SHAPES[SHAPE]
dev = msim.Device(0)
torch.cuda.set_stream(torch.cuda.ExternalStream(dev.stream()))
lib = msim.capi.product()
spec = shape_spec(SHAPE, "t", chunk=8192, weight_scale=0.0)
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
for _ in range(2):
    for layer in range(L):
        eng.decode_attention(layer, q[layer].data_ptr(), o[layer].data_ptr(), 1 / math.sqrt(d))
eng.synchronize()
buf = (C.c_uint64 * (4096 * 8))()
got = C.c_int32()
lib.call("prism_debug_k3_trace", buf, 4096 * 8, C.byref(got))
rows = [buf[i * 8:(i + 1) * 8] for i in range(4096)]
rows = [r for r in rows if r[0] and r[5] >= r[0]]
t0 = min(r[0] for r in rows)
us = lambda x: (x - t0) / 1e3  # noqa: E731
start = [us(r[0]) for r in rows]
pro = [(r[1] - r[0]) / 1e3 for r in rows]
wait = [(r[2] - r[0]) / 1e3 for r in rows]
first = [(r[3] - r[0]) / 1e3 for r in rows]
stream = [(r[4] - r[3]) / 1e3 / max(r[6] - 1, 1) for r in rows]
tail = [(r[5] - r[4]) / 1e3 for r in rows]
done = [us(r[5]) for r in rows]
q = lambda v: f"min {min(v):7.2f} med {st.median(v):7.2f} max {max(v):7.2f}"  # noqa: E731
print(f"{SHAPE} B={B} ctx={CTX}: {len(rows)} CTAs, tiles/CTA {st.median([r[6] for r in rows]):.0f}")
print("CTA start (us)          ", q(start))
print("prologue issued (+us)   ", q(pro))
print("after PDL wait (+us)    ", q(wait))
print("first tile done (+us)   ", q(first))
print("per tile after first(us)", q(stream))
print("last tile -> done (us)  ", q(tail))
print("CTA done (us)           ", q(done))
print(f"launch span {max(done):.2f} us")
