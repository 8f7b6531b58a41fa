"""K4 timeline of one CTA: prefill one llama3.1-8b request to CTX tokens in
CHUNK chunks, run K4 on the last chunk with PRISM_K4_TRACE=1, and print per
tile the times (us, relative) at which the loader issued tile t, the MMA
issued S(t) and P(t)·V(t), and the softmax received S(t) / posted P(t)."""
import ctypes as C
import math
import os
import sys

os.environ["PRISM_K4_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_04021_b200 import msim  # noqa: E402
from paper_2505_04021_b200.configs import shape_spec  # noqa: E402

CHUNK = int(os.environ.get("CHUNK", 2048))
CTX = int(os.environ.get("CTX", 8192))
dev = msim.Device(0)
torch.cuda.set_stream(torch.cuda.ExternalStream(dev.stream()))
lib = msim.capi.product()
spec = shape_spec("llama3.1-8b", "t", chunk=CHUNK, weight_scale=0.0)
gpu = msim.GpuState(0, CTX // 16 + 64)
gpu.ledger.attach_device(dev)
act = gpu.activate(spec)
gpu.finish_activation(act.engine_index)
eng = gpu.engine(act.engine_index)
eng.attach_device(max_step_tokens=CHUNK + 8)
eng.push(1, CTX, 2)
q = torch.randn((CHUNK, 32, 128), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
while True:
    eng.step()
    eng.append_kv_synthetic(0, 32, 1)
    n, first, _ = eng.prefill_info()
    if first + n >= CTX:
        break
for _ in range(3):
    eng.prefill_attention(0, q.data_ptr(), o.data_ptr(), 1 / math.sqrt(128))
eng.synchronize()
R = 16
SHOW = [int(x) for x in os.environ.get('SHOW', '').split(',') if x]
buf = (C.c_uint64 * (R * 1024))()
got = C.c_int32()
lib.call("prism_debug_k4_trace", buf, R * 1024, C.byref(got))
tr = [list(buf[r * 1024:(r + 1) * 1024]) for r in range(R)]
n_tiles = max(i for i in range(1024) if tr[1][i]) + 1
t0 = min(x for row in tr for x in row[:n_tiles] if x)
names = ["load", "S_iss", "PV0_is", "w0_S", "w0_P", "w1_S", "w1_P", "PV1_is", "m_it", "m_P", "m_V", "s_beg", "s_K",
         "e_O", "e_st", "e_tk"]  # e_*: epilogue after tile t (O complete, partial stored, ticket taken)
print("tile " + " ".join(f"{n:>7s}" for n in names) + "   (us from first stamp)")
for t in range(n_tiles):
    row = [(tr[r][t] - t0) / 1e3 if tr[r][t] else float("nan") for r in range(R)]
    if t < 12 or t % 8 == 0 or t == n_tiles - 1 or (SHOW and SHOW[0] <= t < SHOW[1]):
        print(f"{t:4d} " + " ".join(f"{x:7.2f}" for x in row))
mean = lambda xs: sum(xs) / max(len(xs), 1)
d = [(tr[2][t + 1] - tr[2][t]) / 1e3 for t in range(n_tiles - 1)]
for w, (rs, rp) in enumerate(((3, 4), (5, 6))):
    sm = [(tr[rp][t] - tr[rs][t]) / 1e3 for t in range(n_tiles)]
    wait = [(tr[rs][t + 1] - tr[rp][t]) / 1e3 for t in range(n_tiles - 1)]
    print(f"warpgroup {w}: softmax busy per tile {mean(sm):.3f} us, idle between tiles {mean(wait):.3f} us")
p2pv = [(tr[2][t] - tr[4][t]) / 1e3 for t in range(n_tiles)]
s_lat = [(tr[3][t] - tr[1][t]) / 1e3 for t in range(n_tiles)]
print(f"tiles {n_tiles}; mean PV-to-PV {mean(d):.3f} us; P0 posted -> PV0 issued {mean(p2pv):.3f} us; "
      f"S issued -> warpgroup 0 has it {mean(s_lat):.3f} us")
