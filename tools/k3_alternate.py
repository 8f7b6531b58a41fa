"""K3 per-launch time with one pool vs two pools alternating 32-launch groups
(C1 shape, no K1/K2 in between): isolates the cost of touching two models' KV."""
import json, math, os, sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2505_04021_b200 import msim
L, NQ, NKV, D = 32, 32, 8, 128
B, CTX = 64, 2048
dev = msim.Device(0)
torch.cuda.set_stream(torch.cuda.ExternalStream(dev.stream()))
gpu = msim.GpuState(0, 2 * B * (CTX + 600) // 16 + 400)
gpu.ledger.attach_device(dev)
engs = []
for m in range(2):
    spec = msim.ModelSpec.llm(f"m{m}", L, NQ, NKV, D, chunk_size=8192)
    act = gpu.activate(spec); gpu.finish_activation(act.engine_index)
    e = gpu.engine(act.engine_index); e.attach_device(max_step_tokens=8192 + B + 8)
    for i in range(B): e.push(i + 1, CTX - 1, 1_000_000)
    while e.counts()[1] or any(r.prompt_done < r.prompt_tokens for r in e.batch()):
        e.step(); e.append_kv_synthetic(0, L, 1)
    e.step(); e.append_kv_synthetic(0, L, 1)
    engs.append(e)
q = torch.randn((L, B, NQ, D), device="cuda").to(torch.bfloat16); o = torch.empty_like(q)
sc = 1 / math.sqrt(D)
def run(order, reps=4):
    for e in engs:
        for layer in range(L): e.decode_attention(layer, q[layer].data_ptr(), o[layer].data_ptr(), sc)
    dev.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    n = 0
    for _ in range(reps):
        for ei in order:
            for layer in range(L):
                engs[ei].decode_attention(layer, q[layer].data_ptr(), o[layer].data_ptr(), sc); n += 1
    t.record(); t.synchronize()
    return s.elapsed_time(t) / n
print("one engine only :", round(run([0, 0]), 5), "ms/launch")
print("alternating     :", round(run([0, 1]), 5), "ms/launch")
