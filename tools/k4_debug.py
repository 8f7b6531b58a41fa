"""K4 bring-up: one prefill chunk through prism_engine_prefill_attention with
a watchdog thread that prints the kernel's progress words (PRISM_K4_DEBUG=1)
if it does not finish, then checks a few query tokens against the oracle.
  python tools/k4_debug.py [shape] [prompt] [chunk]"""
import ctypes as C
import math
import os
import sys
import threading
import time

os.environ.setdefault("PRISM_K4_DEBUG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2505_04021_b200 import msim  # noqa: E402
from tests import scenarios as S  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "llama3.1-8b"
prompt = int(sys.argv[2]) if len(sys.argv) > 2 else 100
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 512
qs = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
dev = msim.Device(0)
torch.cuda.set_stream(torch.cuda.ExternalStream(dev.stream()))  # producers on the engine stream
lib = msim.capi.product()
gpu = msim.GpuState(0, 2000)
gpu.ledger.attach_device(dev)
spec = S.shape_spec(shape, "dbg", chunk=chunk, weight_scale=0.0)
act = gpu.activate(spec)
gpu.finish_activation(act.engine_index)
eng = gpu.engine(act.engine_index)
eng.attach_device()
eng.push(1, prompt, 2)
L, nkv, nq, d = spec.n_layers, spec.n_kv_heads, spec.n_q_heads, spec.head_dim
gen = torch.Generator(device="cuda").manual_seed(0)
done = threading.Event()


def watchdog():
    while not done.wait(5.0):
        w = (C.c_uint32 * 16)()
        got = C.c_int32()
        lib.call("prism_debug_k4_progress", w, 16, C.byref(got))
        print("K4 progress of CTA 0 (loader Q segment, loader tile, S issued by MMA warp 0 / 1, P.V issued, "
              "softmax 0 has S, posted P, epilogue):",
              list(w)[:8], flush=True)


threading.Thread(target=watchdog, daemon=True).start()
ks, vs = [], []
while True:
    eng.step()
    n_tok, _ = eng.step_info()
    k = (torch.rand((L, n_tok, nkv, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    v = (torch.rand((L, n_tok, nkv, d), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    eng.append_kv(0, L, k.data_ptr(), v.data_ptr())
    ks.append(k[1].cpu())
    vs.append(v[1].cpu())
    n_pf, first, rid = eng.prefill_info()
    print("step: tokens", n_tok, "prefill", n_pf, "first", first, flush=True)
    q = ((torch.rand((max(n_pf, 1), nq, d), generator=gen, device="cuda") * 2 - 1) * qs).to(torch.bfloat16)
    o = torch.full_like(q, float("nan"))
    t0 = time.time()
    eng.prefill_attention(1, q.data_ptr(), o.data_ptr(), 1 / math.sqrt(d))
    eng.synchronize()
    print(f"K4 done in {time.time() - t0:.3f}s", flush=True)
    kk, vv = torch.cat(ks), torch.cat(vs)
    bits = lambda t: t.contiguous().view(torch.int16).numpy().view(np.uint16)  # noqa: E731
    oc = o.float().cpu().numpy()
    nanrows = np.isnan(oc).any(axis=2)  # [token][head]
    if nanrows.any():
        tk, hd = np.nonzero(nanrows)
        print("  NaN rows:", len(tk), "tokens", sorted(set(tk.tolist()))[:20], "heads", sorted(set(hd.tolist())))
    worst = 0.0
    # vectorised fp64 reference for every query token of the chunk
    G = nq // nkv
    qf = q[:n_pf].float().cpu().double().numpy().reshape(n_pf, nkv, G, d)
    kf = kk.float().double().numpy()  # [ctx][nkv][d]
    vf = vv.float().double().numpy()
    sc = np.einsum("ihgd,khd->ihgk", qf, kf[:first + n_pf]) / math.sqrt(d)
    mask = (np.arange(first + n_pf)[None, :] <= (first + np.arange(n_pf))[:, None])  # [i][k]
    sc = np.where(mask[:, None, None, :], sc, -np.inf)
    sc -= sc.max(-1, keepdims=True)
    pr = np.exp(sc)
    pr /= pr.sum(-1, keepdims=True)
    ref = np.einsum("ihgk,khd->ihgd", pr, vf[:first + n_pf]).reshape(n_pf, nq, d)
    err = np.abs(oc[:n_pf] - ref)
    tq = 128 // G
    bad = err > 2e-3 + 1e-2 * np.abs(ref)
    per_tile = [float(err[i:i + tq].max()) for i in range(0, n_pf, tq)]
    print("  max err per q tile:", " ".join(f"{e:.1e}" for e in per_tile))
    print("  bad elements:", int(bad.sum()), "of", bad.size, "bad heads:", sorted(set(np.nonzero(bad)[1].tolist()))[:16])
    worst = float(err.max())
    if first + n_pf >= prompt:
        break
done.set()
print("worst", worst)
