"""Yardstick for K3: FlashInfer's paged decode attention
(BatchDecodeWithPagedKVCacheWrapper, library code) on the same SURVEY §8d
model shapes and the same algorithmic bytes as tools/k3_shapes.py: B decodes
x CTX context, bf16 K/V in an NHD paged cache, one launch per layer, 3 x L
launches back to back timed with CUDA events (mean per launch). PAGE sets the
page size (1 = token-granular like prism's slot tables; 16 = vLLM's default).
Prints one JSON line per shape, fraction of MEASURED_PEAKS.json hbm_gbs."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200.configs import SHAPES  # noqa: E402

import flashinfer  # noqa: E402

B, CTX = int(os.environ.get("B", 64)), int(os.environ.get("CTX", 2048))
PAGE = int(os.environ.get("PAGE", 16))
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
ONLY = os.environ.get("SHAPES")
dev = torch.device("cuda")
for name, (L, nq, nkv, d, _) in SHAPES.items():
    if ONLY and name not in ONLY.split(","):
        continue
    pages_per_seq = math.ceil(CTX / PAGE)
    n_pages = B * pages_per_seq
    # one cache per layer (distinct memory, so L launches stream L x the bytes)
    caches = [torch.randn((n_pages, 2, PAGE, nkv, d), device=dev, dtype=torch.bfloat16) for _ in range(L)]
    perm = torch.randperm(n_pages, device=dev, dtype=torch.int32)  # scattered pages
    indptr = torch.arange(0, B + 1, device=dev, dtype=torch.int32) * pages_per_seq
    last = torch.full((B,), CTX - (pages_per_seq - 1) * PAGE, device=dev, dtype=torch.int32)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD", use_tensor_cores=(nq // nkv) >= 4)
    w.plan(indptr, perm, last, nq, nkv, d, PAGE, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
    q = torch.randn((L, B, nq, d), device=dev, dtype=torch.bfloat16)
    for layer in range(L):  # warm (JIT / first launch)
        w.run(q[layer], caches[layer])
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):  # as tools/k3_shapes.py: 3 passes over the layers, mean per launch
        for layer in range(L):
            w.run(q[layer], caches[layer])
    e.record()
    e.synchronize()
    best = s.elapsed_time(e) / (3 * L)
    nbytes = B * CTX * nkv * d * 4 + 2 * B * nq * d * 2
    print(json.dumps({"shape": name, "impl": "flashinfer", "page": PAGE, "G": nq // nkv, "d": d, "n_kv": nkv,
                      "ms": round(best, 4), "GBps": round(nbytes / best / 1e6, 1),
                      "frac": round(nbytes / best / 1e6 / peak, 4)}), flush=True)
    del caches, w, ws
    torch.cuda.empty_cache()
