"""Does CUDA VMM work (cuMemMap + cuMemSetAccess) slow the GPU down while
kernels run? Times 64 back-to-back K3 launches (C1 shape) with (a) no VMM
activity, (b) 8 single-page maps issued by the launching thread after the
first 8 launches, (c) the same maps issued by a second host thread."""
import json
import math
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402

L, NQ, NKV, D, B, CTX = 32, 32, 8, 128, 64, 2048


def main():
    dev = msim.Device(0)
    gpu = msim.GpuState(0, B * (CTX + 64) // 16 + 4200)
    gpu.ledger.attach_device(dev)
    spec = msim.ModelSpec.llm("m", L, NQ, NKV, D, chunk_size=4096)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device(max_step_tokens=CTX + B + 8)
    for i in range(B):
        eng.push(i + 1, CTX - 1, 1_000_000)
    while eng.counts()[1] or any(r.prompt_done < r.prompt_tokens for r in eng.batch()):
        eng.step()
        eng.append_kv_synthetic(0, L, 1)
    eng.step()
    q = torch.empty((B, NQ, D), dtype=torch.bfloat16, device="cuda")
    o = torch.empty_like(q)
    eng.synth_q(0, 1, 1.0, q.data_ptr())
    stream = torch.cuda.ExternalStream(dev.stream())
    scale = 1 / math.sqrt(D)
    # a second pool on the same ledger to map pages into
    other = msim.alloc_kvcache(gpu.ledger, "other", 131072, 4000)
    handles = []

    def do_maps(n):
        for _ in range(n):
            handles.append(msim.alloc_kv(other, gpu.ledger, 16))

    def run(mode, n_maps=8):
        dev.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        th = None
        t_host = 0.0
        for i in range(64):
            eng.decode_attention(i % L, q.data_ptr(), o.data_ptr(), scale)
            if i == 7 and mode == "inline":
                t0 = time.perf_counter()
                do_maps(n_maps)
                t_host = time.perf_counter() - t0
            if i == 7 and mode == "thread":
                th = threading.Thread(target=do_maps, args=(n_maps,))
                th.start()
        e.record(stream)
        e.synchronize()
        if th:
            th.join()
        for h in handles:
            msim.free_kv(other, gpu.ledger, h.handles)
        handles.clear()
        dev.reclaim(True)
        return s.elapsed_time(e), t_host

    for rep in range(2):
        for mode in ("none", "inline", "thread", "none"):
            ms, th = run(mode)
            print(json.dumps({"rep": rep, "mode": mode, "gpu_ms_64_k3": round(ms, 3),
                              "host_ms_in_maps": round(th * 1e3, 2)}), flush=True)
    print(json.dumps({"vmm_stats": dev.stats()}, default=str)[:2000])


if __name__ == "__main__":
    main()
