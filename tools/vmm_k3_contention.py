"""How long does a page map take on the VMM worker while K3 runs back to
back, and does it slow K3? A side thread maps fresh pages one at a time
(each an urgent map through the worker, waited for) while the main thread
keeps launching C1-shaped K3s. Variant from PRISM_K3 (streamk|mma); stream-K
spread from PRISM_SK_SMS."""
import json
import math
import os
import statistics
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
    dev.quiesce()
    q = torch.empty((B, NQ, D), dtype=torch.bfloat16, device="cuda")
    o = torch.empty_like(q)
    eng.synth_q(0, 1, 1.0, q.data_ptr())
    stream = torch.cuda.ExternalStream(dev.stream())
    scale = 1 / math.sqrt(D)
    other = msim.alloc_kvcache(gpu.ledger, "other", 131072, 4000)
    held = []

    def k3_loop(n):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for i in range(n):
            eng.decode_attention(i % L, q.data_ptr(), o.data_ptr(), scale)
        e.record(stream)
        e.synchronize()
        return s.elapsed_time(e) / n

    def mapper(out, n, stop):
        for _ in range(n):
            if stop.is_set():
                break
            t0 = time.perf_counter()
            held.append(msim.alloc_kv(other, gpu.ledger, 16 * 1))
            out.append((time.perf_counter() - t0) * 1e3)

    k3_loop(64)
    idle_k3 = k3_loop(512)
    dev.reset_stats()
    # maps with the GPU idle
    lat_idle = []
    mapper(lat_idle, 24, threading.Event())
    st0 = dev.stats()
    dev.reset_stats()
    # maps while K3 runs back to back
    lat_busy, stop = [], threading.Event()
    th = threading.Thread(target=mapper, args=(lat_busy, 24, stop))
    dev.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    th.start()
    n = 0
    qdepth = int(os.environ.get("QDEPTH", "256"))  # launches between host syncs
    while th.is_alive() and n < 20000:
        for i in range(32):
            eng.decode_attention(i, q.data_ptr(), o.data_ptr(), scale)
        n += 32
        if n % qdepth == 0:
            ev = torch.cuda.Event()
            ev.record(stream)
            ev.synchronize()
    e.record(stream)
    e.synchronize()
    stop.set()
    th.join()
    busy_k3 = s.elapsed_time(e) / max(n, 1)
    st = dev.stats()
    print(json.dumps({"qdepth": qdepth, "variant": os.environ.get("PRISM_K3", "streamk(default)"), "sk_sms": os.environ.get("PRISM_SK_SMS"),
                      "k3_ms_idle": round(idle_k3, 4), "k3_ms_while_mapping": round(busy_k3, 4), "k3_launches": n,
                      "map_ms_idle_p50": round(statistics.median(lat_idle), 3),
                      "map_ms_busy_p50": round(statistics.median(lat_busy), 3) if lat_busy else None,
                      "map_ms_busy_max": round(max(lat_busy), 3) if lat_busy else None, "maps_busy": len(lat_busy),
                      "premap": os.environ.get("PRISM_PREMAP", "1"), "sk_per_sm": os.environ.get("PRISM_SK_PER_SM"),
                      "idle_us": per_call(st0), "busy_us": per_call(st)}))


def per_call(st):
    return {"create": round(st["create_ns_total"] / max(st["creates"], 1) / 1e3, 1),
            "setaccess": round(st["access_ns_total"] / max(st["access_calls"], 1) / 1e3, 1),
            "map": round(st["map_call_ns_total"] / max(st["access_calls"], 1) / 1e3, 1),
            "creates": st["creates"], "access_calls": st["access_calls"]}


if __name__ == "__main__":
    main()
