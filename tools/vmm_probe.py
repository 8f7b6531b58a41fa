"""CUDA VMM driver-call costs on a B200, idle vs. with the GPU busy on another
stream, and whether each call waits for that work (the call returning while
the kernel still runs means it does not block on the device)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402


def busy(ms):
    """Queue ~ms of matmul work on torch's stream; returns an event at its end."""
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    e = torch.cuda.Event()
    n = max(1, int(ms / 0.7))
    for _ in range(n):
        a = a @ a
        a = a / 64.0
    e.record()
    return e


def measure(label, fn, load_ms):
    torch.cuda.synchronize()
    ev = busy(load_ms) if load_ms else None
    t0 = time.perf_counter()
    fn()
    dt = time.perf_counter() - t0
    still_busy = (not ev.query()) if ev is not None else None
    torch.cuda.synchronize()
    return {"op": label, "load_ms": load_ms, "us_total": round(dt * 1e6, 1), "gpu_still_busy_after": still_busy}


def main():
    out = []
    dev = msim.Device(0)
    for load in (0, 200):
        led = msim.PhysicalLedger(0, 4096)
        led.attach_device(dev)
        pool = msim.alloc_kvcache(led, f"p{load}", 131072, 4096)
        n = 64
        out.append(measure("create x64 (refill_buffer)", lambda: led.refill_buffer(n), load))
        dev.reset_stats()
        holder = {}
        out.append(measure("map x64 contiguous (buffer handles)",
                           lambda: holder.setdefault("r", msim.alloc_kv(pool, led, 16 * n)), load))
        st = dev.stats()
        out.append({"op": "  breakdown", "load_ms": load, "map_call_us": st["map_call_ns_total"] / 1e3,
                    "access_us": st["access_ns_total"] / 1e3, "access_calls": st["access_calls"]})
        out.append(measure("park x64 (free_kv)", lambda: msim.free_kv(pool, led, holder["r"].handles), load))
        out.append(measure("revive x64 (alloc_kv again)",
                           lambda: holder.__setitem__("r2", msim.alloc_kv(pool, led, 16 * n)), load))
        msim.free_kv(pool, led, holder["r2"].handles)
        dev.reset_stats()
        out.append(measure("driver unmap x64 (reclaim)", lambda: dev.reclaim(False) or dev.fence() or dev.reclaim(True),
                           load))
        # single-page maps, each its own SetAccess (the decode pattern)
        dev.reset_stats()
        hs = []

        def singles():
            for _ in range(16):
                hs.append(msim.alloc_kv(pool, led, 16))

        out.append(measure("map x16 one page per call (cache handles)", singles, load))
        st = dev.stats()
        out.append({"op": "  breakdown", "load_ms": load, "map_call_us": st["map_call_ns_total"] / 1e3,
                    "access_us": st["access_ns_total"] / 1e3, "access_calls": st["access_calls"],
                    "create_us": st["create_ns_total"] / 1e3})
        for h in hs:
            msim.free_kv(pool, led, h.handles)
        msim.free_kvcache(led, pool)
    for r in out:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
