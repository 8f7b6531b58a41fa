"""Repeat bench.py's e2e arm (host buffers through the C-ABI) several times in
one process and break each run's host time down (engine step, async issue,
wait for outputs), to find what makes e2e throughput vary between runs."""
import json
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main(reps=int(os.environ.get("REPS", 6)), steps=30):
    torch.cuda.set_device(0)
    mids = bench.placement_for(1, 0)
    dev, gpu, models = bench.setup_gpu(0, mids, reps * (steps + 2) + 16)
    scale = 1.0 / math.sqrt(bench.D)
    n = bench.L * bench.B_PER_MODEL * bench.NKV * bench.D
    nq = bench.L * bench.B_PER_MODEL * bench.NQ * bench.D
    bufs = []
    for _ in models:
        t = [torch.empty(k, dtype=torch.bfloat16).pin_memory() for k in (n, n, nq, nq)]
        for x in t[:3]:
            x.uniform_(-1, 1)
        bufs.append(t)
    print(json.dumps({"cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}), flush=True)
    for rep in range(reps):
        dev.reset_stats()
        t_step = t_issue = t_wait = 0.0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            for m, (hk, hv, hq, ho) in zip(models, bufs):
                a = time.perf_counter()
                m.eng.wait_host()
                b = time.perf_counter()
                m.eng.step()
                c = time.perf_counter()
                m.eng.decode_host_async(hk.data_ptr(), hv.data_ptr(), hq.data_ptr(), ho.data_ptr(), scale)
                d = time.perf_counter()
                t_wait += b - a
                t_step += c - b
                t_issue += d - c
        for m in models:
            m.eng.wait_host()
        sec = time.perf_counter() - t0
        st = dev.stats()
        tok = steps * len(models) * bench.B_PER_MODEL
        print(json.dumps({"rep": rep, "tokens_per_s": round(tok / sec, 1), "ms_per_step": round(sec / steps * 1e3, 3),
                          "host_ms_per_step": {"wait": round(t_wait / steps * 1e3, 3),
                                               "engine_step": round(t_step / steps * 1e3, 3),
                                               "issue": round(t_issue / steps * 1e3, 3)},
                          "maps": st["maps"], "premapped_hits": st["premapped_hits"],
                          "caller_map_ms": round(st["map_ns_total"] / 1e6, 3),
                          "worker_ms": round(st["background_ns_total"] / 1e6, 3)}), flush=True)


if __name__ == "__main__":
    main()
