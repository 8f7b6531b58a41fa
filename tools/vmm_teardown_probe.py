"""Does the exit of a process that held many VMM mappings slow the next
process's VMM calls, and for how long? `heavy`: map N pages and exit.
`sample`: map+unmap one fresh page every 50 ms for S seconds, printing the
latency over time (PRISM_PREMAP=0: each map is a real driver map)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402


def heavy(n):
    dev = msim.Device(0)
    gpu = msim.GpuState(0, n + 64)
    gpu.ledger.attach_device(dev)
    pool = msim.alloc_kvcache(gpu.ledger, "heavy", 131072, n + 16)
    t0 = time.perf_counter()
    msim.alloc_kv_raw(pool, gpu.ledger, 16 * n)
    print(json.dumps({"heavy_pages": n, "map_s": round(time.perf_counter() - t0, 3)}), flush=True)
    os._exit(0)  # exit with everything still mapped


def sample(seconds):
    t_start = time.perf_counter()
    dev = msim.Device(0)
    gpu = msim.GpuState(0, 4096)
    gpu.ledger.attach_device(dev)
    pool = msim.alloc_kvcache(gpu.ledger, "s", 131072, 4096)
    out = []
    while time.perf_counter() - t_start < seconds:
        t0 = time.perf_counter()
        r = msim.alloc_kv(pool, gpu.ledger, 16)
        dt = (time.perf_counter() - t0) * 1e3
        msim.free_kv(pool, gpu.ledger, r.handles)
        dev.reclaim(True)
        out.append((round(time.perf_counter() - t_start, 2), round(dt, 3)))
        time.sleep(0.05)
    buckets = {}
    for t, ms in out:
        buckets.setdefault(int(t // 2) * 2, []).append(ms)
    print(json.dumps({f"{k}s": round(sorted(v)[len(v) // 2], 3) for k, v in sorted(buckets.items())}))


if __name__ == "__main__":
    if sys.argv[1] == "heavy":
        heavy(int(sys.argv[2]))
    else:
        sample(float(sys.argv[2]))
