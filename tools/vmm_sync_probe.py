"""Does a CUDA VMM map (cuMemCreate + cuMemMap + cuMemSetAccess) wait for
GPU work already queued? Times single-page logical maps (a fresh page each,
access set inside the call) with the GPU idle, with a 40 ms spin kernel
running on the VMM device's stream, and with it running on another stream.
Run with PRISM_PREMAP=0 so the background worker stays idle."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402


def main():
    assert os.environ.get("PRISM_PREMAP") == "0", "run with PRISM_PREMAP=0"
    dev = msim.Device(0)
    gpu = msim.GpuState(0, 4096)
    gpu.ledger.attach_device(dev)
    pool = msim.alloc_kvcache(gpu.ledger, "probe", 131072, 4096)  # 16 tokens per page
    vmm_stream = torch.cuda.ExternalStream(dev.stream())
    other = torch.cuda.Stream()
    # spin-kernel calibration: cycles for ~40 ms
    torch.cuda._sleep(1000)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch.cuda._sleep(10_000_000)
    e.record()
    e.synchronize()
    cyc = int(10_000_000 * 40.0 / s.elapsed_time(e))
    held = []

    def one_map():
        t0 = time.perf_counter()
        held.append(msim.alloc_kv(pool, gpu.ledger, 16))
        return (time.perf_counter() - t0) * 1e3

    def unmap_one():
        h = held.pop()
        t0 = time.perf_counter()
        msim.free_kv(pool, gpu.ledger, h.handles)
        dev.reclaim(False)
        return (time.perf_counter() - t0) * 1e3

    out = {}
    for mode in ("idle", "busy_vmm_stream", "busy_other_stream", "idle"):
        times = []
        for _ in range(6):
            torch.cuda.synchronize()
            dev.synchronize()
            if mode == "busy_vmm_stream":
                with torch.cuda.stream(vmm_stream):
                    torch.cuda._sleep(cyc)
            elif mode == "busy_other_stream":
                with torch.cuda.stream(other):
                    torch.cuda._sleep(cyc)
            time.sleep(0.002)  # let the kernel start
            times.append(one_map())
        torch.cuda.synchronize()
        out[mode] = [round(t, 3) for t in times]
        print(json.dumps({"mode": mode, "map_ms": out[mode]}), flush=True)
    st = dev.stats()
    print(json.dumps({k: st[k] for k in ("maps", "creates", "access_calls", "create_ns_total", "map_call_ns_total",
                                          "access_ns_total")}))
    # driver unmap (steal path) while busy
    for mode in ("idle", "busy_other_stream"):
        times = []
        for _ in range(4):
            torch.cuda.synchronize()
            dev.synchronize()
            dev.reclaim(True)
            if mode == "busy_other_stream":
                with torch.cuda.stream(other):
                    torch.cuda._sleep(cyc)
            time.sleep(0.002)
            h = held.pop()
            msim.free_kv(pool, gpu.ledger, h.handles)  # park
            dev.fence()
            time.sleep(0.001)  # the fence on the (idle) VMM stream passes
            t0 = time.perf_counter()
            dev.reclaim(False)  # fence passed long ago -> cuMemUnmap now
            times.append(round((time.perf_counter() - t0) * 1e3, 3))
        torch.cuda.synchronize()
        print(json.dumps({"mode": mode, "reclaim_unmap_ms": times}), flush=True)


if __name__ == "__main__":
    main()
