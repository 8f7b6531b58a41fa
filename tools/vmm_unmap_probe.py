"""Does cuMemUnmap wait for GPU work already queued (an implicit device
synchronisation)? Times cuMemUnmap of a 16 MiB mapping (one handle) with the
GPU idle, and with a ~40 ms spin kernel running on another stream; also the
per-call cost as a function of the number of chunks unmapped in one call.
Uses the driver API directly (cuda-python), no prism code."""
import json
import time

import torch
from cuda.bindings import driver as cu


def ck(r):
    if isinstance(r, tuple):
        err, *rest = r
    else:
        err, rest = r, []
    assert err == cu.CUresult.CUDA_SUCCESS, err
    return rest[0] if len(rest) == 1 else rest


def main():
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    dev = ck(cu.cuCtxGetDevice())
    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = int(dev)
    chunk = 16 << 20
    n = 64
    va = ck(cu.cuMemAddressReserve(chunk * n, 0, 0, 0))
    handles = [ck(cu.cuMemCreate(chunk, prop, 0)) for _ in range(n)]
    acc = cu.CUmemAccessDesc()
    acc.location = prop.location
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE

    def map_all():
        for i, h in enumerate(handles):
            ck(cu.cuMemMap(int(va) + i * chunk, chunk, 0, h, 0))
        ck(cu.cuMemSetAccess(va, chunk * n, [acc], 1))

    torch.cuda._sleep(1000)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch.cuda._sleep(10_000_000)
    e.record()
    e.synchronize()
    cyc = int(10_000_000 * 40.0 / s.elapsed_time(e))
    other = torch.cuda.Stream()
    out = {}
    for busy in (False, True):
        for batch in (1, 8):
            map_all()
            torch.cuda.synchronize()
            ts = []
            for i in range(0, n, batch):
                if busy:
                    with torch.cuda.stream(other):
                        torch.cuda._sleep(cyc)
                    time.sleep(0.002)
                t0 = time.perf_counter()
                ck(cu.cuMemUnmap(int(va) + i * chunk, chunk * batch))
                ts.append((time.perf_counter() - t0) * 1e6)
                if busy:
                    torch.cuda.synchronize()
            ts.sort()
            out[f"{'busy' if busy else 'idle'}_batch{batch}"] = {
                "calls": len(ts), "us_p50": round(ts[len(ts) // 2], 1), "us_max": round(ts[-1], 1)}
    # cuMemMap + cuMemSetAccess of one chunk, GPU idle vs busy
    for busy in (False, True):
        ts = []
        for i, h in enumerate(handles):
            if busy:
                with torch.cuda.stream(other):
                    torch.cuda._sleep(cyc)
                time.sleep(0.002)
            t0 = time.perf_counter()
            ck(cu.cuMemMap(int(va) + i * chunk, chunk, 0, h, 0))
            ck(cu.cuMemSetAccess(int(va) + i * chunk, chunk, [acc], 1))
            ts.append((time.perf_counter() - t0) * 1e6)
            if busy:
                torch.cuda.synchronize()
        ck(cu.cuMemUnmap(va, chunk * n))
        ts.sort()
        out[f"map_access_{'busy' if busy else 'idle'}"] = {
            "calls": len(ts), "us_p50": round(ts[len(ts) // 2], 1), "us_max": round(ts[-1], 1)}
    # cuMemSetAccess: 8 chunks in one call vs one call per chunk (GPU idle)
    for batch in (1, 8):
        ts = []
        for rep in range(4):
            for i, h in enumerate(handles):
                ck(cu.cuMemMap(int(va) + i * chunk, chunk, 0, h, 0))
            t0 = time.perf_counter()
            for i in range(0, n, batch):
                ck(cu.cuMemSetAccess(int(va) + i * chunk, chunk * batch, [acc], 1))
            ts.append((time.perf_counter() - t0) * 1e6 / n)
            ck(cu.cuMemUnmap(va, chunk * n))
        ts.sort()
        out[f"set_access_batch{batch}_us_per_chunk"] = round(ts[len(ts) // 2], 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
