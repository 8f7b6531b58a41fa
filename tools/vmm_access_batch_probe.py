"""Does one cuMemSetAccess over N contiguous 16 MiB chunks cost less than N
calls, with the GPU idle and while HBM-bound kernels run back to back?
Driver API only (cuda-python): per round, N chunks are cuMemMap'ed at
consecutive VAs, made accessible either by N calls or by one call over the
range, then unmapped. The busy phase keeps a side stream saturated with
device-to-device copies (a stand-in for K3's HBM traffic, queue depth ~8 ms).
Prints one JSON line per (state, N, mode) with per-chunk p50 / p99 in us."""
import json
import statistics
import sys
import threading
import time

import torch
from cuda.bindings import driver as cu

CHUNK = 16 << 20
ROUNDS = 24


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


def main():
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    dev = 0
    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = dev
    acc = cu.CUmemAccessDesc()
    acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = dev
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    nmax = 8
    handles = [ck(cu.cuMemCreate(CHUNK, prop, 0)) for _ in range(nmax)]
    va = ck(cu.cuMemAddressReserve(CHUNK * nmax, CHUNK, 0, 0))
    base = int(va)

    def one_round(n, batched):
        nonlocal_base = base
        b0 = nonlocal_base
        for i in range(n):
            ck(cu.cuMemMap(b0 + i * CHUNK, CHUNK, 0, handles[i], 0))
        t0 = time.perf_counter()
        if batched:
            ck(cu.cuMemSetAccess(b0, CHUNK * n, [acc], 1))
        else:
            for i in range(n):
                ck(cu.cuMemSetAccess(b0 + i * CHUNK, CHUNK, [acc], 1))
        us = (time.perf_counter() - t0) * 1e6 / n
        ck(cu.cuMemUnmap(b0, CHUNK * n))
        return us

    def sweep(state):
        for n in (1, 4, 8):
            for batched in ((False, True) if n > 1 else (False,)):
                v = [one_round(n, batched) for _ in range(ROUNDS)]
                v.sort()
                print(json.dumps({"state": state, "chunks": n, "mode": "one call" if batched else "per chunk",
                                  "access_us_per_chunk_p50": round(statistics.median(v), 1),
                                  "access_us_per_chunk_p99": round(v[int(0.99 * (len(v) - 1))], 1)}), flush=True)

    sweep("idle")
    # the serving layout: each pool reserves V x 2 MiB of VA (180 GB) and
    # ~1,300 16 MiB chunks (20 GB of KV) are mapped elsewhere in the process
    big = int(ck(cu.cuMemAddressReserve(85830 * (2 << 20), CHUNK, 0, 0)))
    other = int(ck(cu.cuMemAddressReserve(1300 * CHUNK, CHUNK, 0, 0)))
    extra = []
    for i in range(1300):
        h = ck(cu.cuMemCreate(CHUNK, prop, 0))
        ck(cu.cuMemMap(other + i * CHUNK, CHUNK, 0, h, 0))
        extra.append(h)
    ck(cu.cuMemSetAccess(other, 1300 * CHUNK, [acc], 1))
    base_saved = base
    base = big + 40000 * (2 << 20)
    sweep("idle, 180 GB reservation + 1,300 chunks mapped")
    base = base_saved
    a = torch.empty(1 << 28, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    side = torch.cuda.Stream()
    stop = threading.Event()

    def load():
        with torch.cuda.stream(side):
            while not stop.is_set():
                for _ in range(50):  # ~0.16 ms per copy: ~8 ms queued
                    b.copy_(a)
                side.synchronize()

    th = threading.Thread(target=load)
    th.start()
    time.sleep(0.2)
    sweep("busy")
    stop.set()
    th.join()


if __name__ == "__main__":
    sys.exit(main())
