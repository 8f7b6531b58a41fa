"""Cost of the CUDA VMM calls vs physical handle size (idle GPU): for each
handle size, create / map / set-access / unmap / release REPS handles
laid out contiguously, and report microseconds per call and per 2 MiB.
Also: 8 x 2 MiB handles made accessible by ONE cuMemSetAccess over the run."""
import json
import statistics
import time

from cuda.bindings import driver as d

MIB = 1 << 20


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


def main(reps=16):
    ck(d.cuInit(0))
    dev = ck(d.cuDeviceGet(0))
    ctx = ck(d.cuDevicePrimaryCtxRetain(dev))
    ck(d.cuCtxSetCurrent(ctx))
    prop = d.CUmemAllocationProp()
    prop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = 0
    acc = d.CUmemAccessDesc()
    acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = 0
    acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    out = []
    for size_mib in (2, 4, 8, 16, 32, 64):
        size = size_mib * MIB
        va = ck(d.cuMemAddressReserve(size * reps, 2 * MIB, 0, 0))
        t = {k: [] for k in ("create", "map", "access", "unmap", "release")}
        for rnd in range(3):
            hs = []
            for i in range(reps):
                t0 = time.perf_counter()
                hs.append(ck(d.cuMemCreate(size, prop, 0)))
                t["create"].append(time.perf_counter() - t0)
            for i, h in enumerate(hs):
                t0 = time.perf_counter()
                ck(d.cuMemMap(int(va) + i * size, size, 0, h, 0))
                t["map"].append(time.perf_counter() - t0)
            for i in range(reps):
                t0 = time.perf_counter()
                ck(d.cuMemSetAccess(int(va) + i * size, size, [acc], 1))
                t["access"].append(time.perf_counter() - t0)
            for i in range(reps):
                t0 = time.perf_counter()
                ck(d.cuMemUnmap(int(va) + i * size, size))
                t["unmap"].append(time.perf_counter() - t0)
            for h in hs:
                t0 = time.perf_counter()
                ck(d.cuMemRelease(h))
                t["release"].append(time.perf_counter() - t0)
        ck(d.cuMemAddressFree(va, size * reps))
        med = {k: statistics.median(v) * 1e6 for k, v in t.items()}
        out.append({"handle_MiB": size_mib, "us_per_call": {k: round(v, 1) for k, v in med.items()},
                    "us_per_2MiB": {k: round(v * 2 / size_mib, 1) for k, v in med.items()}})
        print(json.dumps(out[-1]), flush=True)
    # one SetAccess over a run of eight separately mapped 2 MiB handles
    size = 2 * MIB
    va = ck(d.cuMemAddressReserve(size * 8, 2 * MIB, 0, 0))
    tt = []
    for rnd in range(5):
        hs = [ck(d.cuMemCreate(size, prop, 0)) for _ in range(8)]
        for i, h in enumerate(hs):
            ck(d.cuMemMap(int(va) + i * size, size, 0, h, 0))
        t0 = time.perf_counter()
        ck(d.cuMemSetAccess(int(va), 8 * size, [acc], 1))
        tt.append(time.perf_counter() - t0)
        ck(d.cuMemUnmap(int(va), 8 * size))
        for h in hs:
            ck(d.cuMemRelease(h))
    print(json.dumps({"setaccess_8x2MiB_one_call_us": round(statistics.median(tt) * 1e6, 1)}))


if __name__ == "__main__":
    main()
