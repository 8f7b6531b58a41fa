"""Staged weight fan-in across processes:
every rank loads its share of the chunks (chunk i -> rank i % world) from its
own pinned host copy of the weights through its GPU's staging slots, and
writes them into rank 0's target buffer through a CUDA IPC pointer (NVLink
when the ranks sit on different GPUs). Rank 0 checks the bytes and prints
one JSON line (device ms = max over ranks).

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      tools/wload_fanin.py [--mib 1024] [--chunk-mib 8] [--streams 4]

PRISM_WLOAD_DEVICE pins every rank to one GPU (single-GPU boxes: the test
runs 2 ranks on cuda:0 over gloo, PRISM_WLOAD_BACKEND=gloo). Needs
PYTORCH_NO_CUDA_MEMORY_CACHING=1 so the target is a cudaMalloc base pointer
(what CUDA IPC hands out)."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--chunk-mib", type=int, default=8)
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--seed", type=int, default=20251017)
    a = ap.parse_args()
    assert os.environ.get("PYTORCH_NO_CUDA_MEMORY_CACHING") == "1", "set PYTORCH_NO_CUDA_MEMORY_CACHING=1"
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dev = int(os.environ.get("PRISM_WLOAD_DEVICE", os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    backend = os.environ.get("PRISM_WLOAD_BACKEND", "nccl" if world > 1 else "gloo")
    if world > 1:
        dist.init_process_group(backend)
    n = (a.mib << 20) + 12345  # ragged tail chunk
    gen = torch.Generator().manual_seed(a.seed)
    host = torch.randint(0, 256, (n,), dtype=torch.uint8, generator=gen).pin_memory()
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda") if rank == 0 else None
    handle = msim.ipc_handle(dst.data_ptr()) if rank == 0 else None
    if world > 1:
        box = [handle]
        dist.broadcast_object_list(box, src=0)
        handle = box[0]
    ptr = dst.data_ptr() if rank == 0 else msim.ipc_open(dev, handle)
    wl = msim.WeightLoader(dev, a.streams, a.chunk_mib << 20)
    if world > 1:
        dist.barrier()
    wl.load_part(host.data_ptr(), ptr, n, rank, world)
    ms = wl.wait()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()  # every helper's copies are done before rank 0 reads
    if rank == 0:
        ok = bool(torch.equal(dst.cpu(), host))
        print(json.dumps({"fanin_ranks": world, "bytes": n, "chunk_mib": a.chunk_mib, "streams": a.streams,
                          "ms_max_over_ranks": round(ms, 3), "gbs": round(n / ms / 1e6, 2), "bit_exact": ok}),
              flush=True)
    else:
        msim.ipc_close(dev, ptr)
    wl.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
