"""Model weight loading for activation:
the fan-in plan (which helper copies which chunk), the C-ABI surface, and the
measured-bandwidth activation curve. The copies themselves are GPU tests
(tests/test_gpu_weight_load.py)."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_04021_b200 import msim


@pytest.mark.parametrize("n,chunk,parts", [(0, 8, 2), (1, 8, 3), (64, 8, 1), (65, 8, 2), (1000, 7, 8), (8 << 20, 1 << 20, 3)])
def test_fanin_plan_covers_every_byte_once(n, chunk, parts):
    plan = msim.fanin_parts(n, chunk, parts)
    assert len(plan) == parts
    spans = sorted(s for p in plan for s in p)
    pos = 0
    for off, ln in spans:
        assert off == pos and 0 < ln <= chunk
        pos += ln
    assert pos == n
    # round robin: helper loads differ by at most one chunk
    sizes = [len(p) for p in plan]
    assert max(sizes) - min(sizes) <= 1


def test_measured_activation_curve():
    c = msim.measured_activation_curve(50.0, fixed_s=0.1)
    assert c == [(16e9, 0.1 + 16e9 / 50e9), (28e9, 0.1 + 28e9 / 50e9)]


def test_abi_declares_weight_loader(product):
    from paper_2505_04021_b200 import capi
    for name in ("prism_wloader_create", "prism_wloader_load", "prism_wloader_load_part", "prism_wloader_wait",
                 "prism_ipc_handle", "prism_ipc_open", "prism_host_register"):
        assert name in capi.DEVICE_SYMBOLS
        assert hasattr(product.dll, name)


def _rank(rank, world, port, n, chunk, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = msim.fanin_parts(n, chunk, world)[rank]
    got = [None] * world
    dist.all_gather_object(got, mine)
    if rank == 0:
        out.put(sorted(s for p in got for s in p))
    dist.destroy_process_group()


def test_fanin_plan_two_ranks_gloo():
    """Each rank derives its own share independently; together they tile the
    weights exactly (the N-helper fan-in needs no coordination beyond the
    target pointer)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    n, chunk = (3 << 20) + 5, 1 << 18
    procs = [ctx.Process(target=_rank, args=(r, 2, port, n, chunk, q)) for r in range(2)]
    for p in procs:
        p.start()
    spans = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pos = 0
    for off, ln in spans:
        assert off == pos
        pos += ln
    assert pos == n
