"""N>1 path on CPU: world_size-2 gloo. Rank 0 places 24 C4-style models on 2
"GPUs", broadcasts the plan, each rank runs its own shard (host engines on its
own ledger, no data-path collective), and the gathered per-model results
equal a single-process run of the same shards."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_04021_b200 import cluster, msim
from tests import scenarios as S


def _models():
    names = list(S.SHAPES)
    out = []
    for i in range(24):
        spec = S.shape_spec(names[i % len(names)], f"{names[i % len(names)]}#{i}", chunk=256, weight_scale=0.02)
        out.append(msim.ModelDemandPy(spec, rate=0.5 + (i * 7 % 11) * 0.3))
    return out


def run_shard(models) -> dict:
    """Each model: a small fixed request burst on this rank's ledger."""
    if not models:
        return {}
    gpu = msim.GpuState(0, 6000)
    res = {}
    engines = []
    for m in models:
        act = gpu.activate(m.spec)
        gpu.finish_activation(act.engine_index)
        e = gpu.engine(act.engine_index)
        for r in range(4):
            e.push(r + 1, 100 + 37 * r, 20 + r)
        engines.append((m.spec.model_id, e))
    now = 0
    for _ in range(400):
        ran = False
        for mid, e in engines:
            if e.has_runnable_work():
                o = e.step(now_us=now)
                now += o.duration_us
                res.setdefault(mid, []).append([o.duration_us, o.chunk_tokens, o.decode_tokens, o.completions])
                ran = True
        if not ran:
            break
    return {k: S.digest(v) for k, v in res.items()}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    models = _models()
    plan = cluster.plan(models, world, 180 * 10**9) if rank == 0 else None
    plan = cluster.broadcast_plan(plan)
    mine = run_shard(cluster.shard(models, plan, rank))
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        q.put((plan.assignment, gathered))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_sharded_run_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    assignment, gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    models = _models()
    plan = cluster.plan(models, 2, 180 * 10**9)
    assert plan.assignment == assignment
    for rank in range(2):
        assert gathered[rank] == run_shard(cluster.shard(models, plan, rank))
    # every model ran on exactly one rank and the load is split across both
    names = [k for g in gathered for k in g]
    assert sorted(names) == sorted(m.spec.model_id for m in models)
    assert all(len(g) > 0 for g in gathered)
