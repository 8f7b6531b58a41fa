"""Multi-GPU sharding of the hot path by model placement.

One process per GPU. The global scheduler (place_models, Prism Algorithm 1,
run through the C-ABI) assigns every model to a GPU; rank 0 computes the plan
and broadcasts it with torch.distributed (gloo on CPU, nccl on GPUs); each
rank then owns its models' ledger, pools and kernels. There is no collective
on the data path — only this host-side plan exchange and the final
max-over-ranks timing reduction in bench.py.
"""
from __future__ import annotations

from typing import Sequence

from . import msim


def plan(models: Sequence[msim.ModelDemandPy], n_gpus: int, capacity_bytes: int, tau_per_gb: float = 0.05,
         lib=None) -> msim.PlacementPlan:
    """place_models over n_gpus empty GPUs of capacity_bytes each."""
    gpus = [msim.GpuViewPy(g, capacity_bytes, 0, 0.0, capacity_bytes // msim.PAGE_BYTES,
                           capacity_bytes // msim.PAGE_BYTES) for g in range(n_gpus)]
    return msim.place_models(models, gpus, tau_per_gb, lib=lib)


def shard(models: Sequence[msim.ModelDemandPy], placement: msim.PlacementPlan, rank: int) -> list:
    """Models whose (first) part the plan put on `rank`, in input order."""
    return [m for m in models if placement.assignment[m.spec.model_id][0] == rank]


def broadcast_plan(placement_or_none, src: int = 0):
    """Rank `src` passes its plan; every rank returns the same plan."""
    import torch.distributed as dist

    box = [placement_or_none]
    dist.broadcast_object_list(box, src=src)
    return box[0]
