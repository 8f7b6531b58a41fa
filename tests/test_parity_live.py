"""Live differential parity against the compiled reference (needs
oracle/_ref/libmsim_ref.so, built where /root/reference exists): fresh seeds
beyond the golden set, both placements, buffer, weights, caps, misuse."""
import json
import random

import pytest

from paper_2505_04021_b200 import capi, msim
from tests import scenarios as S

pytestmark = pytest.mark.reference


def _norm(x):
    return json.loads(json.dumps(x))


@pytest.mark.parametrize("seed", [101, 202, 303, 404])
@pytest.mark.parametrize("placement", [0, 1])
def test_allocator_fuzz_vs_reference(product, reference, seed, placement):
    rng = random.Random(seed)
    case = dict(seed=seed, placement=placement, capacity=rng.randint(30, 600), vpages=rng.randint(20, 700),
                token_bytes=rng.choice([16 << 10, 131072, 12288, 114688, 57344, 1 << 20]), ops=1500,
                max_n=rng.choice([1, 8, 64, 400]))
    assert _norm(S.allocator_fuzz(product, **case)) == _norm(S.allocator_fuzz(reference, **case))


def test_mapped_page_cap_vs_reference(product, reference):
    def run(lib):
        led = msim.PhysicalLedger(0, 100, lib=lib)
        pool = msim.alloc_kvcache(led, "m", 131072, 100)
        pool.set_mapped_page_cap(5)
        out = [pool.allocatable_tokens(led)]
        r = msim.alloc_kv(pool, led, 70)
        out.append([r.shortfall_pages, len(r.handles)])
        r = msim.alloc_kv(pool, led, 80)
        out.append([r.shortfall_pages, len(r.handles), pool.mapped_pages()])
        pool.set_mapped_page_cap(None)
        out.append(pool.allocatable_tokens(led))
        return out

    assert run(product) == run(reference)


def test_misuse_vs_reference(product, reference):
    def run(lib):
        led = msim.PhysicalLedger(0, 64, lib=lib)
        other = msim.PhysicalLedger(1, 64, lib=lib)
        pool = msim.alloc_kvcache(led, "m", 16 << 10, 10)
        res = []
        r = msim.alloc_kv(pool, led, 5)
        for bad in ([msim.TokenSlotHandle(pool.id(), 9, 0)], [msim.TokenSlotHandle(pool.id(), 0, 127)],
                    [msim.TokenSlotHandle(pool.id(), 10, 0)], [msim.TokenSlotHandle(pool.id() + 1, 0, 0)]):
            try:
                msim.free_kv(pool, led, bad)
                res.append("ok")
            except capi.UsageError as e:
                res.append(e.message)
        try:
            msim.alloc_kv(pool, other, 1)
        except capi.UsageError as e:
            res.append(e.message)
        # partial application before a stale handle, like the reference
        try:
            msim.free_kv(pool, led, r.handles[:2] + r.handles[:1])
        except capi.UsageError as e:
            res.append(e.message)
        res.append([pool.occupied_slots(), pool.mapped_pages()])
        msim.free_kvcache(led, pool)
        for fn in (lambda: msim.free_kvcache(led, pool), lambda: msim.alloc_kv(pool, led, 1)):
            try:
                fn()
            except capi.UsageError as e:
                res.append(e.message)
        try:
            msim.alloc_kvcache(led, "z", 0, 10)
        except capi.UsageError as e:
            res.append(e.message)
        try:
            msim.alloc_kvcache(led, "z", 100, 0)
        except capi.UsageError as e:
            res.append(e.message)
        return res

    assert run(product) == run(reference)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_engine_random_traces_vs_reference(product, reference, seed):
    rng = random.Random(seed)
    shapes = rng.sample(list(S.SHAPES), 3)
    case = dict(name=f"live{seed}", seed=seed, capacity=rng.randint(150, 2000),
                models=[(s, f"{s}@{k}") for k, s in enumerate(shapes)], rate=rng.uniform(1, 10),
                horizon=10.0, prompt=(rng.choice([64, 300, 900]), 0.5), output=(rng.choice([8, 60, 200]), 0.5),
                chunk=rng.choice([32, 128, 512]), steps=400, weight_scale=0.01)
    assert _norm(S.engine_trace(product, **case)) == _norm(S.engine_trace(reference, **case))


def test_throughput_of_vs_reference(product, reference):
    spec = S.shape_spec("llama3.1-8b", "8b")
    spec.token_kv_bytes = 16 << 10
    a = msim.throughput_of(5 * 10**9, spec, 2048, 256, warmup_s=2, window_s=6, lib=product)
    b = msim.throughput_of(5 * 10**9, spec, 2048, 256, warmup_s=2, window_s=6, lib=reference)
    assert a == b


@pytest.mark.parametrize("seed", [7, 8])
def test_placement_random_vs_reference(product, reference, seed):
    case = dict(seed=seed, n_gpus=random.Random(seed).randint(1, 8), n_models=20, tau=0.05, placed_frac=0.5)
    assert _norm(S.placement_case(product, **case)) == _norm(S.placement_case(reference, **case))
