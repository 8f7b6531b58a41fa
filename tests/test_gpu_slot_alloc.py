"""K1 (batched device slot allocator) parity: the GPU-resident slot state,
replaying the pool's op log, must produce exactly the (page, slot) stream of
the host allocator — which is itself bit-exact with the reference
(tests/test_pagealloc_parity.py) — and end in the same occupancy/bitmaps.
"""
import random

import pytest

from paper_2505_04021_b200 import msim

pytestmark = pytest.mark.gpu

CASES = [
    # (seed, token_bytes, vpages, capacity, ops, max_n, placement, sync_every)
    (1, 131072, 600, 600, 400, 40, 0, 1),      # llama-8B shape (tpp 16), sync every op
    (2, 131072, 600, 600, 600, 300, 0, 7),     # batched groups of ops, prefill-sized allocs
    (3, 12288, 300, 300, 500, 900, 0, 5),      # tpp 170 (7 u32 bitmap words), > 1024-token groups
    (4, 114688, 200, 150, 500, 60, 0, 3),      # tpp 18, near-full ledger (shortfalls)
    (5, 32768, 2000, 2000, 300, 2500, 0, 4),   # tpp 64, sub-batching of big allocs
]


def _host_state(pool, vpages):
    return [pool.page_occupied(p) for p in range(vpages)]


@pytest.mark.parametrize("case", CASES)
def test_k1_replay_matches_host(product, device, case):
    seed, tb, vpages, cap, ops, max_n, placement, sync_every = case
    rng = random.Random(seed)
    led = msim.PhysicalLedger(0, cap, lib=product)
    led.attach_device(device)
    pool = msim.alloc_kvcache(led, f"k1-{seed}", tb, vpages, placement)
    pool.attach_mirror()
    tpp = pool.tokens_per_page()
    live = []
    expected = []
    for i in range(ops):
        if not live or rng.random() < 0.55:
            r = msim.alloc_kv(pool, led, rng.randint(1, max_n))
            if r.handles:
                live.append(r.handles)
                expected += [h.page * tpp + h.slot for h in r.handles]
        else:
            k = rng.randrange(len(live))
            grp = live[k]
            if rng.random() < 0.3 and len(grp) > 1:
                cut = rng.randint(1, len(grp) - 1)
                part, live[k] = grp[:cut], grp[cut:]
            else:
                part = live.pop(k)
            msim.free_kv(pool, led, part)
        if (i + 1) % sync_every == 0 or i == ops - 1:
            got = pool.sync_mirror()
            assert got == expected, f"op {i}: first diff at {next(j for j in range(len(got)) if got[j] != expected[j]) if len(got) == len(expected) else 'len'}"
            expected = []
    occ = (pool.lib.prism_pool_read_mirror)
    import ctypes as C

    h_occ = (C.c_uint32 * vpages)()
    words = (tpp + 31) // 32
    h_bits = (C.c_uint32 * (vpages * words))()
    product.call("prism_pool_read_mirror", pool.h, h_occ, vpages, h_bits, vpages * words)
    assert list(h_occ) == _host_state(pool, vpages)
    for grp in live:
        for h in grp:
            assert (h_bits[h.page * words + h.slot // 32] >> (h.slot % 32)) & 1
    assert sum(bin(x).count("1") for x in h_bits) == pool.occupied_slots()
    msim.free_kvcache(led, pool)
