"""Pin the C restatement oracle (oracle/restate/prism_oracle.c) before
trusting it: its allocator must reproduce the reference's golden streams
bit for bit, and its fp64 attention must agree with an independent
implementation (numpy, float64). The attention itself has no reference
counterpart: its parity is pinned only by definition."""
import ctypes as C
import math
import random

import numpy as np
import pytest

import oracle
from tests import scenarios as S


class _Ledger(C.Structure):
    _fields_ = [("capacity", C.c_uint64), ("kv_mapped", C.c_uint64), ("buffer", C.c_uint64),
                ("weights", C.c_uint64)]


def restate_allocator_fuzz(seed, placement, capacity, vpages, token_bytes, ops, max_n):
    """Same op sequence as tests/scenarios.py allocator_fuzz, applied to the
    restatement; ledger, events and weights are kept here in Python exactly as
    reference src/pagealloc.cpp:17-106 defines them."""
    lib = oracle.restate()
    rng = random.Random(seed)
    tpp = (2 << 20) // token_bytes
    led = _Ledger(capacity, 0, 0, 0)
    pool_id = 1
    pool = lib.po_pool_create(pool_id, tpp, vpages, placement)
    events, trace, stream, live = [], [], [], []
    now = 0
    weights_held = False
    weights = 0

    def free_pages():
        return led.capacity - led.kv_mapped - led.buffer - led.weights

    def ev(kind, pages, model="m"):
        events.append([now, model, kind, pages])

    for _ in range(ops):
        now += rng.randint(1, 50)
        u = rng.random()
        if u < 0.05:
            target = rng.randint(0, 12)
            add = 0
            if target > led.buffer:
                add = min(target - led.buffer, free_pages())
                led.buffer += add
                if add:
                    ev("map", add, "")
            trace.append(["refill", add])
        elif u < 0.07:
            if weights_held:
                led.weights -= weights
                weights_held = False
                trace.append(["weights", "released"])
            else:
                pages = rng.randint(0, 8)
                weights_held = pages <= free_pages()
                if weights_held:
                    weights = pages
                    led.weights += pages
                trace.append(["weights", weights_held])
        elif not live or u < 0.55:
            n = rng.randint(1, max_n)
            pg = (C.c_uint32 * n)()
            sl = (C.c_uint32 * n)()
            hits, direct = C.c_uint64(), C.c_uint64()
            short = lib.po_alloc(pool, C.byref(led), n, pg, sl, C.byref(hits), C.byref(direct))
            if short:
                ev("alloc_fail", short)
                trace.append(["alloc", n, short, 0, 0, 0])
            else:
                if hits.value:
                    ev("buffer_hit", hits.value)
                if direct.value:
                    ev("map", direct.value)
                hs = list(zip(pg, sl))
                stream.extend(hs)
                live.append(hs)
                trace.append(["alloc", n, 0, direct.value, hits.value, n])
        else:
            i = rng.randrange(len(live))
            group = live[i]
            if rng.random() < 0.25 and len(group) > 1:
                k = rng.randint(1, len(group) - 1)
                part, live[i] = group[:k], group[k:]
            else:
                part = live.pop(i)
            pg = (C.c_uint32 * len(part))(*[p for p, _ in part])
            sl = (C.c_uint32 * len(part))(*[s for _, s in part])
            # one unmap event per page reaching zero, in handle order
            before = {p: lib.po_page_occupied(pool, p) for p, _ in part}
            left = dict(before)
            order = []
            for p, _ in part:
                left[p] -= 1
                if left[p] == 0:
                    order.append(p)
            assert lib.po_free(pool, C.byref(led), pool_id, pg, sl, len(part)) == len(order)
            for _ in order:
                ev("unmap", 1)
            trace.append(["free", len(part)])
        trace[-1].append(lib.po_mapped(pool))
        trace[-1].append(free_pages())
    # the misuse epilogue of allocator_fuzz: free stream[0] (if live), then
    # its double free and a foreign handle must both be rejected
    if stream:
        p, s = stream[0]
        pg, sl = (C.c_uint32 * 1)(p), (C.c_uint32 * 1)(s)
        if any((p, s) in g for g in live):
            unmapped = lib.po_free(pool, C.byref(led), pool_id, pg, sl, 1)
            for _ in range(unmapped):
                ev("unmap", 1)
        assert lib.po_free(pool, C.byref(led), pool_id, pg, sl, 1) == -1
    assert lib.po_free(pool, C.byref(led), pool_id + 99, (C.c_uint32 * 1)(0), (C.c_uint32 * 1)(0), 1) == -1
    lib.po_pool_destroy(pool)
    return dict(handles=len(stream), handle_digest=S.digest([list(h) for h in stream]),
                trace_digest=S.digest(trace), event_digest=S.digest(events), events=len(events))


@pytest.mark.parametrize("i", range(len(S.ALLOC_CASES)))
def test_restated_allocator_matches_reference_golden(golden, i):
    got = restate_allocator_fuzz(**S.ALLOC_CASES[i])
    ref = golden["allocator"][i]
    assert got["handles"] == ref["handles"]
    assert got["handle_digest"] == ref["handle_digest"]
    assert got["trace_digest"] == ref["trace_digest"]
    assert got["event_digest"] == ref["event_digest"]


def _bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns, round to nearest even."""
    b = x.astype(np.float32).view(np.uint32)
    b = b + 0x7FFF + ((b >> 16) & 1)
    return (b >> 16).astype(np.uint16)


def _f(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("ctx,n_q,n_kv,d", [(1, 4, 1, 64), (37, 32, 8, 128), (300, 14, 2, 64), (129, 28, 4, 128)])
def test_restated_attention_matches_numpy_fp64(ctx, n_q, n_kv, d):
    rng = np.random.default_rng(ctx)
    q = _bf16(rng.standard_normal((n_q, d)).astype(np.float32))
    k = _bf16(rng.standard_normal((ctx, n_kv, d)).astype(np.float32))
    v = _bf16(rng.standard_normal((ctx, n_kv, d)).astype(np.float32))
    scale = 1.0 / math.sqrt(d)
    got = oracle.dense_attention(q, k, v, scale)
    g = n_q // n_kv
    qf, kf, vf = _f(q), _f(k), _f(v)
    ref = np.zeros((n_q, d))
    for h in range(n_q):
        s = kf[:, h // g, :] @ qf[h] * scale
        p = np.exp(s - s.max())
        ref[h] = (p / p.sum()) @ vf[:, h // g, :]
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_synthetic_content_is_layout_free_and_bounded():
    vals = {oracle.synth_bf16(1, 5, p, 3, 0, 2, 7) for p in range(64)}
    assert len(vals) > 40
    for kind in range(3):
        x = _f(np.array([oracle.synth_bf16(9, 1, 0, 0, kind, 0, e) for e in range(512)], dtype=np.uint16))
        assert np.all(x >= -1.0) and np.all(x <= 1.0)  # bf16 rounding can reach 1.0
    # q scaling is exact for powers of two
    a = _f(np.array([oracle.synth_bf16(9, 1, 0, 0, 2, 0, 3, 4.0)], dtype=np.uint16))[0]
    b = _f(np.array([oracle.synth_bf16(9, 1, 0, 0, 2, 0, 3, 1.0)], dtype=np.uint16))[0]
    assert a == 4.0 * b


def test_synthetic_attention_matches_dense_path():
    seed, layer, n_q, n_kv, d = 77, 2, 8, 2, 64
    reqs, ctxs = [3, 9], [5, 40]
    out = oracle.synth_attention(seed, layer, reqs, ctxs, n_q, n_kv, d, 2.0, 0.125)
    for b, (r, L) in enumerate(zip(reqs, ctxs)):
        q = np.array([[oracle.synth_bf16(seed, r, L - 1, layer, 2, h, e, 2.0) for e in range(d)] for h in range(n_q)],
                     dtype=np.uint16)
        k = np.array([[[oracle.synth_bf16(seed, r, t, layer, 0, h, e) for e in range(d)] for h in range(n_kv)]
                      for t in range(L)], dtype=np.uint16)
        v = np.array([[[oracle.synth_bf16(seed, r, t, layer, 1, h, e) for e in range(d)] for h in range(n_kv)]
                      for t in range(L)], dtype=np.uint16)
        np.testing.assert_allclose(out[b], oracle.dense_attention(q, k, v, 0.125), rtol=0, atol=1e-13)
