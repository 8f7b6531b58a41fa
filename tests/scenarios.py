"""Deterministic parity scenarios, driven through the C-ABI of any library
that exports it (the product, or the compiled reference oracle).

Each function returns a JSON-able dict; tools/make_golden.py records the
reference's results in tests/golden/reference_golden.json and the tests
assert the product returns the identical dict (bit-exact: integers exactly,
doubles by repr). Randomness comes from Python's `random.Random(seed)`
(Mersenne Twister, stable across platforms) or from the library's own
seeded generators (synth_trace).
"""
from __future__ import annotations

import hashlib
import json
import random

from paper_2505_04021_b200 import capi, msim
from paper_2505_04021_b200.driver import TraceDriver

PAGE = 2 << 20


def digest(values) -> str:
    return hashlib.sha256(json.dumps(values, separators=(",", ":")).encode()).hexdigest()


# ---------------------------------------------------------------- allocator

ALLOC_CASES = [
    dict(seed=2024, placement=0, capacity=4096, vpages=4096, token_bytes=16 << 10, ops=3000, max_n=300),
    dict(seed=2024, placement=1, capacity=4096, vpages=4096, token_bytes=16 << 10, ops=3000, max_n=300),
    dict(seed=7, placement=0, capacity=40, vpages=64, token_bytes=131072, ops=3000, max_n=64),
    dict(seed=11, placement=0, capacity=300, vpages=300, token_bytes=12288, ops=2000, max_n=600),
    dict(seed=13, placement=1, capacity=120, vpages=90, token_bytes=114688, ops=2000, max_n=40),
    dict(seed=17, placement=0, capacity=2000, vpages=1500, token_bytes=1 << 20, ops=2000, max_n=9),
]


def allocator_fuzz(lib, seed, placement, capacity, vpages, token_bytes, ops, max_n):
    """Random alloc / whole-group free / partial free / buffer refill /
    weight reservation churn on one pool, with the event log recording."""
    rng = random.Random(seed)
    led = msim.PhysicalLedger(0, capacity, lib=lib)
    led.set_recording(True)
    pool = msim.alloc_kvcache(led, "m", token_bytes, vpages, placement)
    live = []  # list of handle lists
    trace = []
    stream = []
    now = 0
    weights_held = False
    for _ in range(ops):
        now += rng.randint(1, 50)
        led.set_time(now)
        u = rng.random()
        if u < 0.05:
            trace.append(["refill", led.refill_buffer(rng.randint(0, 12))])
        elif u < 0.07:
            if weights_held:
                led.release_weight_pages("w")
                weights_held = False
                trace.append(["weights", "released"])
            else:
                weights_held = led.reserve_weight_pages("w", rng.randint(0, 8))
                trace.append(["weights", weights_held])
        elif not live or u < 0.55:
            n = rng.randint(1, max_n)
            buf, res = msim.alloc_kv_raw(pool, led, n)
            hs = [(s.page, s.slot) for s in buf[:res.n_handles]]
            stream.extend(hs)
            trace.append(["alloc", n, res.shortfall_pages, res.pages_mapped, res.buffer_hits, len(hs)])
            if hs:
                live.append(hs)
        else:
            i = rng.randrange(len(live))
            group = live[i]
            if rng.random() < 0.25 and len(group) > 1:
                k = rng.randint(1, len(group) - 1)
                part, live[i] = group[:k], group[k:]
            else:
                part = live.pop(i)
            pid = pool.id()
            msim.free_kv(pool, led, [msim.TokenSlotHandle(pid, p, s) for p, s in part])
            trace.append(["free", len(part)])
        trace[-1].append(pool.mapped_pages())
        trace[-1].append(led.free_pages())
    # misuse: double free of an already freed handle is rejected
    errors = []
    if stream:
        p, s = stream[0]
        still_live = any((p, s) in g for g in live)
        try:
            msim.free_kv(pool, led, [msim.TokenSlotHandle(pool.id(), p, s)])
            if still_live:
                for g in live:
                    if (p, s) in g:
                        g.remove((p, s))
            msim.free_kv(pool, led, [msim.TokenSlotHandle(pool.id(), p, s)])
        except capi.UsageError as e:
            errors.append(e.message)
    try:
        msim.free_kv(pool, led, [msim.TokenSlotHandle(pool.id() + 99, 0, 0)])
    except capi.UsageError as e:
        errors.append(e.message)
    led.check_invariants()
    events = [[e.time_us, e.model_id, e.kind, e.pages] for e in led.events()]
    occ = [pool.page_occupied(p) for p in range(min(vpages, 256))]
    msim.free_kvcache(led, pool)
    return dict(case=dict(seed=seed, placement=placement, capacity=capacity, vpages=vpages,
                          token_bytes=token_bytes, ops=ops, max_n=max_n),
                handles=len(stream), handle_digest=digest(stream), handle_prefix=stream[:64],
                trace_digest=digest(trace), trace_prefix=trace[:40], events=len(events),
                event_digest=digest(events), event_prefix=events[:40], errors=errors, occupancy=occ,
                final_free=led.free_pages(), final_mapped=led.mapped_pages())


def allocator_known_answers(lib):
    """The reference's pagealloc known answers (tests/test_pagealloc.cpp),
    recorded as values (including the 48 KiB tokens_per_page the reference
    computes as 42 although its test expects 43)."""
    out = {}
    led = msim.PhysicalLedger(0, 64, lib=lib)
    pool = msim.alloc_kvcache(led, "m", 16 << 10, 1000)
    out["tpp_16k"] = pool.tokens_per_page()
    out["tpp_48k"] = msim.alloc_kvcache(led, "n", 48 << 10, 10).tokens_per_page()
    try:
        msim.alloc_kvcache(led, "m", 16 << 10, 10)
        out["duplicate"] = "accepted"
    except capi.UsageError as e:
        out["duplicate"] = e.message
    try:
        msim.alloc_kvcache(led, "x", PAGE + 1, 10)
        out["oversize"] = "accepted"
    except capi.UsageError as e:
        out["oversize"] = e.message
    led = msim.PhysicalLedger(0, 64, lib=lib)
    pool = msim.alloc_kvcache(led, "m", 16 << 10, 10)
    r = msim.alloc_kv(pool, led, 130)
    out["alloc130_pages"] = pool.mapped_pages()
    led = msim.PhysicalLedger(0, 64, lib=lib)
    pool = msim.alloc_kvcache(led, "m", 16 << 10, 10)
    a = msim.alloc_kv(pool, led, 128)
    b = msim.alloc_kv(pool, led, 128)
    msim.free_kv(pool, led, a.handles[100:])
    msim.free_kv(pool, led, b.handles[50:])
    c = msim.alloc_kv(pool, led, 20)
    out["most_occupied_pages"] = sorted({h.page for h in c.handles})
    led = msim.PhysicalLedger(0, 4, lib=lib)
    pool = msim.alloc_kvcache(led, "m", 16 << 10, 100)
    r = msim.alloc_kv(pool, led, 6 * 128)
    out["shortfall"] = [r.shortfall_pages, len(r.handles), led.mapped_pages()]
    led = msim.PhysicalLedger(0, 10, lib=lib)
    out["refill"] = [led.refill_buffer(8), led.buffer_pages(), led.refill_buffer(8)]
    pool = msim.alloc_kvcache(led, "m", 16 << 10, 100)
    led.set_recording(True)
    r = msim.alloc_kv(pool, led, 3 * 128)
    r2 = msim.alloc_kv(pool, led, 7 * 128)
    out["buffer_hits"] = [r.buffer_hits, r.pages_mapped, r2.buffer_hits, r2.pages_mapped, led.refill_buffer(8)]
    out["buffer_events"] = [[e.kind, e.pages] for e in led.events()]
    return out


# ---------------------------------------------------------------- engine

from paper_2505_04021_b200.configs import SHAPES, shape_spec  # noqa: E402,F401 (shared with bench.py)


ENGINE_CASES = [
    # C1-like: two llama-8B-shaped pools time-sharing one GPU ledger.
    dict(name="c1", seed=42, capacity=2300, models=[("llama3.1-8b", "a"), ("llama3.1-8b", "b")],
         rate=6.0, horizon=20.0, prompt=(512, 0.3), output=(96, 0.4), chunk=256, steps=700, weight_scale=0.0),
    # C1 under pressure: preemption and prefill pauses.
    dict(name="c1-pressure", seed=5, capacity=230, models=[("llama3.1-8b", "a"), ("llama3.1-8b", "b")],
         rate=8.0, horizon=15.0, prompt=(300, 0.5), output=(80, 0.5), chunk=128, steps=900, weight_scale=0.0),
    # C2-like: the 8 shapes space-sharing one ledger, bursty on/off phases.
    dict(name="c2", seed=42, capacity=9000, models=[(s, s) for s in SHAPES], rate=3.0, horizon=20.0,
         prompt=(256, 0.6), output=(64, 0.6), chunk=128, steps=900, weight_scale=0.05, bursty=True),
    # C3-like: long contexts grown by 512-token chunks.
    dict(name="c3", seed=9, capacity=3000, models=[("llama3.1-8b", "long")], rate=0.8, horizon=10.0,
         prompt=(4096, 0.2), output=(32, 0.3), chunk=512, steps=300, weight_scale=0.0),
]


def engine_trace(lib, name, seed, capacity, models, rate, horizon, prompt, output, chunk, steps, weight_scale,
                 bursty=False):
    """Trace-driven run of engines sharing one GPU ledger: arrivals pushed to
    their engine's local queue, engines stepped round-robin on one serialized
    clock (the driver the reference lacks; SURVEY §7 hard part 6)."""
    gpu = msim.GpuState(0, capacity, lib=lib)
    gpu.ledger.set_recording(True)
    engines = {}
    for shape, mid in models:
        spec = shape_spec(shape, mid, chunk=chunk, weight_scale=weight_scale)
        act = gpu.activate(spec)
        assert act is not None, f"weights of {mid} do not fit"
        gpu.finish_activation(act.engine_index)
        engines[mid] = gpu.engine(act.engine_index)
    profiles = []
    for k, (shape, mid) in enumerate(models):
        if bursty:
            segs = [(t, t + 5.0, rate if (int(t // 5) + k) % 2 == 0 else 0.0) for t in range(0, int(horizon), 5)]
        else:
            segs = [(0.0, horizon, rate)]
        profiles.append(msim.ModelProfile(mid, segs, prompt[0], prompt[1], output[0], output[1]))
    trace = msim.synth_trace(profiles, seed, lib=lib)
    drv = TraceDriver(engines, trace)
    drv.run(steps)
    now = drv.now
    outcomes = [[mid, o.duration_us, o.chunk_tokens, o.decode_tokens, o.first_tokens, o.completions, o.preemptions,
                 o.pages_mapped_direct, o.prefill_paused] for mid, o in drv.outcomes]
    gpu.ledger.check_invariants()
    tables = {}
    for mid, e in engines.items():
        for r in e.batch():
            buf, n = e.request_kv_raw(r.id)
            tables[str(r.id)] = digest([(s.page, s.slot) for s in buf[:n]])
    events = [[ev.time_us, ev.model_id, ev.kind, ev.pages] for ev in gpu.ledger.events()]
    summary = dict(steps=len(outcomes), preemptions=sum(len(o[6]) for o in outcomes),
                   paused=sum(1 for o in outcomes if o[8]), completions=sum(len(o[5]) for o in outcomes),
                   direct_maps=sum(o[7] for o in outcomes))
    return dict(name=name, requests=len(trace), summary=summary, outcome_digest=digest(outcomes),
                outcome_prefix=outcomes[:25], event_digest=digest(events), events=len(events),
                table_digest=digest(sorted(tables.items())), final_mapped=gpu.ledger.mapped_pages(),
                final_free=gpu.ledger.free_pages(), end_us=now)


# C1 exactly as bench.py times it, on the B200-sized ledger: two
# llama3.1-8b pools (weights accounted, 7,659 pages each) on 85,830 pages,
# so every pool's V = 85,830 (reference src/engine.cpp:326-328); 64 prompts
# of 2,047 tokens per model from the seeded C1 trace, prefilled in 4,096-token
# chunks (model A, then model B), then `decode_steps` decode steps
# alternating A / B. The reference runs it through its own engine::step.
C1_FULL = dict(capacity=85_830, decode_steps=60, batch=64, ctx=2048, chunk=4096, weight_bytes=16_060_000_000)


def c1_full_ledger(lib, capacity, decode_steps, batch, ctx, chunk, weight_bytes, device=None, on_step=None):
    gpu = msim.GpuState(0, capacity, lib=lib)
    if device is not None:
        gpu.ledger.attach_device(device)
    gpu.ledger.set_recording(True)
    engines = []
    for mid in ("llama3-8b#0", "llama3-8b#1"):
        prof = msim.ModelProfile(mid, [(0.0, 60.0, 30.0)], prompt_median=ctx - 1, prompt_sigma=0.0,
                                 output_median=256, output_sigma=0.4)
        trace = [e for e in msim.synth_trace([prof], 42, lib=lib) if e.model_id == mid][:batch]
        spec = msim.ModelSpec.llm(mid, 32, 32, 8, 128, weight_bytes=weight_bytes, chunk_size=chunk)
        act = gpu.activate(spec)
        gpu.finish_activation(act.engine_index)
        e = gpu.engine(act.engine_index)
        if device is not None:
            e.attach_device(max_decode_batch=batch, max_step_tokens=chunk + batch + 8)
        for i, ev in enumerate(trace):
            e.push(i + 1, ev.prompt_tokens, 1_000_000)
        engines.append((mid, e))
    outcomes, step_handles = [], []

    def one(mid, e):
        before = {r.id: r.n_slots for r in e.batch()}
        o = e.step()
        outcomes.append([mid, o.duration_us, o.chunk_tokens, o.decode_tokens, o.first_tokens, o.completions,
                         o.preemptions, o.pages_mapped_direct, o.prefill_paused])
        # the step's new handles (per request, in admit order): the handle stream
        new = []
        for r in e.batch():
            k = r.n_slots - before.get(r.id, 0)
            if k:
                buf, n = e.request_kv_raw(r.id)
                new.append([r.id, [(s.page, s.slot) for s in buf[n - k:n]]])
        step_handles.append(digest(new))
        if on_step is not None:
            on_step(mid, e, new)

    for mid, e in engines:
        while e.counts()[1] or any(r.prompt_done < r.prompt_tokens for r in e.batch()):
            one(mid, e)
    for _ in range(decode_steps):
        for mid, e in engines:
            one(mid, e)
    gpu.ledger.check_invariants()
    tables = {}
    for mid, e in engines:
        for r in e.batch():
            buf, n = e.request_kv_raw(r.id)
            tables[f"{mid}/{r.id}"] = digest([(s.page, s.slot) for s in buf[:n]])
    events = [[ev.time_us, ev.model_id, ev.kind, ev.pages] for ev in gpu.ledger.events()]
    return dict(steps=len(outcomes), outcome_digest=digest(outcomes), handle_stream_digest=digest(step_handles),
                event_digest=digest(events), events=len(events), table_digest=digest(sorted(tables.items())),
                mapped=gpu.ledger.mapped_pages(), free=gpu.ledger.free_pages(),
                engines=engines, gpu=gpu)


# ---------------------------------------------------------------- placement

PLACEMENT_CASES = [
    dict(seed=99, n_gpus=8, n_models=24, tau=0.05, placed_frac=0.0),   # C4 shape, cold start
    dict(seed=100, n_gpus=8, n_models=24, tau=0.05, placed_frac=0.7),  # C4 re-placement with migrations
    dict(seed=101, n_gpus=4, n_models=48, tau=0.0, placed_frac=0.5),   # C5 at 4 GPUs
    dict(seed=102, n_gpus=8, n_models=48, tau=0.2, placed_frac=1.0),   # C5 at 8 GPUs
    dict(seed=103, n_gpus=3, n_models=7, tau=0.0, placed_frac=0.0, tp=True),
]


def placement_case(lib, seed, n_gpus, n_models, tau, placed_frac, tp=False):
    rng = random.Random(seed)
    names = list(SHAPES)
    models = []
    for i in range(n_models):
        shape = names[i % len(names)]
        spec = shape_spec(shape, f"{shape}#{i}", ttft=rng.choice([0.04, 0.07, 0.1, 0.13, 1.0]))
        if tp and i % 3 == 0:
            spec.tp_degree = 2
        rate = rng.paretovariate(1.2) * 0.5  # long tail
        cur = []
        if rng.random() < placed_frac:
            cur = rng.sample(range(n_gpus), spec.tp_degree)
        models.append(msim.ModelDemandPy(spec, rate, cur))
    cap = 180 * 10**9 if not tp else 40 * 10**9
    gpus = [msim.GpuViewPy(g, cap, 0, 0.0, cap // PAGE, cap // PAGE) for g in range(n_gpus)]
    try:
        plan = msim.place_models(models, gpus, tau, lib=lib)
    except capi.PlacementError as e:
        return dict(seed=seed, error=e.message)
    return dict(seed=seed, assignment=plan.assignment, migrations=plan.migrations,
                kvpr_after=[repr(x) for x in plan.kvpr_after], max_kvpr=repr(plan.max_kvpr_after),
                critical=[plan.critical_gpu, repr(plan.critical_shared_before_bytes),
                          repr(plan.critical_last_weight_bytes)])


def eviction_cases(lib):
    rng = random.Random(4242)
    out = []
    for case in range(20):
        gpus = []
        for g in range(3):
            res = {}
            for k in range(rng.randint(0, 6)):
                res[f"m{g}.{k}"] = msim.ResidentModel(rng.choice([2.0, 9.0, 10.0, 30.0, 120.0]),
                                                      rng.choice([0.5, 1.0, 2.0, 10.0]),
                                                      rng.randint(1, 20) * 10**9, rng.randint(100, 9000))
            gpus.append(msim.GpuViewPy(g, 80 * 10**9, sum(r.weight_bytes for r in res.values()), 0.0, 40000,
                                       rng.randint(0, 12000), PAGE, res))
        ev = msim.eviction_tick(gpus, 10.0, 8000, lib=lib)
        spec = shape_spec("llama3.1-8b", "new", ttft=1.0)
        arr = msim.activate_on_arrival(spec, gpus, lib=lib)
        spec.tp_degree = 2
        arr_tp = msim.activate_on_arrival_tp(spec, gpus, lib=lib)
        out.append([ev, arr, arr_tp])
    return out


# ---------------------------------------------------------------- admission

ADMISSION_CASES = [dict(seed=s, n=n) for s, n in ((5, 8), (17, 40), (23, 256), (31, 120))]


def admission_case(lib, seed, n):
    rng = random.Random(seed)
    q = []
    for i in range(n):
        arr = round(rng.uniform(0.0, 5.0), 3)
        q.append(msim.QueuedRequest(i + 1, rng.choice("abcd"), arr, rng.randint(16, 4096),
                                    rng.choice([0.04, 0.1, 0.5, 1.0, 2.0]), rng.uniform(0.01, 0.6)))
    admit, deferred = msim.moore_hodgson(q, 1.0, lib=lib)
    budget = {m: rng.randint(0, n) for m in "abcd"}

    def gate(r):
        if budget[r.model_id] <= 0:
            return 1
        budget[r.model_id] -= 1
        return 0

    sent = msim.dispatch(admit, gate, lib=lib)
    merged = msim.requeue_deferred(deferred, [r for r in q if r.id % 3 == 0], lib=lib)
    return dict(seed=seed, admit=[r.id for r in admit], deferred=[r.id for r in deferred], dispatched=sent,
                requeued=[r.id for r in merged])


# ---------------------------------------------------------------- traces

TRACE_CASES = [
    dict(name="c1", seed=42, models=[("a", [(0, 60, 30.0)], 2048, 0.0, 256, 0.4),
                                     ("b", [(0, 60, 30.0)], 2048, 0.0, 256, 0.4)]),
    dict(name="c2", seed=42, models=[(s, [(t, t + 10, 12.0 if (t // 10 + k) % 2 == 0 else 0.0)
                                          for t in range(0, 60, 10)], 1024, 0.6, 256, 0.6)
                                     for k, s in enumerate(SHAPES)]),
    dict(name="c5", seed=42, models=[(f"m{k}", [(t, t + 60, (5.0 if (t // 60) % 2 else 1.0) * (1 + k % 3))
                                               for t in range(0, 300, 60)], 512, 0.5, 128, 0.5)
                                     for k in range(48)]),
]


def trace_case(lib, name, seed, models):
    profiles = [msim.ModelProfile(m, segs, pm, ps, om, os_) for m, segs, pm, ps, om, os_ in models]
    t = msim.synth_trace(profiles, seed, lib=lib)
    rows = [[repr(e.arrival_s), e.model_id, e.prompt_tokens, e.output_tokens] for e in t]
    scaled = msim.scale_trace(t[:200], 3, seed, lib=lib)
    srows = [[repr(e.arrival_s), e.model_id, e.prompt_tokens, e.output_tokens] for e in scaled]
    return dict(name=name, n=len(rows), digest=digest(rows), prefix=rows[:12], scaled_digest=digest(srows))
