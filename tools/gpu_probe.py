"""First-contact GPU probe: engine + K1/K2/K3 correctness against the
oracles, and rough timings. Run on a B200 via gpurun."""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2505_04021_b200 import msim  # noqa: E402

SEED = 20251017


def check_engine(n_req=12, prompt=300, output=40, layers=4, n_q=32, n_kv=8, d=128, chunk=128, cap_pages=512):
    dev = msim.Device(0)
    gpu = msim.GpuState(0, cap_pages)
    gpu.ledger.attach_device(dev)
    gpu.ledger.refill_buffer(8)
    spec = msim.ModelSpec.llm("m8b", layers, n_q, n_kv, d, weight_bytes=0, chunk_size=chunk)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device()
    for i in range(n_req):
        eng.push(100 + i, prompt + 7 * i, output + i)
    scale = 1.0 / math.sqrt(d)
    worst = 0.0
    steps = 0
    checked = 0
    while True:
        b, q = eng.counts()
        if b == 0 and q == 0:
            break
        before = {r.id: r.n_slots for r in eng.batch()}
        out = eng.step()
        steps += 1
        eng.append_kv_synthetic(0, layers, SEED)
        n_tok, n_dec = eng.step_info()
        dev_slots = eng.step_slots()
        assert len(dev_slots) == n_tok, (len(dev_slots), n_tok)
        # host view of the slots allocated this step: prefill tokens then decodes
        tp = (2 << 20) // spec.token_kv_bytes
        host_step = []
        after = {r.id: r for r in eng.batch()}
        if out.chunk_tokens:
            pre = [r for r in after.values() if r.id not in before or r.n_slots - before.get(r.id, 0) > 1]
            for r in pre:
                hs = eng.request_kv(r.id)[before.get(r.id, 0):]
                host_step += [h.page * tp + h.slot for h in hs]
        for rid in eng.step_decode_ids():
            if rid in after:
                h = eng.request_kv(rid)[-1]
                host_step.append(h.page * tp + h.slot)
        if not out.completions and host_step != dev_slots:
            print("STEP SLOT MISMATCH step", steps, "chunk", out.chunk_tokens, "host", host_step[:20], "dev",
                  dev_slots[:20], len(host_step), len(dev_slots))
            raise SystemExit(1)
        # host handles of this step's slots, in allocation order
        ids = eng.step_decode_ids()
        if n_dec and steps % 3 == 0:
            qb = torch.empty((n_dec, n_q, d), dtype=torch.bfloat16, device="cuda")
            ob = torch.empty_like(qb)
            ctx = []
            batch = {r.id: r for r in eng.batch()}
            for rid in ids:
                ctx.append(batch[rid].live_slots() if rid in batch else None)
            for layer in range(layers):
                eng.synth_q(layer, SEED, 4.0, qb.data_ptr())
                eng.decode_attention(layer, qb.data_ptr(), ob.data_ptr(), scale)
                eng.synchronize()
                keep = [i for i, c in enumerate(ctx) if c is not None]
                ref = oracle.synth_attention(SEED, layer, [ids[i] for i in keep], [ctx[i] for i in keep], n_q, n_kv,
                                             d, 4.0, scale)
                got = ob.float().cpu().numpy()[keep]
                err = np.abs(got - ref).max()
                worst = max(worst, float(err))
                checked += 1
        # block table row == host handles for every batch request
        for r in eng.batch():
            host = eng.request_kv(r.id)
            tpp = 16 if d == 128 and n_kv == 8 and layers == 32 else None
            row = eng.table_row(r.table_row, len(host))
            tp = (2 << 20) // spec.token_kv_bytes
            exp = [h.page * tp + h.slot for h in host]
            if row != exp:
                bad = [i for i in range(len(exp)) if row[i] != exp[i]]
                print("MISMATCH req", r.id, "prompt", r.prompt_tokens, "done", r.prompt_done, "gen", r.generated,
                      "row", r.table_row, "n", len(exp), "bad idx", bad[:10], "got", [row[i] for i in bad[:10]],
                      "exp", [exp[i] for i in bad[:10]], "step", steps)
                raise SystemExit(1)
    st = dev.stats()
    print(f"engine ok: steps={steps} attention checks={checked} max_abs_err={worst:.3e} dev_stats={st}")
    return worst


def bench_attention(B=64, ctx=2048, layers=32, n_q=32, n_kv=8, d=128, reps=20):
    """C1-shaped steady decode: K3 for all layers; GB/s of K+V reads."""
    dev = msim.Device(0)
    tb = 2 * layers * n_kv * d * 2
    tpp = (2 << 20) // tb
    need_pages = (B * (ctx + reps + 8)) // tpp + 64
    gpu = msim.GpuState(0, need_pages + 16)
    gpu.ledger.attach_device(dev)
    spec = msim.ModelSpec.llm("m8b", layers, n_q, n_kv, d, chunk_size=4096)
    act = gpu.activate(spec)
    gpu.finish_activation(act.engine_index)
    eng = gpu.engine(act.engine_index)
    eng.attach_device(max_step_tokens=ctx + B + 8)
    for i in range(B):
        eng.push(i + 1, ctx - 1, 10000)
    t0 = time.time()
    for i in range(B):
        eng.step()
        eng.append_kv_synthetic(0, layers, SEED)
    eng.synchronize()
    print(f"prefill {B} x {ctx-1} in {time.time()-t0:.2f}s")
    qb = torch.empty((B, n_q, d), dtype=torch.bfloat16, device="cuda")
    ob = torch.empty_like(qb)
    scale = 1.0 / math.sqrt(d)
    res = {}
    for chunk in (0, 256, 512, 1024):
        eng.step()
        eng.append_kv_synthetic(0, layers, SEED)
        n_tok, n_dec = eng.step_info()
        eng.synth_q(0, SEED, 1.0, qb.data_ptr())
        for _ in range(3):
            for layer in range(layers):
                eng.decode_attention(layer, qb.data_ptr(), ob.data_ptr(), scale, chunk)
        eng.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.ExternalStream(dev.stream())
        s.record(stream)
        for _ in range(reps):
            for layer in range(layers):
                eng.decode_attention(layer, qb.data_ptr(), ob.data_ptr(), scale, chunk)
        e.record(stream)
        e.synchronize()
        ms = s.elapsed_time(e) / reps
        ctxs = [r.live_slots() for r in eng.batch()]
        kv_bytes = sum(ctxs) * n_kv * d * 2 * 2 * layers + 2 * B * n_q * d * 2 * layers
        res[chunk] = kv_bytes / ms / 1e6
        print(f"chunk={chunk}: {ms:.3f} ms per {layers}-layer step -> {kv_bytes/ms/1e6:.1f} GB/s")
    # correctness at this size for one layer sample
    eng.synth_q(5, SEED, 4.0, qb.data_ptr())
    eng.decode_attention(5, qb.data_ptr(), ob.data_ptr(), scale)
    eng.synchronize()
    ids = eng.step_decode_ids()
    batch = {r.id: r for r in eng.batch()}
    sel = ids[:8]
    ref = oracle.synth_attention(SEED, 5, sel, [batch[i].live_slots() for i in sel], n_q, n_kv, d, 4.0, scale)
    got = ob.float().cpu().numpy()[:8]
    print("full-size sample max_abs_err", float(np.abs(got - ref).max()))
    return res


def vmm_probe(n=256):
    dev = msim.Device(0)
    led = msim.PhysicalLedger(0, 4096)
    led.attach_device(dev)
    pool = msim.alloc_kvcache(led, "p", 131072, 4096)
    t0 = time.perf_counter()
    led.refill_buffer(n)
    t1 = time.perf_counter()
    r = msim.alloc_kv(pool, led, 16 * n)
    t2 = time.perf_counter()
    msim.free_kv(pool, led, r.handles)
    t3 = time.perf_counter()
    r = msim.alloc_kv(pool, led, 16 * n)  # revive pending pages in place
    t4 = time.perf_counter()
    msim.free_kv(pool, led, r.handles)
    dev.reclaim(True)
    t5 = time.perf_counter()
    r = msim.alloc_kv(pool, led, 16 * 64)  # from the recycle cache (64 handles)
    t6 = time.perf_counter()
    print(f"create(buffer) {(t1-t0)/n*1e6:.1f} us/page; map from buffer {(t2-t1)/n*1e6:.1f}; "
          f"free(pending) {(t3-t2)/n*1e6:.1f}; revive {(t4-t3)/n*1e6:.1f}; unmap {(t5-t4)/n*1e6:.1f}; "
          f"map from cache {(t6-t5)/64*1e6:.1f} us/page")
    msim.free_kv(pool, led, r.handles)
    dev.reclaim(True)
    # does cuMemUnmap block behind a kernel running on another stream?
    x = torch.empty(1 << 28, device="cuda")
    r = msim.alloc_kv(pool, led, 16 * 32)
    msim.free_kv(pool, led, r.handles)
    dev.fence()
    dev.synchronize()
    torch.cuda.synchronize()
    for _ in range(40):
        x.mul_(1.0001)
    t0 = time.perf_counter()
    dev.reclaim(False)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"unmap 32 pages while another stream is busy: {(t1-t0)*1e3:.2f} ms (then {(t2-t1)*1e3:.2f} ms to drain); "
          f"stats {dev.stats()}")
    dev.reset_stats()
    t0 = time.perf_counter()
    r = msim.alloc_kv(pool, led, 16 * n)
    t1 = time.perf_counter()
    msim.free_kv(pool, led, r.handles)
    t2 = time.perf_counter()
    dev.reclaim(True)
    t3 = time.perf_counter()
    print(f"map {n} pages: {(t1-t0)/n*1e6:.1f} us/page; free: {(t2-t1)/n*1e6:.1f} us/page; "
          f"reclaim(unmap): {(t3-t2)/n*1e6:.1f} us/page; stats {dev.stats()}")
    # does cuMemUnmap block on a running kernel?
    x = torch.empty(1 << 28, device="cuda")
    r = msim.alloc_kv(pool, led, 16 * 64)
    msim.free_kv(pool, led, r.handles)
    torch.cuda.synchronize()
    for _ in range(20):
        x.mul_(1.0001)  # ~ms of work queued on torch's stream
    t0 = time.perf_counter()
    dev.reclaim(True)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"reclaim(wait) with busy GPU: {(t1-t0)*1e3:.2f} ms; remaining sync {(t2-t1)*1e3:.2f} ms")
    dev.close()


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0))
    vmm_probe()
    bench_attention()
    check_engine(layers=24, n_q=14, n_kv=2, d=64, prompt=200, output=30, chunk=64, n_req=6)
    check_engine(layers=36, n_q=16, n_kv=2, d=128, prompt=100, output=30, chunk=64, n_req=6)
    bench_attention(B=16, ctx=32768, reps=3)
