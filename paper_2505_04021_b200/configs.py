"""BASELINE.json workload shapes shared by bench.py, tools/ and tests/.

SHAPES: the eight model shapes of SURVEY §8d (configs C2/C4/C5);
c5_case: config 5 ("48 models with 5x minute-scale rate swings on
1/2/4/8 GPUs, measuring SLO attainment") as simcore input."""
from __future__ import annotations

from . import msim

SHAPES = {  # (L, n_q, n_kv, d, weight GB)
    "qwen2.5-0.5b": (24, 14, 2, 64, 0.99),
    "llama3.2-1b": (16, 32, 8, 64, 2.47),
    "qwen2.5-1.5b": (28, 12, 2, 128, 3.09),
    "qwen2.5-3b": (36, 16, 2, 128, 6.17),
    "llama3.2-3b": (28, 24, 8, 128, 6.43),
    "qwen2.5-7b": (28, 28, 4, 128, 15.23),
    "mistral-7b": (32, 32, 8, 128, 14.5),
    "llama3.1-8b": (32, 32, 8, 128, 16.06),
}

B200_LEDGER_PAGES = 85_830  # 180 GB usable / 2 MiB


def shape_spec(name, model_id=None, chunk=512, weight_scale=1.0, ttft=1.0) -> msim.ModelSpec:
    L, nq, nkv, d, wgb = SHAPES[name]
    return msim.ModelSpec.llm(model_id or name, L, nq, nkv, d, weight_bytes=int(wgb * 1e9 * weight_scale),
                              chunk_size=chunk, ttft_slo_s=ttft)


def slo_of(name):
    """SPEC simcore ranges (TTFT 0.04-0.13 s, TPOT 5.2-50.9 ms), growing with
    the model's weight size."""
    frac = SHAPES[name][4] / 16.06
    return 0.04 + 0.09 * frac, 0.0052 + 0.0457 * frac


def slo_models(copies, shapes=None):
    out = []
    for name in shapes or SHAPES:
        for c in range(copies):
            ttft, tpot = slo_of(name)
            spec = shape_spec(name, f"{name}#{c}", chunk=512, ttft=ttft)
            spec.tpot_slo_s = tpot
            out.append(spec)
    return out


def c5_case(copies=6, horizon=240.0, base_rate=0.25):
    """Every shape x `copies` (48 models at 6), per-minute segments
    alternating r and 5r (phase-shifted per model). Returns ((spec, demand
    rate) pairs, synth_trace profiles)."""
    profiles, models = [], []
    for i, spec in enumerate(slo_models(copies)):
        segs, t, k = [], 0.0, i % 2
        while t < horizon:
            segs.append((t, min(t + 60.0, horizon), base_rate * (5.0 if k % 2 else 1.0)))
            t += 60.0
            k += 1
        profiles.append(msim.ModelProfile(spec.model_id, segs, 384.0, 0.6, 96.0, 0.6))
        models.append((spec, base_rate * 3.0))
    return models, profiles


def c2_case(rate=3.0, horizon=80.0):
    """Config 2 ("8 models (1B-8B shapes) space-sharing 1 B200 with bursty
    trace forcing frequent page map/unmap across models"): one model per
    shape, 10 s on / 10 s off with alternating phase. Returns ((spec,
    demand rate) pairs, synth_trace profiles)."""
    specs = slo_models(1)
    prof = []
    for i, s in enumerate(specs):
        segs = [(float(t), float(t) + 10.0, rate) for t in range(10 * (i % 2), int(horizon), 20)]
        prof.append(msim.ModelProfile(s.model_id, segs, 256.0, 0.6, 64.0, 0.6))
    return [(s, rate / 2) for s in specs], prof


def c4_case(copies=3, horizon=120.0, total_rate=24.0, zipf=1.2, idle_every=3):
    """Config 4 ("24 models of mixed size placed across 8 x B200 by the
    global scheduler, long-tail synthetic trace with idle periods"): every
    shape x `copies`; model k (popularity rank) gets total_rate * k^-zipf /
    H; every `idle_every`-th model alternates 20 s on / 20 s idle."""
    specs = slo_models(copies)
    w = [(k + 1) ** -zipf for k in range(len(specs))]
    h = sum(w)
    prof, models = [], []
    for k, s in enumerate(specs):
        r = total_rate * w[k] / h
        if idle_every and k % idle_every == idle_every - 1:
            segs = [(float(t), float(t) + 20.0, r) for t in range(0, int(horizon), 40)]
        else:
            segs = [(0.0, horizon, r)]
        prof.append(msim.ModelProfile(s.model_id, segs, 384.0, 0.6, 96.0, 0.6))
        models.append((s, r))
    return models, prof
