"""Deterministic trace driver: arrivals -> engines -> iterations on one GPU.

The reference defines the pieces (engine::step, the schedulers) but no loop
that composes them over a trace (its simcore module is spec-only,
SPEC.md:514-580; SURVEY §7 hard part 6). This is the single composition
order used everywhere in this repo — parity scenarios (tests/scenarios.py),
the page-churn measurement in bench.py — so both backends see identical
request streams:

  * arrivals whose time has come are pushed (in trace order) to their
    model's engine local queue;
  * engines are visited in registration order; each one with runnable work
    takes one step at the current clock, which then advances by the step's
    modelled duration (iterations on one GPU are serialized, SPEC.md
    enginemodel "Open Questions");
  * when no engine can run, the clock jumps to the next arrival.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

from . import msim


class TraceDriver:
    def __init__(self, engines: dict, trace: Sequence[msim.TraceEvent], params: Optional[msim.EngineParams] = None,
                 on_step: Optional[Callable] = None):
        self.engines = engines          # model_id -> msim.Engine (iteration order = dict order)
        self.trace = list(trace)
        self.params = params or msim.EngineParams()
        self.on_step = on_step          # called as on_step(model_id, engine, outcome) after each step
        self.now = 0
        self.next = 0
        self.request_id = 0
        self.outcomes = []
        # per request id: [model, arrival_us, output_tokens, first_token_us, completion_us]
        self.requests = {}

    def admit_arrivals(self) -> None:
        while self.next < len(self.trace) and int(self.trace[self.next].arrival_s * 1e6) <= self.now:
            ev = self.trace[self.next]
            self.request_id += 1
            self.engines[ev.model_id].push(self.request_id, ev.prompt_tokens, ev.output_tokens)
            self.requests[self.request_id] = [ev.model_id, int(ev.arrival_s * 1e6), ev.output_tokens, None, None]
            self.next += 1

    def _record(self, o) -> None:
        # Tokens of a step become visible when the step ends (self.now).
        for rid in o.first_tokens:
            self.requests[rid][3] = self.now
        for rid in o.completions:
            self.requests[rid][4] = self.now
        for rid in o.preemptions:  # restarts from scratch: its first token comes again
            self.requests[rid][3] = None

    def slo_attainment(self, ttft_slo_s: dict, tpot_slo_s: dict, scale: float = 1.0) -> dict:
        """SPEC simcore metrics: TTFT = first token -
        arrival; TPOT = (completion - first token) / (output_tokens - 1).
        Returns per model {'ttft': fraction on time, 'tpot': ..., 'n': done}
        over completed requests, SLOs scaled by `scale`."""
        out = {}
        for rid, (mid, arr, n_out, first, done) in self.requests.items():
            if done is None or first is None:
                continue
            m = out.setdefault(mid, {"n": 0, "ttft_ok": 0, "tpot_ok": 0})
            m["n"] += 1
            if (first - arr) / 1e6 <= ttft_slo_s[mid] * scale:
                m["ttft_ok"] += 1
            tpot = (done - first) / 1e6 / (n_out - 1) if n_out > 1 else 0.0
            if tpot <= tpot_slo_s[mid] * scale:
                m["tpot_ok"] += 1
        return {mid: {"n": v["n"], "ttft": v["ttft_ok"] / v["n"], "tpot": v["tpot_ok"] / v["n"]}
                for mid, v in out.items()}

    def run(self, max_rounds: int) -> list:
        for _ in range(max_rounds):
            self.admit_arrivals()
            ran = False
            for mid, e in self.engines.items():
                if not e.has_runnable_work():
                    continue
                o = e.step(self.params, self.now)
                self.now += o.duration_us
                ran = True
                self.outcomes.append((mid, o))
                self._record(o)
                if self.on_step:
                    self.on_step(mid, e, o)
            if not ran:
                if self.next >= len(self.trace):
                    break
                self.now = max(self.now, int(self.trace[self.next].arrival_s * 1e6))
        return self.outcomes
