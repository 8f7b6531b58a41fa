"""Reproduce a scheduler-driven device run (prism_sim_run_device) of one
scenario: python tools/debug_serving.py c5 [copies horizon measured chunk_pages]"""
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402
from paper_2505_04021_b200.configs import B200_LEDGER_PAGES, c2_case, c4_case, c5_case  # noqa: E402

case = sys.argv[1]
copies = int(sys.argv[2]) if len(sys.argv) > 2 else 6
horizon = float(sys.argv[3]) if len(sys.argv) > 3 else 120.0
measured = bool(int(sys.argv[4])) if len(sys.argv) > 4 else True
chunk_pages = int(sys.argv[5]) if len(sys.argv) > 5 else 0
if case == "c5":
    models, prof = c5_case(copies=copies, horizon=horizon)
    n = 1
elif case == "c2":
    models, prof = c2_case(horizon=horizon)
    n = 1
else:
    models, prof = c4_case(copies=copies, horizon=horizon)
    n = 8
trace = msim.synth_trace(prof, 42)
cfg = msim.SimConfig(n_gpus=n, capacity_pages=B200_LEDGER_PAGES)
t = time.time()
try:
    r = msim.simulate(cfg, models, trace, serving=msim.ServingConfig(measured=measured, chunk_pages=chunk_pages,
                                                                     owned=[0]))
    print(case, copies, horizon, measured, chunk_pages, "OK", r.summary, r.serving, round(time.time() - t, 1))
except Exception:
    print(case, copies, horizon, measured, chunk_pages, "FAIL", round(time.time() - t, 1))
    traceback.print_exc()
