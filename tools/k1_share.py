"""K1's share of the data path on the C2 shapes: the
scheduler-driven C2 serving run (simcore + K1 / K2 / K4 / K3 per iteration on
the device, measured clock; bench.py serving_gpu) for HORIZON seconds of
trace. Run it under ncu's launch list to get per-kernel time shares:
  ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 20000
      --launch-count 8000 --csv --log-file gpurun_out/k1_share.csv python tools/k1_share.py
  python tools/ncu_summary.py launches gpurun_out/k1_share.csv profiles/r02_k1_share_c2.md"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402
from paper_2505_04021_b200.configs import B200_LEDGER_PAGES, c2_case  # noqa: E402

HORIZON = float(os.environ.get("HORIZON", 40.0))
models, prof = c2_case(horizon=HORIZON)
trace = msim.synth_trace(prof, 20251017)
cfg = msim.SimConfig(n_gpus=1, capacity_pages=B200_LEDGER_PAGES)
r = msim.simulate(cfg, models, trace, serving=msim.ServingConfig(measured=True))
s = r.serving
print({k: s[k] for k in ("iterations", "k2_launches", "k3_launches", "k4_launches", "gpu_us")})
