"""K3 timelines inside bench.py's C1 step loop (2 models, K1 + K2 + 32 K3
per model step): PRISM_K3_TRACE_LAUNCH picks which launch is stamped; this
runs the bench workload for a few steps and prints the per-CTA summary of the
selected launch (first of a model group = unchained, or a mid-group one)."""
import ctypes as C
import math
import os
import statistics as st
import sys

os.environ["PRISM_K3_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.set_device(0)
mids = bench.placement_for(1, 0)
dev, gpu, models = bench.setup_gpu(0, mids, 64)
lib = bench.msim.capi.product() if hasattr(bench, "msim") else None
from paper_2505_04021_b200 import msim  # noqa: E402

lib = msim.capi.product()
q = [torch.randn((bench.L, bench.B_PER_MODEL, bench.NQ, bench.D), device="cuda").to(torch.bfloat16) for _ in models]
o = [torch.empty_like(x) for x in q]
torch.cuda.synchronize()
bench.run_steps(models, int(os.environ.get("STEPS", 6)), q, o, 1 / math.sqrt(bench.D))
dev.synchronize()
buf = (C.c_uint64 * (4096 * 8))()
got = C.c_int32()
lib.call("prism_debug_k3_trace", buf, 4096 * 8, C.byref(got))
rows = [buf[i * 8:(i + 1) * 8] for i in range(4096)]
rows = [r for r in rows if r[0] and r[5] >= r[0]]
t0 = min(r[0] for r in rows)
qf = lambda v: f"min {min(v):7.2f} med {st.median(v):7.2f} max {max(v):7.2f}"  # noqa: E731
print("launch", os.environ.get("PRISM_K3_TRACE_LAUNCH"), len(rows), "CTAs")
print("CTA start (us)          ", qf([(r[0] - t0) / 1e3 for r in rows]))
print("after PDL wait (+us)    ", qf([(r[2] - r[0]) / 1e3 for r in rows]))
print("first tile done (+us)   ", qf([(r[3] - r[0]) / 1e3 for r in rows]))
print("per tile after first(us)", qf([(r[4] - r[3]) / 1e3 / max(r[6] - 1, 1) for r in rows]))
print("last tile -> done (us)  ", qf([(r[5] - r[4]) / 1e3 for r in rows]))
print("CTA done (us)           ", qf([(r[5] - t0) / 1e3 for r in rows]))
