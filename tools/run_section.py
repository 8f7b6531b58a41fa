"""Run one bench.py section by name on the GPU box and print its JSON
(development helper: `python tools/run_section.py serving_gpu`)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for name in sys.argv[1:]:
    t = time.time()
    r = getattr(bench, name)()
    print(json.dumps({"section": name, "wall_s": round(time.time() - t, 1), "result": r}), flush=True)
