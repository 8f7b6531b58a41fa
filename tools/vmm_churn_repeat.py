"""C2 page churn (bench.page_churn_c2) repeated inside ONE process: separates
per-process / per-VA driver warm-up from steady-state map/unmap cost."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    reps = int(os.environ.get("REPS", "3"))
    for i in range(reps):
        r = bench.page_churn_c2()
        print(json.dumps({"rep": i, "amortised_us_per_page_op": r["amortised_us_per_page_op"],
                          "breakdown": r["breakdown_us_per_page_op"], "driver_unmaps": r["driver_unmaps"],
                          "access_calls": r["access_calls"], "wall_s": r["wall_s"]}), flush=True)


if __name__ == "__main__":
    main()
