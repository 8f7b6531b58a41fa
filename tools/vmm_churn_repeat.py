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
        keys = ("amortised_us_per_page_op", "caller_wait_us_per_page_op", "background_us_per_page_op",
                "breakdown_us_per_page_op", "urgent_chunks", "steals", "reserve_steals", "driver_unmaps", "driver_creates",
                "access_calls", "driver_call_us", "wall_s")
        print(json.dumps({"rep": i, "urgent_steal_batch": os.environ.get("PRISM_VMM_URGENT_STEAL_BATCH", "8"),
                          "reserve_chunks": os.environ.get("PRISM_VMM_RESERVE_CHUNKS", "8"),
                          **{k: r[k] for k in keys if k in r}}), flush=True)


if __name__ == "__main__":
    main()
