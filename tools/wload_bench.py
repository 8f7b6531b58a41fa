"""WeightLoader bandwidth sweep on one GPU: naive (one cudaMemcpyAsync) vs
chunked multi-stream loads from pinned host memory, and the staged path a
fan-in helper uses (host -> staging -> target). GiB= sets the buffer size."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04021_b200 import msim  # noqa: E402


def main():
    n = int(float(os.environ.get("GIB", "4")) * (1 << 30))
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    host[:: 4096] = 7
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = []

    def run(kind, streams, chunk_mib, reps=3):
        wl = msim.WeightLoader(0, streams, chunk_mib << 20)
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            if kind == "naive":
                wl.load_naive(host.data_ptr(), dst.data_ptr(), n)
            elif kind == "chunked":
                wl.load(host.data_ptr(), dst.data_ptr(), n)
            else:
                wl.load_part(host.data_ptr(), dst.data_ptr(), n, 0, 1)
            ms = wl.wait()
            best = ms if best is None else min(best, ms)
        wl.close()
        r = {"kind": kind, "streams": streams, "chunk_mib": chunk_mib, "ms": round(best, 2),
             "gbs": round(n / best / 1e6, 2)}
        out.append(r)
        print(json.dumps(r), flush=True)

    run("naive", 1, 8)
    for streams in (1, 2, 4, 8):
        for chunk in (2, 8, 32):
            run("chunked", streams, chunk)
    for streams in (2, 4):
        run("staged", streams, 8)
    best = max((r for r in out if r["kind"] == "chunked"), key=lambda r: r["gbs"])
    naive = out[0]
    for name, wb in (("llama3.1-8b", 16.06e9), ("14B", 28e9)):
        print(json.dumps({"model": name, "weight_bytes": wb, "naive_s": round(wb / naive["gbs"] / 1e9, 3),
                          "chunked_s": round(wb / best["gbs"] / 1e9, 3)}), flush=True)


if __name__ == "__main__":
    main()
