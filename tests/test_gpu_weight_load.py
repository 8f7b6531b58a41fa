"""WeightLoader on the GPU: every load path is bit-exact
(byte-identical to the pinned host source) for ragged sizes, chunk sizes and
stream counts; the staged fan-in tiles the target across helpers, in one
process and across two processes through CUDA IPC (tools/wload_fanin.py)."""
import json
import os
import subprocess
import sys

import pytest
import torch

from paper_2505_04021_b200 import msim

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _host(n, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).pin_memory()


@pytest.mark.parametrize("n,chunk,streams", [(1, 1 << 20, 1), ((8 << 20) + 3, 1 << 20, 4),
                                             ((64 << 20) + 4097, 8 << 20, 8), (40 << 20, 40 << 20, 2)])
def test_load_paths_bit_exact(n, chunk, streams):
    host = _host(n, n)
    wl = msim.WeightLoader(0, streams, chunk)
    for mode in ("load", "naive"):
        dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        (wl.load if mode == "load" else wl.load_naive)(host.data_ptr(), dst.data_ptr(), n)
        ms = wl.wait()
        assert ms >= 0.0
        assert torch.equal(dst.cpu(), host), mode
    wl.close()


@pytest.mark.parametrize("parts", [1, 2, 3, 5])
def test_fanin_parts_tile_target(parts):
    n, chunk = (24 << 20) + 777, 2 << 20
    host = _host(n, 7)
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    helpers = [msim.WeightLoader(0, 2, chunk) for _ in range(parts)]
    for p, wl in enumerate(helpers):
        wl.load_part(host.data_ptr(), dst.data_ptr(), n, p, parts)
    for wl in helpers:
        wl.wait()
    assert torch.equal(dst.cpu(), host)
    # one helper alone writes exactly its planned spans
    if parts > 1:
        dst.zero_()
        torch.cuda.synchronize()
        helpers[1].load_part(host.data_ptr(), dst.data_ptr(), n, 1, parts)
        helpers[1].wait()
        got, ref = dst.cpu(), torch.zeros(n, dtype=torch.uint8)
        for off, ln in msim.fanin_parts(n, chunk, parts)[1]:
            ref[off:off + ln] = host[off:off + ln]
        assert torch.equal(got, ref)
    for wl in helpers:
        wl.close()


def test_bad_arguments_raise():
    from paper_2505_04021_b200 import capi
    with pytest.raises(capi.PrismError):
        msim.WeightLoader(0, 0, 1 << 20)
    wl = msim.WeightLoader(0, 1, 1 << 20)
    with pytest.raises(capi.PrismError):
        wl.load_part(0, 0, 16, 0, 1)
    host = _host(16, 1)
    dst = torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(capi.PrismError):
        wl.load_part(host.data_ptr(), dst.data_ptr(), 16, 2, 2)
    wl.close()


def test_fanin_two_processes_ipc():
    env = dict(os.environ, PRISM_WLOAD_BACKEND="gloo", PRISM_WLOAD_DEVICE="0", PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29541", "tools/wload_fanin.py", "--mib", "96", "--chunk-mib", "4"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    res = json.loads(lines[0])
    assert res["bit_exact"] and res["fanin_ranks"] == 2
