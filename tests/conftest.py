import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "reference: needs the compiled reference oracle (oracle/_ref)")


@pytest.fixture(scope="session")
def product():
    from paper_2505_04021_b200 import capi

    return capi.product()


@pytest.fixture(scope="session")
def reference():
    import oracle

    if not oracle.have_reference():
        pytest.skip("oracle/_ref/libmsim_ref.so not built (needs /root/reference at build time)")
    return oracle.reference()


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def device(product):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_04021_b200 import msim

    dev = msim.Device(0, lib=product)
    # Device pointers handed to the engine must be ready on its stream (the
    # engine's kernels do not wait for other streams): run the tests' torch
    # work (K/V / q producers, output reads) on that same stream.
    prev = torch.cuda.current_stream()
    torch.cuda.set_stream(torch.cuda.ExternalStream(dev.stream()))
    yield dev
    torch.cuda.set_stream(prev)
    dev.close()
