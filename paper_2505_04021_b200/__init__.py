"""prism-b200: B200-native elastic KV cache + paged GQA decode attention for
Prism (arXiv 2505.04021).

The product is the shared library ``libprism_b200.so`` (host C++ runtime with
the reference's msim:: API, CUDA VMM pools, sm_100a kernels) behind the C-ABI
in ``include/prism_capi.h``. This package only binds it (``capi``) and mirrors
the reference interface in Python (``msim``). Importing it loads the library
and fails loudly when it has not been built — there is no fallback path.
"""
from . import capi
from .capi import PrismError, UsageError, ParseError, PlacementError, CudaError

__all__ = ["capi", "msim", "PrismError", "UsageError", "ParseError", "PlacementError", "CudaError", "lib"]


def lib() -> "capi.Lib":
    """The product C-ABI library (raises FileNotFoundError when unbuilt)."""
    return capi.product()


from . import msim  # noqa: E402  (after capi)
