"""paper_2604_00048_b200 -- B200-native hot path of the differentiable
heteroscedastic Whittaker layer (arXiv 2604.00048).

The compute lives in ``libwhit.so`` (hand-written sm_100a CUDA behind the C-ABI
of ``include/libwhit.h``); this package is the thin binding:

* ``_lib``      ctypes marshalling for every C entry point (same names);
* ``autograd``  ``WhittakerFn`` / ``smooth`` -- the torch autograd shim.

Importing fails loudly (ImportError) when the shared library is missing.
"""
from ._lib import (  # noqa: F401
    WHIT_F32,
    WHIT_F64,
    WhitError,
    Workspace,
    whit_backward,
    whit_backward_bands,
    whit_grad_w,
    whit_failures,
    whit_forward_bands,
    whit_forward_mse,
    whit_forward_times,
    whit_forward_times_bands,
    whit_forward_wbits,
    whit_pack_mask,
    whit_posterior_variance,
    whit_ws_bytes_bands,
    whit_forward,
    whit_host_ws_bytes,
    whit_run_host,
    whit_run_host_bands,
    whit_ws_bytes,
    whit_wbits_detected,
    whit_twist_groups,
)
from .autograd import WhittakerFn, smooth  # noqa: F401

__all__ = ["smooth", "WhittakerFn", "Workspace", "whit_forward", "whit_backward", "whit_failures",
           "whit_ws_bytes", "whit_forward_bands", "whit_backward_bands", "whit_grad_w",
           "whit_ws_bytes_bands", "whit_forward_mse", "whit_forward_times", "whit_forward_times_bands", "whit_forward_wbits", "whit_pack_mask", "whit_posterior_variance", "whit_host_ws_bytes", "whit_run_host", "whit_run_host_bands", "whit_wbits_detected", "whit_twist_groups", "WhitError", "WHIT_F32", "WHIT_F64"]
