"""B200-native SWARM per-stage hot path (arXiv 2301.11913).

Drop-in for the reference's codec API (``swarmsim`` / ``_swarmsim``,
/root/reference/proj/bindings/module.cpp:143-163): same names, arguments and
exceptions, computed by hand-written sm_100a kernels in ``libswarm_b200.so``
(C-ABI: include/swarm_b200.h).  ``ops`` exposes the same kernels on torch
device tensors; ``stage`` is the per-peer stage executor.

Importing never falls back to a CPU path: if the native library or the
extension module is missing the import fails.
"""
from ._swarmsim_b200 import (  # noqa: F401 — the reference-compatible surface
    ConfigError,
    LayerShape,
    NoPeerAvailable,
    ParseError,
    QuantizedTensor,
    activation_payload_bits,
    bottleneck_decompress,
    bottleneck_forward,
    compressed_payload_bits,
    dequantize_blockwise,
    flops_per_stage,
    layer_norm,
    maxout_k,
    params_per_layer,
    preset,
    preset_names,
    quantize_blockwise,
)
from . import _lib  # noqa: F401

_lib.lib()  # load libswarm_b200.so now: fail at import, not at first use

__version__ = "0.1.0"
