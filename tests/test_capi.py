"""CPU: the C-ABI library loads, exports every symbol include/swarm_b200.h
declares, and the reference-compatible Python surface imports.  No compute
calls (there is no GPU here); host-only arithmetic (payload accounting) is
checked against the reference's values."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "swarm_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(swarm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_codec_and_gemm():
    names = declared_functions()
    for must in ("swarm_quantize_blockwise", "swarm_dequantize_blockwise", "swarm_maxout_forward",
                 "swarm_layer_norm_forward", "swarm_gemm_bf16"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2301_11913_b200 import _lib
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes signature table covers the whole header
    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_version_and_error_without_gpu():
    from paper_2301_11913_b200 import _lib
    L = _lib.lib()
    assert L.swarm_version() == 1
    assert isinstance(L.swarm_launch_count(), int)


def test_reference_surface_imports():
    import paper_2301_11913_b200 as sw
    for name in ("quantize_blockwise", "dequantize_blockwise", "maxout_k", "layer_norm", "compressed_payload_bits",
                 "QuantizedTensor", "ConfigError", "LayerShape", "preset", "preset_names", "params_per_layer",
                 "activation_payload_bits", "flops_per_stage"):
        assert hasattr(sw, name), name
    assert issubclass(sw.ConfigError, ValueError)


def test_payload_bits_match_reference(golden):
    import paper_2301_11913_b200 as sw
    for name, d, L, b in [("base", 768, 512, 1), ("xxlarge", 4096, 512, 1), ("gpt3", 12288, 512, 1),
                          ("ours", 4096, 512, 1), ("configC_B4", 2048, 512, 4)]:
        s = sw.LayerShape()
        s.d_model, s.d_ffn, s.n_heads, s.seq_len, s.batch = d, 4 * d, 1, L, b
        s.activation_bytes_per_element = 2.0
        exp = golden["payload_bits"][name]
        assert sw.compressed_payload_bits(s, "none") == exp["none"]
        assert sw.compressed_payload_bits(s, "int8") == exp["int8"]
        assert sw.compressed_payload_bits(s, "bottleneck", 0.25) == exp["bottleneck_0.25"]
        assert sw.compressed_payload_bits(s, "maxout", 2.0) == exp["maxout_2"]
        assert sw.compressed_payload_bits(s, "int8") * 2 == sw.activation_payload_bits(s)  # acceptance #8
    with pytest.raises(sw.ConfigError):
        sw.compressed_payload_bits(sw.preset("xxlarge"), "bottleneck", 1.5)
    with pytest.raises(sw.ConfigError):
        sw.compressed_payload_bits(sw.preset("xxlarge"), "zip")


def test_cost_model_convention():
    import paper_2301_11913_b200 as sw
    s = sw.preset("base")
    assert sw.params_per_layer(s) == 4 * 768 * 768 + 2 * 768 * 3072
    assert sw.flops_per_stage(s, True) == 3 * 2 * sw.params_per_layer(s) * 512


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2301_11913_b200 as sw
    with pytest.raises(RuntimeError):
        sw.quantize_blockwise([1.0, 2.0], 2)
    with pytest.raises(sw.ConfigError):  # validation happens before any device work, like the reference
        sw.quantize_blockwise([1.0], 0)
