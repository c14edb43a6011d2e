"""CPU proof step for the arithmetic dequantize (csrc/codec.cu deq_f32_fast):
scripts/deq_exhaustive.c replays its fp32 operations for every code and every
fp32 mantissa of the scale in a binade and compares with the reference's fp64
value (compression.cpp:34) rounded once to f32 / bf16.  The GPU kernel itself
is checked bit-exactly in tests/test_codec_gpu.py."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc absent")
@pytest.mark.parametrize("expb", [127, 64])
def test_deq_arith_exhaustive_binade(tmp_path, expb):
    exe = tmp_path / "deq_exhaustive"
    subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "scripts", "deq_exhaustive.c"), "-lm"], check=True)
    out = subprocess.run([str(exe), str(expb)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "f32 mismatches 0 bf16 mismatches 0" in out.stdout
