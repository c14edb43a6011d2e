"""GPU: every attention path of the stage executor against the fp64 block oracle at BASELINE
configs[2]'s shape (d 2048, 16 heads, seq 512, microbatch 4).  The default path (one-pass forward
storing the log2-sum-exp, the one-kernel backward recomputing P) is covered by
tests/test_stage_gpu.py::test_one_block_at_baseline_shape; this reruns that test with each
alternative selected (the selection is read once per process, hence a subprocess per path):
  SWARM_ATTN_LSE=0        the forward stores P, the one-kernel backward reads it
  SWARM_ATTN_BWD_FUSED=0  score-gradient kernel + batched dQ / dK / dV GEMMs over the stored P
  SWARM_ATTN_PV=0         P V as a separate GEMM after the fused score kernel (unfused backward)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("env", [{"SWARM_ATTN_LSE": "0"}, {"SWARM_ATTN_BWD_FUSED": "0"}, {"SWARM_ATTN_PV": "0"}])
def test_attention_path_matches_oracle_at_baseline_shape(cuda, env):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_stage_gpu.py::test_one_block_at_baseline_shape[configs2]"],
                       cwd=root, env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (env, r.stdout[-2000:], r.stderr[-2000:])
    assert "1 passed" in r.stdout, r.stdout[-500:]
