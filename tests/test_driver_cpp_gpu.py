"""GPU: the C++ test binary (tests/cpp/driver_test.cpp) runs the tiny SWARM
pipeline through the C-ABI alone — the host driver walks the engine's records,
issues the visits, moves the wire messages and all-reduces, no Python in the
process — and its results match the Python orchestrator (PyEngineExecutor, an
independent host implementation over torch) run on the same token pool, and a
sequential replay of the visits it ran.
"""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "driver_test")


def rel(a, b):
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def read_out(path):
    with open(path, "rb") as f:
        S, T, npool, ntok, done, nlog = np.frombuffer(f.read(48), np.int64)
        tok = np.frombuffer(f.read(4 * npool * ntok), np.int32).reshape(npool, ntok)
        tgt = np.frombuffer(f.read(4 * npool * ntok), np.int32).reshape(npool, ntok)
        loss = float(np.frombuffer(f.read(4), np.float32)[0])
        log = [tuple(int(v) for v in np.frombuffer(f.read(40), np.int64)) for _ in range(nlog)]
        peers = {}
        while hdr := f.read(16):
            pid, n = np.frombuffer(hdr, np.int64)
            g = np.frombuffer(f.read(4 * n), np.float32)
            p = np.frombuffer(f.read(4 * n), np.float32)
            peers[int(pid)] = (g, p)
    return dict(S=int(S), T=int(T), done=int(done), tok=tok, tgt=tgt, loss=loss, log=log, peers=peers)


@pytest.mark.parametrize("S,tpp,lanes,ticks", [(2, 2, 1, 0), (2, 2, 2, 0), (4, 1, 1, 0), (2, 2, 1, 1)])
def test_cpp_binary_matches_python_orchestrator(cuda, tmp_path, S, tpp, lanes, ticks):
    import torch
    from paper_2301_11913_b200.executor import PyEngineExecutor, sequential_reference_grads
    from paper_2301_11913_b200.swarm import PRESETS
    assert os.path.exists(BIN), "tests/cpp/driver_test not built (paper_2301_11913_b200/csrc/Makefile)"
    out = tmp_path / "run.bin"
    N = 9
    r = subprocess.run([BIN, "--stages", str(S), "--tpp", str(tpp), "--microbatches", str(N), "--lanes", str(lanes),
                        "--ticks", str(ticks), "--out", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    c = read_out(out)
    assert c["done"] == N
    # the same model / schedule / pool in the Python orchestrator (driver_test.cpp's settings)
    py = PyEngineExecutor(PRESETS["tiny"], S, trainers_per_peer=tpp, seed=11, lr=1e-3, lanes=lanes,
                          tokens=torch.from_numpy(c["tok"].copy()), targets=torch.from_numpy(c["tgt"].copy()),
                          allreduce_period=10.0 if ticks else 0.0, allreduce_stall=0.1 if ticks else 0.0)
    assert py.run(N) == N
    py.finish()
    py.flush_wgrad()
    torch.cuda.synchronize()
    assert [(t, k, s, int(b), p) for t, k, s, b, p in py.visit_log] == c["log"]
    assert abs(c["loss"] - py.loss_sum.item()) <= 1e-5 * abs(py.loss_sum.item())
    for pid, (g, p) in c["peers"].items():
        st = py.stages[pid]
        tol = 1e-4 if ticks else 1e-5
        assert rel(torch.from_numpy(g.copy()).cuda(), st.grads()) <= tol, pid
        assert rel(torch.from_numpy(p.copy()).cuda(), st.params()) <= (1e-4 if ticks else 1e-7), pid
    if not ticks:  # and both equal a sequential replay of the visits (weights fixed without ticks)
        ref = sequential_reference_grads(py)
        for pid, (g, _) in c["peers"].items():
            assert rel(torch.from_numpy(g.copy()).cuda(), ref[pid]) <= 1e-4, pid
