"""CPU: the reference-compatible cost model (swarmsim::cost_model, built into the
B200 library) against the unmodified reference compiled in oracle/_ref —
stage_cost / square_cube_ratio must agree to the last bit (same formulas, same
order) — and the B200 calibration helper."""
import ctypes as C
import random

import numpy as np
import pytest


def _ref():
    import oracle as O
    if O.ref is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return O.ref


def test_stage_cost_matches_reference():
    ref = _ref()
    from paper_2301_11913_b200 import _swarmsim_b200 as M
    rng = random.Random(5)
    for _ in range(200):
        h = rng.choice([4, 8, 12, 16, 32])
        d = h * rng.choice([32, 64, 128])
        shape = [d, 4 * d, h, rng.choice([128, 512, 2048]), rng.randint(1, 8), rng.randint(1, 16)]
        act = rng.choice([1.0, 2.0, 0.5])
        dev = [10 ** rng.uniform(12, 15.5), 10 ** rng.uniform(8, 12), 10 ** rng.uniform(8, 12), rng.uniform(0, 1e-3)]
        for overlap in (0, 1):
            out = np.zeros(6)
            assert ref.ref_stage_cost((C.c_int64 * 6)(*shape), act, (C.c_double * 4)(*dev), overlap,
                                      out.ctypes.data_as(C.c_void_p)) == 0
            s = M.LayerShape()
            s.d_model, s.d_ffn, s.n_heads, s.seq_len, s.batch, s.layers_per_stage = shape
            s.activation_bytes_per_element = act
            p = M.DeviceProfile()
            p.effective_flops, p.upload_bps, p.download_bps, p.rtt_seconds = dev
            c = M.stage_cost(s, p, bool(overlap))
            assert (c.compute_seconds, c.comm_seconds, c.total_seconds, c.idle_fraction, c.utilization) == \
                tuple(out[:5])
            assert M.square_cube_ratio(s) == out[5]


def test_calibrated_profile_reproduces_the_measured_visit():
    from paper_2301_11913_b200 import _swarmsim_b200 as M
    s = M.LayerShape()
    s.d_model, s.d_ffn, s.n_heads, s.seq_len, s.batch, s.layers_per_stage = 2048, 8192, 16, 512, 4, 8
    s.activation_bytes_per_element = 1.0  # int8 wire
    p = M.calibrated_profile(s, 6.5e-3, 300e9, 5e-6)
    assert p.effective_flops == pytest.approx(M.flops_per_stage(s, True) / 6.5e-3)
    c = M.stage_cost(s, p, False)
    assert c.compute_seconds == pytest.approx(6.5e-3)
    assert c.comm_seconds == pytest.approx(2 * 2048 * 4 * 512 * 8 / 300e9 + 1e-5)
    with pytest.raises(ValueError):
        M.calibrated_profile(s, 0.0, 1e9)
