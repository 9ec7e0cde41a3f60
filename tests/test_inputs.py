"""Host-side checks of the synthetic input generator (inputs/), which both the
oracle and the product consume.  Device/host identity is checked in
tests/test_gpu_parity.py (-m gpu)."""
import numpy as np

import inputs


def test_traces_are_deterministic_quantised_and_in_range():
    a = inputs.synth_traces_host(5, 8784, seed=5)
    b = inputs.synth_traces_host(5, 8784, seed=5)
    assert a.tobytes() == b.tobytes()
    assert a.shape == (5, 8784) and a.dtype == np.float32
    assert np.all(a >= 0) and np.all(a < 4096)
    assert np.all(a * 64 == np.round(a * 64))          # multiples of 1/64 (exact in fp32/fp64)
    # shards are independent of how the batch is cut (trace0 offset)
    c = inputs.synth_traces_host(2, 8784, seed=5, trace0=3)
    assert c.tobytes() == a[3:5].tobytes()
    assert not np.array_equal(a[0], a[1])


def test_paper_mode_shape():
    """C1/C2 'paper-shaped' region: mean 550, amplitude 150, sigma 10."""
    x = inputs.synth_traces_host(1, 24 * 365, seed=0, mode=inputs.MODE_PAPER)[0]
    assert abs(x.mean() - 550) < 2 and 690 < x.max() < 760 and 340 < x.min() < 410


def test_profiles_satisfy_spec_invariants():
    """limits strictly increasing, avg_power <= 1.05*limit, thr > 0."""
    for shape in inputs.SHAPES:
        for lim in (inputs.LIMITS_7, inputs.LIMITS_9):
            p = inputs.make_profile(shape, lim)
            assert np.all(np.diff(p.limit_w) > 0) and p.K >= 2
            assert np.all(p.avg_power_w > 0) and np.all(p.avg_power_w <= 1.05 * p.limit_w)
            assert np.all(p.throughput_sps > 0) and np.all(np.diff(p.throughput_sps) >= 0)
    b = inputs.make_profile("bert", inputs.LIMITS_9)
    assert b.avg_power_w[-1] == b.avg_power_w[-2] and b.throughput_sps[-1] == b.throughput_sps[-2]


def test_profile_ids_cover_all_shapes():
    pid = inputs.profile_ids_host(3000, seed=4, n_profiles=3)
    assert set(np.unique(pid)) == {0, 1, 2}
