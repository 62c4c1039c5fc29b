"""The checker every parity claim goes through (oracle.tolerance_check, R8) must
reject what the north-star bar rejects: a relative L2 error above 1e-5, and a single element
above its per-element bound 1e-4 * max_c s_c(i) * sum_j (|x_re,j| + |x_im,j|) even when the
relative L2 error is tiny.  (no test showed it ever fails.)"""
import numpy as np

import oracle as orc


def _case(n=64, m=48, B=2, seed=0):
    rng = np.random.default_rng(seed)
    y_ref = (rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))) * 10.0
    scales = rng.uniform(0.01, 0.1, (n, 4)).astype(np.float32)
    x = (rng.standard_normal((B, m)) + 1j * rng.standard_normal((B, m))).astype(np.complex64)
    return y_ref, scales, x


def test_identical_passes():
    y_ref, sc, x = _case()
    ok, rel, worst = orc.tolerance_check(y_ref.astype(np.complex64), y_ref, sc, x)
    assert ok and rel < 1e-7 and worst < 1e-2


def test_relative_l2_just_above_bar_is_rejected():
    y_ref, sc, x = _case()
    ok, rel, _ = orc.tolerance_check(y_ref * (1 + 2e-5), y_ref, sc, x)
    assert not ok and abs(rel - 2e-5) < 1e-9
    ok, rel, _ = orc.tolerance_check(y_ref * (1 + 5e-6), y_ref, sc, x)
    assert ok and abs(rel - 5e-6) < 1e-9


def test_single_element_above_its_bound_is_rejected_despite_tiny_rel_l2():
    n, m = 1000, 4
    y_ref = np.full((1, n), 1e6 + 1e6j)
    sc = np.ones((n, 4), np.float32)
    sc[7] = [0.5, 0.25, 0.125, 0.5]            # max_c s_c(7) = 0.5
    x = np.array([[1 + 1j, -1 + 0j, 0 - 2j, 0.5 + 0.5j]], np.complex64)
    l1 = 2 + 1 + 2 + 1                         # sum_j |re| + |im| = 6
    bound = 1e-4 * 0.5 * l1                    # row 7: 3e-4
    for part in (1, 1j):                       # re and im are bounded separately
        y = y_ref.copy()
        y[0, 7] += 1.01 * bound * part
        ok, rel, worst = orc.tolerance_check(y, y_ref, sc, x)
        assert rel < 1e-9 and not ok and abs(worst - 1.01) < 1e-6
        y = y_ref.copy()
        y[0, 7] += 0.99 * bound * part
        ok, rel, worst = orc.tolerance_check(y, y_ref, sc, x)
        assert ok and abs(worst - 0.99) < 1e-6


def test_per_tensor_scales_and_row_subset():
    y_ref, _, x = _case(n=10, B=1)
    sc = np.array([0.1, 0.2, 0.3, 0.4], np.float32)
    l1 = np.sum(np.abs(x.real) + np.abs(x.imag))
    y = y_ref.copy()
    y[0, 3] += 1.5 * 1e-4 * 0.4 * l1
    ok, _, worst = orc.tolerance_check(y, y_ref, sc, x)
    assert not ok and abs(worst - 1.5) < 1e-4
    # sampled rows: the bound of each sampled row uses that row's scales
    rows = np.array([5, 2])
    sc_rows = np.ones((10, 4), np.float32)
    sc_rows[2] = 1e-3
    yr = y_ref[:, rows].copy()
    yr[0, 1] += 2e-4 * l1 * 1e-3  # 2x row 2's bound, far below row 5's
    ok, _, worst = orc.tolerance_check(yr, y_ref[:, rows], sc_rows, x, rows)
    assert not ok and abs(worst - 2.0) < 1e-3
