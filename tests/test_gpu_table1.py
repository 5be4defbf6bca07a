"""GPU: Table 1 (bench::table1_genp, bench.cpp:107-140) at the acceptance scale
(tests/acceptance.cpp:51-73: n = 64, 100 trials, CirculantSign, seed 20260825) on the reference's
own illblock systems (tests/golden t1/*): both refinement levels as batched Left-side launches.
The GPU's samples must pass the acceptance gates, accept/reject exactly where the reference does,
and follow the reference's residual distribution (geometric-mean ratio within 2x; the contrast arm
is catastrophic on both sides: median >= 10)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_table1_acceptance_scale(rl, golden):
    from paper_1212_4560_b200.table1 import acceptance_criterion1, table1_genp_systems
    A, b, ref = golden["t1/A"], golden["t1/b"], golden["t1/samples"]
    rows = table1_genp_systems(A, b, seed=20260825, size_index=0)
    assert [(r.n, r.refine, r.stats.n_trials) for r in rows] == [(64, 0, 100), (64, 1, 100)]
    assert acceptance_criterion1(rows)
    g0, g1 = np.array(rows[0].stats.samples), np.array(rows[1].stats.samples)
    raw = np.array(rows[0].raw_stats.samples)
    assert np.array_equal(g0 <= 1e-7, ref[:, 0] <= 1e-7) and np.array_equal(g1 <= 1e-7, ref[:, 1] <= 1e-7)
    for col, ours in ((0, g0), (1, g1)):
        r = np.log(np.maximum(ours, 1e-300) / np.maximum(ref[:, col], 1e-300))
        assert np.exp(np.mean(r)) <= 2.0 and np.exp(np.mean(r)) >= 0.5, (col, np.exp(np.mean(r)))
    assert np.median(raw) >= 10.0 and np.median(ref[:, 2]) >= 10.0
