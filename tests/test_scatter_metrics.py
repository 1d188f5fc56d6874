"""Target strength, far-field deviation (the paper's Delta_sct) and the
far-field CSV against the reference (scatter.py:411-452): its own unit
tests (pkg/tests/test_scatter.py TestTargetStrength / TestDeviation /
test_far_field_csv) and a golden file written by the real reference
(tests/golden/make_ts_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden


def _s():
    from paper_1711_01897_b200 import scatter
    return scatter


def test_reference_golden_values_and_csv(tmp_path):
    s, g = _s(), golden("ts")
    ts = s.target_strength(g["u"], 1.5 - 0.5j, 75.0)
    assert np.array_equal(ts, g["ts"])  # includes the -inf of the silent sample
    assert s.deviation(g["u"], g["ref"]) == float(g["dev"])
    p = tmp_path / "far.csv"
    s.write_far_field_csv(p, g["angles"], g["u"], 1.5 - 0.5j, 75.0)
    assert p.read_text() == str(g["csv"])


def test_target_strength_reference_cases():
    s = _s()
    assert s.target_strength(1.0 / 50.0, 1.0, 50.0) == pytest.approx(0.0)
    assert s.target_strength(1.0, 1.0, 20000.0) == pytest.approx(86.0206, abs=1e-4)
    base = s.target_strength(0.01, 1.0, 100.0)
    assert s.target_strength(0.02, 1.0, 100.0) - base == pytest.approx(6.0206, abs=1e-4)
    assert s.target_strength(0.0, 1.0, 100.0) == -np.inf
    assert isinstance(s.target_strength(0.5, 1.0, 10.0), float)


def test_target_strength_validation():
    from paper_1711_01897_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        _s().target_strength(1.0, 0.0, 100.0)
    with pytest.raises(ConfigError):
        _s().target_strength(1.0, 1.0, -5.0)


def test_deviation_reference_cases(rng):
    from paper_1711_01897_b200.errors import ConfigError
    s = _s()
    u = rng.standard_normal(10) + 1j * rng.standard_normal(10)
    assert s.deviation(u, u) == 0.0
    assert s.deviation(1.01 * u, u) == pytest.approx(0.01, rel=1e-10)
    with pytest.raises(ZeroDivisionError, match="index 2"):
        s.deviation(np.ones(4), np.array([1.0, 2.0, 0.0, 3.0]))
    with pytest.raises(ConfigError):
        s.deviation(np.ones(3), np.ones(4))
