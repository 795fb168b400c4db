"""Host-side checks of the seeded input generators (synth/)."""
import numpy as np
import pytest

from synth import CONFIGS, make_config, mask_count
from synth.generate import fibre_mask, uniform_mask


def test_mask_counts_match_config_table():
    """exact observed counts, round-half-up(SR·n) (reading R12)."""
    assert mask_count(0.30, 8000) == 2400
    assert mask_count(0.10, 256 * 256 * 31) == 203162
    assert mask_count(0.05, 144 * 176 * 3 * 50) == 190080
    assert mask_count(0.05, 64 ** 4 * 32) == 26843546
    assert int(np.floor(0.70 * 214 * 61 * 4 + 0.5)) == 36551


@pytest.mark.parametrize("name", ["C1", "C2", "C2s", "C3s", "C4s", "C5s"])
def test_config_shapes_and_counts(name):
    p = make_config(name)
    assert p.truth.shape == (p.n,) and p.mask.shape == (p.n,)
    assert p.truth.dtype == np.dtype(CONFIGS[name]["dtype"])
    assert int(p.mask.sum()) == p.recipe["mask"]["observed"]
    obs = p.mask.astype(bool)
    assert np.array_equal(p.observed[obs], p.truth[obs])
    assert np.all(p.observed[~obs] == 0)
    assert np.array_equal(p.ranks, p.ranks.T) and np.all(np.diag(p.ranks) == 0)


def test_generators_are_deterministic():
    a, b = make_config("C3s", seed=3), make_config("C3s", seed=3)
    assert np.array_equal(a.truth, b.truth) and np.array_equal(a.mask, b.mask)
    assert np.array_equal(a.G0, b.G0)
    c = make_config("C3s", seed=4)
    assert not np.array_equal(a.G0, c.G0)


def test_fibre_mask_structure():
    """FM protocol: whole mode-3 fibres missing, exact fibre count."""
    dims = (4, 5, 6)
    m = fibre_mask(dims, 2, 10, seed=0).reshape(dims, order="F")
    per_fibre = m.sum(axis=2)
    assert set(np.unique(per_fibre)) <= {0, 6}
    assert int((per_fibre == 0).sum()) == 10


def test_uniform_mask_exact():
    m = uniform_mask(1000, 370, seed=1)
    assert int(m.sum()) == 370


def test_C4_fibre_counts():
    p = make_config("C4")
    assert p.recipe["mask"]["fibres"] == 52216
    assert p.recipe["mask"]["missing_fibres"] == 36551
    assert int(p.mask.sum()) == 2255760
