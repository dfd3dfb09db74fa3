"""Host-side indicator validation (validate.py) against the reference's
validate_indicator (dist.py:224-248): every golden indicator of
tests/golden/golden_derived.npz is accepted or rejected exactly as the
unmodified reference did.  CPU only (no kernel runs)."""

import numpy as np
import pytest

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200.validate import collapse, is_binary_bracketing, validate_indicator
from golden import builders as bld
from golden_io import load

CASES = [c for c in load("derived") if c.meta.get("nbad")]


def _dist(case):
    fam = case.meta["family"]
    inp = {k[3:]: case[k] for k in case if k.startswith("in_")}
    return bld.make_dist(sd, fam, inp, case.meta)


def _ind(case, prefix):
    return {k[len(prefix):]: case[k] for k in case if k.startswith(prefix)}


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c.meta['family']}-{c.meta['idx']}")
def test_validate_matches_reference(case):
    d = _dist(case)
    validate_indicator(d, _ind(case, "sample_"))  # a sample is a valid structure
    for b in range(case.meta["nbad"]):
        ind = _ind(case, f"bad{b}_")
        if np.isnan(case.bad_logprob[b]):
            with pytest.raises(sd.InvalidProblem):
                validate_indicator(d, ind)
        else:
            validate_indicator(d, ind)


def test_collapse_and_bracketing():
    assert collapse([0, 1, 1, 0, 1, 2, 2, 0]) == (1, 1, 2)
    assert collapse([0, 0]) == ()
    assert is_binary_bracketing({(0, 0)}, 1)
    assert is_binary_bracketing({(0, 2), (0, 1), (0, 0), (1, 1), (2, 2)}, 3)
    assert not is_binary_bracketing({(0, 2), (0, 0), (1, 1), (2, 2), (1, 2), (0, 1)}, 3)
    assert not is_binary_bracketing({(0, 2), (0, 0), (1, 1), (2, 2), (0, 0)}, 3)


def test_missing_part_is_invalid():
    d = sd.LinearChainCRF(np.zeros(2), np.zeros((1, 2, 2)))
    with pytest.raises(sd.InvalidProblem):
        validate_indicator(d, {"init": np.array([1.0, 0.0])})
