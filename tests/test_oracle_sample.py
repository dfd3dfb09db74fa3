"""Pin the oracle's samplers to the reference: same seed -> the same
structures as structdist.sample_info(d, seed, num=2) (golden_sample.npz)."""

import numpy as np
import pytest

from golden_io import inputs, load
from oracle import sd_oracle as O

CASES = load("sample")


def _draws(case, fn):
    rng = np.random.default_rng(int(case.meta["seed"]))
    return [fn(rng) for _ in range(2)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: str(c.meta))
def test_oracle_samples_match_reference(case):
    x = inputs(case)
    fam = case.meta["family"]
    if fam == "chain":
        for r, tags in enumerate(_draws(case, lambda g: O.chain_sample(x["init"], x["transitions"], g))):
            ind = case[f"sample{r}_transitions"]
            assert case[f"sample{r}_init"][tags[0]] == 1
            for t in range(len(tags) - 1):
                assert ind[t, tags[t], tags[t + 1]] == 1
            assert ind.sum() == len(tags) - 1
    elif fam == "alignment":
        for r, path in enumerate(_draws(case, lambda g: O.nw_sample(x["move_potentials"], g))):
            mask = np.zeros_like(x["move_potentials"])
            ii, jj = np.nonzero(path >= 0)
            mask[ii, jj, path[ii, jj]] = 1
            np.testing.assert_array_equal(mask, case[f"sample{r}_move_potentials"])
    elif fam == "ctc":
        lab = O.ctc_labels(np.asarray(x["target"])[None])[0]
        for r, states in enumerate(_draws(case, lambda g: O.ctc_sample(x["frame_potentials"], x["target"], g))):
            mask = np.zeros_like(x["frame_potentials"])
            mask[np.arange(len(states)), lab[states]] = 1
            np.testing.assert_array_equal(mask, case[f"sample{r}_frame_potentials"])
    elif fam == "tree":
        for r, lab in enumerate(_draws(case, lambda g: O.tree_sample(x["span_potentials"], g))):
            mask = np.zeros_like(x["span_potentials"])
            ii, jj = np.nonzero(lab >= 0)
            mask[ii, jj, lab[ii, jj]] = 1
            np.testing.assert_array_equal(mask, case[f"sample{r}_span_potentials"])
    elif fam == "spanning":
        single = bool(case.meta["single"])
        for r, heads in enumerate(_draws(case, lambda g: O.eisner_sample(x["adjacency"], single, g))):
            mask = np.zeros_like(x["adjacency"])
            d = np.arange(1, len(heads))
            mask[heads[1:], d] = 1
            np.testing.assert_array_equal(mask, case[f"sample{r}_adjacency"])
        heads = O.eisner_decode(x["adjacency"], single)
        mask = np.zeros_like(x["adjacency"])
        mask[heads[1:], np.arange(1, len(heads))] = 1
        np.testing.assert_array_equal(mask, case["eisner_max"])


def test_stream_equals_per_pick_draws():
    """The GPU consumes one pre-drawn Gumbel stream; numpy's Generator gives
    the same values whether drawn per pick or in one call."""
    a = np.random.default_rng(5)
    per = np.concatenate([a.gumbel(size=k) for k in (3, 1, 2, 7, 1)])
    np.testing.assert_array_equal(per, np.random.default_rng(5).gumbel(size=14))


@pytest.mark.parametrize("case", load("wilson"), ids=lambda c: str(c.meta))
def test_oracle_wilson_matches_reference(case):
    adj = inputs(case)["adjacency"]
    single = bool(case.meta["single"])
    rng = np.random.default_rng(int(case.meta["seed"]))
    for r in range(2):
        heads = O.wilson_sample(adj, single, rng)
        mask = np.zeros_like(adj)
        mask[heads[1:], np.arange(1, len(heads))] = 1
        np.testing.assert_array_equal(mask, case[f"sample{r}_adjacency"])


@pytest.mark.parametrize("case", load("colbourn"), ids=lambda c: str(c.meta))
def test_oracle_colbourn_matches_reference(case):
    adj = inputs(case)["adjacency"]
    single = bool(case.meta["single"])
    rng = np.random.default_rng(int(case.meta["seed"]))
    for r in range(2):
        heads, fell = O.colbourn_sample(adj, single, rng)
        assert fell == case.meta["algo"].endswith("wilson-fallback")
        mask = np.zeros_like(adj)
        mask[heads[1:], np.arange(1, len(heads))] = 1
        np.testing.assert_array_equal(mask, case[f"sample{r}_adjacency"])


@pytest.mark.parametrize("case", load("sample2"), ids=lambda c: str(c.meta))
def test_oracle_semimarkov_pcfg_samples_match_reference(case):
    x = inputs(case)
    rng = np.random.default_rng(int(case.meta["seed"]))
    for r in range(2):
        if case.meta["family"] == "semi_markov":
            th = x["segment_potentials"]
            mask = np.zeros_like(th)
            for s0, w, p, l in O.sm_sample(th, rng):
                mask[s0, w - 1, p, l] = 1
            np.testing.assert_array_equal(mask, case[f"sample{r}_segment_potentials"])
        else:
            mask = O.pcfg_sample(x["root"], x["binary_rules"], x["emissions"], rng)
            np.testing.assert_array_equal(mask, case[f"sample{r}_sticky"])
