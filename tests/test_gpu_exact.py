"""GPU parity of the exact mode (set_precision("fp64"): float64 potentials to
the sdb_*_f64 entry points) against the float64 oracle at the reference's own
tolerances.  Inputs are nudged off the fp32 grid so a silent fp32 round trip
would show."""

import numpy as np
import pytest

import paper_2308_03291_b200 as sd
from gpu_util import need_gpu
from golden.builders import family_inputs, make_dist
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu

RT, AT = 1e-9, 1e-11


@pytest.fixture(autouse=True)
def exact_mode():
    sd.set_precision("fp64")
    yield
    sd.set_precision("fp32")


def _off_grid(inp, seed):
    rng = np.random.default_rng(seed)
    out = {}
    for k, v in inp.items():
        v = np.asarray(v)
        if v.dtype.kind == "f":
            fin = np.isfinite(v)
            v = v.astype(np.float64).copy()
            v[fin] += 1e-9 * rng.standard_normal(fin.sum())
        out[k] = v
    return out


def _close(got, want):
    np.testing.assert_allclose(np.asarray(got, dtype=np.float64), want, rtol=RT, atol=AT)


@pytest.mark.parametrize("n,m", [(12, 5), (1, 3), (40, 32)])
def test_exact_chain(n, m):
    need_gpu()
    inp = _off_grid(family_inputs("chain", 11, dict(n=n, m=m)), 1)
    d = make_dist(sd, "chain", inp)
    z, pi, pt = O.chain_marginals(inp["init"][None], inp["transitions"][None])
    _close(sd.log_partition(d), z[0])
    mg = sd.marginals(d)
    _close(mg["init"], pi[0])
    _close(mg["transitions"], pt[0])
    assert sd.get_precision() == "fp64"


def test_exact_semi_markov():
    need_gpu()
    inp = _off_grid(family_inputs("semi_markov", 12, dict(n=10, s=3, m=4)), 2)
    d = make_dist(sd, "semi_markov", inp)
    z, mg = O.sm_marginals(inp["segment_potentials"])
    _close(sd.log_partition(d), z)
    _close(sd.marginals(d)["segment_potentials"], mg)


@pytest.mark.parametrize("n,m", [(9, 7), (30, 33)])
def test_exact_alignment(n, m):
    need_gpu()
    inp = _off_grid(family_inputs("alignment", 13, dict(n=n, m=m)), 3)
    d = make_dist(sd, "alignment", inp)
    z, mg = O.nw_marginals(inp["move_potentials"])
    _close(sd.log_partition(d), z)
    _close(sd.marginals(d)["move_potentials"], mg)


def test_exact_ctc():
    need_gpu()
    inp = _off_grid(family_inputs("ctc", 14, dict(T=12, V=6, L=4)), 4)
    d = make_dist(sd, "ctc", inp)
    z, mg = O.ctc_marginals(inp["frame_potentials"][None], np.asarray(inp["target"])[None])
    _close(sd.log_partition(d), z[0])
    _close(sd.marginals(d)["frame_potentials"], mg[0])


def test_exact_tree():
    need_gpu()
    inp = _off_grid(family_inputs("tree", 15, dict(n=8, m=3)), 5)
    d = make_dist(sd, "tree", inp)
    z, mg = O.tree_marginals(inp["span_potentials"])
    _close(sd.log_partition(d), z)
    _close(sd.marginals(d)["span_potentials"], mg)


def test_exact_pcfg_gradients():
    need_gpu()
    inp = _off_grid(family_inputs("pcfg", 16, dict(n=6, nt=3, pt=3)), 6)
    d = make_dist(sd, "pcfg", inp)
    z, g = O.pcfg_gradients(inp["root"], inp["binary_rules"], inp["emissions"])
    _close(sd.log_partition(d), z)
    pm = sd.potential_marginals(d)
    for k in ("root", "binary_rules", "emissions", "sticky"):
        _close(pm[k], g[k])


@pytest.mark.parametrize("projective", [False, True])
@pytest.mark.parametrize("single", [False, True])
def test_exact_spanning(projective, single):
    need_gpu()
    inp = _off_grid(family_inputs("spanning", 17, dict(n=9)), 7)
    d = make_dist(sd, "spanning", inp, dict(projective=projective, single=single))
    adj = inp["adjacency"]
    if projective:
        z, mg = O.eisner_log_partition(adj, single), O.eisner_marginals(adj, single)
    else:
        z, mg = O.mtt_log_partition(adj, single), O.mtt_marginals(adj, single)
    if isinstance(mg, tuple):
        mg = mg[1]
    _close(sd.log_partition(d), z)
    _close(sd.marginals(d)["adjacency"], mg)


def test_exact_entropy_and_statuses():
    need_gpu()
    inp = _off_grid(family_inputs("chain", 18, dict(n=7, m=4)), 8)
    p = make_dist(sd, "chain", inp)
    z, pi, pt = O.chain_marginals(inp["init"][None], inp["transitions"][None])
    h = z[0] - (np.sum(pi[0] * inp["init"]) + np.sum(pt[0] * inp["transitions"]))
    _close(sd.entropy(p), h)
    bad = dict(inp)
    bad["transitions"] = bad["transitions"].copy()
    bad["transitions"][2, 1, 1] = -np.inf
    bad["transitions"][:, :, :] = -np.inf  # no sequence at all
    assert sd.log_partition(make_dist(sd, "chain", bad)) == -np.inf
    with pytest.raises(sd.VacuousDistribution):
        sd.marginals(make_dist(sd, "chain", bad))


@pytest.mark.parametrize("family,dims", [("alignment", dict(n=40, m=30)), ("ctc", dict(T=60, V=8, L=10)),
                                         ("chain", dict(n=50, m=6))])
def test_auto_exact_large_magnitudes(family, dims):
    """fp32 mode (the default), potentials ~400 nats: the API routes the call to the exact
    kernels by itself (dist.AUTO_EXACT_NATS), so the results keep the reference's
    tolerances where the fp32 kernels would drift past 1e-4."""
    need_gpu()
    sd.set_precision("fp32")
    inp = family_inputs(family, 19, dims)
    inp = {k: (np.asarray(v) * 400.0 if np.asarray(v).dtype.kind == "f" else v) for k, v in inp.items()}
    d = make_dist(sd, family, inp)
    if family == "alignment":
        z, mg = O.nw_marginals(inp["move_potentials"])
        key = "move_potentials"
    elif family == "ctc":
        z, mg = O.ctc_marginals(inp["frame_potentials"][None], np.asarray(inp["target"])[None])
        z, mg = z[0], mg[0]
        key = "frame_potentials"
    else:
        z, pi, pt = O.chain_marginals(inp["init"][None], inp["transitions"][None])
        z, mg = z[0], pt[0]
        key = "transitions"
    _close(sd.log_partition(d), z)
    _close(sd.marginals(d)[key], mg)
    assert sd.get_precision() == "fp32"  # the switch is scoped to the call
