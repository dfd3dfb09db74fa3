"""Host logic of the exact mode (no GPU): the precision switch, what it
routes, and that the refshim restores the previous mode on undo."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import backends, kernels as K, ragged


@pytest.fixture(autouse=True)
def restore():
    yield
    sd.set_precision("fp32")


def test_switch_values():
    assert sd.get_precision() == "fp32"
    sd.set_precision("fp64")
    assert sd.get_precision() == "fp64" and backends.pot_dtype() == torch.float64
    sd.set_precision("fp32")
    assert backends.pot_dtype() == torch.float32
    with pytest.raises(ValueError):
        sd.set_precision("fp16")


def test_exact_dispatch_is_by_dtype():
    assert K.exact(torch.zeros(2, dtype=torch.float64))
    assert not K.exact(torch.zeros(2, dtype=torch.float32))
    assert not K.exact(np.zeros(2))


def test_exact_mode_pads_ragged_chains():
    ds = [sd.LinearChainCRF(np.zeros(3), np.zeros((n - 1, 3, 3))) for n in (4, 6)]
    sd.set_precision("fp64")
    assert not ragged.native_ragged(ds)  # the fp64 chain kernel takes same-length groups


def test_refshim_restores_precision():
    from paper_2308_03291_b200 import refshim

    class _Mod:  # the attributes install() replaces, on stand-in modules
        pass

    fake = _Mod()
    fake.errors = type("E", (), {"VacuousDistribution": ValueError, "InvalidProblem": TypeError,
                                 "UnsupportedInference": KeyError})
    names = {"chain": ["forward_log_partition", "chain_marginals", "chain_argmax", "semi_markov_log_partition",
                       "semi_markov_marginals", "semi_markov_argmax"],
             "alignment": ["nw_log_partition", "nw_marginals", "nw_argmax", "ctc_log_partition", "ctc_marginals",
                           "ctc_argmax"],
             "constituency": ["cky_log_partition", "tree_marginals", "tree_argmax", "pcfg_inside", "pcfg_gradients",
                              "pcfg_argmax", "pcfg_max_score"],
             "spanning": ["span_log_partition", "span_marginals", "span_argmax"]}
    for mod, fns in names.items():
        m = _Mod()
        for f in fns:
            setattr(m, f, None)
        setattr(fake, mod, m)
    undo = refshim.install(fake, exact=True, warm=False)  # host logic only: no device bring-up
    assert sd.get_precision() == "fp64"
    undo()
    assert sd.get_precision() == "fp32" and fake.chain.chain_marginals is None


def test_auto_exact_detection():
    """dist._large: potentials past AUTO_EXACT_NATS (finite entries only) send a call to the
    exact kernels; -inf structure zeros do not."""
    from paper_2308_03291_b200 import dist as gd

    small = sd.LinearChainCRF(np.zeros(3), np.full((2, 3, 3), -5.0))
    th = np.full((2, 3, 3), -np.inf)
    th[:, 0, 0] = 1.0
    masked = sd.LinearChainCRF(np.zeros(3), th)
    big = sd.LinearChainCRF(np.zeros(3), np.full((2, 3, 3), -2.0 * gd.AUTO_EXACT_NATS))
    assert not gd._large([small]) and not gd._large([masked])
    assert gd._large([small, big])


def test_exact_scope_is_per_thread():
    """dist._run / _argmax switch to the exact kernels through a per-thread scope: another
    thread (and the process default) keeps its precision."""
    import threading

    seen = {}

    def other():
        seen["other"] = backends.exact_now()

    with backends.exact_scope():
        assert backends.exact_now() and sd.get_precision() == "fp32"
        t = threading.Thread(target=other)
        t.start()
        t.join()
    assert seen["other"] is False and not backends.exact_now()
