"""The reference-side binding (paper_2308_03291_b200.refshim, INTEGRATION.md
section 2) exercised on the UNMODIFIED reference installed in baseline/_ref:
after install(), the reference's own public calls run on the sm_100a kernels
and agree with what the reference computed before (rtol 1e-4), with the
reference's own exception classes."""
import os
import sys

import numpy as np
import pytest

from golden import builders as bld
from gpu_util import ATOL, RTOL, need_gpu

pytestmark = pytest.mark.gpu
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "structdist")):
        pytest.skip("unmodified reference not installed (tools/install_reference.sh)")
    sys.path.insert(0, REF)
    import structdist

    return structdist


def _cases(sd):
    init, tr = bld.chain(3, 9, 4)
    fp, tg = bld.ctc(4, 10, 5, 3)
    r, ru, e = bld.pcfg(5, 6, 3, 3)
    return [sd.LinearChainCRF(init, tr), sd.SemiMarkovCRF(bld.semi_markov(1, 7, 3, 3)),
            sd.MonotoneAlignmentCRF(bld.alignment(2, 6, 5)), sd.CTCDist(fp, tg), sd.TreeCRF(bld.tree(6, 7, 3)),
            sd.PCFG(r, ru, e), sd.SpanningTreeCRF(bld.spanning(7, 6)),
            sd.SpanningTreeCRF(bld.spanning(8, 6), projective=True, single_root_edge=True)]


def test_refshim_routes_reference_api(ref):
    need_gpu()
    from paper_2308_03291_b200 import refshim

    sd = ref
    cases = _cases(sd)
    want = [(sd.log_partition(d), sd.marginals(d), sd.argmax_info(d)) for d in cases]
    undo = refshim.install(sd)
    try:
        for d, (z, mg, (ind, score, algo)) in zip(cases, want):
            assert abs(sd.log_partition(d) - z) <= RTOL * max(1.0, abs(z))
            got = sd.marginals(d)
            for k in mg:
                np.testing.assert_allclose(got[k], mg[k], rtol=RTOL, atol=ATOL)
            gi, gs, ga = sd.argmax_info(d)
            assert ga == algo
            for k in ind:
                np.testing.assert_array_equal(gi[k], ind[k])
            assert abs(gs - score) <= 1e-9 * max(1.0, abs(score))
        vac = sd.LinearChainCRF(np.zeros(2), np.full((2, 2, 2), -np.inf))
        assert sd.log_partition(vac) == -np.inf
        with pytest.raises(sd.VacuousDistribution):
            sd.marginals(vac)
    finally:
        undo()
