"""GPU parity: monotone alignment (alignment.py:62-167) through the C-ABI."""

import numpy as np
import pytest
import torch

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import kernels as K
from golden_io import inputs, load
from gpu_util import ATOL, NEG_INF, RTOL, close_logz, dev, need_gpu
from golden.builders import alignment, batch_alignment
from oracle import sd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", load("alignment"), ids=lambda c: str(c.meta))
def test_alignment_golden(case):
    need_gpu()
    d = sd.MonotoneAlignmentCRF(inputs(case)["move_potentials"])
    close_logz(sd.log_partition(d), case.logz)
    marg, algo = sd.marginals_info(d)
    assert algo == "needleman-wunsch"
    case.check_marg("move_potentials", marg["move_potentials"], RTOL, ATOL)
    ind, score, algo = sd.argmax_info(d)
    assert algo == "max-plus-needleman-wunsch"
    np.testing.assert_array_equal(ind["move_potentials"], case["argmax_move_potentials"])
    assert score == float(case.argmax_score)


@pytest.mark.parametrize("B,n,m", [(3, 512, 128), (4, 40, 31), (2, 33, 32), (5, 7, 70), (2, 1, 1), (3, 100, 200)])
def test_alignment_batched_vs_oracle(B, n, m):
    need_gpu()
    th = batch_alignment(1000, B, n, m)
    logz, marg, st = K.nw_fb(dev(th))
    assert (st.cpu().numpy() == 0).all()
    lz_only, _, _ = K.nw_fb(dev(th), marginals=False)
    for b in range(B):
        z, mg = O.nw_marginals(th[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        assert abs(lz_only[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
    path, score, st2 = K.nw_viterbi(dev(th))
    for b in range(min(B, 2)):
        mask, sc = O.nw_argmax(th[b])
        p = path[b].cpu().numpy()
        got = np.zeros_like(mask)
        ii, jj = np.nonzero(p >= 0)
        got[ii, jj, p[ii, jj]] = 1
        np.testing.assert_array_equal(got, mask)  # bit-exact argmax
        assert score[b].item() == sc


def test_alignment_config_invariants():
    """C2a shape (B=256, 512x128): every alignment path crosses each
    anti-diagonal band once -> marginal flow conservation: sum of marginals
    of moves INTO row i cells equals 1 summed appropriately; we check the
    cheapest size-independent identity: total expected DOWN moves = n and
    RIGHT moves = m minus expected DIAG moves."""
    need_gpu()
    B, n, m = 256, 512, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    th = torch.randn(B, n + 1, m + 1, 3, device="cuda", generator=g)
    th[:, 0, :, 0] = NEG_INF
    th[:, 0, :, 1] = NEG_INF
    th[:, :, 0, 0] = NEG_INF
    th[:, :, 0, 2] = NEG_INF
    logz, marg, st = K.nw_fb(th)
    assert (st == 0).all()
    md = marg.double()
    diag, down, right = md[..., 0].sum((1, 2)), md[..., 1].sum((1, 2)), md[..., 2].sum((1, 2))
    assert torch.allclose(diag + down, torch.full_like(diag, n), rtol=1e-4)
    assert torch.allclose(diag + right, torch.full_like(diag, m), rtol=1e-4)


def test_alignment_status():
    need_gpu()
    th = batch_alignment(5, 3, 6, 5)
    th[1, 1:, :, :] = NEG_INF  # nothing reaches row >= 1
    th[2, 3, 3, 1] = np.nan
    logz, marg, st = K.nw_fb(dev(th))
    assert st.cpu().tolist() == [0, 1, 2]
    assert logz[1].item() == NEG_INF
    assert float(marg[1].abs().sum()) == 0.0


# Shapes on the meet-in-the-middle path (n >= 40 (NW-1) + 32), including
# m + 1 a multiple of 32 (no padding lanes), one padding-heavy strip, and
# many strips.
@pytest.mark.parametrize("B,n,m", [(2, 32, 5), (3, 100, 63), (2, 80, 32), (2, 300, 200), (2, 400, 287),
                                   (2, 201, 127), (3, 513, 129)])
def test_alignment_mitm_vs_oracle(B, n, m):
    need_gpu()
    th = batch_alignment(2000 + n + m, B, n, m)
    logz, marg, st = K.nw_fb(dev(th))
    assert (st.cpu().numpy() == 0).all()
    for b in range(B):
        z, mg = O.nw_marginals(th[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)


def test_alignment_mitm_masked_and_vacuous():
    """Banded alignment (cells far from the diagonal forbidden), a vacuous
    instance and an invalid one, all on the meet-in-the-middle path."""
    need_gpu()
    n, m = 160, 96
    th = batch_alignment(77, 4, n, m)
    ii, jj = np.meshgrid(np.arange(n + 1), np.arange(m + 1), indexing="ij")
    band = np.abs(ii * m - jj * n) > 12 * n
    th[0][band] = NEG_INF
    th[1, :, 50, :] = NEG_INF  # column 50 unreachable -> no path
    th[2, 70, 40, 0] = np.inf
    logz, marg, st = K.nw_fb(dev(th))
    assert st.cpu().tolist() == [0, 1, 2, 0]
    assert logz[1].item() == NEG_INF and float(marg[1].abs().sum()) == 0.0
    for b in (0, 3):
        z, mg = O.nw_marginals(th[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("n,m", [(200, 64), (152, 128), (33, 32)])
def test_alignment_mitm_edge_column(n, m):
    """m % 32 == 0: column m is handled outside the strips (suffix sums for
    beta, prefix sums of the entry marginals for its DOWN moves).  Masks and
    bad values placed in that column must behave exactly as anywhere else."""
    need_gpu()
    th = batch_alignment(31 + n + m, 6, n, m)
    th[1, n // 3, m, 1] = NEG_INF        # no DOWN through (n/3, m): enter below
    th[2, n // 2, m, 1] = np.nan         # invalid
    th[3, :n, m, 0] = NEG_INF            # enter column m only by RIGHT ...
    th[3, :n // 2, m, 2] = NEG_INF       # ... in the lower half
    th[4, 0, m, 0] = np.inf              # an unused move, still invalid
    th[5, :, m, 0] = NEG_INF             # column m unreachable -> vacuous
    th[5, :, m, 2] = NEG_INF
    logz, marg, st = K.nw_fb(dev(th))
    assert st.cpu().tolist() == [0, 0, 2, 0, 2, 1]
    assert logz[5].item() == NEG_INF and float(marg[5].abs().sum()) == 0.0
    for b in (0, 1, 3):
        z, mg = O.nw_marginals(th[b])
        assert abs(logz[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("B,n,m", [(2, 20, 400), (2, 360, 370), (3, 5, 1000)])
def test_alignment_general_shapes(B, n, m):
    """m > 351 runs the anti-diagonal fp64 kernel (nw_gen.cu): same results,
    same argmax tie-breaking, same statuses as the strip kernels."""
    need_gpu()
    th = batch_alignment(4000 + n + m, B, n, m)
    th[B - 1, n // 2, :, 1] = NEG_INF  # a row no path can enter by DOWN
    logz, marg, st = K.nw_fb(dev(th))
    lz_only, _, st0 = K.nw_fb(dev(th), marginals=False)
    path, score, st2 = K.nw_viterbi(dev(th))
    for b in range(B):
        z, mg = O.nw_marginals(th[b])
        assert st[b].item() == st0[b].item() == st2[b].item() == (0 if z > NEG_INF else 1)
        if z == NEG_INF:
            continue
        assert abs(logz[b].item() - z) <= RTOL * abs(z) and abs(lz_only[b].item() - z) <= RTOL * abs(z)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
        mask, sc = O.nw_argmax(th[b])
        p = path[b].cpu().numpy()
        got = np.zeros_like(mask)
        ii, jj = np.nonzero(p >= 0)
        got[ii, jj, p[ii, jj]] = 1
        np.testing.assert_array_equal(got, mask)
        assert score[b].item() == sc
    bad = th.copy()
    bad[0, 3, 7, 2] = np.nan
    assert K.nw_fb(dev(bad))[2][0].item() == 2
    d = sd.MonotoneAlignmentCRF(th[0])  # through the public API
    assert abs(sd.log_partition(d) - O.nw_marginals(th[0])[0]) <= RTOL * abs(float(logz[0]))


def test_run_host_batch_matches_device_call():
    """kernels.run_host_batch (pinned host slices, H2D / kernels / D2H
    overlapped on separate streams) returns exactly the device call's result."""
    need_gpu()
    th = batch_alignment(1500, 11, 40, 24)
    lz, mg, st = K.nw_fb(dev(th))
    host_in = [torch.as_tensor(th, dtype=torch.float32).pin_memory()]
    host_out = [torch.empty(tuple(lz.shape), dtype=lz.dtype).pin_memory(),
                torch.empty(tuple(mg.shape), dtype=mg.dtype).pin_memory()]
    K.run_host_batch(lambda t: K.nw_fb(t)[:2], host_in, host_out, torch.device("cuda", 0), chunks=4)
    torch.cuda.synchronize()
    assert torch.equal(host_out[0], lz.cpu()) and torch.equal(host_out[1], mg.cpu())
    # explicit (uneven) slice sizes
    for h in host_out:
        h.zero_()
    K.run_host_batch(lambda t: K.nw_fb(t)[:2], host_in, host_out, torch.device("cuda", 0), chunks=[5, 4, 2])
    torch.cuda.synchronize()
    assert torch.equal(host_out[0], lz.cpu()) and torch.equal(host_out[1], mg.cpu())


@pytest.mark.parametrize("scale,exact", [(25.0, False), (400.0, True)])
def test_alignment_large_magnitudes(scale, exact):
    """Move log-potentials scaled to |theta| ~ 25 nats (|log Z| ~ 1e4) through the
    meet-in-the-middle kernel: integer offsets keep fp32 at the parity bar.  Per-step
    rounding grows like |theta| 2^-24; at ~400 nats float64 potentials take the exact
    kernels."""
    need_gpu()
    th = (batch_alignment(2100, 2, 200, 64) * scale).astype(np.float32).astype(np.float64)
    x = torch.as_tensor(th, dtype=torch.float64 if exact else torch.float32, device="cuda")
    logz, marg, st = K.nw_fb(x)
    for b in range(2):
        z, mg = O.nw_marginals(th[b])
        np.testing.assert_allclose(logz[b].item(), z, rtol=RTOL)
        np.testing.assert_allclose(marg[b].cpu().numpy(), mg, rtol=RTOL, atol=ATOL)
