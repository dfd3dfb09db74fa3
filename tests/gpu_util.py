"""Helpers for the -m gpu parity tests."""
import numpy as np
import pytest
import torch

NEG_INF = float("-inf")

# parity bar (BASELINE.json north_star): fp32 path within rtol 1e-4 of the
# float64 reference, with an absolute floor for tiny marginals
RTOL = 1e-4
ATOL = 1e-6


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def close_logz(got, want, rtol=RTOL):
    got, want = float(got), float(want)
    if want == NEG_INF:
        assert got == NEG_INF, (got, want)
    else:
        assert abs(got - want) <= rtol * max(1.0, abs(want)), (got, want)


def dev(x, dtype=torch.float32):
    return torch.as_tensor(np.asarray(x), dtype=dtype).cuda()
