"""paper_2308_03291_b200 -- B200-native structured-inference core.

Drop-in for the hot path of the reference `structdist` 0.1.0 (SynJax,
arXiv 2308.03291): log-partition, marginals and argmax of linear-chain and
semi-Markov CRFs, monotone alignment / CTC, CKY Tree-CRF / PCFG and
projective / non-projective spanning trees, computed by hand-written sm_100a
CUDA kernels behind a C-ABI (include/sdb200.h, `_sdb200.so`).

The public surface mirrors `structdist/__init__.py:11-80`.
"""

from . import kernels  # noqa: F401  (batched device entry points)
from . import sharding  # noqa: F401  (multi-GPU batch sharding)
from . import problemfile  # noqa: F401  (problem documents, batched loader)
from .dist import (
    argmax,
    argmax_info,
    batch_map,
    cross_entropy,
    cross_entropy_info,
    entropy,
    entropy_info,
    kl_divergence,
    kl_divergence_info,
    log_partition,
    log_partition_info,
    log_prob,
    log_prob_info,
    marginals,
    marginals_info,
    masked_dot,
    potential_marginals,
    sample,
    sample_info,
    structure_score,
)
from .dist import get_precision, set_precision  # noqa: F401  (exact fp64 mode)
from .dist import warmup  # noqa: F401  (one-time CUDA context / module bring-up)
from .errors import (
    InvalidProblem,
    SamplerStepLimit,
    StructDistError,
    UnsupportedInference,
    VacuousDistribution,
)
from .sharding import run_sharded, sharded_batch_map  # noqa: F401
from .families import (
    FAMILIES,
    PCFG,
    CTCDist,
    LinearChainCRF,
    MonotoneAlignmentCRF,
    OneToOneMatching,
    SemiMarkovCRF,
    SpanningTreeCRF,
    TreeCRF,
    undirected_to_directed,
)

__version__ = "0.1.0"
