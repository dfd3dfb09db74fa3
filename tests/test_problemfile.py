"""Problem documents (problemfile.py): the fast batched decoder accepts and
rejects exactly what the unmodified reference accepted / rejected on the
fixtures it wrote (tests/golden/problems/, make_problems.py), decodes the
same tensors, and writes byte-identical documents.  CPU only."""
import glob
import json
import os

import numpy as np
import pytest

import paper_2308_03291_b200 as sd
from paper_2308_03291_b200 import problemfile as pf

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "problems")
VERDICTS = json.load(open(os.path.join(HERE, "verdicts.json")))


def _slow_decode(v):  # problemfile.py:24-34, for comparison
    if isinstance(v, list):
        return [_slow_decode(x) for x in v]
    return float("-inf") if v == "-inf" else float(v)


@pytest.mark.parametrize("name", sorted(VERDICTS))
def test_loader_matches_reference_verdicts(name):
    path = os.path.join(HERE, name + ".json")
    want = VERDICTS[name]
    if not want["ok"]:
        with pytest.raises(sd.InvalidProblem) as ei:
            pf.problem_to_distribution(pf.load_problem(path))
        if name == "bad_json":
            assert str(ei.value).startswith("cannot parse")
        else:
            assert str(ei.value) == want["error"]
        return
    doc = pf.load_problem(path)
    d = pf.problem_to_distribution(doc)
    assert d.family == want["family"]
    raw = json.load(open(path))
    for k, v in d.potentials().items():
        if k in raw["potentials"]:
            np.testing.assert_array_equal(v, np.asarray(_slow_decode(raw["potentials"][k])))
    ind = pf.document_indicator(doc)
    out = os.path.join("/tmp", f"sdb_pf_{os.getpid()}_{name}.json")
    pf.dump_problem(pf.distribution_to_problem(d, ind), out)
    assert open(out).read() == open(path).read()  # byte-identical document
    os.remove(out)


def test_load_problems_batch():
    paths = sorted(p for p in glob.glob(os.path.join(HERE, "*.json")) if not os.path.basename(p).startswith(("bad", "verd")))
    got = pf.load_problems(paths)
    assert len(got) == len(paths) and all(ind is not None for _, ind in got)
