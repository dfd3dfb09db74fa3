"""Problem-document fixtures written by the UNMODIFIED reference's
problemfile.py (distribution_to_problem + dump_problem), plus malformed
documents and the reference's verdict on each (tests/golden/problems/).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_problems.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
import builders as bld  # noqa: E402
import structdist as sd  # noqa: E402
from structdist import problemfile as pf  # noqa: E402

OUT = os.path.join(HERE, "problems")
os.makedirs(OUT, exist_ok=True)
verdicts = {}


def write(name, doc_or_text):
    path = os.path.join(OUT, name + ".json")
    if isinstance(doc_or_text, str):
        with open(path, "w") as fh:
            fh.write(doc_or_text)
    else:
        pf.dump_problem(doc_or_text, path)
    try:
        d = pf.problem_to_distribution(pf.load_problem(path))
        verdicts[name] = {"ok": True, "family": d.family, "logz": float(sd.log_partition(d))}
    except sd.InvalidProblem as e:
        verdicts[name] = {"ok": False, "error": str(e)}


r, ru, e = bld.pcfg(3, 4, 2, 2)
fp, tg = bld.ctc(4, 6, 4, 2)
dists = {
    "chain": sd.LinearChainCRF(*bld.chain(1, 5, 3)),
    "semi_markov": sd.SemiMarkovCRF(bld.semi_markov(2, 5, 2, 2)),
    "alignment": sd.MonotoneAlignmentCRF(bld.alignment(3, 4, 3)),
    "ctc": sd.CTCDist(fp, tg),
    "tree": sd.TreeCRF(bld.tree(5, 4, 2)),
    "pcfg": sd.PCFG(r, ru, e),
    "pcfg_sticky": sd.PCFG(r, ru, e, np.where(np.eye(4) > 0, 0.0, 0.0)),
    "spanning": sd.SpanningTreeCRF(bld.spanning(6, 4)),
    "spanning_proj": sd.SpanningTreeCRF(bld.spanning(7, 4), projective=True, single_root_edge=True),
}
for name, d in dists.items():
    ind = sd.argmax(d)
    write(name, pf.distribution_to_problem(d, ind))
good = pf.distribution_to_problem(dists["chain"])
bad = {
    "bad_string": json.dumps(dict(good, potentials=dict(good["potentials"], init=["x", 0.0, 1.0]))),
    "bad_bool": json.dumps(dict(good, potentials=dict(good["potentials"], init=[True, 0.0, 1.0]))),
    "bad_null": json.dumps(dict(good, potentials=dict(good["potentials"], init=[None, 0.0, 1.0]))),
    "bad_family": json.dumps(dict(good, family="nope")),
    "bad_config": json.dumps(dict(good, config={"n": 5})),
    "bad_shape": json.dumps(dict(good, config={"n": 6, "m": 3})),
    "bad_json": "{not json",
    "bad_inf": json.dumps(dict(good, potentials=dict(good["potentials"], init=["inf", 0.0, 1.0]))),
}
for name, text in bad.items():
    write(name, text)
with open(os.path.join(OUT, "verdicts.json"), "w") as fh:
    json.dump(verdicts, fh, indent=1, sort_keys=True)
print(json.dumps(verdicts, indent=1)[:1500])
