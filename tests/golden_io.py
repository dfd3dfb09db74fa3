"""Load the committed golden vectors (tests/golden/golden_<family>.npz) made
by tests/golden/make_golden.py from the unmodified reference."""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
sys.path.insert(0, GOLDEN)

import builders  # noqa: E402,F401


class Case(dict):
    """Attribute access over one case's arrays plus its meta dict."""

    def __init__(self, meta, arrays):
        super().__init__(arrays)
        self.meta = meta

    def __getattr__(self, k):
        try:
            return self[k]
        except KeyError as e:
            raise AttributeError(k) from e

    @property
    def vacuous(self):
        return bool(self["vacuous"])

    def marg(self, key):
        return self.get(f"marg_{key}")

    def check_marg(self, key, got, rtol=1e-4, atol=1e-6, prefix="marg_"):
        """Compare a full marginal array against the golden (full or
        subsampled + sum).  Returns max abs error.  prefix "pmarg_" selects
        the potential_marginals goldens."""
        flat = np.asarray(got, dtype=np.float64).ravel()
        if f"{prefix}{key}" in self:
            ref = np.asarray(self[f"{prefix}{key}"]).ravel()
            np.testing.assert_allclose(flat, ref, rtol=rtol, atol=atol)
            return float(np.max(np.abs(flat - ref))) if flat.size else 0.0
        ix = self[f"{prefix}{key}_idx"]
        ref = self[f"{prefix}{key}_val"]
        np.testing.assert_allclose(flat[ix], ref, rtol=rtol, atol=atol)
        s = float(self[f"{prefix}{key}_sum"])
        assert abs(flat.sum() - s) <= rtol * abs(s) + atol * flat.size ** 0.5
        return float(np.max(np.abs(flat[ix] - ref)))


def load(family):
    z = np.load(os.path.join(GOLDEN, f"golden_{family}.npz"))
    meta = json.loads(str(z["meta_json"]))
    cases = []
    for m in meta:
        pre = f"c{m['idx']:03d}__"
        arrays = {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
        cases.append(Case(m, arrays))
    return cases


def inputs(case):
    """Rebuild the inputs of a case (stored for small cases, regenerated from
    the seed by builders.py for scale cases)."""
    m = case.meta
    fam = m["family"]
    if not m.get("scale"):
        return {k[3:]: case[k] for k in case if k.startswith("in_")}
    b = builders
    if fam == "chain":
        init, tr = b.chain(m["seed"], m["n"], m["m"])
        return {"init": init, "transitions": tr}
    if fam == "semi_markov":
        return {"segment_potentials": b.semi_markov(m["seed"], m["n"], m["s"], m["m"])}
    if fam == "alignment":
        return {"move_potentials": b.alignment(m["seed"], m["n"], m["m"])}
    if fam == "ctc":
        fp, tg = b.ctc(m["seed"], m["T"], m["V"], m["L"])
        return {"frame_potentials": fp, "target": np.array(tg)}
    if fam == "tree":
        return {"span_potentials": b.tree(m["seed"], m["n"], m["m"])}
    if fam == "pcfg":
        r, ru, e = b.pcfg(m["seed"], m["n"], m["nt"], m["pt"])
        return {"root": r, "binary_rules": ru, "emissions": e}
    if fam == "spanning":
        return {"adjacency": b.spanning(m["seed"], m["n"], m.get("directed", True))}
    raise KeyError(fam)
