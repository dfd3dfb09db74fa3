"""pytest plugin: run the reference's OWN test-suite with its family
functions routed onto the sm_100a kernels (paper_2308_03291_b200.refshim).

    PYTHONPATH=baseline/_ref:tools/refsuite:. python -m pytest -p refsuite_plugin baseline/_ref/tests

(tools/run_refsuite.sh).  The reference is imported unchanged; only the
module attributes its dispatch reads are replaced."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import structdist  # noqa: E402  (the unmodified reference)

from paper_2308_03291_b200 import refshim  # noqa: E402

_EXACT = os.environ.get("SDB_REFSUITE_EXACT", "0") == "1"  # fp64 entry points (set_precision("fp64"))
_undo = refshim.install(structdist, exact=_EXACT)


def pytest_report_header(config):
    return ["structdist family functions routed onto the sm_100a kernels (paper_2308_03291_b200.refshim)"
            + (" -- exact fp64 mode" if _EXACT else ""),
            f"structdist from {os.path.dirname(structdist.__file__)}"]
