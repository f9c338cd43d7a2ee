"""pytest plugin (test infrastructure): run the REFERENCE's own test suite
with the CUDA engine installed into the reference package.

Loaded with `-p tests.ref_engine_plugin` by tests/test_reference_suite.py.
At import -- before the reference's test modules import
`from gridshift.modeseek import meanshiftpp, meanshiftpp_step, ...` -- it
puts the reference install (baseline/_ref) on sys.path, calls
paper_2104_00303_b200.install(gridshift) and wraps the patched surfaces
with call counters, written to $GS_REF_CALLS at the end of the session, so
the caller can prove the CUDA engine (not the reference's numpy) answered.
"""

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
for p in (str(ROOT), str(REF)):
    if p not in sys.path:
        sys.path.insert(0, p)

import gridshift  # noqa: E402  (the reference package, from baseline/_ref)
import gridshift.modeseek as _ms  # noqa: E402
import gridshift.track as _tr  # noqa: E402

import paper_2104_00303_b200 as _gs  # noqa: E402

_gs.install(gridshift)
CALLS = {"meanshiftpp": 0, "meanshiftpp_step": 0, "extract_clusters": 0}


def _count(name, fn):
    def wrapped(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)
    wrapped.__gridshift_b200__ = True
    return wrapped


_engine = _count("meanshiftpp", _ms.meanshiftpp)
_ms.ENGINES["meanshiftpp"] = _engine
_ms.meanshiftpp = _engine
_tr.meanshiftpp = _engine
_ms.meanshiftpp_step = _count("meanshiftpp_step", _ms.meanshiftpp_step)
_ms.extract_clusters = _count("extract_clusters", _ms.extract_clusters)


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("GS_REF_CALLS")
    if out:
        Path(out).write_text(json.dumps(CALLS))
