import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running test")


def pytest_sessionfinish(session, exitstatus):
    """Write the C-att-5 diagnostics (max abs / max rel / bound use) of every GPU-vs-oracle
    comparison this session made, for profiles/."""
    try:
        from tests.helpers import DIAGNOSTICS
    except Exception:
        return
    if not DIAGNOSTICS:
        return
    import json
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    worst = {k: max(d[k] for d in DIAGNOSTICS) for k in ("max_abs", "max_rel", "max_bound_use")}
    json.dump({"tolerance": "abs(x - r) <= 2e-3 + 1e-2 abs(r) per element [C-att-5]",
               "comparisons": len(DIAGNOSTICS), "worst": worst, "all": DIAGNOSTICS},
              open(os.path.join(out, "parity_diagnostics.json"), "w"), indent=1)
