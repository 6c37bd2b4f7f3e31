"""The attention kernel resolves each CTA's first work item before its grid dependency,
publishes it as soon as the dependency resolves and validates it beside the first loads by
reloading the work-list words it was built from (include/taper.h ordering contract).  In
practice the words match (the admission finished long before), so the failure path -- the
item runs, its epilogue discards it, and the first claim is resolved again as the next
record -- is rarely taken; a test build forces it in every CTA
(-DTAPER_DBG_FORCE_RERESOLVE=1).  Its outputs must equal the product build's bit for bit,
whatever the item type (row mode, swap mode, local items) or the rank's head count."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RUN = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
import synth
from tests.helpers import Case
rng = np.random.default_rng(31)
b = synth.make_batch([5000, 300, 4097, 65, 2200], [11, 1, 3, 2, 6],
                     rng.integers(1, 700, size=23).tolist(), 1e3, 0.0, rng=rng)
case = Case(b, seed=6)
outs = {}
for heads in ((0, 8), (3, 4)):
    adm, out, lse = case.run_gpu(policy="eager", heads=heads)
    outs[heads] = (adm.slot_admitted.cpu(), out, lse)
torch.save(outs, sys.argv[1])
"""


def _run(lib, path):
    env = dict(os.environ)
    env.pop("TAPER_LIB", None)
    if lib:
        env["TAPER_LIB"] = lib
    subprocess.run([sys.executable, "-c", _RUN, path, ROOT], env=env, check=True, cwd=ROOT, timeout=600)
    return torch.load(path)


def test_forced_reresolve_is_bitwise_identical(tmp_path):
    from paper_2605_06914_b200 import build as B
    lib = os.path.join(ROOT, "build", "libtaper_reresolve.so")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    B.build(force=True, defines=["TAPER_DBG_FORCE_RERESOLVE=1"], out=lib)
    ref = _run(None, str(tmp_path / "product.pt"))
    got = _run(lib, str(tmp_path / "reresolve.pt"))
    for heads in ref:
        m_r, o_r, l_r = ref[heads]
        m_g, o_g, l_g = got[heads]
        assert torch.equal(m_r, m_g)
        adm = m_r[:o_r.shape[0]].bool()
        assert adm.sum() > 0
        assert torch.equal(o_r[adm], o_g[adm]), heads
        assert torch.equal(l_r[adm], l_g[adm]), heads
