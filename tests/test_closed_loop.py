"""NEXT-2 closed-loop harness (scripts/closed_loop.py), host logic on CPU: the literal
Alg. 1 oracle admits, and a linear step-time model (App. C.1, cascade-aware context)
stands in for the B200 step.  Checks the metric definitions (App. D) and the
directional behaviour the paper reports: Eager buys throughput and loses attainment under
load (the throughput trap, Sec. 2.2), TAPER keeps the SLO while admitting more than Off."""
import importlib.util
import os
import sys

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location("closed_loop", os.path.join(ROOT, "scripts", "closed_loop.py"))
CL = importlib.util.module_from_spec(_spec)
sys.modules["closed_loop"] = CL  # dataclasses resolve their module by name
_spec.loader.exec_module(CL)

# a B200-like predictor with the synthetic non-attention part (scripts/closed_loop.py)
MODEL = (0.707 + CL.REST[0], 0.0107 + CL.REST[1], 4.07e-5)


def _drivers():
    def admit_fn(b, policy, rho, model):
        kind, cap = CL.POLICY_ARGS[policy]
        o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                         model, kind, cap, rho, ctx="per_request")
        assert (o.req_width >= 1).all()  # every active request advances (L128)
        return o.slot_admitted.astype(bool), o.T_S

    def step_fn(b, adm):
        return MODEL[0] + MODEL[1] * int(adm.sum()) + MODEL[2] * CL.context_per_request(b, adm)

    return admit_fn, step_fn


@pytest.fixture(scope="module")
def results():
    admit_fn, step_fn = _drivers()
    return {p: CL.run(p, admit_fn, step_fn, 900, seed=1, model=MODEL) for p in ("off", "eager", "taper")}


def test_metric_definitions(results):
    for r in results.values():
        assert 0.0 <= r["attainment"] <= 1.0
        assert r["goodput_tok_s"] <= r["throughput_tok_s"] + 1e-9
        assert r["finished"] > 50


def test_throughput_trap_directional(results):
    off, eager, taper = results["off"], results["eager"], results["taper"]
    assert off["admission_rate"] == 0.0 and eager["admission_rate"] == 1.0
    assert 0.0 < taper["admission_rate"] < 1.0
    assert eager["attainment"] < taper["attainment"]
    assert taper["attainment"] >= 0.9
    assert taper["goodput_tok_s"] > eager["goodput_tok_s"]


def test_rolling_refit_recovers_the_step_model():
    """App. C.2 (L337): OLS on the last 200 observed steps recovers the true (a, b, c)
    from a biased starting model (exact linear clock, so the fit is exact)."""
    admit_fn, step_fn = _drivers()
    r = CL.run("taper", admit_fn, step_fn, 400, seed=2, model=(5.0, 0.05, 1e-5), refit=True)
    np.testing.assert_allclose(r["final_model"], MODEL, rtol=1e-6)
    assert abs(r["predictor_rel_err_median"]) < 1e-6


def test_table1_ablations_run_and_behave():
    """Table 1 ablation switches: without the slack budget the planner
    admits every ready branch (= Eager's admission); without per-step replanning a request's
    width is held for its whole phase; a constant predictor prices every sequence alike."""
    admit_fn, step_fn = _drivers()
    res = {a: CL.run("taper", admit_fn, step_fn, 500, seed=3, model=MODEL, ablation=a)
           for a in CL.ABLATIONS}
    eager = CL.run("eager", admit_fn, step_fn, 500, seed=3, model=MODEL)
    assert res["noslack"]["admission_rate"] == 1.0
    assert res["noslack"]["throughput_tok_s"] == pytest.approx(eager["throughput_tok_s"])
    for r in res.values():
        assert 0.0 <= r["attainment"] <= 1.0 and r["finished"] > 20
    taper = CL.run("taper", admit_fn, step_fn, 500, seed=3, model=MODEL)
    # a phase's first step admits its fresh branches (Lloc = 1, the cheapest candidates), and
    # without replanning that width is held while the load builds: the controller cannot
    # contract mid-phase (the paper's failure mode at load transitions)
    assert res["noreplan"]["admission_rate"] >= taper["admission_rate"]
    assert res["noreplan"]["attainment"] <= taper["attainment"]
    assert 0.0 < res["const"]["admission_rate"] < 1.0


def test_canonical_first_is_cap_per_request():
    import synth
    b = synth.make_batch([100, 50], [3, 2], [7, 2, 9, 4, 4], 1e3, 0.0)
    m = CL.canonical_first(b, 0, 2)
    assert m.tolist() == [True, True, False, False, False]  # local 7, 2, 9 -> slots 1, 0
    m = CL.canonical_first(b, 1, 1)
    assert m.tolist() == [False, False, False, True, False]  # tie 4, 4 -> lower slot
