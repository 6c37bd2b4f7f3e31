"""NEXT-1 rolling refit behind the C ABI (taper_latency_observe / taper_latency_refit,
include/taper.h): App. C.1 "Fitting" -- OLS of T(S) = a + b n + c L (L316)
over the most recent 200 observed steps.  Host code, no GPU.  Pinned against numpy's
least-squares solver on the same window, exact recovery of a noiseless model, the window
semantics, and the monotonicity guard (L341)."""
import numpy as np
import pytest

from paper_2605_06914_b200 import taper as T


def _fill(w, rng, k, model, noise=0.0):
    obs = []
    for _ in range(k):
        n = float(rng.integers(1, 513))
        L = float(rng.integers(128, 8193)) * n / 4
        t = model[0] + model[1] * n + model[2] * L + noise * rng.standard_normal()
        w.observe(n, L, t)
        obs.append((n, L, t))
    return obs


def test_noiseless_window_recovers_the_model():
    w = T.LatencyWindow()
    true = (0.7, 0.0107, 4.07e-5)
    _fill(w, np.random.default_rng(0), 120, true)
    model, fit = w.refit((12.0, 0.03, 2e-5))
    np.testing.assert_allclose(model, true, rtol=1e-9)
    assert fit["r2"] == pytest.approx(1.0) and fit["mape"] < 1e-12


def test_rolling_window_matches_lstsq_on_the_last_200():
    w = T.LatencyWindow()
    obs = _fill(w, np.random.default_rng(1), 340, (2.0, 0.02, 3e-5), noise=0.3)
    assert w.count == T.TAPER_LATENCY_WINDOW
    last = np.array(obs[-T.TAPER_LATENCY_WINDOW:])
    X = np.c_[np.ones(len(last)), last[:, 0], last[:, 1]]
    ref, *_ = np.linalg.lstsq(X, last[:, 2], rcond=None)
    model, fit = w.refit((12.0, 0.03, 2e-5))
    np.testing.assert_allclose(model, ref, rtol=1e-7)
    pred = X @ ref
    assert fit["mape"] == pytest.approx(np.mean(np.abs(last[:, 2] - pred) / last[:, 2]), rel=1e-9)
    assert fit["rmse_ms"] == pytest.approx(np.sqrt(np.mean((last[:, 2] - pred) ** 2)), rel=1e-9)


def test_non_monotone_or_degenerate_fits_are_refused():
    w = T.LatencyWindow()
    _fill(w, np.random.default_rng(2), 50, (5.0, -0.01, 1e-5))  # b < 0: T not monotone
    with pytest.raises(T.TaperError, match="monotone"):
        w.refit((12.0, 0.03, 2e-5))
    w2 = T.LatencyWindow()
    for L in (1000.0, 2000.0, 3000.0, 4000.0):
        w2.observe(8.0, L, 1.0 + 1e-3 * L)  # n constant: b not identifiable
    with pytest.raises(T.TaperError):
        w2.refit((12.0, 0.03, 2e-5))
    with pytest.raises(T.TaperError):
        T.LatencyWindow().refit((12.0, 0.03, 2e-5))  # empty window
