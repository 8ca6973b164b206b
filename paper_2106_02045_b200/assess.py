"""Accuracy and convergence statistics of fit results (
Table 1, Fig. 8 of PAPER.md:264-284).  Vectorised numpy over result arrays --
post-processing, not on the timed path."""
from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

from .io_formats import STOP_NAMES

NOT_CONVERGED = 3


@dataclass(frozen=True)
class AccuracyStats:
    """errors in units of sigma_true over converged fits."""

    position_median: float
    position_mean: float
    position_std: float
    sigma_median: float
    sigma_mean: float
    sigma_std: float
    n_fits: int
    n_excluded: int

    def as_dict(self):
        return asdict(self)


def accuracy(params: np.ndarray, status: np.ndarray, truth: np.ndarray) -> AccuracyStats:
    """SPEC.md:424-432.  params (n, 3|4), status (n,), truth (n, >=3) [x, y, sigma, ...].
    Position errors |x^-x|/s_true and |y^-y|/s_true pooled; sigma error ||s^|-s_true|/s_true;
    NotConverged fits excluded."""
    params = np.asarray(params, np.float64)
    truth = np.asarray(truth, np.float64)
    if len(params) != len(truth):
        raise ValueError("MismatchedLengths: results and truths must align by index")
    ok = (np.asarray(status) & 7) != NOT_CONVERGED
    p, t = params[ok], truth[ok]
    s_true = t[:, 2]
    pos = np.concatenate([np.abs(p[:, 0] - t[:, 0]) / s_true, np.abs(p[:, 1] - t[:, 1]) / s_true])
    sig = np.abs(np.abs(p[:, 2]) - s_true) / s_true
    f = lambda a, fn: float(fn(a)) if a.size else float("nan")  # noqa: E731
    return AccuracyStats(f(pos, np.median), f(pos, np.mean), f(pos, np.std), f(sig, np.median), f(sig, np.mean),
                         f(sig, np.std), int(ok.sum()), int((~ok).sum()))


def expected_error_ratio(stats: AccuracyStats, n_signal: float) -> float:
    """mean position error / (1/sqrt(N_signal))."""
    if not n_signal > 0:
        raise ValueError("n_signal must be > 0")
    return stats.position_mean * np.sqrt(n_signal)


def iteration_stats(status: np.ndarray, iterations: np.ndarray, max_iterations: int = 20) -> dict:
    """histogram of iterations_used (0..max) and stop-reason tallies
    (no-improvement stops counted separately inside the MinDelta family)."""
    status = np.asarray(status, np.uint8)
    it = np.asarray(iterations, np.int64)
    hist = np.bincount(np.clip(it, 0, max_iterations), minlength=max_iterations + 1)
    stops = np.bincount(status & 7, minlength=5)
    return {
        "histogram": hist.tolist(),
        "mode": int(np.argmax(hist)) if hist.sum() else 0,
        "mean": float(it.mean()) if it.size else float("nan"),
        "stop_reasons": {name: int(stops[k]) for k, name in enumerate(STOP_NAMES)},
        "no_improvement": int(((status & 0x80) != 0).sum()),
        "invalid_input": int(((status & 0x40) != 0).sum()),
        "n_fits": int(status.size),
    }
