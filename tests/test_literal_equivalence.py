"""The contract oracle replays the paper's method: statistical equivalence with a literal replay.

The contract oracle (oracle/oracle.cpp) follows the numerics contract so that the
CUDA path can match it bit for bit: Philox4x32-10 with a table-driven log and a shared-block
Box-Muller (NC-3), Alg. 2 on shifted running sums with one shared reciprocal (NC-6).  None of
that is in the paper.  These tests pin the contract oracle to a second replay written as the
paper prints it (oracle/literal.cpp): the C++ standard library's normals and integers, and
Alg. 2 recomputed from the cost history on every Observe, σ̂² = (1/σ̂0² + |C_b|/σ̃²)⁻¹ and
μ̂ = σ̂²(μ̂0/σ̂0² + Sum(C_b)/σ̃²), θ̂_b ~ N(μ̂_b, σ̂_b²) (Alg. 1).

Two replays with different random streams cannot agree trial by trial; they must agree in
distribution.  For each workload both replay the same trials independently and we require:
  * two-sample KS on the per-trial total cost, energy and time: p > 1e-3;
  * chi-square (contingency) on the final batch size: p > 1e-3;
  * per-recurrence mean cost: |z_t| < 4.5 for every t (a family-wise false-alarm rate of
    ~1.4e-3 over 200 recurrences; a per-t 4σ bound would false-alarm in ~1.3% of seeds);
  * per-arm share of all decisions (one share vector per trial, so trials are the
    independent units): |z| < 4.5.
A negative control shows the comparison has the power to see a wrong sampler: the literal
replay with σ̂_b doubled (or halved) in the draw must fail it.

Any future revision of the numerics contract must keep this file green.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2208_06102_b200 import synth

THREADS = max(1, min(16, os.cpu_count() or 1))
N_TRIALS = 10_000
ALPHA = 1e-3
Z_MAX = 4.5


@pytest.fixture(scope="module")
def literal():
    from oracle import literal as L

    L.build()
    return L


def _cases():
    """CFG1 (ResNet-18-like, 8 x 6, R = 50), two CFG2 workloads (R = 200) and the CFG4 drift
    scenario (windowed posterior, N = 10, 200 slices; §6.4)."""
    (c1,) = synth.config("cfg1", trials=N_TRIALS)
    ds2 = synth.make_workload("deepspeech2", 2208)
    sa = synth.make_workload("bert_sa", 2208)
    (c4,) = synth.config("cfg4", trials=N_TRIALS)
    return {
        "cfg1": (c1.workload, c1.cells[0], c1.recurrences),
        "cfg2_deepspeech2": (ds2, synth.cell(seed=2210), 200),
        "cfg2_bert_sa": (sa, synth.cell(seed=2210), 200),
        "cfg4_drift": (c4.workload, c4.cells[0], c4.recurrences),
    }


CASES = _cases()


def _replays(oracle, literal, key, sigma_scale=1.0):
    w, c, R = CASES[key]
    a = oracle.replay(w, c, R, np.arange(N_TRIALS), threads=THREADS, logs=True)
    b = literal.replay(w, dict(c, seed=c["seed"] + 7919), R, N_TRIALS, threads=THREADS,
                       sigma_scale=sigma_scale)
    return w, R, a, b


def _compare(w, R, a, b):
    """p-values / z-scores of every comparison (dict)."""
    from scipy import stats

    res = {}
    for k in ("tot_cost", "tot_energy", "tot_time"):
        res["ks_" + k] = stats.ks_2samp(a[k], b[k]).pvalue
    B = len(w["batch_sizes"])
    ca = np.bincount(a["final_arm"], minlength=B)
    cb = np.bincount(b["final_arm"], minlength=B)
    keep = (ca + cb) >= 10                      # pool sparse categories into one
    table = np.array([np.append(ca[keep], ca[~keep].sum()), np.append(cb[keep], cb[~keep].sum())])
    table = table[:, table.sum(0) > 0]
    res["chi2_final_arm"] = stats.chi2_contingency(table).pvalue if table.shape[1] > 1 else 1.0
    ya, yb = a["cost_log"], b["cost_log"]
    se = np.sqrt(ya.var(0, ddof=1) / len(ya) + yb.var(0, ddof=1) / len(yb))
    d = ya.mean(0) - yb.mean(0)
    res["z_curve"] = float(np.max(np.abs(np.where(se > 0, d / np.where(se > 0, se, 1), 0))))
    arms_a = (a["log"] & 0xFF).astype(np.int64)
    arms_b = b["arm_log"].astype(np.int64)
    sa = np.stack([(arms_a == k).mean(1) for k in range(B)], 1)
    sb = np.stack([(arms_b == k).mean(1) for k in range(B)], 1)
    se = np.sqrt(sa.var(0, ddof=1) / len(sa) + sb.var(0, ddof=1) / len(sb))
    d = sa.mean(0) - sb.mean(0)
    res["z_arm_share"] = float(np.max(np.abs(np.where(se > 0, d / np.where(se > 0, se, 1), 0))))
    return res


def _passes(res):
    return (all(v > ALPHA for k, v in res.items() if k.startswith(("ks_", "chi2_")))
            and res["z_curve"] < Z_MAX and res["z_arm_share"] < Z_MAX)


@pytest.mark.parametrize("key", list(CASES))
def test_contract_replay_is_the_literal_replay_in_distribution(oracle, literal, key):
    """Alg. 1-3 with the contract's sampler and Observe arithmetic (NC-3/NC-6) vs the paper's
    literal Alg. 1-3 with library normals."""
    w, R, a, b = _replays(oracle, literal, key)
    res = _compare(w, R, a, b)
    assert _passes(res), res
    # the two replays are independent streams: they must not be trivially identical
    assert not np.array_equal(a["tot_cost"], b["tot_cost"])


@pytest.mark.parametrize("scale", [2.0, 0.5])
def test_comparison_detects_a_wrong_sampler(oracle, literal, scale):
    """Negative control: θ̂_b drawn with σ̂_b scaled by 2 or 1/2 (a plausible sampler slip: a
    variance used as a standard deviation, a dropped factor) fails the comparison."""
    w, R, a, b = _replays(oracle, literal, "cfg2_deepspeech2", sigma_scale=scale)
    res = _compare(w, R, a, b)
    assert not _passes(res), res
    assert res["ks_tot_cost"] < 1e-6, res


# ------------------------------------------------------------------ Observe, call by call
def _alg2_exact(xs, window, prior_mean, prior_var):
    """Alg. 2 in exact rational arithmetic: σ̃² = Var(C_b) (n−1 divisor, R-Q6),
    σ̂² = (1/σ̂0² + |C_b|/σ̃²)⁻¹, μ̂ = σ̂²(μ̂0/σ̂0² + Sum(C_b)/σ̃²); flat prior: 1/σ̂0² = 0."""
    C = [Fraction(x) for x in (xs[-window:] if window else xs)]
    n = len(C)
    mean = sum(C) / n
    s2 = sum((c - mean) ** 2 for c in C) / (n - 1)
    if s2 == 0:
        return None
    prec0 = Fraction(0) if math.isinf(prior_var) else 1 / Fraction(prior_var)
    var = 1 / (prec0 + n / s2)
    mu = var * (Fraction(prior_mean) * prec0 + sum(C) / s2)
    return float(mu), float(var), float(s2), float(mean)


def _replay_histories(oracle, n_hist=60):
    """Per-arm cost histories taken from contract-oracle replays (costs, stops and spreads
    shaped like the real Observe inputs), plus a few synthetic ones."""
    hists = []
    for name, seed in (("deepspeech2", 3), ("bert_qa", 4), ("generic16", 5)):
        w = synth.make_workload(name, seed)
        o = oracle.replay(w, synth.cell(seed=seed), 150, range(20), logs=True)
        for j in range(20):
            arms = o["log"][j] & 0xFF
            for b in np.unique(arms):
                h = o["cost_log"][j][arms == b]
                if len(h) >= 2:
                    hists.append(h)
    rng = np.random.default_rng(17)
    for _ in range(40):                          # relative spreads from 1e-5 to 0.3
        m = rng.uniform(1e3, 1e7)
        hists.append(rng.normal(m, m * 10 ** rng.uniform(-5, -0.5), size=rng.integers(2, 60)))
    return hists[:: max(1, len(hists) // n_hist)]


@pytest.mark.parametrize("window,prior", [(0, (0.0, math.inf)), (10, (0.0, math.inf)),
                                          (0, (5e5, 1e10))])
def test_observe_matches_alg2_exactly_within_1e12(oracle, literal, window, prior):
    """Every Observe of the contract (NC-6: shifted running sums, one shared reciprocal) gives
    Alg. 2's μ̂ and σ̂² within 1e-12 relative of the exact rational value of the printed formula,
    on every prefix of replay-shaped cost histories.  The literal fp64 formula is checked too."""
    worst_c = worst_l = 0.0
    n_checked = 0
    for h in _replay_histories(oracle):
        for m in range(2, len(h) + 1):
            xs = list(h[:m])
            ex = _alg2_exact(xs, window, *prior)
            if ex is None:                             # zero variance: the floor decides (R-Q7)
                continue
            mu, var, s2, mean = ex
            if s2 < 1e-12 * (1 + mean * mean) * 2:   # the zero-variance floor (R-Q7) decides
                continue
            r = oracle.posterior(xs, window, *prior)
            rl = literal.posterior(xs, window, *prior)
            worst_c = max(worst_c, abs(r["mu"] - mu) / abs(mu), abs(r["var"] - var) / var)
            worst_l = max(worst_l, abs(rl["mu"] - mu) / abs(mu), abs(rl["var"] - var) / var)
            n_checked += 1
    assert n_checked > 300
    print(f"checked {n_checked} Observe calls: contract {worst_c:.2e}, literal {worst_l:.2e}")
    assert worst_c < 1e-12, worst_c
    assert worst_l < 1e-12, worst_l


# ------------------------------------------------------------------ P8: the Thompson argmin
def test_p8_zero_variance_picks_the_smallest_mean(oracle):
    """SPEC S:L261 / Alg. 1 argmin: with σ̂ = 0 every sample is its mean, so the
    arm with mean 3 of {5, 3, 9} is picked at every (trial, recurrence); equal means go to the
    lower index (R-Q17)."""
    for i in range(2000):
        assert oracle.thompson_argmin(7, i, i % 97, [5.0, 3.0, 9.0], [0.0, 0.0, 0.0]) == 1
        assert oracle.thompson_argmin(7, i, 3, [4.0, 2.0, 2.0, 8.0], [0.0] * 4) == 1
        assert oracle.thompson_argmin(7, i, 3, [9.0, 5.0, 3.0, 3.0], [0.0] * 4, arms=[0, 1, 3]) == 3


def test_p8_never_picks_the_far_worse_arm(oracle):
    """N(10, 1) vs N(20, 1): the worse arm wins with probability Φ(−10/√2) ≈ 7.7e-13,
    so in 10^5 draws (trials x recurrences, either arm order) it never does."""
    for i in range(50_000):
        assert oracle.thompson_argmin(11, i, 2 * (i % 500), [10.0, 20.0], [1.0, 1.0]) == 0
        assert oracle.thompson_argmin(11, i, 2 * (i % 500) + 1, [20.0, 10.0], [1.0, 1.0]) == 1


def test_p8_single_arm(oracle):
    """a single arm is always chosen, whatever its posterior."""
    for i in range(500):
        assert oracle.thompson_argmin(3, i, i, [1e9], [1e9]) == 0
        assert oracle.thompson_argmin(3, i, i, [1.0, -5.0, 2.0], [1.0, 1.0, 1.0], arms=[2]) == 2


def test_p8_pick_frequencies(oracle):
    """Alg. 1 picks arm b with probability P(θ̂_b = min): two arms N(0,1) and N(0.5,1) give
    P(first) = Φ(0.5/√2) = 0.6382; three identical arms give 1/3 each (each arm has its own
    normal: a shared z would always tie and pick arm 0); a zero-variance arm at 1 against N(0,1)
    gives P(N(0,1) < 1) = Φ(1) = 0.8413.  Binomial / chi-square at 1e-4."""
    from scipy import stats

    n = 40_000
    picks = np.array([oracle.thompson_argmin(21, i, 5, [0.0, 0.5], [1.0, 1.0]) for i in range(n)])
    p = 0.5 * (1 + math.erf(0.5 / math.sqrt(2) / math.sqrt(2)))
    assert stats.binomtest(int((picks == 0).sum()), n, p).pvalue > 1e-4
    picks = np.array([oracle.thompson_argmin(22, i, 6, [1.0] * 3, [2.0] * 3) for i in range(n)])
    assert stats.chisquare(np.bincount(picks, minlength=3)).pvalue > 1e-4
    picks = np.array([oracle.thompson_argmin(23, i, 7, [1.0, 0.0], [0.0, 1.0]) for i in range(n)])
    p = 0.5 * (1 + math.erf(1 / math.sqrt(2)))
    assert stats.binomtest(int((picks == 1).sum()), n, p).pvalue > 1e-4
