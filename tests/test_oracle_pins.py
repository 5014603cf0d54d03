"""Pins for the CPU oracle: what the paper, SPEC's worked examples and mathematics fix.

Each test names the passage it pins (P:L = PAPER.md line, S:L = SPEC.md line) and
is chosen so that a plausible slip in the oracle (a dropped term, a wrong sign or
index, a transposed operand, a wrong tie-break) fails at least one of them.
"""
import json
import math
import os
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

from paper_2208_06102_b200 import synth
from tests.conftest import GOLDEN


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def trace(batch_sizes, b0, power_limits, max_power, avg_power, throughput, pool,
          max_epochs=30, charge_profiling=0):
    return {"batch_sizes": np.array(batch_sizes, np.int32), "b0": b0,
            "power_limits": np.array(power_limits, float), "max_power": float(max_power),
            "max_epochs": max_epochs, "charge_profiling": charge_profiling,
            "avg_power": np.array(avg_power, float), "throughput": np.array(throughput, float),
            "pool": np.array(pool, np.int32)}


# ------------------------------------------------------------------ RNG
def test_philox_known_answers(oracle):
    """Random123 KAT vectors for Philox4x32-10 (tests/golden/philox_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        assert oracle.philox(v[0:4], v[4:6]) == v[6:10]
        n += 1
    assert n == 3


def test_uniform_boundaries(oracle):
    """NC-3: u1 = (a + 1) 2^-32 in (0,1], v = b 2^-32 in [0,1); extreme words map exactly."""
    assert oracle.uniforms(0, 0) == (2.0**-32, 0.0)
    u, v = oracle.uniforms(2**32 - 1, 2**32 - 1)
    assert u == 1.0 and v == 1.0 - 2.0**-32
    u, v = oracle.uniforms((1 << 31) - 1, 1 << 31)
    assert u == 0.5 and v == 0.5


def _ulp_err(got, ref: Decimal):
    r = float(ref)
    return abs(Decimal(got) - ref) / Decimal(math.ulp(r))


def test_zlog_accuracy(oracle):
    """NC-3: zlog_fdlibm (the table generator) is fdlibm's log, < 1 ulp; the sampler's
    table-driven zlog is < 2 ulp; both checked against a 40-digit decimal ln, and zlog is
    never positive on (0, 1] (so sqrt(-2 log u1) is real)."""
    getcontext().prec = 40
    rng = np.random.default_rng(7)
    xs = [1.0, 0.5, 0.25, 2.0**-52, 2.0**-52 * 3, 0.7071067811865476, 0.7071067811865475,
          1.0 - 2.0**-52, 0.9999, 0.75, 0.1, 1e-10]
    for w in rng.integers(0, 2**32, size=3000, dtype=np.int64):
        xs.append(oracle.uniforms(int(w), 0)[0])
    xs += list(rng.random(1000) + 1e-300)
    worst = worst_fd = 0
    for x in xs:
        got = oracle.zlog(x)
        if x == 1.0:
            assert got == 0.0 and oracle.zlog_fdlibm(x) == 0.0
            continue
        ref = Decimal(x).ln()
        worst = max(worst, _ulp_err(got, ref))
        worst_fd = max(worst_fd, _ulp_err(oracle.zlog_fdlibm(x), ref))
        if x <= 1.0:
            assert got <= 0.0
    assert worst_fd <= 1, worst_fd
    assert worst <= 2, worst


def _sin_cos_pi(m):
    """sin, cos of pi*m/2^51 by exact rational reduction and a 50-digit Taylor series."""
    getcontext().prec = 50
    x = Fraction(m, 2**51)
    PI = Decimal("3.14159265358979323846264338327950288419716939937510582097494")
    a = Decimal(x.numerator) / Decimal(x.denominator) * PI
    s, c, term_s, term_c = Decimal(0), Decimal(0), a, Decimal(1)
    for k in range(60):
        s += term_s
        c += term_c
        term_s = -term_s * a * a / ((2 * k + 2) * (2 * k + 3))
        term_c = -term_c * a * a / ((2 * k + 1) * (2 * k + 2))
    return s, c


def test_zsincospi_within_one_ulp(oracle):
    """Contract sin/cos(2*pi*v) vs an exact-reduction Taylor reference (<= 1 ulp)."""
    rng = np.random.default_rng(11)
    ms = [0, 1, 2**49, 2**50, 2**50 + 1, 2**51, 3 * 2**49, 2**52 - 1, 2**51 - 1, 2**49 - 1,
          3 * 2**50, 7 * 2**49]
    ms += [int(v) for v in rng.integers(0, 2**52, size=1500, dtype=np.int64)]
    worst = 0
    for m in ms:
        s, c = oracle.zsincospi(m)
        rs, rc = _sin_cos_pi(m)
        for got, ref in ((s, rs), (c, rc)):
            if abs(ref) < Decimal("1e-40"):        # exact zeros of sin/cos
                assert got == 0.0
                continue
            worst = max(worst, _ulp_err(got, ref))
    assert worst <= 1, worst


def test_normals_are_standard_normal(oracle):
    """Q21: the Box-Muller pair is N(0,1) x N(0,1): mean, variance, KS, independence."""
    from scipy import stats

    z = np.array([oracle.normal_pair(1234, i, 3, 1) for i in range(60000)])
    n = z.size
    flat = z.ravel()
    assert abs(flat.mean()) < 5 / math.sqrt(n)
    assert abs(flat.var() - 1) < 5 * math.sqrt(2 / n)
    assert stats.kstest(flat, "norm").pvalue > 1e-4
    assert abs(np.corrcoef(z[:, 0], z[:, 1])[0, 1]) < 5 / math.sqrt(len(z))
    # the pair is keyed by (trial, recurrence, arm pair): changing any key changes it, and the
    # two pairs that share a Philox block are independent
    a = oracle.normal_pair(1234, 5, 3, 1)
    assert a != oracle.normal_pair(1234, 6, 3, 1)
    assert a != oracle.normal_pair(1234, 5, 4, 1)
    assert a != oracle.normal_pair(1234, 5, 3, 2)
    assert a != oracle.normal_pair(1235, 5, 3, 1)
    zz = np.array([oracle.normal_pair(99, i, 2, 0) + oracle.normal_pair(99, i, 2, 1) for i in range(20000)])
    c = np.corrcoef(zz.T)
    assert np.all(np.abs(c[np.triu_indices(4, 1)]) < 5 / math.sqrt(len(zz)))


def test_replica_draw_is_uniform(oracle):
    """Q15: replicas resampled uniformly with replacement (chi-square)."""
    from scipy import stats

    K = 4
    r = np.array([oracle.replica(99, i, 7, K) for i in range(40000)])
    assert r.min() >= 0 and r.max() < K
    counts = np.bincount(r, minlength=K)
    assert stats.chisquare(counts).pvalue > 1e-4


# ------------------------------------------------------------------ step 1 (Eq. 7)
def _one_arm(ex, eta):
    w = trace([32], 0, ex["power_limits"], ex["max_power"], [ex["avg_power"]], [ex["throughput"]],
              [[[10]]])
    return w, synth.cell(eta=eta)


def test_plo_spec_worked_example(oracle):
    """Eq. 7 on SPEC's table; p* = 150 W at eta = .5, 250 W at 0, 100 W at 1."""
    ex = load("spec_plo_example.json")
    for case in ex["cases"]:
        w, c = _one_arm(ex, case["eta"])
        st = oracle.step1(w, c)
        assert st["pstar"][0] == case["pstar"]
        if "costs" in case:
            assert st["c1"][0] == pytest.approx(case["costs"][case["pstar"]], rel=1e-15)
        if "c1" in case:
            assert st["c1"][0] == pytest.approx(case["c1"], rel=1e-15)


def test_plo_matches_brute_force(oracle):
    """S:L624 / P14: per-arm p* equals the exhaustive min over (b,p) restricted to {b}."""
    rng = np.random.default_rng(5)
    for it in range(50):
        B, P = int(rng.integers(1, 9)), int(rng.integers(1, 7))
        pl = np.sort(rng.choice(np.arange(100, 260, 10), size=P, replace=False)).astype(float)
        A = rng.uniform(60, pl.max(), size=(B, P))
        Th = rng.uniform(0.01, 0.1, size=(B, P))
        if it % 5 == 0:            # force exact ties: duplicate a column
            A[:, -1] = A[:, 0]
            Th[:, -1] = Th[:, 0]
        eta = float(rng.choice([0.0, 0.25, 0.5, 1.0]))
        MP = float(pl.max() + rng.choice([0, 30]))
        w = trace(list(range(8, 8 * B + 1, 8)), 0, pl, MP, A, Th, np.full((1, B, 1), 5))
        st = oracle.step1(w, synth.cell(eta=eta))
        for b in range(B):
            costs = [Fraction(eta) * Fraction(A[b, p]) + (1 - Fraction(eta)) * Fraction(MP) for p in range(P)]
            costs = [cst / Fraction(Th[b, p]) for p, cst in enumerate(costs)]
            m = min(costs)
            # the contract evaluates in fp64: the chosen p must be exactly optimal or
            # within fp64 rounding of the exact optimum, and ties go to the smaller p
            chosen = st["pstar"][b]
            assert float(costs[chosen]) == pytest.approx(float(m), rel=1e-14)
            exact_ties = [p for p in range(P) if costs[p] == m]
            if len(exact_ties) > 1 and chosen in exact_ties:
                assert chosen == exact_ties[0]


def test_eta_endpoints(oracle):
    """eta = 1 makes cost == ETA (bitwise), eta = 0 makes cost == MAXPOWER*TTA."""
    w = synth.make_workload("deepspeech2", 3)
    st1 = oracle.step1(w, synth.cell(eta=1.0))
    assert np.array_equal(st1["c1"], st1["e1"])
    A, Th = w["avg_power"], w["throughput"]
    assert np.array_equal(st1["pstar"], np.argmin(A / Th, axis=1))
    st0 = oracle.step1(w, synth.cell(eta=0.0))
    np.testing.assert_allclose(st0["c1"], w["max_power"] * st0["t1"], rtol=1e-15)
    assert np.array_equal(st0["pstar"], np.argmax(Th, axis=1))


def test_profiling_epoch_example(oracle):
    """P={100,200}, Th={.01,.02}, A={100,200} -> 75 s and 10000 J; P=1 -> a regular epoch."""
    w = trace([32], 0, [100, 200], 200, [[100, 200]], [[0.01, 0.02]], [[[5]]])
    st = oracle.step1(w, synth.cell(eta=0.5))
    assert st["t_prof"][0] == 75.0 and st["e_prof"][0] == 10000.0
    assert st["c_prof"][0] == 0.5 * 10000.0 + 0.5 * 200 * 75.0
    w = trace([32], 0, [150], 200, [[120]], [[0.013]], [[[5]]])
    st = oracle.step1(w, synth.cell(eta=0.3))
    assert st["t_prof"][0] == st["t1"][0] and st["e_prof"][0] == st["e1"][0]
    assert st["c_prof"][0] == pytest.approx(st["c1"][0], rel=1e-15)


def test_known_optimum_and_pareto(oracle):
    """P:L822 / P15: opt(s) is the exhaustive min over (b,p) of Ebar(b)*c(b,p), and for
    eta in (0,1) it lies on the (TTA, ETA) Pareto front of the grid."""
    for name in synth.SIX:
        w = synth.make_workload(name, 9)
        A, Th, pool = w["avg_power"], w["throughput"], w["pool"][0]
        ebar = np.array([row[row > 0].mean() if (row > 0).any() else np.nan for row in pool])
        tta = ebar[:, None] / Th
        eta_ = ebar[:, None] * A / Th
        for eta in (0.2, 0.5, 0.8):
            st = oracle.step1(w, synth.cell(eta=eta))
            cost = eta * eta_ + (1 - eta) * w["max_power"] * tta
            b, p = np.unravel_index(np.nanargmin(cost), cost.shape)
            assert st["opt_arm"][0] == b
            assert st["opt"][0] == pytest.approx(np.nanmin(cost), rel=1e-12)
            dominated = (tta <= tta[b, p]) & (eta_ <= eta_[b, p]) & ((tta < tta[b, p]) | (eta_ < eta_[b, p]))
            assert not np.any(dominated[~np.isnan(tta)])


# ------------------------------------------------------------------ Observe (Alg. 2)
def test_posterior_worked_examples(oracle):
    """{10,14} -> 8/4/12; prior (0,100); window 3 over 5,50,52,54."""
    for case in load("posterior_examples.json")["cases"]:
        pv = math.inf if case["prior_var"] == "inf" else case["prior_var"]
        r = oracle.posterior(case["xs"], case["window"], case["prior_mean"], pv)
        for k in ("s2", "var", "mu"):
            assert r[k] == pytest.approx(case[k], rel=1e-12, abs=1e-12)
        assert r["sigma"] == pytest.approx(math.sqrt(case["var"]), rel=1e-12)


def test_posterior_closed_form(oracle):
    """P4: flat prior gives mean and s^2/n (numpy mean / var(ddof=1)); a proper prior gives
    the conjugate normal posterior; a window keeps only the last N observations."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = int(rng.integers(2, 40))
        xs = rng.normal(rng.uniform(1e3, 1e6), rng.uniform(1, 1e4), size=n)
        r = oracle.posterior(xs)
        assert r["mu"] == pytest.approx(xs.mean(), rel=1e-9)
        assert r["var"] == pytest.approx(xs.var(ddof=1) / n, rel=1e-9)
        N = int(rng.integers(2, 12))
        r = oracle.posterior(xs, window=N)
        tail = xs[-N:]
        if len(tail) >= 2:
            assert r["mu"] == pytest.approx(tail.mean(), rel=1e-9)
            assert r["s2"] == pytest.approx(tail.var(ddof=1), rel=1e-7)
        m0, v0 = rng.uniform(0, 1e6), rng.uniform(1, 1e8)
        r = oracle.posterior(xs, 0, m0, v0)
        s2 = xs.var(ddof=1)
        var = 1.0 / (1.0 / v0 + n / s2)
        assert r["var"] == pytest.approx(var, rel=1e-9)
        assert r["mu"] == pytest.approx(var * (m0 / v0 + xs.sum() / s2), rel=1e-9)
    assert oracle.posterior([5.0]) is None       # one observation: no variance yet (R-Q6)
    r = oracle.posterior([7.0, 7.0, 7.0])          # zero variance: floored (R-Q7)
    assert r["mu"] == 7.0 and 0 < r["sigma"] < 1e-4


# ------------------------------------------------------------------ whole-trial pins
def _micro(key):
    g = load("micro_traces.json")
    t = g["trace"]
    w = trace(t["batch_sizes"], t["b0"], t["power_limits"], t["max_power"], t["avg_power"],
              t["throughput"], t["pool"], t["max_epochs"], g[key]["charge_profiling"])
    return g, w


def test_micro_trace_step1(oracle):
    g, w = _micro("W1")
    st = oracle.step1(w, synth.cell(eta=1.0))
    d = g["derived"]
    assert list(st["pstar"]) == d["pstar"]
    np.testing.assert_allclose(st["c1"], d["c1"], rtol=1e-15)
    np.testing.assert_allclose(st["c_prof"], d["c_prof"], rtol=1e-15)
    np.testing.assert_allclose(st["t_prof"], d["t_prof"], rtol=1e-15)
    assert st["opt"][0] == d["opt"] and st["opt_arm"][0] == d["opt_arm"]


@pytest.mark.parametrize("key", ["W1", "W2"])
def test_micro_traces(oracle, key):
    """W1 / W2: hand-computed decisions, charges, stops and regret."""
    g, w = _micro(key)
    exp = g[key]
    for seed in (1, 2, 3):
        o = oracle.replay(w, synth.cell(eta=1.0, beta=2.0, seed=seed), 8, [0, 1, 2], logs=True)
        for j in range(3):
            log = o["log"][j]
            assert [int(x & 0xFF) for x in log] == exp["arms"]
            assert [int(x >> 8 & 0xFF) for x in log] == [0] * 8
            flags = [int(x >> 16) for x in log]
            assert [f & 1 for f in flags] == exp["stopped"]
            assert [(f >> 3) & 1 for f in flags] == exp["ts"]
            if "profiled" in exp:
                assert [(f >> 2) & 1 for f in flags] == exp["profiled"]
            np.testing.assert_allclose(o["cost_log"][j], exp["costs"], rtol=1e-13)
            assert o["tot_cost"][j] == pytest.approx(exp["total_cost"], rel=1e-13)
        if "pseudo_regret" in exp:
            np.testing.assert_allclose(o["curves"][:, 3] / 3, exp["pseudo_regret"], atol=1e-9)
            t_stop = exp["stopped"].index(1)
            assert o["time_log"][0][t_stop] == pytest.approx(exp["stop_time"], rel=1e-13)
            assert o["energy_log"][0][t_stop] == pytest.approx(exp["stop_energy"], rel=1e-13)


def test_pruning_walk(oracle):
    """P10 / S:L333-334 / Alg. 3: B={8,16,32,64,128}, b0=32; 8 and 128 never converge.
    Round 1 visits 32, 16, 8 (fail), 64, 128 (fail); round 2 starts at the cheapest
    survivor (64) and walks down 32, 16; then Thompson sampling over {16,32,64}."""
    A = [[100, 100]] * 5
    Th = [[1, 1], [1, 1], [1, 1], [2, 2], [1, 1]]
    pool = [[[0], [10], [10], [10], [0]]]
    w = trace([8, 16, 32, 64, 128], 2, [100, 200], 200, A, Th, pool, max_epochs=20)
    o = oracle.replay(w, synth.cell(eta=1.0, beta=math.inf), 40, range(20), logs=True)
    for log in o["log"]:
        arms = [int(x & 0xFF) for x in log]
        assert arms[:8] == [2, 1, 0, 3, 4, 3, 2, 1]
        assert set(arms[8:]) <= {1, 2, 3}
        assert [int(x >> 19) & 1 for x in log[:8]] == [0] * 8
        assert all(int(x >> 19) & 1 for x in log[8:])
        conv = [int(x >> 17) & 1 for x in log[:5]]
        assert conv == [1, 1, 0, 1, 0]


def test_single_arm_closed_form(oracle):
    """P:L1123-1126 / P11: with B = {b0} Zeus only tunes p; K = 1 gives a closed form."""
    w = trace([64], 0, [100, 150, 200], 250, [[90, 120, 150]], [[0.01, 0.013, 0.014]], [[[7]]],
              charge_profiling=1)
    cel = synth.cell(eta=0.4, beta=2.0)
    st = oracle.step1(w, cel)
    R = 25
    o = oracle.replay(w, cel, R, range(10), logs=True)
    assert np.all((o["log"] & 0xFF) == 0)
    E, c1, cp = 7, st["c1"][0], st["c_prof"][0]
    np.testing.assert_allclose(o["tot_cost"], cp + (E - 1) * c1 + (R - 1) * E * c1, rtol=1e-13)
    assert np.all(o["n_stop"] == 0)


def test_early_stop_never_overcharges(oracle):
    """P:L559 / P9: every charge is <= beta * (min cost of earlier converged runs), exactly;
    a stopped run is charged exactly the threshold and counts as not converged."""
    for name, beta in (("deepspeech2", 2.0), ("bert_sa", 1.5), ("resnet18", 3.0)):
        w = synth.make_workload(name, 4)
        cel = synth.cell(beta=beta, seed=8)
        o = oracle.replay(w, cel, 120, range(40), logs=True)
        for j in range(40):
            best = math.inf
            for t in range(120):
                f = int(o["log"][j, t]) >> 16
                C = o["cost_log"][j, t]
                thr = beta * best
                assert C <= thr
                if f & 1:
                    assert C == thr and not (f & 2)
                if f & 2:
                    best = min(best, C)


def test_cost_identity_every_decision(oracle):
    """S:L46 / Eq. 2: C = eta*ETA + (1-eta)*MAXPOWER*TTA for every charged run, stopped or not."""
    for name, eta in (("resnet18", 0.5), ("neumf", 0.0), ("bert_qa", 1.0), ("shufflenet_v2", 0.3)):
        w = synth.make_workload(name, 2)
        o = oracle.replay(w, synth.cell(eta=eta, beta=1.5, seed=3), 60, range(30), logs=True)
        rhs = eta * o["energy_log"] + (1 - eta) * w["max_power"] * o["time_log"]
        np.testing.assert_allclose(o["cost_log"], rhs, rtol=1e-12)


def test_pseudo_regret_nonnegative_and_plateaus(oracle):
    """Eqs. 8-9 / P13: per-decision pseudo-regret >= 0; cumulative is non-decreasing."""
    for name in synth.SIX:
        w = synth.make_workload(name, 1)
        st = oracle.step1(w, synth.cell())
        assert np.all(st["regret"] >= 0)
        o = oracle.replay(w, synth.cell(seed=4), 150, range(50))
        assert np.all(o["curves"][:, 3] >= 0)
        assert np.all(np.diff(np.cumsum(o["curves"][:, 3])) >= 0)


def test_thompson_sampling_converges(oracle):
    """Directional (P17): on a stationary trace late choices are near-optimal
    (pseudo-regret per decision a few % of the optimum and far below the pruning phase)."""
    for name, seed in (("generic16", 1), ("resnet18", 2), ("deepspeech2", 3)):
        w = synth.make_workload(name, seed)
        opt = oracle.step1(w, synth.cell())["opt"][0]
        o = oracle.replay(w, synth.cell(seed=6), 300, range(200))
        late = o["curves"][-50:]
        assert late[:, 6].sum() == late.shape[0] * 200          # all trials in TS by then
        assert late[:, 3].mean() / 200 < 0.05 * opt
        assert late[:, 3].mean() < 0.2 * o["curves"][:20, 3].mean()


def test_determinism_and_shard_independence(oracle):
    """P16: same seed -> bitwise same; any split of the trial range gives the same per-trial
    results (counter-based RNG keyed by the global trial index); constant slices == stationary."""
    w = synth.make_workload("bert_sa", 5)
    cel = synth.cell(window=10, seed=77)
    a = oracle.replay(w, cel, 80, range(64))
    b = oracle.replay(w, cel, 80, range(64), threads=4)
    c1 = oracle.replay(w, cel, 80, range(0, 23))
    c2 = oracle.replay(w, cel, 80, range(23, 64))
    for k in ("digest", "tot_cost", "tot_energy", "tot_time", "n_stop", "final_arm"):
        assert np.array_equal(a[k], b[k])
        assert np.array_equal(a[k], np.concatenate([c1[k], c2[k]]))
    np.testing.assert_allclose(a["curves"], c1["curves"] + c2["curves"], rtol=1e-12)
    w4 = dict(w)
    w4["pool"] = np.repeat(w["pool"], 4, axis=0)
    d = oracle.replay(w4, cel, 80, range(64))
    assert np.array_equal(a["digest"], d["digest"]) and np.array_equal(a["tot_cost"], d["tot_cost"])


def test_validation_lists_every_violation(oracle):
    """validate returns every violated invariant, not just the first."""
    w = synth.make_workload("bert_qa", 0)
    w = dict(w)
    w["b0"] = 17
    w["max_power"] = 10.0
    rc, msg = oracle.validate(w, synth.cell(eta=1.5, beta=1.0, window=1))
    assert rc == 1
    for frag in ("default batch size", "max power", "eta", "beta", "window"):
        assert frag in msg, (frag, msg)
    w2 = synth.make_workload("bert_qa", 0)
    w2 = dict(w2)
    w2["pool"] = np.zeros_like(w2["pool"])
    rc, msg = oracle.validate(w2, synth.cell())
    assert rc == 1 and "no converged replica" in msg
    assert oracle.validate(synth.make_workload("bert_qa", 0), synth.cell())[0] == 0


# ------------------------------------------------------------------ §6.1 baselines
def test_default_baseline_closed_form(oracle):
    """P:L787 Default = (b0, MAXPOWER) every recurrence, no profiling, no early stop:
    each charge is E_run * c(b0, max p), the cost identity holds, and nothing is pruned."""
    w = synth.make_workload("resnet50", 3)
    cel = synth.cell(eta=0.3, beta=1.5, seed=4, policy="default")
    R = 40
    o = oracle.replay(w, cel, R, range(25), logs=True)
    P = len(w["power_limits"])
    assert np.all((o["log"] & 0xFF) == w["b0"]) and np.all(((o["log"] >> 8) & 0xFF) == P - 1)
    A, Th = w["avg_power"][w["b0"], -1], w["throughput"][w["b0"], -1]
    c = (0.3 * A + 0.7 * w["max_power"]) / Th
    E = w["pool"][0, w["b0"]]
    assert set(np.round(o["cost_log"].ravel() / c, 9)) <= set(E.astype(float))
    np.testing.assert_allclose(o["cost_log"], 0.3 * o["energy_log"] + 0.7 * w["max_power"] * o["time_log"],
                               rtol=1e-12)
    assert np.all(o["n_stop"] == 0) and o["curves"][:, 6].sum() == 0


def test_grid_search_enumeration_and_pruning(oracle):
    """one (b, p) per recurrence, b then p ascending, a failed run
    prunes the rest of its batch size, then the cheapest converged configuration is exploited."""
    A = [[100, 100]] * 5
    Th = [[1, 1], [1, 1], [1, 1], [2, 2], [1, 1]]
    pool = [[[0], [10], [10], [10], [0]]]
    w = trace([8, 16, 32, 64, 128], 2, [100, 200], 200, A, Th, pool, max_epochs=20)
    o = oracle.replay(w, synth.cell(eta=1.0, policy="grid_search"), 20, range(3), logs=True)
    for log in o["log"]:
        bp = [(int(x & 0xFF), int(x >> 8 & 0xFF)) for x in log]
        assert bp[:8] == [(0, 0), (1, 0), (1, 1), (2, 0), (2, 1), (3, 0), (3, 1), (4, 0)]
        assert bp[8:] == [(3, 0)] * 12          # cheapest (c = 50) first found at p index 0
    np.testing.assert_allclose(o["cost_log"][0, :8], [20 * 100, 1000, 1000, 1000, 1000, 500, 500, 2000])


def test_zeus_beats_baselines_directionally(oracle):
    """S:L627, S:L631 (directional, never parity): on the six synthetic workloads Zeus's
    cumulative pseudo-regret is below Grid Search's, and its last-five-recurrence energy is
    below Default's."""
    wins_gs = wins_def = 0
    for job in synth.config("f1", trials=60):
        res = {c["policy"]: oracle.replay(job.workload, c, job.recurrences, range(60)) for c in job.cells}
        zeus, default, gs = res[0], res[1], res[2]
        wins_gs += zeus["curves"][:, 3].sum() < gs["curves"][:, 3].sum()
        wins_def += zeus["curves"][-5:, 1].sum() < default["curves"][-5:, 1].sum()
    assert wins_gs >= 5 and wins_def >= 5


# ------------------------------------------------------------------ Pareto front
def test_pareto_spec_example(oracle):
    """{(10 s, 100 J), (12 s, 90 J), (11 s, 120 J)} -> {(10,100), (12,90)}; expressed
    as three batch sizes at one power limit with Ebar = 1 (TTA = 1/Th, ETA = A/Th)."""
    Th = [[0.1], [1 / 12], [1 / 11]]
    A = [[10.0], [90 / 12], [120 / 11]]
    w = trace([8, 16, 32], 0, [100], 100, A, Th, [[[1], [1], [1]]])
    assert oracle.pareto(w).ravel().tolist() == [1, 1, 0]


def test_pareto_brute_force_and_scalarisation(oracle):
    """Definition by exhaustive dominance in exact rationals; the eta-optimal configuration of
    every eta in (0,1) and both endpoints (min TTA, min ETA) are on the front."""
    for name in synth.SIX:
        w = synth.make_workload(name, 11)
        m = oracle.pareto(w)
        pool = w["pool"][0]
        B, P = m.shape
        pts = {}
        for b in range(B):
            conv = pool[b][pool[b] > 0]
            if len(conv) == 0:
                continue
            eb = Fraction(int(conv.sum()), len(conv))
            for p in range(P):
                pts[(b, p)] = (eb / Fraction(w["throughput"][b, p]),
                               eb * Fraction(w["avg_power"][b, p]) / Fraction(w["throughput"][b, p]))
        for (b, p), (t, e) in pts.items():
            dom = any(t2 <= t and e2 <= e and (t2 < t or e2 < e) for (b2, p2), (t2, e2) in pts.items())
            assert m[b, p] == (0 if dom else 1), (name, b, p)
        assert m[min(pts, key=lambda k: pts[k][0])] == 1 and m[min(pts, key=lambda k: pts[k][1])] == 1
        for eta in (0.1, 0.5, 0.9):
            st = oracle.step1(w, synth.cell(eta=eta))
            b = st["opt_arm"][0]
            assert m[b, st["pstar"][b]] == 1


# ------------------------------------------------------------------ concurrent submissions (f3)
def test_concurrency_sequential_schedule_is_identical(oracle):
    """S:L445 / acceptance 10: an arrival schedule without overlap (every run done
    before the next submission) reproduces the sequential replay bit-exactly."""
    for name, window in (("deepspeech2", 0), ("bert_sa", 10)):
        w = synth.make_workload(name, 2)
        R = 90
        base = synth.cell(seed=12, window=window)
        seq = dict(base, arrivals=np.arange(R) * 1e9)
        a = oracle.replay(w, base, R, range(40), logs=True)
        b = oracle.replay(w, seq, R, range(40), logs=True)
        for k in ("log", "tot_cost", "tot_time", "digest", "n_stop"):
            assert np.array_equal(a[k], b[k]), k


def test_concurrency_pruning_runs_best_known(oracle):
    """during pruning a submission that overlaps the walk's outstanding run takes the
    best-known batch size (b0 before anything converged); the walk resumes with the results
    in completion order (W1 trace: the arm-32 run takes 6 x 4/3 = 8 s)."""
    g = load("micro_traces.json")
    t = g["trace"]
    w = trace(t["batch_sizes"], t["b0"], t["power_limits"], t["max_power"], t["avg_power"],
              t["throughput"], t["pool"], t["max_epochs"], 0)
    arr = np.array([0.0, 0.1, 100, 100.5, 200, 300, 300.2, 400, 500, 600])
    o = oracle.replay(w, synth.cell(eta=1.0, beta=2.0, seed=3, arrivals=arr), len(arr), [0, 1], logs=True)
    arms = [int(x & 0xFF) for x in o["log"][0]]
    # t0 walk: 32; t1 overlaps it: best-known = none -> start 32; t2 walk down: 16 (done at 110);
    # t3 overlaps: best-known = 32 (720); t4 walk up: 64 -> stopped at 2*720
    assert arms[:5] == [1, 1, 0, 1, 2]
    assert int(o["log"][0][4] >> 16) & 1


def test_concurrency_overlap_is_valid_and_deterministic(oracle):
    """Heavy overlap (up to the 8-run cap): decisions stay valid, charges stay under the
    threshold of their submission time, and the replay is deterministic."""
    w = synth.make_workload("resnet50", 3)
    R = 120
    rng = np.random.default_rng(4)
    arr = np.cumsum(rng.exponential(0.25 * 40 / w["throughput"].max(), size=R))
    cel = synth.cell(seed=21, arrivals=arr)
    a = oracle.replay(w, cel, R, range(30), logs=True)
    b = oracle.replay(w, cel, R, range(30), logs=True, threads=3)
    assert np.array_equal(a["digest"], b["digest"])
    np.testing.assert_allclose(a["cost_log"], 0.5 * a["energy_log"] + 0.5 * w["max_power"] * a["time_log"],
                               rtol=1e-12)
    seq = oracle.replay(w, synth.cell(seed=21), R, range(30))
    assert not np.array_equal(a["digest"], seq["digest"])


# ------------------------------------------------------------------ variant readings
def _variant_cell(ablation, **kw):
    c = synth.cell(**kw)
    c["ablation"] = ablation
    return c


@pytest.mark.parametrize("key", ["W1_retry", "W1_epoch"])
def test_micro_trace_variants(oracle, key):
    """R-Q4v / R-Q1v on W1, computed by hand: per-recurrence arms, costs,
    totals, decision and stop counts, and the charged time and energy of epoch-boundary stops."""
    g, w = _micro(key)
    exp = g[key]
    for seed in (1, 2):
        o = oracle.replay(w, _variant_cell(exp["ablation"], eta=1.0, beta=exp["beta"], seed=seed), 8,
                          [0], logs=True)
        log = o["log"][0]
        assert [int(x & 0xFF) for x in log] == exp["arms"]
        assert [int(x >> 16) for x in log] == exp["final_flags"]
        np.testing.assert_allclose(o["cost_log"][0], exp["costs"], rtol=1e-13)
        assert o["tot_cost"][0] == pytest.approx(exp["total_cost"], rel=1e-13)
        assert o["counters"][0] == exp["decisions"] and o["counters"][4] == exp["stops"]
        if "stop_times" in exp:
            ts = [t for t in range(8) if int(log[t] >> 16) & 1]
            np.testing.assert_allclose(o["time_log"][0][ts], exp["stop_times"], rtol=1e-13)
            np.testing.assert_allclose(o["energy_log"][0][ts], exp["stop_energies"], rtol=1e-13)


@pytest.mark.parametrize("ablation", [4, 8, 16, 4 | 8 | 16, 1 | 4, 2 | 8])
def test_variants_act_only_through_the_stop(oracle, ablation):
    """Every variant reading changes what happens after an early stop, or which threshold
    stops a run: with beta = inf (no early stop) each is bit-identical to the base
    replay (same draws: attempt 0 uses the base counters)."""
    w = synth.make_workload("deepspeech2", 5)
    kw = dict(beta=math.inf, seed=13, window=10 if ablation & 16 else 0)
    a = oracle.replay(w, _variant_cell(ablation, **kw), 150, range(40), logs=True)
    b = oracle.replay(w, _variant_cell(ablation & 3, **kw), 150, range(40), logs=True)
    for k in ("log", "tot_cost", "digest", "n_stop"):
        assert np.array_equal(a[k], b[k]), k


def test_windowed_best_full_window_is_the_global_best(oracle):
    """R-Q5v with N >= R recurrences covers every earlier run: identical to the global best."""
    w = synth.make_workload("bert_sa", 2208, slices=40, drift=True)
    R = 40
    a = oracle.replay(w, _variant_cell(16, beta=1.5, seed=5, window=R), R, range(60), logs=True)
    b = oracle.replay(w, _variant_cell(0, beta=1.5, seed=5, window=R), R, range(60), logs=True)
    for k in ("log", "tot_cost", "digest", "n_stop"):
        assert np.array_equal(a[k], b[k]), k


def test_windowed_best_threshold(oracle):
    """R-Q5v from the logs: every run is charged at most beta * min(converged costs of the last
    N recurrences), a stopped run exactly that (continuous truncation), and the window matters
    (some charge exceeds beta * the global best)."""
    w = synth.make_workload("bert_sa", 2208, slices=120, drift=True)
    R, N, beta = 120, 10, 1.5
    o = oracle.replay(w, _variant_cell(16, beta=beta, seed=6, window=N), R, range(80), logs=True)
    above_global = 0
    for j in range(80):
        conv = []
        for t in range(R):
            f = int(o["log"][j, t]) >> 16
            C = o["cost_log"][j, t]
            thr = beta * min([c for u, c in conv if u >= t - N], default=math.inf)
            gthr = beta * min([c for _, c in conv], default=math.inf)
            assert C <= thr
            if f & 1:
                assert C == thr and not (f & 2)
            above_global += C > gthr
            if f & 2:
                conv.append((t, C))
    assert above_global > 0


def test_epoch_boundary_stop(oracle):
    """R-Q1v from the logs: a stopped run ends at the first epoch boundary whose accumulated
    cost exceeds thr = beta * best: C > thr >= C - c1(b) (cost per epoch at p*), and C minus the
    first epoch is a whole number of epochs; runs are never stopped in their last epoch."""
    for name in ("deepspeech2", "bert_qa", "resnet18"):
        w = synth.make_workload(name, 9)
        beta = 1.3
        cel = _variant_cell(8, beta=beta, seed=7)
        st = oracle.step1(w, cel)
        o = oracle.replay(w, cel, 100, range(40), logs=True)
        n_stopped = 0
        for j in range(40):
            best = math.inf
            for t in range(100):
                x = int(o["log"][j, t])
                b, f, C = x & 0xFF, x >> 16, o["cost_log"][j, t]
                thr = beta * best
                if f & 1:
                    n_stopped += 1
                    c1 = st["c1"][b]
                    c0 = st["c_prof"][b] if f & 4 else c1
                    assert C > thr >= C - c1 or (C == c0 and c0 > thr)
                    k = (C - c0) / c1
                    assert abs(k - round(k)) < 1e-9
                if f & 2:
                    best = min(best, C)
        assert n_stopped > 0


def test_retry_recurrences(oracle):
    """R-Q4v: every retry follows a stop (decisions - R <= stops), a recurrence only ends on a
    stop when Thompson sampling has run out of arms, and without any stop the replay is the
    base replay's."""
    w = synth.make_workload("shufflenet_v2", 3)
    R, n = 150, 40
    o = oracle.replay(w, _variant_cell(4, beta=1.3, seed=11), R, range(n), logs=True)
    base = oracle.replay(w, _variant_cell(0, beta=1.3, seed=11), R, range(n), logs=True)
    assert o["counters"][0] > R * n                     # some recurrences retried
    assert o["counters"][0] - R * n <= o["counters"][4]
    for j in range(n):
        for t in range(R):
            f = int(o["log"][j, t]) >> 16
            if f & 1:                                    # ended on a stop: TS with no arm left
                assert f & 8
    same = o["n_stop"] == 0
    assert np.array_equal(o["digest"][same], base["digest"][same])


def test_variant_validation(oracle):
    w = synth.make_workload("bert_qa", 0)
    assert "windowed best needs window" in oracle.validate(w, _variant_cell(16))[1]
    assert "sequential" in oracle.validate(w, _variant_cell(4, arrivals=np.arange(10.0)))[1]
    assert "subset" in oracle.validate(w, _variant_cell(32))[1]
    assert oracle.validate(w, _variant_cell(4 | 8 | 16, window=5))[0] == 0
