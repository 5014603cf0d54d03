"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): every (batch size, power limit) decision and
early-stop event bit-exact -- checked through the per-decision log (CFG1) and
the FNV-1a digest of (b_t, p_t, flags) per trial (all configs) -- and per-trial
totals bit-exact (NC-8: both sides sum in recurrence order); curves summed over
trials within 1e-9 relative of the oracle's fp64 sums.  The GPU curves are exact
fixed-point sums rounded once (include/zeus_sim.h curves_fixed), so between GPU runs
-- any layout, shard split or world size -- they are compared bit for bit.
"""
import math

import numpy as np
import pytest

from paper_2208_06102_b200 import synth

pytestmark = pytest.mark.gpu

CURVE_RTOL = 1e-9


@pytest.fixture(scope="module")
def zs():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2208_06102_b200 import build, zeus_sim

    build.build()
    return zeus_sim


def oracle_threads(oracle):
    return max(1, min(64, oracle.hardware_threads()))


def run_gpu(zs, w, cells, trials, R, shard=(0, -1), log=False, want=None, layout=0, draw=0):
    sim = zs.Simulation(w, cells, trials, R, shard=shard, log=log, layout=layout,
                        draw=draw).load_profile().run()
    keys = ["curves", "curves_fixed", "tot_cost", "tot_energy", "tot_time", "digest", "n_stop", "final_arm",
            "counters", "pstar_index", "c1", "t1", "e1", "c_prof", "t_prof", "e_prof", "opt_cost",
            "opt_arm"] + (["log"] if log else [])
    out = sim.results(want=want or keys)
    out["R"] = sim.R
    out["n"] = sim.shard_n // len(cells)
    out["kernel_launches"] = out.get("kernel_launches", 0)
    sim.close()
    return out


def compare_cell(oracle, g, w, cell, ci, trials_idx, R, n_shard, full_curves=True, logs=False,
                 shard_begin=0):
    """Per-trial bit-exact + curves within 1e-9 for cell ci of a GPU result."""
    o = oracle.replay(w, cell, R, trials_idx, threads=oracle_threads(oracle), logs=logs)
    pos = np.asarray(trials_idx) - shard_begin + ci * n_shard
    for k in ("tot_cost", "tot_energy", "tot_time", "digest", "n_stop", "final_arm"):
        got, exp = g[k][pos], o[k]
        if not np.array_equal(got, exp):
            bad = np.nonzero(got != exp)[0]
            raise AssertionError(f"{k}: {len(bad)} of {len(exp)} trials differ, first trial "
                                 f"{trials_idx[bad[0]]}: gpu {got[bad[0]]!r} oracle {exp[bad[0]]!r}")
    if logs:
        gl = g["log"][pos]
        if not np.array_equal(gl, o["log"]):
            bad = np.argwhere(gl != o["log"])[0]
            raise AssertionError(f"log differs at trial {trials_idx[bad[0]]} t={bad[1]}: "
                                 f"gpu {gl[tuple(bad)]:#x} oracle {o['log'][tuple(bad)]:#x}")
    if full_curves:
        gc, oc = g["curves"][ci], o["curves"]
        np.testing.assert_allclose(gc[:, :4], oc[:, :4], rtol=CURVE_RTOL, atol=0)
        assert np.array_equal(gc[:, 4:], oc[:, 4:])
        if len(g["curves"]) == 1:
            assert np.array_equal(g["counters"][:9], o["counters"])   # events of the method
            assert g["counters"][9] <= g["counters"][2]                  # work the screen left
    return o


def compare_step1(oracle, g, w, cells):
    for ci, c in enumerate(cells):
        st = oracle.step1(w, c)
        assert np.array_equal(g["pstar_index"][ci], st["pstar"])
        for k in ("c1", "t1", "e1", "c_prof", "t_prof", "e_prof"):
            assert np.array_equal(g[k][ci], st[k]), k
        assert np.array_equal(g["opt_cost"][ci], st["opt"])
        assert np.array_equal(g["opt_arm"][ci], st["opt_arm"])


# ------------------------------------------------------------------ configs
def test_cfg1_full_log_bit_exact(zs, oracle):
    (job,) = synth.config("cfg1")
    g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences, log=True)
    compare_step1(oracle, g, job.workload, job.cells)
    compare_cell(oracle, g, job.workload, job.cells[0], 0, np.arange(job.trials), job.recurrences,
                 job.trials, logs=True)


def test_cfg2_six_workloads_all_trials(zs, oracle):
    for job in synth.config("cfg2"):
        g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences)
        compare_step1(oracle, g, job.workload, job.cells)
        compare_cell(oracle, g, job.workload, job.cells[0], 0, np.arange(job.trials),
                     job.recurrences, job.trials)


def test_cfg3_sweep_all_trials(zs, oracle):
    """CFG3 in full (the bench's launch: six workloads x 44 (eta, beta) cells x 10^4 trials x 200
    recurrences, 5.3e8 decisions, the early split): every trial of every cell bit-exact, every
    cell's curves within CURVE_RTOL (counts exact)."""
    for job in synth.config("cfg3"):
        g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences)
        compare_step1(oracle, g, job.workload, job.cells)
        for ci, c in enumerate(job.cells):
            compare_cell(oracle, g, job.workload, c, ci, np.arange(job.trials), job.recurrences,
                         job.trials)


@pytest.mark.parametrize("name", ["cfg4", "cfg4_38"])
def test_cfg4_drift_window(zs, oracle, name):
    (job,) = synth.config(name)
    g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences)
    compare_step1(oracle, g, job.workload, job.cells)
    compare_cell(oracle, g, job.workload, job.cells[0], 0, np.arange(job.trials), job.recurrences,
                 job.trials)


def test_cfg5_full_size_sampled(zs, oracle):
    """BASELINE size (10^7 trials x 1000 recurrences, the bench's launch): every 100th trial
    bit-exact (10^8 decisions); curves checked by properties that hold at any size."""
    (job,) = synth.config("cfg5")
    g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences,
                want=["curves", "tot_cost", "tot_energy", "tot_time", "digest", "n_stop",
                      "final_arm", "counters"])
    idx = np.arange(0, job.trials, 100)
    o = compare_cell(oracle, g, job.workload, job.cells[0], 0, idx, job.recurrences, job.trials,
                     full_curves=False)
    c = g["curves"][0]
    n = job.trials
    assert np.all(c[:, 4:] <= n) and np.all(c[:, 4:] >= 0)
    assert np.all(c[:, 3] >= 0)
    np.testing.assert_allclose(c[:, 0].sum(), g["tot_cost"].sum(), rtol=1e-9)
    np.testing.assert_allclose(c[:, 1].sum(), g["tot_energy"].sum(), rtol=1e-9)
    assert c[:, 4].sum() == g["n_stop"].sum() == g["counters"][4]
    assert g["counters"][0] == n * job.recurrences
    # Thompson-sampling picks: every sampled or forced decision, and every decision once the
    # pruning stage (at most 2|B| recurrences, Alg. 3) is over -- exact integer sums
    B = len(job.workload["batch_sizes"])
    assert c[:, 6].sum() == g["counters"][1] + g["counters"][6]
    assert np.all(c[2 * B:, 6] == n)
    assert c[:, 5].sum() <= n * job.recurrences
    # the 1-in-100 sample's curves estimate the full curves (statistical, loose)
    np.testing.assert_allclose(o["curves"][-100:, 0].sum() * 100, c[-100:, 0].sum(), rtol=0.02)


# ------------------------------------------------------------------ edge cases
def test_micro_traces_gpu(zs, oracle):
    import json
    import os

    from tests.conftest import GOLDEN

    g = json.load(open(os.path.join(GOLDEN, "micro_traces.json")))
    t = g["trace"]
    for key in ("W1", "W2"):
        w = {"batch_sizes": np.array(t["batch_sizes"], np.int32), "b0": t["b0"],
             "power_limits": np.array(t["power_limits"], float), "max_power": t["max_power"],
             "max_epochs": t["max_epochs"], "charge_profiling": g[key]["charge_profiling"],
             "avg_power": np.array(t["avg_power"], float), "throughput": np.array(t["throughput"], float),
             "pool": np.array(t["pool"], np.int32)}
        cell = synth.cell(eta=1.0, beta=2.0, seed=5)
        r = run_gpu(zs, w, [cell], 50, 8, log=True)
        assert [int(x & 0xFF) for x in r["log"][0]] == g[key]["arms"]
        np.testing.assert_allclose(r["tot_cost"], g[key]["total_cost"], rtol=1e-13)
        compare_cell(oracle, r, w, cell, 0, np.arange(50), 8, 50, logs=True)


def _random_trace(rng, B, P, S, K, fail=0.2):
    bs = np.cumsum(rng.integers(1, 9, size=B)).astype(np.int32) * 8
    pl = np.sort(rng.choice(np.arange(50, 400), size=P, replace=False)).astype(float)
    MP = float(pl.max())
    A = rng.uniform(30, MP, size=(B, P))
    Th = rng.uniform(1e-3, 1e-1, size=(B, P))
    pool = rng.integers(1, 60, size=(S, B, K)).astype(np.int32)
    pool[rng.random(pool.shape) < fail] = 0
    pool[:, 0, 0] = np.maximum(pool[:, 0, 0], 1)
    return {"batch_sizes": bs, "b0": int(rng.integers(B)), "power_limits": pl, "max_power": MP,
            "max_epochs": 80, "charge_profiling": int(rng.integers(2)), "avg_power": A,
            "throughput": Th, "pool": pool}


@pytest.mark.parametrize("B,P,S,K,window,beta,trials,R", [
    (1, 1, 1, 1, 0, 2.0, 37, 9),          # single arm (HPO case), ragged tail
    (32, 64, 1, 4, 0, 2.0, 130, 40),      # maximum sizes
    (32, 7, 5, 3, 2, 1.5, 65, 33),        # max arms, smallest window, S not dividing R
    (7, 5, 3, 2, 4, math.inf, 200, 25),   # no early stop
    (16, 16, 1, 4, 10, 3.0, 1, 100),      # one trial
    (5, 3, 1, 1, 0, 1.0000001, 96, 20),   # beta just above 1: stops everywhere
    (9, 7, 1, 4, 0, 2.0, 300, 0),         # R = 0 -> auto 2|B||P|
    (32, 8, 1, 4, 0, 2.0, 200, 100),      # two phases with 32 arms (16 pairs, 8 quads)
    (17, 5, 2, 3, 0, 2.0, 150, 60),       # odd arm count, two phases, two slices
    (3, 4, 1, 2, 0, math.inf, 130, 30),   # two phases, two pairs, no early stop
])
@pytest.mark.parametrize("layout,draw", [(0, 0), (0, 2), (3, 0), (4, 0)])
def test_random_traces_edge_cases(zs, oracle, B, P, S, K, window, beta, trials, R, layout, draw):
    rng = np.random.default_rng(B * 1000 + P)
    w = _random_trace(rng, B, P, S, K)
    cells = [synth.cell(eta=e, beta=beta, window=window, seed=int(rng.integers(2**63)),
                        prior_mean=pm, prior_var=pv)
             for e, pm, pv in ((0.0, 0.0, math.inf), (1.0, 500.0, 1e6), (0.37, 0.0, math.inf))]
    g = run_gpu(zs, w, cells, trials, R, log=True, layout=layout, draw=draw)
    Rr = g["R"]
    assert Rr == (R if R > 0 else 2 * B * P)
    compare_step1(oracle, g, w, cells)
    for ci, c in enumerate(cells):
        compare_cell(oracle, g, w, c, ci, np.arange(trials), Rr, trials, logs=True)


def test_empty_shard_and_sharding_invariance(zs, oracle):
    """P16: per-trial results do not depend on the shard split (global-index RNG keys)."""
    (job,) = synth.config("cfg4", trials=3000)
    w, cells, R = job.workload, job.cells, job.recurrences
    full = run_gpu(zs, w, cells, 3000, R)
    parts = [run_gpu(zs, w, cells, 3000, R, shard=(b, e)) for b, e in ((0, 1111), (1111, 2048), (2048, 3000))]
    for k in ("tot_cost", "digest", "tot_time", "n_stop", "final_arm"):
        assert np.array_equal(full[k], np.concatenate([p[k] for p in parts]))
    # the curves' fixed-point sums add exactly; rounded once they are the full run's bits
    assert np.array_equal(_fixed_value(full["curves_fixed"]),
                          _fixed_value(sum(p["curves_fixed"] for p in parts)))
    import torch

    sim = zs.Simulation(w, cells, 3000, R).load_profile()
    fx = torch.from_numpy(sum(p["curves_fixed"] for p in parts)).cuda()
    cv = torch.zeros((len(cells), R, 7), dtype=torch.float64, device="cuda")
    sim.curves_from_fixed(fx, cv)
    sim.close()
    assert np.array_equal(cv.cpu().numpy(), full["curves"])
    empty = run_gpu(zs, w, cells, 3000, R, shard=(5000, 6000))
    assert empty["n"] == 0 and np.all(empty["curves"] == 0)


def test_results_into_device_buffers(zs):
    import torch

    (job,) = synth.config("cfg1")
    sim = zs.Simulation(job.workload, job.cells, job.trials, job.recurrences).load_profile()
    stream = torch.cuda.Stream()
    sim.run(stream)
    dev = torch.zeros((1, sim.R, 7), dtype=torch.float64, device="cuda")
    out = sim.results(want=["curves"])
    out2 = sim.results(want=[], out={"curves": dev})
    np.testing.assert_array_equal(dev.cpu().numpy(), out["curves"])
    assert out2["replay_ms"] > 0
    sim.close()


def test_results_async_device_buffers(zs):
    """zeus_sim_results_async: the replay outputs enqueued into device buffers on the run's
    stream (no synchronisation) equal zeus_sim_results'; host destinations and step-1 tables
    are refused before anything is queued."""
    import torch

    (job,) = synth.config("cfg4", trials=3000)
    sim = zs.Simulation(job.workload, job.cells, job.trials, job.recurrences).load_profile()
    stream = torch.cuda.Stream()
    sim.run(stream)
    ref = sim.results(want=["curves", "curves_fixed", "tot_cost", "digest", "counters"])
    sim.run(stream)                                  # a second run: the same bits
    n = sim.shard_n
    dev = {"curves": torch.zeros((1, sim.R, 7), dtype=torch.float64, device="cuda"),
           "curves_fixed": torch.zeros((1, sim.R, 7, 3), dtype=torch.int64, device="cuda"),
           "tot_cost": torch.zeros(n, dtype=torch.float64, device="cuda"),
           "digest": torch.zeros(n, dtype=torch.int64, device="cuda"),
           "counters": torch.zeros(14, dtype=torch.int64, device="cuda")}
    r = sim.results(want=[], out=dev, enqueue_only=True)
    assert r["kernel_launches"] > 0
    stream.synchronize()
    for k, v in dev.items():
        assert np.array_equal(v.cpu().numpy().view(np.asarray(ref[k]).dtype).reshape(np.shape(ref[k])),
                              np.asarray(ref[k])), k
    with pytest.raises(zs.ZeusError, match="neither device nor pinned"):
        sim.results(want=["tot_cost"], enqueue_only=True)          # pageable numpy
    pinned = torch.zeros(n, dtype=torch.float64).pin_memory()
    sim.results(want=[], out={"tot_cost": pinned}, enqueue_only=True)
    stream.synchronize()
    assert np.array_equal(pinned.numpy(), np.asarray(ref["tot_cost"]))
    with pytest.raises(zs.ZeusError, match="replay outputs only"):
        sim.results(want=["c1"], enqueue_only=True)
    sim.close()


def test_errors_are_reported(zs):
    (job,) = synth.config("cfg1")
    w = dict(job.workload)
    bad = synth.cell(eta=2.0, beta=0.5, window=1)
    with pytest.raises(zs.ZeusError) as e:
        zs.Simulation(w, [bad], 10, 5)
    for frag in ("eta", "beta", "window"):
        assert frag in str(e.value)
    sim = zs.Simulation(w, job.cells, 10, 5)
    with pytest.raises(zs.ZeusError, match="ZEUS_E_STATE"):
        sim.run()
    w2 = dict(w)
    w2["pool"] = np.zeros_like(w["pool"])
    sim2 = zs.Simulation(w2, job.cells, 10, 5)
    with pytest.raises(zs.ZeusError, match="NO_CONVERGENT_ARM"):
        sim2.load_profile()


@pytest.mark.parametrize("name", ["cfg1", "cfg4_38", "cfg5"])
def test_schedules_bit_identical(zs, oracle, name):
    """layout 1 (one pass, thread per trial), layout 2 (pruning phase, regroup, Thompson
    phase), layout 3 (lane group per trial) and layout 4 (layout 2 with the early split) give
    the same bits for every trial and decision."""
    (job,) = synth.config(name, trials=2000 if name != "cfg5" else 700)
    outs = [run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences, log=True, layout=l, draw=d)
            for l, d in ((1, 0), (2, 1), (3, 0), (2, 0), (2, 2), (4, 0), (4, 2))]
    for o in outs[1:]:
        for k in ("log", "tot_cost", "tot_energy", "tot_time", "digest", "n_stop", "final_arm"):
            assert np.array_equal(outs[0][k], o[k]), k
        assert np.array_equal(outs[0]["counters"][:9], o["counters"][:9])
        assert np.array_equal(outs[0]["curves"], o["curves"])          # exact sums: same bits
    # evaluated work: lane groups transform every survivor pair (each with its own Philox
    # block); the bound screen of the one-pass and Thompson-phase kernels
    # transforms at most as many, and far fewer once the posteriors separate
    c1, c2, c3, c4, c5, c6, c7 = (o["counters"] for o in outs)
    assert c3[9] == c3[2] and c3[10] == c3[2]
    for c in (c1, c2):
        assert c[9] <= c[2] and c[10] >= c[8]
        if name == "cfg5":
            assert c[9] < 0.6 * c[2]
    # certified fp32 draw: every Thompson-phase draw is either certified or
    # sent to the exact fallback; draw = 2 sends all of them
    # (windowed cells take it in replay_kernel's exact phase B, the others in thompson_kernel)
    ts_b = c4[12] + c4[13]
    assert ts_b > 0 and c5[12] == 0 and c5[13] == ts_b
    assert c6[12] + c6[13] == ts_b and c7[12] == 0 and c7[13] == ts_b   # early split: same draws
    assert c4[13] <= 0.01 * ts_b
    assert c1[12] + c1[13] > 0                  # the one-pass kernel certifies too (draw 0)
    assert c2[12] + c2[13] == 0                 # draw 1: the exact screen only
    compare_cell(oracle, outs[1], job.workload, job.cells[0], 0, np.arange(job.trials),
                 job.recurrences, job.trials, logs=True)


def test_f1_baselines_same_replay(zs, oracle):
    """Default and Grid Search (§6.1) replayed in the same launch
    as Zeus on the six workloads, T = 2|B||P|; every trial bit-exact vs the oracle."""
    for job in synth.config("f1", trials=3000):
        g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences, log=True)
        assert g["kernel_launches"] >= 3
        for ci, c in enumerate(job.cells):
            compare_cell(oracle, g, job.workload, c, ci, np.arange(job.trials), job.recurrences,
                         job.trials, logs=True)


def test_concurrent_handles_different_footprints(zs, oracle):
    """Handles with different shared-memory footprints (B = 6 windowed vs B = 16) run
    concurrently on separate streams; each stays bit-exact."""
    import torch

    jobs = [synth.config("cfg4_38", trials=500)[0], synth.config("cfg5", trials=500)[0],
            synth.config("cfg2", trials=500)[3]]
    sims = [zs.Simulation(j.workload, j.cells, j.trials, j.recurrences).load_profile() for j in jobs]
    streams = [torch.cuda.Stream() for _ in jobs]
    for sm, st in zip(sims, streams):
        sm.run(st)
    for sm, j in zip(sims, jobs):
        g = sm.results(want=["digest", "tot_cost", "tot_energy", "tot_time", "n_stop", "final_arm",
                             "curves", "counters"])
        compare_cell(oracle, g, j.workload, j.cells[0], 0, np.arange(j.trials), j.recurrences,
                     j.trials)
        sm.close()


def test_f4_pareto_front(zs, oracle):
    """the (TTA, ETA) Pareto front of every slice equals the oracle's."""
    for name in ("cfg2", "cfg4_38"):
        for job in synth.config(name, trials=10):
            sim = zs.Simulation(job.workload, job.cells, job.trials, job.recurrences).load_profile()
            g = sim.results(want=["pareto"])
            sim.close()
            for s in range(job.workload["pool"].shape[0]):
                assert np.array_equal(g["pareto"][s], oracle.pareto(job.workload, s)), (name, s)


@pytest.mark.parametrize("draw", [0, 2])
def test_f2_ablations(zs, oracle, draw):
    """the ablations of P:L1076-1077 (no early stop = beta inf, no pruning,
    no JIT profiling) in the same launch as full Zeus; every trial bit-exact vs the oracle, with the
    certified draw (0) and with every Thompson draw through its exact fallback (2)."""
    for job in synth.config("f2", trials=2000)[:3]:
        g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences, log=True, draw=draw)
        for ci, c in enumerate(job.cells):
            compare_cell(oracle, g, job.workload, c, ci, np.arange(job.trials), job.recurrences,
                         job.trials, logs=True)


def test_layout4_with_ablation_and_policy_cells(zs, oracle):
    """Layout 4 (the early split) asked for on launches it does not apply to -- ablation cells
    (the exact phase B), the Default / Grid Search policies next to Zeus (f1) -- gives every
    trial the oracle's bits."""
    for name in ("f2", "f1"):
        for job in synth.config(name, trials=1500)[:2]:
            g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences, log=True, layout=4)
            for ci, c in enumerate(job.cells):
                compare_cell(oracle, g, job.workload, c, ci, np.arange(job.trials), job.recurrences,
                             job.trials, logs=True)


@pytest.mark.parametrize("draw", [0, 2])
def test_f3_concurrent_submissions(zs, oracle, draw):
    """concurrent submissions under Poisson arrival schedules (§4.4
    P:L634-646) next to the sequential cell in one launch; every trial bit-exact."""
    for job in synth.config("f3", trials=2000)[:3]:
        g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences, log=True, draw=draw)
        for ci, c in enumerate(job.cells):
            compare_cell(oracle, g, job.workload, c, ci, np.arange(job.trials), job.recurrences,
                         job.trials, logs=True)
    # the drift config with a window, heavy overlap
    (job,) = synth.config("cfg4_38", trials=1500)
    c = dict(job.cells[0], arrivals=synth.arrival_schedule(job.workload, job.recurrences, 0.3, 5))
    g = run_gpu(zs, job.workload, [c], job.trials, job.recurrences, log=True, draw=draw)
    compare_cell(oracle, g, job.workload, c, 0, np.arange(job.trials), job.recurrences, job.trials,
                 logs=True)


@pytest.mark.parametrize("draw", [0, 2])
def test_f2v_variant_readings(zs, oracle, draw):
    """SURVEY §8(f) f2, the variant readings of P:L559 (DESIGN.md R-Q4v retry, R-Q1v epoch-boundary
    stop, R-Q5v windowed best under drift), each in the same launch as the base cell: every
    trial and logged decision bit-exact vs the oracle, curves within 1e-9."""
    jobs = synth.config("f2v", trials=1500)
    for job in (jobs[0], jobs[3], jobs[6]):
        g = run_gpu(zs, job.workload, job.cells, job.trials, job.recurrences, log=True, draw=draw)
        decisions = 0
        for ci, c in enumerate(job.cells):
            o = compare_cell(oracle, g, job.workload, c, ci, np.arange(job.trials), job.recurrences,
                             job.trials, logs=True)
            decisions += o["counters"][0]
        assert g["counters"][0] == decisions          # retries are decisions


def test_cuda_graph_runs_identical(zs):
    """zeus_run_opts.graph: the captured run, replayed, gives the bits of the direct launches;
    reloading the same-shaped trace keeps the graph valid, a new shape recaptures it."""
    want = ["digest", "tot_cost", "final_arm", "curves", "counters"]
    for name, trials in (("cfg1", 300), ("cfg4_38", 400), ("cfg5", 600)):
        (job,) = synth.config(name, trials=trials)
        direct = zs.Simulation(job.workload, job.cells, job.trials, job.recurrences).load_profile()
        ref = direct.run().results(want=want)
        direct.close()
        g = zs.Simulation(job.workload, job.cells, job.trials, job.recurrences, graph=True).load_profile()
        for rep in range(3):
            if rep == 2:
                g.load_profile()                     # same trace again: same buffers, same graph
            out = g.run().results(want=want)
            for k in want:
                if k == "curves":
                    np.testing.assert_allclose(out[k], ref[k], rtol=1e-12)
                else:
                    assert np.array_equal(out[k], ref[k]), (name, rep, k)
        g.close()


def test_cuda_graph_with_early_split_and_async_results(zs):
    """A captured run of the early-split schedule (layout 4: pruning-only phase A, (quads, t0)
    regroup, thompson_kernel<..., EARLY>) replays with the direct launches' bits, and its outputs
    handed over by zeus_sim_results_async match."""
    import torch

    want = ["digest", "tot_cost", "curves"]
    job = synth.config("cfg3", trials=1500)[0]
    cells = job.cells[:3]
    direct = zs.Simulation(job.workload, cells, job.trials, job.recurrences, layout=4).load_profile()
    ref = direct.run().results(want=want)
    direct.close()
    g = zs.Simulation(job.workload, cells, job.trials, job.recurrences, layout=4, graph=True).load_profile()
    stream = torch.cuda.Stream()
    for _ in range(2):
        g.run(stream)
        dev = {"digest": torch.zeros(g.shard_n, dtype=torch.int64, device="cuda"),
               "tot_cost": torch.zeros(g.shard_n, dtype=torch.float64, device="cuda"),
               "curves": torch.zeros((len(cells), g.R, 7), dtype=torch.float64, device="cuda")}
        g.results(want=[], out=dev, enqueue_only=True)
        stream.synchronize()
        assert np.array_equal(dev["digest"].cpu().numpy().view(np.uint64), ref["digest"])
        assert np.array_equal(dev["tot_cost"].cpu().numpy(), ref["tot_cost"])
        assert np.array_equal(dev["curves"].cpu().numpy(), ref["curves"])
    g.close()


def test_cuda_graph_reload_new_values_same_shape(zs):
    """A same-shaped reload with different values keeps the captured graph only where nothing
    captured changed: a trace 64x slower changes the curves' fixed-point scale F (a kernel
    argument), so the graph is recaptured, and the run equals a fresh handle's."""
    want = ["digest", "tot_cost", "curves", "curves_fixed"]
    (job,) = synth.config("cfg4_38", trials=500)
    w2 = dict(job.workload)
    w2["throughput"] = np.asarray(job.workload["throughput"]) / 64.0      # every cost 64x: F - 6
    direct = zs.Simulation(w2, job.cells, job.trials, job.recurrences).load_profile()
    ref = direct.run().results(want=want)
    direct.close()
    g = zs.Simulation(job.workload, job.cells, job.trials, job.recurrences, graph=True).load_profile()
    f0 = g.run().results(want=want)["curve_scale_bits"]
    g.w = w2
    out = g.load_profile().run().results(want=want)
    g.close()
    assert out["curve_scale_bits"] == ref["curve_scale_bits"] != f0
    for k in want:
        assert np.array_equal(out[k], ref[k]), k


def test_bound_screen_every_path(zs, oracle):
    """a trace whose posteriors stay wide (32 arms, few recurrences, large beta)
    drives the bound screen through all of its paths -- screened-out pairs, parked residuals
    and redrawn ones past the two slots (counter [10] above [8]) -- bit-exact vs the oracle."""
    rng = np.random.default_rng(77)
    w = _random_trace(rng, 32, 4, 1, 4, fail=0.05)
    cells = [synth.cell(eta=0.5, beta=50.0, seed=int(rng.integers(2**63)), prior_mean=0.0,
                        prior_var=math.inf)]
    trials, R = 400, 90
    for layout in (1, 2):
        g = run_gpu(zs, w, cells, trials, R, log=True, layout=layout, draw=1)
        c = g["counters"]
        assert c[9] < c[2]                       # pairs screened out
        assert c[10] > c[8]                      # a third residual redrew its block
        compare_cell(oracle, g, w, cells[0], 0, np.arange(trials), R, trials, logs=True)


def test_round_key_kernels_match_multicell_launch(zs):
    """a one-cell launch runs the RK kernels (Philox round keys in the kernel
    parameters), a multi-cell launch the kernels that derive them from the key; the same cell
    in both gives the same bits, in both schedules (phase A/B and one pass)."""
    want = ["digest", "tot_cost", "tot_energy", "tot_time", "final_arm", "n_stop"]
    (job,) = synth.config("cfg5", trials=3000)
    other = synth.cell(eta=0.3, beta=3.0, seed=99)
    for layout in (1, 2):
        one = zs.Simulation(job.workload, job.cells, job.trials, 300, layout=layout).load_profile()
        a = one.run().results(want=want)
        one.close()
        two = zs.Simulation(job.workload, [job.cells[0], other], job.trials, 300,
                            layout=layout).load_profile()
        b = two.run().results(want=want)
        two.close()
        for k in want:
            assert np.array_equal(np.asarray(a[k]).reshape(-1)[:job.trials],
                                  np.asarray(b[k]).reshape(-1)[:job.trials]), (layout, k)


@pytest.mark.parametrize("B,P,S,K,window,beta,trials,R", [
    (32, 8, 1, 4, 0, 2.0, 200, 100),      # 32 arms: 16 pairs, 8 quads, three-residual redraws
    (17, 5, 2, 3, 4, 2.0, 150, 60),       # odd arm count, window, two slices
    (6, 7, 40, 4, 10, 2.0, 300, 40),      # drift-shaped: one slice per recurrence, window N = 10
    (3, 4, 1, 2, 0, math.inf, 130, 30),   # two pairs, no early stop
])
@pytest.mark.parametrize("layout,draw", [(1, 0), (2, 0), (2, 1), (2, 2), (4, 0), (4, 2)])
def test_random_traces_one_cell(zs, oracle, B, P, S, K, window, beta, trials, R, layout, draw):
    """One-cell launches run the RK kernels (round keys in the parameters, the
    record cache with write-back in the Thompson phase); edge shapes in both schedules,
    every decision bit-exact vs the oracle."""
    rng = np.random.default_rng(B * 7919 + S)
    w = _random_trace(rng, B, P, S, K)
    cell = synth.cell(eta=0.6, beta=beta, window=window, seed=int(rng.integers(2**63)))
    g = run_gpu(zs, w, [cell], trials, R, log=True, layout=layout, draw=draw)
    compare_step1(oracle, g, w, [cell])
    compare_cell(oracle, g, w, cell, 0, np.arange(trials), R, trials, logs=True)


def test_certified_draw_bounds(zs):
    """the two measured bounds behind the certified fp32 draw hold for EVERY
    32-bit word -- |r32 - r| <= e_r(a) for all 2^32 radius words and |cos32 - cos|, |sin32 - sin|
    <= kAng for all 2^32 angle words, against the contract's fp64 values (NC-3)."""
    out = zs.zeus_sim_certify_bounds(0)
    assert out[0] <= 1.0, f"radius bound exceeded: ratio {out[0]}"
    assert 6.66 < out[1] <= out[5]
    assert out[2] <= out[4] and out[3] <= out[4], out
    assert out[2] > 0.5 * out[4] and out[3] > 0.5 * out[4]      # the bound is measured, not loose
    # the composed per-arm bound (argmin keys vs the contract's theta), 2^28 seeded samples
    assert 0.0 < out[6] <= 1.0, f"theta bound exceeded: ratio {out[6]}"


def test_certified_draw_multicell_and_drift(zs, oracle):
    """The certified draw in multi-cell launches (keys derived in-kernel, no RK), a proper prior
    and a drifting trace without a window: draw 0, 1 and 2 give the oracle's bits."""
    rng = np.random.default_rng(2024)
    w = _random_trace(rng, 12, 6, 5, 4)
    cells = [synth.cell(eta=0.3, beta=2.0, seed=11, prior_mean=500.0, prior_var=1e4),
             synth.cell(eta=0.8, beta=math.inf, seed=12)]
    trials, R = 600, 150
    ref = None
    for d in (0, 1, 2):
        g = run_gpu(zs, w, cells, trials, R, log=True, layout=2, draw=d)
        for ci, c in enumerate(cells):
            compare_cell(oracle, g, w, c, ci, np.arange(trials), R, trials, logs=True, full_curves=False)
        if ref is None:
            ref = g
        assert np.array_equal(ref["curves"], g["curves"])


def test_reload_is_stream_ordered(zs, oracle):
    """include/zeus_sim.h "Async": load_profile enqueues its copies on the handle's stream after
    the run in flight there, so run(A) -> load_profile(B) -> results() returns A's replay, and the
    next run (on another stream) replays B.  No call synchronises the device."""
    import torch

    (job,) = synth.config("cfg5", trials=20000)
    wa = job.workload
    wb = dict(wa)
    wb["pool"] = np.ascontiguousarray(np.maximum(1, wa["pool"][:, ::-1, :]))   # another trace, same shape
    R = 400
    ref_a = run_gpu(zs, wa, job.cells, 20000, R)
    ref_b = run_gpu(zs, wb, job.cells, 20000, R)
    assert not np.array_equal(ref_a["digest"], ref_b["digest"])
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    sim = zs.Simulation(wa, job.cells, 20000, R).load_profile()
    sim.run(s1)
    sim.w = wb
    sim.load_profile()                      # while the first run is still in flight on s1
    ga = sim.results(want=["digest", "tot_cost", "curves"])
    assert np.array_equal(ga["digest"], ref_a["digest"]) and np.array_equal(ga["curves"], ref_a["curves"])
    sim.run(s2)
    gb = sim.results(want=["digest", "tot_cost", "tot_energy", "tot_time", "n_stop", "final_arm",
                           "curves", "c1"])
    assert np.array_equal(gb["digest"], ref_b["digest"]) and np.array_equal(gb["curves"], ref_b["curves"])
    sim.close()
    compare_cell(oracle, gb, wb, job.cells[0], 0, np.arange(0, 20000, 97), R, 20000, full_curves=False)


def test_results_validates_before_copying(zs):
    """A failing results() call (log without log_mode; replay outputs before any run) returns
    ZEUS_E_STATE without writing any caller buffer; step-1 tables and the Pareto masks are
    available before the first run (computed on request)."""
    (job,) = synth.config("cfg1")
    sim = zs.Simulation(job.workload, job.cells, job.trials, job.recurrences).load_profile()
    sentinel = np.full((1, sim.R, 7), 7.0)
    with pytest.raises(zs.ZeusError, match="ZEUS_E_STATE"):
        sim.results(want=[], out={"curves": sentinel})
    assert np.all(sentinel == 7.0)
    t = sim.results(want=["c1", "pareto", "opt_cost"])
    assert np.all(t["c1"] > 0) and t["pareto"].any()
    sim.run()
    log = np.full((sim.shard_n, sim.R), 5, np.uint32)
    with pytest.raises(zs.ZeusError, match="log_mode"):
        sim.results(want=[], out={"curves": sentinel, "log": log})
    assert np.all(sentinel == 7.0) and np.all(log == 5)
    sim.close()


def test_two_ranks_through_bench_match_one(tmp_path):
    """SURVEY §8(e) on one GPU: bench.py's real step under torchrun with 2 ranks sharing the GPU
    over gloo (shard_range, zeus_sim_run, the fixed-point all-reduce, max-over-ranks timing) gives
    per-trial digests and costs equal to one rank's, and curves with the same bits."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    common = ["--config", "cfg5", "--trials", "30000", "--steps", "1", "--warmup", "3",
              "--scaling", "strong", "--no-cpu-baseline", "--e2e-steps", "1"]
    env = dict(os.environ, ZEUS_DIST_BACKEND="gloo")
    one = tmp_path / "one"
    two = tmp_path / "two"
    r1 = subprocess.run([sys.executable, "bench.py", *common, "--dump", str(one)], cwd=root, env=env,
                        capture_output=True, text=True, timeout=900)
    assert r1.returncode == 0, r1.stderr[-2000:]
    r2 = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                         "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                         *common, "--dump", str(two)], cwd=root, env=env, capture_output=True, text=True,
                        timeout=900)
    assert r2.returncode == 0, r2.stderr[-2000:]
    line = [l for l in r2.stdout.splitlines() if l.startswith("{")][-1]
    import json

    assert json.loads(line)["n_gpus"] == 2
    a = np.load(one / "rank0_job0.npz")
    b0, b1 = np.load(two / "rank0_job0.npz"), np.load(two / "rank1_job0.npz")
    assert int(b0["begin"]) == 0 and int(b0["end"]) == int(b1["begin"]) and int(b1["end"]) == 30000
    for k in ("digest", "tot_cost", "n_stop", "final_arm"):
        assert np.array_equal(a[k], np.concatenate([b0[k], b1[k]])), k
    for b in (b0, b1):                      # every rank holds the all-reduced curves
        assert np.array_equal(_fixed_value(b["curves_fixed"]), _fixed_value(a["curves_fixed"]))
        assert np.array_equal(b["curves"], a["curves"])


def _fixed_value(fx):
    """The integers the limbs represent (limb sums are not canonical: carries differ)."""
    return np.array([int(l0) + (int(l1) << 26) + (int(l2) << 52) for l0, l1, l2 in fx.reshape(-1, 3)],
                    dtype=object)
