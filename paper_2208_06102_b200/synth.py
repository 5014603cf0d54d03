"""Seeded synthetic traces and the five benchmark configurations.

INPUT GENERATION ONLY: this module holds none of the method's arithmetic (no
cost metric, no argmin, no sampling, no posterior).  It writes the two traces
the paper's replay consumes (§6.1) -- the power trace
(AvgPower, Throughput per (b, p)) and the training trace (epochs-to-target per
(b, seed), with K = 4 seeds) -- shaped as DESIGN.md §5 states, and
the (eta, beta, N, seed) cells of CFG1..CFG5 (BASELINE.json ``configs``).
Both the CUDA path and the oracle consume exactly these arrays.
"""
from __future__ import annotations

import math
import zlib
from dataclasses import dataclass, field

import numpy as np

P_IDLE = 70.0  # W, idle draw


@dataclass(frozen=True)
class Shape:
    """Per-workload generator constants (proposals; the shape constraints are cited in DESIGN.md §5)."""

    name: str
    batch_sizes: tuple
    b0: int                 # default batch size (Table 1)
    dataset: float          # samples per epoch
    rho: float              # saturated samples/s
    h: float                # half-saturation batch size
    e_w: float              # epochs at the best batch size
    kappa: float            # convexity of Epochs(b) in log2 b (App. C)
    b_star: float           # epoch-optimal batch size
    tau: float = 30.0       # W, power-curve knee
    power_limits: tuple = tuple(range(100, 251, 25))   # V100 range
    max_power: float = 250.0


# Table 1 workloads; b0 from the table, 𝓑 per SURVEY §8(d).
WORKLOADS = {
    "deepspeech2": Shape("deepspeech2", (8, 16, 24, 32, 48, 64, 96, 128, 192), 192,
                         28539, 180.0, 48.0, 25.0, 0.12, 32.0, 35.0),
    "bert_qa": Shape("bert_qa", (8, 12, 16, 24, 32, 48), 32, 88641, 120.0, 16.0, 3.0, 0.2, 16.0),
    "bert_sa": Shape("bert_sa", (8, 16, 32, 64, 128, 256), 128, 25000, 400.0, 32.0, 4.0, 0.2, 32.0),
    "resnet50": Shape("resnet50", (8, 16, 32, 64, 128, 256), 256, 1281167, 1200.0, 64.0, 40.0, 0.1, 64.0),
    "shufflenet_v2": Shape("shufflenet_v2", (16, 32, 64, 128, 256, 512, 1024, 2048), 1024,
                           50000, 9000.0, 256.0, 60.0, 0.08, 128.0),
    "neumf": Shape("neumf", (64, 128, 256, 512, 1024, 2048, 4096, 8192), 1024,
                   994169, 1.5e6, 1024.0, 10.0, 0.1, 512.0),
    # CFG1: a ResNet-18-like single job, 8 sizes x 6 limits
    "resnet18": Shape("resnet18", (8, 16, 32, 64, 128, 256, 512, 1024), 256, 50000, 8000.0, 64.0,
                      20.0, 0.15, 64.0, 30.0, (100, 130, 160, 190, 220, 250)),
    # CFG5: generic scale job, 16 half-octave sizes x 16 limits
    "generic16": Shape("generic16", (8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512, 768, 1024,
                                     1536, 2048), 256, 50000, 9000.0, 128.0, 30.0, 0.1, 96.0, 30.0,
                       tuple(range(100, 251, 10))),
}
SIX = ("deepspeech2", "bert_qa", "bert_sa", "resnet50", "shufflenet_v2", "neumf")


def _rng(seed: int, name: str, salt: str = "") -> np.random.Generator:
    return np.random.default_rng([seed, zlib.crc32((name + salt).encode())])


def _fail_prob(b: float, b_star: float) -> float:
    """Replicas fail more often far above b* ("too large ... loss of accuracy")."""
    up = 0.35 * (math.log2(b / b_star) - 1.5)
    down = 0.3 * (math.log2(b_star / b) - 2.0)
    return float(min(0.95, max(0.0, up, down)))


def make_workload(name: str, seed: int = 0, slices: int = 1, replicas: int = 4,
                  drift: bool = False, charge_profiling: int = 1) -> dict:
    """Power trace + training trace for one workload (dict of numpy arrays)."""
    sh = WORKLOADS[name]
    bs = np.array(sh.batch_sizes, dtype=np.float64)
    pl = np.array(sh.power_limits, dtype=np.float64)
    B, P = len(bs), len(pl)
    b0 = sh.batch_sizes.index(sh.b0)
    # throughput: saturating in b, increasing-concave in p; epochs/s
    g = (1.0 - np.exp(-(pl - P_IDLE) / sh.tau)) / (1.0 - math.exp(-(sh.max_power - P_IDLE) / sh.tau))
    th_max = sh.rho * bs / (bs + sh.h) / sh.dataset
    th = th_max[:, None] * g[None, :]
    # average power: ~90 W light load .. ~210 W heavy load, capped by the limit
    p_dem = 90.0 + 120.0 * bs / (bs + sh.h)
    A = np.minimum(0.97 * pl[None, :], p_dem[:, None])
    rng = _rng(seed, name, "pool")
    pool = np.zeros((slices, B, replicas), dtype=np.int32)
    ebar_max = 0.0
    ebars = []
    for s in range(slices):
        if drift:
            # §6.4: the optimum jumps (a spike at 30% of the slices) then drifts back
            frac = s / max(1, slices - 1)
            if frac < 0.3:
                b_star = 32.0
            else:
                b_star = 2.0 ** (7.0 - (frac - 0.3) / 0.7)   # 128 -> 64, log-linear
            e_w = sh.e_w * (1.0 + 0.05 * math.sin(2 * math.pi * s / max(1, slices)))
        else:
            b_star, e_w = sh.b_star, sh.e_w
        eb = e_w * (1.0 + sh.kappa * np.log2(bs / b_star) ** 2)
        ebars.append((eb, b_star))
        ebar_max = max(ebar_max, float(eb.max()))
    max_epochs = int(math.ceil(3.0 * ebar_max))
    for s, (eb, b_star) in enumerate(ebars):
        for b in range(B):
            noise = np.exp(0.05 * rng.standard_normal(replicas))   # <~14% spread
            E = np.maximum(1, np.rint(eb[b] * noise)).astype(np.int64)
            E = np.minimum(E, max_epochs)
            if b != b0:   # b0 "consistently achieves the target"
                fail = rng.random(replicas) < _fail_prob(bs[b], b_star)
                E[fail] = 0
            pool[s, b] = E
    return {
        "name": name, "batch_sizes": np.array(sh.batch_sizes, np.int32), "b0": b0,
        "power_limits": pl, "max_power": sh.max_power, "max_epochs": max_epochs,
        "charge_profiling": charge_profiling, "avg_power": np.ascontiguousarray(A),
        "throughput": np.ascontiguousarray(th), "pool": pool,
    }


POLICIES = {"zeus": 0, "default": 1, "grid_search": 2}   # §6.1 baselines


ABLATIONS = {"no_pruning": 1, "no_jit": 2,            # P:L1076-1077 (β = ∞ is "no early stop")
             "retry": 4, "epoch_stop": 8, "windowed_best": 16}   # readings of P:L559 (R-Q4v/1v/5v)


def cell(eta=0.5, beta=2.0, window=0, seed=1, prior_mean=0.0, prior_var=math.inf,
         policy="zeus", ablation=0, arrivals=None) -> dict:
    """One sweep cell; defaults are the paper's η = 0.5, β = 2 and a flat prior.
    ``arrivals``: optional [R] submission times (s) for concurrent submissions (§4.4)."""
    if isinstance(ablation, str):
        ablation = sum(ABLATIONS[a] for a in ablation.split("+") if a)
    c = {"eta": float(eta), "beta": float(beta), "window": int(window), "seed": int(seed),
         "prior_mean": float(prior_mean), "prior_var": float(prior_var),
         "policy": POLICIES[policy] if isinstance(policy, str) else int(policy),
         "ablation": int(ablation)}
    if arrivals is not None:
        c["arrivals"] = np.ascontiguousarray(arrivals, dtype=np.float64)
    return c


def arrival_schedule(workload: dict, R: int, overlap: float, seed: int) -> np.ndarray:
    """Poisson submissions whose mean gap is ``overlap`` x the TTA of b0 at the highest power
    limit with mean epochs (overlap < 1: later jobs start before earlier ones finish, as in
    the Alibaba job groups of §6.3)."""
    b0 = workload["b0"]
    pool = workload["pool"][0, b0]
    tta = float(pool[pool > 0].mean()) / float(workload["throughput"][b0, -1])
    rng = _rng(seed, workload["name"], "arrivals")
    return np.cumsum(rng.exponential(overlap * tta, size=R))


@dataclass
class Job:
    workload: dict
    cells: list
    recurrences: int
    trials: int          # global trials per cell
    extra: dict = field(default_factory=dict)

    @property
    def decisions(self) -> int:
        return len(self.cells) * self.trials * self.recurrences


def config(name: str, seed: int = 2208, trials: int | None = None) -> list[Job]:
    """CFG1..CFG5 of BASELINE.json as concrete synthetic jobs."""
    if name == "cfg1":
        return [Job(make_workload("resnet18", seed), [cell(seed=seed + 1)], 50, trials or 100)]
    if name == "cfg2":
        return [Job(make_workload(w, seed), [cell(seed=seed + 2)], 200, trials or 10_000) for w in SIX]
    if name == "cfg3":
        etas = [round(0.1 * i, 1) for i in range(11)]
        betas = [1.5, 2.0, 3.0, math.inf]
        cells = [cell(eta=e, beta=b, seed=seed + 3) for e in etas for b in betas]
        return [Job(make_workload(w, seed), cells, 200, trials or 10_000) for w in SIX]
    if name == "cfg4":
        return [Job(make_workload("bert_sa", seed, slices=200, drift=True),
                    [cell(window=10, seed=seed + 4)], 200, trials or 100_000)]
    if name == "cfg4_38":
        return [Job(make_workload("bert_sa", seed, slices=38, drift=True),
                    [cell(window=10, seed=seed + 4)], 38, trials or 100_000)]
    if name == "f1":   # Zeus vs the §6.1 baselines on the six workloads, T = 2|B||P|
        jobs = []
        for w in SIX:
            wl = make_workload(w, seed)
            R = 2 * len(wl["batch_sizes"]) * len(wl["power_limits"])
            jobs.append(Job(wl, [cell(seed=seed + 6, policy=p) for p in POLICIES], R, trials or 10_000))
        return jobs
    if name == "f2":   # ablations of Fig. eval-breakdown on the six workloads
        abl = [cell(seed=seed + 7), cell(seed=seed + 7, beta=math.inf),
               cell(seed=seed + 7, ablation="no_pruning"), cell(seed=seed + 7, ablation="no_jit")]
        return [Job(make_workload(w, seed), abl, 200, trials or 10_000) for w in SIX]
    if name == "f2v":  # the variant readings of P:L559 (R-Q4v retry, R-Q1v epoch-boundary stop)
        var = [cell(seed=seed + 9), cell(seed=seed + 9, ablation="retry"),
               cell(seed=seed + 9, ablation="epoch_stop"), cell(seed=seed + 9, ablation="retry+epoch_stop")]
        jobs = [Job(make_workload(w, seed), var, 200, trials or 10_000) for w in SIX]
        # R-Q5v windowed best under drift (§6.4's optimum shift, window N = 10)
        drift = [cell(window=10, seed=seed + 9), cell(window=10, seed=seed + 9, ablation="windowed_best"),
                 cell(window=10, seed=seed + 9, ablation="windowed_best+retry+epoch_stop")]
        jobs.append(Job(make_workload("bert_sa", seed, slices=200, drift=True), drift, 200, trials or 10_000))
        return jobs
    if name == "f3":   # concurrent submissions (§4.4): sequential, mild, heavy overlap
        jobs = []
        for w in SIX:
            wl = make_workload(w, seed)
            cells = [cell(seed=seed + 8)] + [cell(seed=seed + 8, arrivals=arrival_schedule(wl, 200, ov, seed))
                                             for ov in (1.0, 0.25)]
            jobs.append(Job(wl, cells, 200, trials or 10_000))
        return jobs
    if name == "cfg5":
        return [Job(make_workload("generic16", seed), [cell(seed=seed + 5)], 1000,
                    trials or 10_000_000)]
    raise KeyError(name)


CONFIGS = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")
NEXT = ("f1", "f2", "f2v", "f3")   # SURVEY §8(f) rows built on the same replay
