"""ctypes access to the C++ oracle (oracle/liboracle.so) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  It never touches the CUDA library and
the CUDA path never touches it.  See oracle.h for the meaning of every field.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.cpp")

# NC-1: plain -O2, no contraction, no fast-math.
CXXFLAGS = ["-O2", "-ffp-contract=off", "-std=c++17", "-Wall", "-shared", "-fPIC", "-pthread"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
        os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))
    ):
        subprocess.check_call(["g++", *CXXFLAGS, "-o", LIB_PATH, SRC])
    return LIB_PATH


class Trace(C.Structure):
    _fields_ = [
        ("num_batch_sizes", C.c_int32),
        ("batch_sizes", C.POINTER(C.c_int32)),
        ("default_bs_index", C.c_int32),
        ("num_power_limits", C.c_int32),
        ("power_limits_w", C.POINTER(C.c_double)),
        ("max_power_w", C.c_double),
        ("max_epochs", C.c_int32),
        ("charge_profiling", C.c_int32),
        ("avg_power_w", C.POINTER(C.c_double)),
        ("throughput_eps", C.POINTER(C.c_double)),
        ("num_slices", C.c_int32),
        ("replicas", C.c_int32),
        ("epochs_to_target", C.POINTER(C.c_int32)),
    ]


class Cell(C.Structure):
    _fields_ = [
        ("eta", C.c_double),
        ("beta", C.c_double),
        ("window", C.c_int32),
        ("prior_mean", C.c_double),
        ("prior_var", C.c_double),
        ("seed", C.c_uint64),
        ("policy", C.c_int32),
        ("ablation", C.c_int32),
        ("arrivals", C.POINTER(C.c_double)),
    ]


class Tables(C.Structure):
    _fields_ = [
        ("pstar", C.POINTER(C.c_int32)),
        ("c1", C.POINTER(C.c_double)),
        ("t1", C.POINTER(C.c_double)),
        ("e1", C.POINTER(C.c_double)),
        ("c_prof", C.POINTER(C.c_double)),
        ("t_prof", C.POINTER(C.c_double)),
        ("e_prof", C.POINTER(C.c_double)),
        ("ebar", C.POINTER(C.c_double)),
        ("opt", C.POINTER(C.c_double)),
        ("opt_arm", C.POINTER(C.c_int32)),
        ("regret", C.POINTER(C.c_double)),
    ]


class Out(C.Structure):
    _fields_ = [
        ("tot_cost", C.POINTER(C.c_double)),
        ("tot_energy", C.POINTER(C.c_double)),
        ("tot_time", C.POINTER(C.c_double)),
        ("digest", C.POINTER(C.c_uint64)),
        ("n_stop", C.POINTER(C.c_int32)),
        ("final_arm", C.POINTER(C.c_int32)),
        ("log", C.POINTER(C.c_uint32)),
        ("cost_log", C.POINTER(C.c_double)),
        ("energy_log", C.POINTER(C.c_double)),
        ("time_log", C.POINTER(C.c_double)),
        ("curves", C.POINTER(C.c_double)),
        ("counters", C.POINTER(C.c_int64)),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.oracle_validate.argtypes = [C.POINTER(Trace), C.POINTER(Cell), C.c_char_p, C.c_int32]
        L.oracle_step1.argtypes = [C.POINTER(Trace), C.POINTER(Cell), C.POINTER(Tables)]
        L.oracle_replay.argtypes = [C.POINTER(Trace), C.POINTER(Cell), C.c_int32,
                                    C.POINTER(C.c_int64), C.c_int64, C.c_int32, C.POINTER(Out)]
        L.oracle_philox4x32_10.argtypes = [C.POINTER(C.c_uint32)] * 3
        L.oracle_zlog.argtypes = [C.c_double]
        L.oracle_zlog.restype = C.c_double
        L.oracle_zlog_fdlibm.argtypes = [C.c_double]
        L.oracle_zlog_fdlibm.restype = C.c_double
        L.oracle_zsincospi.argtypes = [C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.oracle_uniforms.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.oracle_normal_pair.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_int32,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.oracle_replica.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_int32]
        L.oracle_replica.restype = C.c_uint32
        L.oracle_thompson_argmin.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_uint32,
                                             C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.oracle_thompson_argmin.restype = C.c_int32
        L.oracle_posterior.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32, C.c_double,
                                       C.c_double] + [C.POINTER(C.c_double)] * 4
        L.oracle_hardware_threads.restype = C.c_int32
        L.oracle_zlog_batch.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64]
        L.oracle_zsincospi_batch.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                             C.POINTER(C.c_double), C.c_int64]
        L.oracle_normal_batch.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                          C.c_int32, C.POINTER(C.c_double)]
        L.oracle_pareto.argtypes = [C.POINTER(Trace), C.c_int32, C.POINTER(C.c_uint8)]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


class _Held:
    """Keeps numpy arrays alive while a ctypes struct points into them."""

    def __init__(self, w):
        self.bs = np.ascontiguousarray(w["batch_sizes"], dtype=np.int32)
        self.pl = np.ascontiguousarray(w["power_limits"], dtype=np.float64)
        self.A = np.ascontiguousarray(w["avg_power"], dtype=np.float64)
        self.Th = np.ascontiguousarray(w["throughput"], dtype=np.float64)
        self.pool = np.ascontiguousarray(w["pool"], dtype=np.int32)
        S, B, K = self.pool.shape
        self.tr = Trace(len(self.bs), _p(self.bs, C.c_int32), int(w["b0"]), len(self.pl),
                        _p(self.pl, C.c_double), float(w["max_power"]), int(w["max_epochs"]),
                        int(w.get("charge_profiling", 1)), _p(self.A, C.c_double),
                        _p(self.Th, C.c_double), S, K, _p(self.pool, C.c_int32))


def _cell(c):
    arr = c.get("arrivals")
    cc = Cell(float(c["eta"]), float(c["beta"]), int(c.get("window", 0)),
              float(c.get("prior_mean", 0.0)), float(c.get("prior_var", np.inf)),
              int(c.get("seed", 0)), int(c.get("policy", 0)), int(c.get("ablation", 0)), None)
    if arr is not None:
        cc._arr = np.ascontiguousarray(arr, dtype=np.float64)   # kept alive with the struct
        cc.arrivals = _p(cc._arr, C.c_double)
    return cc


def validate(w, c):
    h = _Held(w)
    cc = _cell(c)
    buf = C.create_string_buffer(4096)
    rc = lib().oracle_validate(C.byref(h.tr), C.byref(cc), buf, 4096)
    return rc, buf.value.decode()


def step1(w, c):
    h = _Held(w)
    cc = _cell(c)
    S, B, _ = h.pool.shape
    o = {k: np.zeros(B) for k in ("c1", "t1", "e1", "c_prof", "t_prof", "e_prof")}
    o["pstar"] = np.zeros(B, np.int32)
    o["ebar"] = np.zeros((S, B))
    o["regret"] = np.zeros((S, B))
    o["opt"] = np.zeros(S)
    o["opt_arm"] = np.zeros(S, np.int32)
    t = Tables(_p(o["pstar"], C.c_int32), *[_p(o[k], C.c_double) for k in ("c1", "t1", "e1", "c_prof", "t_prof", "e_prof")],
               _p(o["ebar"], C.c_double), _p(o["opt"], C.c_double), _p(o["opt_arm"], C.c_int32),
               _p(o["regret"], C.c_double))
    rc = lib().oracle_step1(C.byref(h.tr), C.byref(cc), C.byref(t))
    if rc != 0:
        raise ValueError(validate(w, c)[1])
    return o


def replay(w, c, R, trials, threads=1, logs=False, curves=True):
    """Replays the given global trial indices; returns a dict of numpy arrays."""
    h = _Held(w)
    cc = _cell(c)
    trials = np.ascontiguousarray(trials, dtype=np.int64)
    n = len(trials)
    o = {
        "tot_cost": np.zeros(n), "tot_energy": np.zeros(n), "tot_time": np.zeros(n),
        "digest": np.zeros(n, np.uint64), "n_stop": np.zeros(n, np.int32),
        "final_arm": np.zeros(n, np.int32), "counters": np.zeros(9, np.int64),
    }
    o["curves"] = np.zeros((R, 7)) if curves else None
    if logs:
        o["log"] = np.zeros((n, R), np.uint32)
        o["cost_log"] = np.zeros((n, R))
        o["energy_log"] = np.zeros((n, R))
        o["time_log"] = np.zeros((n, R))
    g = lambda k, ct: _p(o.get(k), ct)  # noqa: E731
    out = Out(g("tot_cost", C.c_double), g("tot_energy", C.c_double), g("tot_time", C.c_double),
              g("digest", C.c_uint64), g("n_stop", C.c_int32), g("final_arm", C.c_int32),
              g("log", C.c_uint32), g("cost_log", C.c_double), g("energy_log", C.c_double),
              g("time_log", C.c_double), g("curves", C.c_double), g("counters", C.c_int64))
    rc = lib().oracle_replay(C.byref(h.tr), C.byref(cc), int(R), _p(trials, C.c_int64), n,
                             int(threads), C.byref(out))
    if rc != 0:
        raise ValueError(validate(w, c)[1] or "bad R / n")
    return o


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return list(o)


def zlog(x):
    return lib().oracle_zlog(float(x))


def zlog_fdlibm(x):
    return lib().oracle_zlog_fdlibm(float(x))


def zsincospi(m52):
    s, c = C.c_double(), C.c_double()
    lib().oracle_zsincospi(int(m52), C.byref(s), C.byref(c))
    return s.value, c.value


def uniforms(a, b):
    u, v = C.c_double(), C.c_double()
    lib().oracle_uniforms(int(a), int(b), C.byref(u), C.byref(v))
    return u.value, v.value


def normal_pair(seed, trial, t, k):
    a, b = C.c_double(), C.c_double()
    lib().oracle_normal_pair(int(seed), int(trial), int(t), int(k), C.byref(a), C.byref(b))
    return a.value, b.value


def replica(seed, trial, t, K):
    return lib().oracle_replica(int(seed), int(trial), int(t), int(K))


def thompson_argmin(seed, trial, t, mu, sigma, arms=None):
    """Alg. 1 Predict as the replay runs it: the arm picked among ``arms`` (default: all)."""
    mu = np.ascontiguousarray(mu, np.float64)
    sigma = np.ascontiguousarray(sigma, np.float64)
    B = len(mu)
    mask = sum(1 << a for a in (range(B) if arms is None else arms))
    return int(lib().oracle_thompson_argmin(int(seed), int(trial), int(t), B, mask,
                                            _p(mu, C.c_double), _p(sigma, C.c_double)))


def posterior(xs, window=0, prior_mean=0.0, prior_var=np.inf):
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    mu, sg, s2, var = (C.c_double() for _ in range(4))
    rc = lib().oracle_posterior(_p(xs, C.c_double), len(xs), int(window), float(prior_mean),
                                float(prior_var), C.byref(mu), C.byref(sg), C.byref(s2), C.byref(var))
    if rc != 0:
        return None
    return {"mu": mu.value, "sigma": sg.value, "s2": s2.value, "var": var.value}


def pareto(w, s=0):
    """Pareto-front mask [B][P] of slice s's (TTA, ETA) grid."""
    h = _Held(w)
    B, P = len(h.bs), len(h.pl)
    m = np.zeros((B, P), np.uint8)
    if lib().oracle_pareto(C.byref(h.tr), int(s), _p(m, C.c_uint8)) != 0:
        raise ValueError("bad slice")
    return m


def zlog_batch(x):
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    lib().oracle_zlog_batch(_p(x, C.c_double), _p(y, C.c_double), len(x))
    return y


def zsincospi_batch(m):
    m = np.ascontiguousarray(m, np.uint64)
    s, c = np.empty(len(m)), np.empty(len(m))
    lib().oracle_zsincospi_batch(_p(m, C.c_uint64), _p(s, C.c_double), _p(c, C.c_double), len(m))
    return s, c


def normal_batch(seed, trial0, n, t, k, threads=1):
    """[n][2]: the Box-Muller pair k of trials trial0 .. trial0+n-1 at recurrence t (NC-3)."""
    out = np.empty((n, 2))
    lib().oracle_normal_batch(int(seed), int(trial0), int(n), int(t), int(k), int(threads),
                              _p(out, C.c_double))
    return out


def hardware_threads():
    return int(lib().oracle_hardware_threads())
