"""ctypes access to the literal replay (oracle/libliteral.so) -- TEST INFRASTRUCTURE ONLY.

The literal replay writes Alg. 1-3 as the paper prints them, with library random numbers
(see literal.cpp).  Only tests/ load it: it is the paper-side reference against which the
contract oracle's replay is checked statistically.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libliteral.so")
SRC = os.path.join(HERE, "literal.cpp")
CXXFLAGS = ["-O2", "-std=c++17", "-Wall", "-shared", "-fPIC", "-pthread"]


def build(force: bool = False) -> str:
    hdr = os.path.join(HERE, "literal.h")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC), os.path.getmtime(hdr)):
        subprocess.check_call(["g++", *CXXFLAGS, "-o", LIB_PATH, SRC])
    return LIB_PATH


class Trace(C.Structure):
    _fields_ = [
        ("num_batch_sizes", C.c_int32), ("batch_sizes", C.POINTER(C.c_int32)),
        ("default_bs_index", C.c_int32), ("num_power_limits", C.c_int32),
        ("power_limits_w", C.POINTER(C.c_double)), ("max_power_w", C.c_double),
        ("max_epochs", C.c_int32), ("charge_profiling", C.c_int32),
        ("avg_power_w", C.POINTER(C.c_double)), ("throughput_eps", C.POINTER(C.c_double)),
        ("num_slices", C.c_int32), ("replicas", C.c_int32),
        ("epochs_to_target", C.POINTER(C.c_int32)),
    ]


class Cell(C.Structure):
    _fields_ = [("eta", C.c_double), ("beta", C.c_double), ("window", C.c_int32),
                ("prior_mean", C.c_double), ("prior_var", C.c_double), ("seed", C.c_uint64)]


class Out(C.Structure):
    _fields_ = [("tot_cost", C.POINTER(C.c_double)), ("tot_energy", C.POINTER(C.c_double)),
                ("tot_time", C.POINTER(C.c_double)), ("n_stop", C.POINTER(C.c_int32)),
                ("final_arm", C.POINTER(C.c_int32)), ("cost_log", C.POINTER(C.c_double)),
                ("arm_log", C.POINTER(C.c_int32))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.literal_replay.argtypes = [C.POINTER(Trace), C.POINTER(Cell), C.c_int32, C.c_int64,
                                     C.c_int64, C.c_int32, C.c_double, C.POINTER(Out)]
        L.literal_posterior.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32, C.c_double,
                                        C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def replay(w, c, R, n, trial0=0, threads=1, logs=True, sigma_scale=1.0):
    """Replays trials trial0 .. trial0+n-1 of workload ``w`` under cell ``c`` (synth dicts)."""
    bs = np.ascontiguousarray(w["batch_sizes"], np.int32)
    pl = np.ascontiguousarray(w["power_limits"], np.float64)
    A = np.ascontiguousarray(w["avg_power"], np.float64)
    Th = np.ascontiguousarray(w["throughput"], np.float64)
    pool = np.ascontiguousarray(w["pool"], np.int32)
    S, B, K = pool.shape
    tr = Trace(len(bs), _p(bs, C.c_int32), int(w["b0"]), len(pl), _p(pl, C.c_double),
               float(w["max_power"]), int(w["max_epochs"]), int(w.get("charge_profiling", 1)),
               _p(A, C.c_double), _p(Th, C.c_double), S, K, _p(pool, C.c_int32))
    cc = Cell(float(c["eta"]), float(c["beta"]), int(c.get("window", 0)),
              float(c.get("prior_mean", 0.0)), float(c.get("prior_var", np.inf)), int(c.get("seed", 0)))
    o = {"tot_cost": np.zeros(n), "tot_energy": np.zeros(n), "tot_time": np.zeros(n),
         "n_stop": np.zeros(n, np.int32), "final_arm": np.zeros(n, np.int32)}
    if logs:
        o["cost_log"] = np.zeros((n, R))
        o["arm_log"] = np.zeros((n, R), np.int32)
    out = Out(_p(o["tot_cost"], C.c_double), _p(o["tot_energy"], C.c_double),
              _p(o["tot_time"], C.c_double), _p(o["n_stop"], C.c_int32), _p(o["final_arm"], C.c_int32),
              _p(o.get("cost_log"), C.c_double), _p(o.get("arm_log"), C.c_int32))
    if lib().literal_replay(C.byref(tr), C.byref(cc), int(R), int(trial0), int(n), int(threads),
                            float(sigma_scale), C.byref(out)) != 0:
        raise ValueError("bad arguments")
    return o


def posterior(xs, window=0, prior_mean=0.0, prior_var=np.inf):
    xs = np.ascontiguousarray(xs, np.float64)
    mu, var = C.c_double(), C.c_double()
    if lib().literal_posterior(_p(xs, C.c_double), len(xs), int(window), float(prior_mean),
                               float(prior_var), C.byref(mu), C.byref(var)) != 0:
        return None
    return {"mu": mu.value, "var": var.value}
