"""Thin Python binding of the C ABI in include/zeus_sim.h (argument marshalling only).

The functions ``zeus_sim_create / zeus_sim_load_profile / zeus_sim_run /
zeus_sim_results / zeus_sim_destroy / zeus_sim_last_error`` keep the C names;
``Simulation`` bundles them for one job.  Every step of the replay runs in
the CUDA library; if ``libzeus_sim.so`` is missing or no GPU is usable the
calls raise -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ZEUS_SIM_LIB selects an alternative build of the same ABI (kernel A/B experiments only)
LIB_PATH = os.environ.get("ZEUS_SIM_LIB") or os.path.join(HERE, "libzeus_sim.so")

ZEUS_OK = 0
STATUS = {0: "ZEUS_OK", 1: "ZEUS_E_INVALID", 2: "ZEUS_E_STATE", 3: "ZEUS_E_NO_CONVERGENT_ARM",
          4: "ZEUS_E_CUDA", 5: "ZEUS_E_NOMEM", 6: "ZEUS_E_UNSUPPORTED"}
CURVE_Q = 7
COUNTERS = 14
EXPORTS = ("zeus_sim_create", "zeus_sim_load_profile", "zeus_sim_run", "zeus_sim_results",
           "zeus_sim_results_async", "zeus_sim_destroy", "zeus_sim_last_error", "zeus_sim_shape", "zeus_sim_curves_from_fixed",
           "zeus_sim_certify_bounds")
CURVE_LIMBS = 3


class ZeusError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class zeus_job(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("num_batch_sizes", C.c_int32),
                ("batch_sizes", C.POINTER(C.c_int32)), ("default_bs_index", C.c_int32),
                ("num_power_limits", C.c_int32), ("power_limits_w", C.POINTER(C.c_double)),
                ("max_power_w", C.c_double), ("max_epochs", C.c_int32),
                ("charge_profiling", C.c_int32)]


class zeus_cell(C.Structure):
    _fields_ = [("eta", C.c_double), ("beta", C.c_double), ("window", C.c_int32),
                ("prior_mean", C.c_double), ("prior_var", C.c_double), ("seed", C.c_uint64),
                ("trials", C.c_int64), ("policy", C.c_int32), ("ablation", C.c_int32),
                ("arrivals", C.POINTER(C.c_double))]


class zeus_run_opts(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("recurrences", C.c_int32),
                ("shard_begin", C.c_int64), ("shard_end", C.c_int64), ("log_mode", C.c_int32),
                ("layout", C.c_int32), ("graph", C.c_int32), ("draw", C.c_int32)]


class zeus_results(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("curves", C.c_void_p), ("curves_fixed", C.c_void_p),
                ("tot_cost", C.c_void_p),
                ("tot_energy", C.c_void_p), ("tot_time", C.c_void_p), ("digest", C.c_void_p),
                ("n_stop", C.c_void_p), ("final_arm", C.c_void_p), ("pstar_index", C.c_void_p),
                ("c1", C.c_void_p), ("t1", C.c_void_p), ("e1", C.c_void_p), ("c_prof", C.c_void_p),
                ("t_prof", C.c_void_p), ("e_prof", C.c_void_p), ("opt_cost", C.c_void_p),
                ("opt_arm", C.c_void_p), ("pareto", C.c_void_p), ("log", C.c_void_p),
                ("counters", C.c_void_p),
                ("step1_ms", C.c_float), ("replay_ms", C.c_float), ("reduce_ms", C.c_float),
                ("kernel_launches", C.c_int32), ("curve_scale_bits", C.c_int32)]


_lib = None


def lib():
    """Loads libzeus_sim.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.zeus_sim_create.argtypes = [C.POINTER(zeus_job), C.POINTER(zeus_cell), C.c_int32,
                                      C.POINTER(zeus_run_opts), C.c_int32, C.POINTER(C.c_void_p)]
        L.zeus_sim_load_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                            C.c_int32, C.c_void_p]
        L.zeus_sim_run.argtypes = [C.c_void_p, C.c_void_p]
        L.zeus_sim_results.argtypes = [C.c_void_p, C.POINTER(zeus_results)]
        L.zeus_sim_results_async.argtypes = [C.c_void_p, C.POINTER(zeus_results)]
        L.zeus_sim_destroy.argtypes = [C.c_void_p]
        L.zeus_sim_destroy.restype = None
        L.zeus_sim_last_error.argtypes = [C.c_void_p]
        L.zeus_sim_last_error.restype = C.c_char_p
        L.zeus_sim_shape.argtypes = [C.c_void_p] + [C.c_void_p] * 5
        L.zeus_sim_curves_from_fixed.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.zeus_sim_certify_bounds.argtypes = [C.c_int32, C.c_void_p]
        for f in ("zeus_sim_create", "zeus_sim_load_profile", "zeus_sim_run", "zeus_sim_results", "zeus_sim_results_async",
                  "zeus_sim_shape", "zeus_sim_curves_from_fixed", "zeus_sim_certify_bounds"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(rc, handle):
    if rc != ZEUS_OK:
        raise ZeusError(rc, lib().zeus_sim_last_error(handle).decode())


# ------------------------------------------------------------------ C-named calls
def zeus_sim_create(job: zeus_job, cells, opts: zeus_run_opts, cuda_device: int = 0):
    arr = (zeus_cell * len(cells))(*cells)
    h = C.c_void_p()
    _check(lib().zeus_sim_create(C.byref(job), arr, len(cells), C.byref(opts), cuda_device,
                                 C.byref(h)), None)
    return h


def zeus_sim_load_profile(h, avg_power_w, throughput_eps, num_slices, replicas, epochs_to_target):
    _check(lib().zeus_sim_load_profile(h, _ptr(avg_power_w), _ptr(throughput_eps), num_slices,
                                       replicas, _ptr(epochs_to_target)), h)


def zeus_sim_run(h, cuda_stream=None):
    _check(lib().zeus_sim_run(h, C.c_void_p(cuda_stream or 0)), h)


def zeus_sim_results(h, res: zeus_results):
    _check(lib().zeus_sim_results(h, C.byref(res)), h)
    return res


def zeus_sim_results_async(h, res: zeus_results):
    _check(lib().zeus_sim_results_async(h, C.byref(res)), h)
    return res


def zeus_sim_curves_from_fixed(h, curves_fixed, curves):
    _check(lib().zeus_sim_curves_from_fixed(h, _ptr(curves_fixed), _ptr(curves)), h)


def zeus_sim_certify_bounds(cuda_device: int = 0):
    """Exhaustive check of the certified draw's error bounds (include/zeus_sim.h): 8 doubles."""
    out = np.zeros(8)
    _check(lib().zeus_sim_certify_bounds(int(cuda_device), _ptr(out)), None)
    return out


def zeus_sim_destroy(h):
    if h:
        lib().zeus_sim_destroy(h)


def zeus_sim_last_error(h=None) -> str:
    return lib().zeus_sim_last_error(h).decode()


def _ptr(a):
    """Address of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


# ------------------------------------------------------------------ one job
class Simulation:
    """One job (power + training trace) with its cells, on one GPU.

    ``workload`` is the dict produced by ``synth.make_workload``; ``cells`` are
    ``synth.cell`` dicts.  ``shard`` is this rank's global trial range.
    """

    def __init__(self, workload, cells, trials, recurrences=0, shard=(0, -1), log=False,
                 device=0, layout=0, graph=False, draw=0):
        self.w = workload
        bs = np.ascontiguousarray(workload["batch_sizes"], dtype=np.int32)
        pl = np.ascontiguousarray(workload["power_limits"], dtype=np.float64)
        self._keep = [bs, pl]
        job = zeus_job(C.sizeof(zeus_job), len(bs), bs.ctypes.data_as(C.POINTER(C.c_int32)),
                       int(workload["b0"]), len(pl), pl.ctypes.data_as(C.POINTER(C.c_double)),
                       float(workload["max_power"]), int(workload["max_epochs"]),
                       int(workload.get("charge_profiling", 1)))
        cs = []
        for c in cells:
            arr = c.get("arrivals")
            ptr = None
            if arr is not None:
                arr = np.ascontiguousarray(arr, dtype=np.float64)
                self._keep.append(arr)
                ptr = arr.ctypes.data_as(C.POINTER(C.c_double))
            cs.append(zeus_cell(float(c["eta"]), float(c["beta"]), int(c.get("window", 0)),
                                float(c.get("prior_mean", 0.0)), float(c.get("prior_var", math.inf)),
                                int(c.get("seed", 0)), int(trials), int(c.get("policy", 0)),
                                int(c.get("ablation", 0)), ptr))
        opts = zeus_run_opts(C.sizeof(zeus_run_opts), int(recurrences), int(shard[0]),
                             int(shard[1]), 1 if log else 0, int(layout), 1 if graph else 0,
                             int(draw))
        self.h = zeus_sim_create(job, cs, opts, device)
        R, n, nc, B, S = (C.c_int32(), C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32())
        lib().zeus_sim_shape(self.h, C.byref(R), C.byref(n), C.byref(nc), C.byref(B), None)
        self.R, self.shard_n, self.ncells, self.B = R.value, n.value, nc.value, B.value
        self.P = len(pl)
        self.log = log
        self.S = None

    def load_profile(self):
        w = self.w
        A = np.ascontiguousarray(w["avg_power"], dtype=np.float64)
        Th = np.ascontiguousarray(w["throughput"], dtype=np.float64)
        pool = np.ascontiguousarray(w["pool"], dtype=np.int32)
        S, _, K = pool.shape
        zeus_sim_load_profile(self.h, A, Th, S, K, pool)
        self.S = S
        return self

    def run(self, stream=None):
        """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None (legacy default)."""
        if stream is not None and hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        zeus_sim_run(self.h, stream)
        return self

    def results(self, want=("curves", "tot_cost", "tot_energy", "tot_time", "digest", "n_stop",
                            "final_arm", "counters"), out=None, enqueue_only=False):
        """Copies outputs into host numpy arrays (default) or into caller buffers given in
        ``out`` (numpy arrays or torch tensors, host or device).  enqueue_only: the replay
        outputs into the device or pinned host buffers of ``out`` on the run's stream, without
        waiting (zeus_sim_results_async; no timings)."""
        nc, R, n, B, S = self.ncells, self.R, self.shard_n, self.B, self.S
        shapes = {"curves": ((nc, R, CURVE_Q), np.float64),
                  "curves_fixed": ((nc, R, CURVE_Q, CURVE_LIMBS), np.int64), "tot_cost": ((n,), np.float64),
                  "tot_energy": ((n,), np.float64), "tot_time": ((n,), np.float64),
                  "digest": ((n,), np.uint64), "n_stop": ((n,), np.int32),
                  "final_arm": ((n,), np.int32), "pstar_index": ((nc, B), np.int32),
                  "c1": ((nc, B), np.float64), "t1": ((nc, B), np.float64),
                  "e1": ((nc, B), np.float64), "c_prof": ((nc, B), np.float64),
                  "t_prof": ((nc, B), np.float64), "e_prof": ((nc, B), np.float64),
                  "opt_cost": ((nc, S), np.float64), "opt_arm": ((nc, S), np.int32),
                  "pareto": ((S, B, self.P), np.uint8),
                  "log": ((n, R), np.uint32), "counters": ((COUNTERS,), np.int64)}
        bufs = dict(out or {})
        for k in want:
            if k not in bufs:
                shp, dt = shapes[k]
                bufs[k] = np.zeros(shp, dt)
        res = zeus_results()
        res.struct_size = C.sizeof(zeus_results)
        for k, v in bufs.items():
            setattr(res, k, _ptr(v).value if v is not None else None)
        if enqueue_only:
            zeus_sim_results_async(self.h, res)
            bufs["kernel_launches"] = res.kernel_launches
            bufs["curve_scale_bits"] = res.curve_scale_bits
            return bufs
        zeus_sim_results(self.h, res)
        bufs["step1_ms"] = res.step1_ms
        bufs["replay_ms"] = res.replay_ms
        bufs["reduce_ms"] = res.reduce_ms
        bufs["kernel_launches"] = res.kernel_launches
        bufs["curve_scale_bits"] = res.curve_scale_bits
        return bufs

    def curves_from_fixed(self, curves_fixed, curves):
        """Device tensors: curves [cells][R][7] from (all-reduced) curves_fixed [cells][R][7][3]."""
        zeus_sim_curves_from_fixed(self.h, curves_fixed, curves)
        return curves

    def close(self):
        zeus_sim_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.close()
        except Exception:
            pass
