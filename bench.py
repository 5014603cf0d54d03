"""Benchmark: simulated bandit decisions/sec (trials x recurrences) of the batched
Zeus replay on B200 (BASELINE.json ``metric``).

One step = one pass of the whole hot path over the bench
workload: step 1 (Eq. 7) for every cell, the replay kernel over every trial of
this rank for R recurrences, the curve reduction, and -- at N > 1 -- the NCCL
all-reduce of the curves.  Default workload: CFG5 (10^7 trials x 1000
recurrences, 16 batch sizes x 16 power limits) per GPU ("scaling": "weak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.  ``--impl reference`` times the CPU oracle
(the reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2208_06102_b200 import synth  # noqa: E402
from paper_2208_06102_b200.sharding import reduce_curves, shard_range  # noqa: E402

METRIC = "simulated bandit decisions/sec (trials x recurrences) at 1/2/4/8 B200 vs roofline"
UNIT = "decisions/s"
SM_COUNT = 148
ISSUE_LANES_PER_CLK_SM = 128      # 4 SMSPs x 1 warp-instruction x 32 lanes
FP64_LANES_PER_CLK_SM = 64        # DFMA/DADD/DMUL lanes per SM per clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg5", choices=list(synth.CONFIGS) + ["cfg4_38"] + list(synth.NEXT))
    ap.add_argument("--trials", type=int, default=None, help="trials per cell per GPU (default: the config's)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--layout", type=int, default=0)
    ap.add_argument("--graph", type=int, default=0, choices=(0, 1),
                    help="1: each handle's run is one CUDA-graph launch (zeus_run_opts.graph)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--dump", default=None,
                    help="directory: each rank writes rank<r>.npz (shard, per-trial digests and "
                         "costs, curves) after the timed steps (multi-rank parity tests)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:   # first sample before timing starts
                time.sleep(0.05)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ work model
PIPES = ("fp64", "alu", "fma", "total")
# lanes per clock per SM of each pipe (B200: 4 SMSPs; DESIGN.md §8 derives them from the guides and
# tools/peaks.cu): the FP64 unit, the alu pipe (LOP3/IADD3/SHF/SEL/ISETP), the fma pipe (IMAD*),
# and issue (one warp-instruction per SMSP per clock)
PIPE_LANES = {"fp64": 64, "alu": 64, "fma": 64, "total": ISSUE_LANES_PER_CLK_SM}


def _work_model():
    return json.load(open(os.path.join(ROOT, "tools", "work_model.json")))


def method_work(counters):
    """the algorithmic lane-instructions of the METHOD's events, by pipe.  Alg. 1
    samples every survivor, so every survivor pair is one Box-Muller transform
    (counter [2]), every quad with a survivor one Philox block ([8]), every normal used one
    θ = fma + argmin step ([3]); every decision ([0]) does the serial contract work (lookup,
    charge, early stop, Observe + posterior, totals, digest, curve contributions), a quarter of
    a replica Philox block and its share of the warp curve reduction.  Costs per primitive:
    sm_100a SASS of the contract functions (tools/work_model.json).  The counters are the
    oracle-checked event counts, so W does not depend on what the kernel skipped."""
    wm = _work_model()
    c = [int(x) for x in counters]
    dec, pairs, normals, blocks = c[0], c[2], c[3], c[8]
    return {k: pairs * wm["bm"][k] + blocks * wm["philox"][k] + normals * wm["theta"][k]
            + dec * (wm["serial"][k] + wm["philox"][k] / 4.0 + wm["curves"][k]) for k in PIPES}


def evaluated_work(counters):
    """The work this build evaluated for the same events: the fp64 Box-Muller transforms it
    performed ([9]), the Philox blocks it drew ([10]), and [11] either the pairs the bound screen
    handled or -- when the Thompson phase ran the certified draw ([12] + [13] > 0,
    §7.9) -- the pairs transformed in fp32 with their bound and packed-key argmin update."""
    wm = _work_model()
    c = [int(x) for x in counters]
    dec, pairs, normals = c[0], c[2], c[3]
    bm_done, blocks_done, handled = c[9], c[10], c[11]
    certified = len(c) > 13 and c[12] + c[13] > 0
    per_pair = wm["fpair"] if certified else wm["screen"]
    used = normals * bm_done / max(1, pairs)
    return {k: bm_done * wm["bm"][k] + blocks_done * wm["philox"][k] + handled * per_pair[k]
            + used * wm["theta"][k] + dec * (wm["serial"][k] + wm["philox"][k] / 4.0 + wm["curves"][k])
            for k in PIPES}


def roofline_of(counters, launch_s, clock_hz, dram_bytes, single):
    """t_bound = max over {FP64 unit, alu pipe, fma pipe, issue, HBM} of work / peak (SURVEY
    §8(d)); frac = t_bound / t_measured.  `achieved` / `peak` are those of the binding resource."""
    W = method_work(counters)
    E = evaluated_work(counters)
    peaks = {k: PIPE_LANES[k] * SM_COUNT * clock_hz for k in PIPES}
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9 \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6.65e12
    t_pipe = {k: W[k] / peaks[k] for k in PIPES}
    t_hbm = (dram_bytes or 0.0) / hbm
    bind = max(t_pipe, key=t_pipe.get)
    dec = max(1, int(counters[0]))
    name = {"total": "issue", "alu": "alu pipe", "fma": "fma pipe", "fp64": "FP64 unit"}
    return {"bound": "alu", "binding": name[bind],
            "achieved": W[bind] / launch_s / 1e12, "peak": peaks[bind] / 1e12, "unit": "T lane-inst/s",
            "frac": t_pipe[bind] / launch_s, "traffic": None,
            "kernel": "replay (phase A + regroup + phase B kernels)" if single else "whole step",
            "launch_ms": launch_s * 1e3,
            "method_work_per_decision": {k: W[k] / dec for k in PIPES},
            "pipes": {name[k]: {"achieved": W[k] / launch_s / 1e12, "peak": peaks[k] / 1e12,
                                "frac": t_pipe[k] / launch_s} for k in PIPES},
            "hbm": {"bytes": dram_bytes, "t_bound_ms": 1e3 * t_hbm},
            "evaluated": {"work_per_decision": E["total"] / dec,
                          "achieved": E["total"] / launch_s / 1e12,
                          "frac_of_issue": E["total"] / launch_s / peaks["total"]},
            "peak_basis": f"lanes/clk/SM: FP64 64, alu 64, fma 64, issue {ISSUE_LANES_PER_CLK_SM} "
                          f"(tools/peaks.cu, DESIGN.md §8) x {SM_COUNT} SMs x median SM clock under "
                          f"load {clock_hz / 1e6:.0f} MHz"}


# ------------------------------------------------------------------ reference arm (oracle)
def cpu_sample(job, seconds, threads):
    """Times the oracle, as it stands, on a bounded prefix of the workload's trials."""
    from oracle import oracle as O

    w, c, R = job.workload, job.cells[0], job.recurrences
    n = max(threads, 16)
    while True:
        t0 = time.perf_counter()
        O.replay(w, c, R, np.arange(n), threads=threads, curves=True)
        dt = time.perf_counter() - t0
        if dt >= seconds or n >= job.trials:
            return n, dt
        n = min(job.trials, int(n * max(2.0, min(10.0, 1.2 * seconds / max(dt, 1e-3)))))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(args, jobs, seconds):
    """the oracle as it stands on the host's cores.  The whole workload (every job,
    cell and trial) when it takes at most ~2 * `seconds` on all threads, else a bounded prefix of
    the first cell's trials; plus the 1-thread rate on a small prefix and the CPU model."""
    from oracle import oracle as O

    threads = os.cpu_count() or 1
    job = jobs[0]
    n, dt = cpu_sample(job, min(seconds, 4.0), threads)            # rate estimate
    rate = n * job.recurrences / dt
    total = sum(len(jb.cells) * jb.trials * jb.recurrences for jb in jobs)
    if total / rate <= 2.0 * seconds:
        t0 = time.perf_counter()
        for jb in jobs:
            for c in jb.cells:
                O.replay(jb.workload, c, jb.recurrences, np.arange(jb.trials), threads=threads, curves=True)
        dt = time.perf_counter() - t0
        value, sample, full = total / dt, f"the whole {args.config} workload ({total:.3g} decisions), {dt:.1f} s", True
    else:
        n, dt = cpu_sample(job, seconds, threads)
        value, full = n * job.recurrences / dt, False
        sample = (f"first {n} of {job.trials} trials x {job.recurrences} recurrences of {args.config} "
                  f"({job.workload['name']}, cell 0), {dt:.1f} s")
    n1, dt1 = cpu_sample(job, min(3.0, seconds / 4), 1)
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
            "full_workload": full, "value_1thread": n1 * job.recurrences / dt1,
            "sample_1thread": f"first {n1} trials of cell 0, {dt1:.1f} s on 1 thread", "cpu_model": cpu_model()}


def reference_main(args, rank, world):
    if rank != 0:
        return
    jobs = synth.config(args.config, trials=args.trials)
    job = jobs[0]
    threads = os.cpu_count() or 1
    per_step_s = min(args.cpu_seconds, max(1.0, min(15.0, 90.0 / max(1, args.steps + args.warmup))))
    n, _ = cpu_sample(job, per_step_s, threads)
    from oracle import oracle as O

    for _ in range(args.warmup):
        O.replay(job.workload, job.cells[0], job.recurrences, np.arange(n), threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.replay(job.workload, job.cells[0], job.recurrences, np.arange(n), threads=threads)
        times.append(time.perf_counter() - t0)
    dps = n * job.recurrences * len(times) / sum(times)
    sample = (f"first {n} of {job.trials} trials x {job.recurrences} recurrences of "
              f"{args.config} ({job.workload['name']}), per step")
    line = {"impl": "reference", "metric": METRIC, "value": dps, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, job, 1),
            "cpu_baseline": {"value": dps, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": dps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, jobs, world):
    jobs = jobs if isinstance(jobs, list) else [jobs]
    job = jobs[0]
    w = job.workload
    names = ",".join(j.workload["name"] for j in jobs)
    return {"workload": f"{args.config}: {names} synthetic trace(s), {len(w['batch_sizes'])} batch sizes x "
                        f"{len(w['power_limits'])} power limits, {len(job.cells)} cell(s) per job, "
                        f"{job.recurrences} recurrences",
            "jobs": len(jobs),
            "trials_per_gpu_per_cell": job.trials if args.scaling == "weak" else job.trials // world,
            "cells": len(job.cells), "recurrences": job.recurrences,
            "batch_sizes": len(w["batch_sizes"]), "power_limits": len(w["power_limits"]),
            "slices": int(w["pool"].shape[0]), "replicas": int(w["pool"].shape[2]),
            "eta": job.cells[0]["eta"], "beta": job.cells[0]["beta"], "window": job.cells[0]["window"],
            "l2": "flushed between timed steps (256 MiB memset); inputs are KB-sized tables staged to smem",
            "cuda_graph": bool(args.graph),
            "parallelism": f"trials sharded over {world} GPU(s), NCCL all-reduce of curves"}


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        import torch

        if args.impl == "ours":
            torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
        # NCCL over NVLink for the curve all-reduce; ZEUS_DIST_BACKEND=gloo lets several ranks
        # share one GPU when the multi-rank path itself is under test
        backend = os.environ.get("ZEUS_DIST_BACKEND", "nccl" if args.impl == "ours" else "gloo")
        dist.init_process_group(backend)
    if args.impl == "reference":
        reference_main(args, rank, world)
        if dist:
            dist.destroy_process_group()
        return

    import torch

    from paper_2208_06102_b200 import build
    from paper_2208_06102_b200.zeus_sim import Simulation

    if local == 0:                                   # one builder per node; the others wait
        build.build()
    if dist:
        dist.barrier()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    jobs = synth.config(args.config, trials=args.trials)
    job = jobs[0]
    sims, streams, curves, fixed = [], [], [], []
    for jb in jobs:                                  # one handle and one stream per job
        total, begin, end = shard_range(jb.trials, world, rank, args.scaling)
        sm = Simulation(jb.workload, jb.cells, total, jb.recurrences, shard=(begin, end),
                        device=local, layout=args.layout, graph=bool(args.graph)).load_profile()
        sims.append(sm)
        streams.append(torch.cuda.Stream(device=dev))
        curves.append(torch.zeros((sm.ncells, sm.R, 7), dtype=torch.float64, device=dev))
        fixed.append(torch.zeros((sm.ncells, sm.R, 7, 3), dtype=torch.int64, device=dev))
    main = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    launches = []

    def step():
        """All jobs of the config concurrently (one stream each); curves all-reduced (a8)."""
        start = torch.cuda.Event()
        start.record(main)
        outs = []
        for sm, st, cv in zip(sims, streams, curves):
            st.wait_event(start)
            sm.run(st)
        for sm, st, cv, fx in zip(sims, streams, curves, fixed):
            with torch.cuda.stream(st):
                # one job: synchronous, for the replay's event time (the roofline); several: the
                # curves handed over in stream order (zeus_sim_results_async), no host round trip
                # per job; their counters are read once after the timed steps
                if len(sims) == 1:
                    r = sm.results(want=["counters"], out={"curves": cv, "curves_fixed": fx})
                else:
                    r = sm.results(want=[], out={"curves": cv, "curves_fixed": fx}, enqueue_only=True)
                if dist:                             # a8: exact all-reduce, then one rounding
                    reduce_curves(fx)
                    sm.curves_from_fixed(fx, cv)
            outs.append(r)
            main.wait_stream(st)
        launches.append(sum(r["kernel_launches"] for r in outs))
        return outs

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    replay_ms, counters = [], None
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            with torch.cuda.stream(main):
                flush.zero_()                        # L2 flush outside the timed events
            ev[i][0].record(main)
            outs = step()
            ev[i][1].record(main)
            replay_ms.append(sum(r["replay_ms"] for r in outs) if len(outs) == 1 else None)
        torch.cuda.synchronize()
    # the event counters of the last step (every run resets them)
    counters = np.sum([sm.results(want=["counters"])["counters"] for sm in sims], axis=0)
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    single = len(sims) == 1
    t_local = torch.tensor([sum(step_ms), sum(replay_ms) if single else sum(step_ms)],
                           dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms, replay_total = float(t_local[0]), float(t_local[1])
    dec_per_step = sum(sm.shard_n * sm.R for sm in sims) * world   # shards are equal across ranks
    if args.scaling == "strong":
        dec_per_step = sum(jb.trials * len(jb.cells) * sm.R for jb, sm in zip(jobs, sims))
    value = dec_per_step * args.steps / (total_ms / 1e3)
    clocks = clk.summary()

    # ---- e2e: public API with host buffers, H2D of the traces and D2H of the results every step
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 3))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    from paper_2208_06102_b200 import zeus_sim as Z

    h2d = d2h = 0
    staged = []
    for jb, sm in zip(jobs, sims):
        w = jb.workload
        A_h, Th_h, pool_h = pin(w["avg_power"]), pin(w["throughput"]), pin(w["pool"].astype(np.int32))
        n_out = sm.shard_n
        host_out = {"curves": pin(np.zeros((sm.ncells, sm.R, 7))), "tot_cost": pin(np.zeros(n_out)),
                    "tot_energy": pin(np.zeros(n_out)), "tot_time": pin(np.zeros(n_out)),
                    "digest": pin(np.zeros(n_out, np.uint64))}
        h2d += A_h.nbytes + Th_h.nbytes + pool_h.nbytes
        d2h += sum(a.nbytes for a in host_out.values())
        # the C-named calls with their argument structs built once (the per-step calls then
        # marshal nothing): zeus_sim_load_profile / zeus_sim_run / zeus_sim_results
        res = Z.zeus_results()                      # pinned host destinations (zeus_sim_results_async)
        res.struct_size = Z.C.sizeof(Z.zeus_results)
        for k, v in host_out.items():
            setattr(res, k, Z._ptr(v).value)
        staged.append((A_h, Th_h, pool_h, host_out, res))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    calls = [(sm.h, st.cuda_stream, Z._ptr(A_h), Z._ptr(Th_h), pool_h.shape[0], pool_h.shape[2], Z._ptr(pool_h))
             for sm, st, (A_h, Th_h, pool_h, _, _) in zip(sims, streams, staged)]
    for _ in range(e2e_steps):
        for h, stream, A_p, Th_p, S_n, K_n, pool_p in calls:
            Z._check(Z.lib().zeus_sim_load_profile(h, A_p, Th_p, S_n, K_n, pool_p), h)
            Z._check(Z.lib().zeus_sim_run(h, Z.C.c_void_p(stream)), h)
        for sm, fx, cv, (A_h, Th_h, pool_h, host_out, res) in zip(sims, fixed, curves, staged):
            if dist:
                sm.results(want=[], out=dict(host_out, curves=None, curves_fixed=fx))
                reduce_curves(fx)
                sm.curves_from_fixed(fx, cv)
                torch.from_numpy(host_out["curves"]).copy_(cv.cpu())
            else:                                # every job's copies queued, then one wait
                Z.zeus_sim_results_async(sm.h, res)
        torch.cuda.synchronize()                 # this step's results are in host memory
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = dec_per_step * e2e_steps / float(e2e_s[0])

    # ---- roofline of the dominant kernel group (the replay): the method's work
    # over the replay's CUDA-event duration on its launching stream (whole step for multi-job
    # configs); traffic from the committed ncu capture of this build (profiles/replay_traffic.json)
    launch_s = replay_total / args.steps / 1e3
    clock_hz = (clocks["sm_mhz"] or 1965.0) * 1e6
    roofline = roofline_of(counters, launch_s, clock_hz, None, single)
    prof = os.path.join(ROOT, "profiles", "replay_traffic.json")
    if os.path.exists(prof) and args.config == "cfg5":
        tr = json.load(open(prof))
        roofline["traffic"] = tr["dram_bytes_per_decision"] * dec_per_step / world
        roofline["traffic_source"] = tr.get("source")
        roofline["hbm"] = {"bytes": roofline["traffic"],
                           "t_bound_ms": 1e3 * roofline["traffic"] / (json.load(open(os.path.join(
                               ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9)
                           if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None}
    if os.path.exists(os.path.join(ROOT, "profiles", "replay_executed.json")) and args.config == "cfg5":
        ex = json.load(open(os.path.join(ROOT, "profiles", "replay_executed.json")))
        roofline["executed"] = ex

    if args.dump:                                    # per-rank outputs for the parity tests
        os.makedirs(args.dump, exist_ok=True)
        for i, (jb, sm) in enumerate(zip(jobs, sims)):
            total, begin, end = shard_range(jb.trials, world, rank, args.scaling)
            o = sm.results(want=["digest", "tot_cost", "n_stop", "final_arm"])
            np.savez(os.path.join(args.dump, f"rank{rank}_job{i}.npz"), begin=begin, end=end,
                     total=total, digest=o["digest"], tot_cost=o["tot_cost"], n_stop=o["n_stop"],
                     final_arm=o["final_arm"], curves=curves[i].cpu().numpy(),
                     curves_fixed=fixed[i].cpu().numpy())

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generator, DESIGN.md §5)",
                "config": workload_config(args, jobs, world), "clocks": clocks,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "steps": e2e_steps},
                "gpu_launches": int(sum(launches[-args.steps:])), "roofline": roofline,
                "replay_ms_per_step": replay_total / args.steps, "jobs": len(jobs),
                "counters_per_step": [int(x) for x in counters]}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args, jobs, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    for sm in sims:
        sm.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
