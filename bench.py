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
def work_per_launch(counters, _unused=None):
    """Algorithmic lane-instructions of one launch: the work the replay evaluated x per-primitive
    sm_100a SASS costs of the contract (tools/work_model.json):
      per Box-Muller transform evaluated      bm
      per Philox block evaluated              philox (a block feeds two pairs, NC-3)
      per survivor pair bound-screened        screen
      per normal used in a transformed pair   theta = fma + argmin step
      per decision                            the serial contract work (lookup, charge, early
                                              stop, Observe and posterior, totals, digest, curve
                                              contributions) + a quarter replica Philox block +
                                              this decision's share of the warp curve reduction
    Transforms the bound screen proved unnecessary are not counted (counters [9..11])."""
    wm = json.load(open(os.path.join(ROOT, "tools", "work_model.json")))
    c = [int(x) for x in counters]
    dec, pairs, normals = c[0], c[2], c[3]
    bm_done, blocks_done, screened = c[9], c[10], c[11]
    used = normals * bm_done / max(1, pairs)
    per_dec = {k: wm["serial"][k] + wm["philox"][k] / 4.0 + wm["curves"][k] for k in ("fp64", "total")}
    return {k: bm_done * wm["bm"][k] + blocks_done * wm["philox"][k] + screened * wm["screen"][k]
            + used * wm["theta"][k] + dec * per_dec[k] for k in ("fp64", "total")}


# ------------------------------------------------------------------ reference arm (oracle)
def cpu_sample(job, seconds, threads):
    """Times the oracle, as it stands, on a bounded prefix of the workload's trials."""
    from oracle import oracle as O

    w, c, R = job.workload, job.cells[0], job.recurrences
    n = max(threads, 64)
    while True:
        t0 = time.perf_counter()
        O.replay(w, c, R, np.arange(n), threads=threads, curves=True)
        dt = time.perf_counter() - t0
        if dt >= seconds or n >= job.trials:
            return n, dt
        n = min(job.trials, int(n * max(2.0, min(10.0, 1.2 * seconds / max(dt, 1e-3)))))


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
                             "sample": sample},
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

    build.build()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    jobs = synth.config(args.config, trials=args.trials)
    job = jobs[0]
    sims, streams, curves = [], [], []
    for jb in jobs:                                  # one handle and one stream per job
        total, begin, end = shard_range(jb.trials, world, rank, args.scaling)
        sm = Simulation(jb.workload, jb.cells, total, jb.recurrences, shard=(begin, end),
                        device=local, layout=args.layout, graph=bool(args.graph)).load_profile()
        sims.append(sm)
        streams.append(torch.cuda.Stream(device=dev))
        curves.append(torch.zeros((sm.ncells, sm.R, 7), dtype=torch.float64, device=dev))
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
        for sm, st, cv in zip(sims, streams, curves):
            with torch.cuda.stream(st):
                r = sm.results(want=["counters"], out={"curves": cv})
                reduce_curves(cv)
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
            counters = np.sum([r["counters"] for r in outs], axis=0)
        torch.cuda.synchronize()
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
        staged.append((A_h, Th_h, pool_h, host_out))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        for sm, st, (A_h, Th_h, pool_h, host_out) in zip(sims, streams, staged):
            Z.zeus_sim_load_profile(sm.h, A_h, Th_h, pool_h.shape[0], pool_h.shape[2], pool_h)
            sm.run(st)
        for sm, (A_h, Th_h, pool_h, host_out) in zip(sims, staged):
            sm.results(want=[], out=host_out)
            if dist:
                cur_h = torch.from_numpy(host_out["curves"])
                cur_h.copy_(reduce_curves(cur_h.to(dev)).cpu())
    torch.cuda.synchronize()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = dec_per_step * e2e_steps / float(e2e_s[0])

    # ---- roofline of the dominant kernel group (the replay): algorithmic lane-instructions /
    # its CUDA-event duration on the launching stream (whole step for multi-job configs)
    work = work_per_launch(counters, None)
    launch_s = replay_total / args.steps / 1e3
    clock_hz = (clocks["sm_mhz"] or 1965.0) * 1e6
    peak_issue = ISSUE_LANES_PER_CLK_SM * SM_COUNT * clock_hz
    peak_fp64 = FP64_LANES_PER_CLK_SM * SM_COUNT * clock_hz
    ach_issue, ach_fp64 = work["total"] / launch_s, work["fp64"] / launch_s
    prof = os.path.join(ROOT, "profiles", "replay_traffic.json")
    traffic = None
    if os.path.exists(prof):
        tr = json.load(open(prof))
        traffic = tr["dram_bytes_per_decision"] * dec_per_step / world
    roofline = {"bound": "alu", "achieved": ach_issue / 1e12, "peak": peak_issue / 1e12,
                "unit": "T lane-inst/s", "frac": ach_issue / peak_issue, "traffic": traffic,
                "kernel": "replay (phase A + regroup + phase B kernels)" if single else "whole step",
                "launch_ms": launch_s * 1e3,
                "work_per_decision": work["total"] / max(1, int(counters[0])),
                "peak_basis": f"issue: {ISSUE_LANES_PER_CLK_SM} lanes/clk/SM x {SM_COUNT} SMs x "
                              f"median SM clock under load {clock_hz / 1e6:.0f} MHz",
                "fp64": {"achieved": ach_fp64 / 1e12, "peak": peak_fp64 / 1e12,
                         "frac": ach_fp64 / peak_fp64,
                         "peak_basis": f"{FP64_LANES_PER_CLK_SM} FP64 lanes/clk/SM (measured "
                                       "1.82e13 DFMA lane/s at 1965 MHz, tools/peaks.cu)"}}

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
            threads = os.cpu_count() or 1
            n, dt = cpu_sample(job, args.cpu_seconds, threads)
            line["cpu_baseline"] = {"value": n * job.recurrences / dt, "unit": UNIT, "cores": threads,
                                    "kind": "oracle",
                                    "sample": f"first {n} trials x {job.recurrences} recurrences of "
                                              f"{args.config}, {dt:.1f} s on {threads} threads"}
        print(json.dumps(line), flush=True)
    for sm in sims:
        sm.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
