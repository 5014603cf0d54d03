"""Host-side breakdown of bench.py's e2e loop (public API, pinned host buffers) for one config:
per step, the wall time of the enqueue loop (load_profile + run per job), of the results loop
(synchronises and copies), and of the whole step, next to the device-timed step.
usage: python tools/e2e_probe.py [config] [steps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2208_06102_b200 import synth  # noqa: E402
from paper_2208_06102_b200 import zeus_sim as Z  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
jobs = synth.config(cfg)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
sims, streams, staged = [], [], []
for jb in jobs:
    sm = Z.Simulation(jb.workload, jb.cells, jb.trials, jb.recurrences, device=0).load_profile()
    sims.append(sm)
    streams.append(torch.cuda.Stream())
    w = jb.workload
    n = sm.shard_n
    out = {"curves": pin(np.zeros((sm.ncells, sm.R, 7))), "tot_cost": pin(np.zeros(n)),
           "tot_energy": pin(np.zeros(n)), "tot_time": pin(np.zeros(n)), "digest": pin(np.zeros(n, np.uint64))}
    staged.append((pin(w["avg_power"]), pin(w["throughput"]), pin(w["pool"].astype(np.int32)), out))


def one(mode):
    t0 = time.perf_counter()
    for sm, st, (A, Th, pool, out) in zip(sims, streams, staged):
        if mode != "noload":
            Z.zeus_sim_load_profile(sm.h, A, Th, pool.shape[0], pool.shape[2], pool)
        sm.run(st)
    t1 = time.perf_counter()
    for sm, (A, Th, pool, out) in zip(sims, staged):
        sm.results(want=[], out=out)
    t2 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t2 - t0) * 1e3


def per_call():
    """host time of each call type per job (median over steps), after a device sync"""
    tl, tr, ts = [], [], []
    for _ in range(steps):
        torch.cuda.synchronize()
        for sm, st, (A, Th, pool, out) in zip(sims, streams, staged):
            t0 = time.perf_counter()
            Z.zeus_sim_load_profile(sm.h, A, Th, pool.shape[0], pool.shape[2], pool)
            t1 = time.perf_counter()
            sm.run(st)
            t2 = time.perf_counter()
            tl.append(t1 - t0)
            tr.append(t2 - t1)
        torch.cuda.synchronize()
        for sm, (A, Th, pool, out) in zip(sims, staged):
            t0 = time.perf_counter()
            sm.results(want=[], out=out)
            ts.append(time.perf_counter() - t0)
    print(f"{cfg} per call (host, us): load_profile {np.median(tl) * 1e6:.1f}, run {np.median(tr) * 1e6:.1f}, "
          f"results after sync {np.median(ts) * 1e6:.1f}")


per_call()
for mode in ("full", "noload"):
    for _ in range(3):
        one(mode)
    torch.cuda.synchronize()
    r = np.array([one(mode) for _ in range(steps)])
    dec = sum(sm.shard_n * sm.R for sm in sims)
    print(f"{cfg} {mode}: enqueue {np.median(r[:, 0]):.3f} ms, results {np.median(r[:, 1]):.3f} ms, "
          f"step {np.median(r[:, 2]):.3f} ms (median of {steps}) -> {dec / np.median(r[:, 2]) * 1e3:.3g} dec/s")
# device-timed step (events around the runs on one stream each)
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
main = torch.cuda.current_stream()
ts = []
for _ in range(steps):
    s0.record(main)
    for sm, st in zip(sims, streams):
        st.wait_event(s0)
        sm.run(st)
    for st in streams:
        main.wait_stream(st)
    s1.record(main)
    torch.cuda.synchronize()
    ts.append(s0.elapsed_time(s1))
print(f"{cfg} device step (runs only) {np.median(ts):.3f} ms")
