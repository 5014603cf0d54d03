"""Do the jobs of a multi-job config overlap on the GPU?  Times one job alone, then all jobs
enqueued on their own streams, device-timed with events (python tools/concurrency_probe.py cfg2)."""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_06102_b200 import synth  # noqa: E402
from paper_2208_06102_b200.zeus_sim import Simulation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
jobs = synth.config(name)
sims = [Simulation(j.workload, j.cells, j.trials, j.recurrences).load_profile() for j in jobs]
streams = [torch.cuda.Stream() for _ in sims]
main = torch.cuda.current_stream()


def run(idx, reps=20):
    for _ in range(3):
        for i in idx:
            sims[i].run(streams[i])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps):
        ev = torch.cuda.Event()
        ev.record(main)
        for i in idx:
            streams[i].wait_event(ev)
            sims[i].run(streams[i])
        for i in idx:
            main.wait_stream(streams[i])
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for i in range(len(sims)):
    print(f"{name} job {i} alone: {run([i]):.3f} ms")
print(f"{name} all {len(sims)} jobs, one stream each, runs only (no results): {run(list(range(len(sims)))):.3f} ms")
