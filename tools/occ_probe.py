"""Device-timed replay of one cell of a small-arm workload at throughput scale (1e6 trials x 1000
recurrences): a configuration whose shared memory does not cap residency, for occupancy A/Bs
(python tools/occ_probe.py [workload] [trials] [R])."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_06102_b200 import synth  # noqa: E402
from paper_2208_06102_b200.zeus_sim import Simulation  # noqa: E402

wname = sys.argv[1] if len(sys.argv) > 1 else "deepspeech2"
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
R = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
w = synth.make_workload(wname, 2208)
sim = Simulation(w, [synth.cell(seed=7)], trials, R).load_profile()
for _ in range(2):
    sim.run()
torch.cuda.synchronize()
ms = []
for _ in range(3):
    r = sim.run().results(want=["counters"])
    ms.append(r["replay_ms"])
print(f"{wname} B={len(w['batch_sizes'])} trials={trials} R={R}: replay {min(ms):.2f} ms, "
      f"{trials * R / (min(ms) / 1e3):.4g} decisions/s")
