"""N > 1 host logic on CPU: world_size-2 gloo ranks shard the trials, replay their
shard (with the oracle, which stands in for the GPU library here), and all-reduce
the curves' fixed-point limbs; the result must equal one rank replaying everything,
bit for bit.  The fixed-point encoding mirrors include/zeus_sim.h
(curves_fixed): Q = RN(v 2^F), limbs Q = l0 + l1 2^26 + l2 2^52."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_06102_b200 import synth
from paper_2208_06102_b200.sharding import reduce_curves, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


F = 30


def _fixed(cost_log):
    """[trials][R] per-trial values -> [R][3] int64 limb sums (what the kernels accumulate)."""
    Q = np.rint(cost_log * 2.0 ** F).astype(np.int64)
    limbs = np.stack([Q & ((1 << 26) - 1), (Q >> 26) & ((1 << 26) - 1), Q >> 52], axis=-1)
    return limbs.sum(axis=0)


def _to_float(fx):
    return np.array([float((int(a) + (int(b) << 26) + (int(c) << 52))) * 2.0 ** -F for a, b, c in fx])


def _worker(rank, world, port, scaling, per, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    (job,) = synth.config("cfg4", trials=per)
    total, b, e = shard_range(per, world, rank, scaling)
    o = O.replay(job.workload, job.cells[0], job.recurrences, np.arange(b, e), logs=True)
    fx = torch.from_numpy(_fixed(o["cost_log"]))
    reduce_curves(fx)
    digests = [None] * world
    dist.all_gather_object(digests, o["digest"].tolist())
    if rank == 0:
        q.put((total, fx.numpy(), sum(digests, [])))
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_two_rank_shards_match_single_rank(oracle, scaling):
    per = 301
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, scaling, per, q)) for r in range(2)]
    for p in procs:
        p.start()
    total, fx, digests = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (job,) = synth.config("cfg4", trials=per)
    ref = oracle.replay(job.workload, job.cells[0], job.recurrences, np.arange(total), logs=True)
    assert total == (2 * per if scaling == "weak" else per)
    assert np.array_equal(np.array(digests, dtype=np.uint64), ref["digest"])
    assert np.array_equal(fx, _fixed(ref["cost_log"]))          # bitwise, any world size
    np.testing.assert_allclose(_to_float(fx), ref["curves"][:, 0], rtol=1e-12)


def test_shard_range_partitions():
    for world in (1, 2, 3, 8):
        for n in (0, 1, 7, 100):
            spans = [shard_range(n, world, r, "strong") for r in range(world)]
            assert spans[0][1] == 0 and spans[-1][2] == n
            assert all(spans[i][2] == spans[i + 1][1] for i in range(world - 1))
            weak = [shard_range(n, world, r, "weak") for r in range(world)]
            assert weak[-1][2] == n * world and all(w[0] == n * world for w in weak)
