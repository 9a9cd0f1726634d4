"""bench.py's multi-GPU path is replicas only: one independent
array per rank, max-over-ranks time, whole-job keys/s.  The host-side logic is
exercised here with two gloo processes on CPU (the GPU legs need real devices)."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    r, w, local = bench.dist_setup(want_nccl=False)
    seed = bench.replica_seed(r)
    slowest = bench.max_over_ranks(10.0 + r, w, "cpu")
    seeds = [None] * w
    dist.all_gather_object(seeds, seed)
    out[r] = (r, w, local, seeds, slowest, bench.job_value(w, 1000, 4, slowest))
    dist.barrier()
    dist.destroy_process_group()


def test_two_replica_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    for r in range(world):
        rr, w, local, seeds, slowest, value = out[r]
        assert (rr, w, local) == (r, world, r)
        assert seeds == [bench.SEED, O.derive_seed(bench.SEED, 1, 0)]   # each rank its own array
        assert seeds[0] != seeds[1]
        assert slowest == 11.0                                          # the job's time = the slowest rank
        assert value == pytest.approx(world * 1000 * 4 / 11.0e-3)       # whole-job keys/s
