"""N>1 host path on CPU: world_size-2 gloo processes shard the batch with
parallel.shard_range, each computes its shard (test-only stand-in: the fp64
oracle -- the CUDA path needs a GPU), outputs are all-gathered with
parallel.gather_batch and must equal the unsharded result bit for bit; the
max-over-ranks timing reduction is checked too."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1809_07851_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import oracle
    import synth
    r, w, _ = parallel.init("gloo")
    assert (r, w) == (rank, world)
    cfg = synth.custom(B, 3, 4, 10, 9, 3, seed=5)
    I, W = synth.make_inputs(cfg)          # globally drawn, identical on every rank
    lo, hi = parallel.shard_range(B, r, w)
    local = torch.from_numpy(oracle.conv_fp64(I[lo:hi].contiguous(), W))
    full = parallel.gather_batch(local, B, w)
    t = parallel.max_over_ranks(1.0 + r)
    parallel.barrier()
    if r == 0:
        ref = oracle.conv_fp64(I, W)
        q.put((bool(np.array_equal(full.numpy(), ref)), t))
    torch.distributed.destroy_process_group()


@pytest.mark.parametrize("B", [4, 5])
def test_gloo_world2_shard_gather(B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    assert t == 2.0


def test_shard_range_partitions():
    for B in (1, 7, 64, 128):
        for world in (1, 2, 3, 4, 8):
            spans = [parallel.shard_range(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard_range(4, 2, 2)
