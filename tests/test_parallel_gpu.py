"""Batch-sharded multi-GPU path on the CUDA kernels, on one device.

Two spawned ranks (gloo for the gathers -- the data path has no collective) each take
their images parallel.shard_range(B, k, 2) of ONE global seeded draw, plan B_k images,
transform the kernels locally and run the whole CUDA forward through the C-ABI.  The
gathered output must equal the unsharded forward bit for bit for every contraction mode:
every per-image quantity (including the F16X3 per-image U scale) is independent of the
rest of the batch, so sharding changes no arithmetic.  The ranks share cuda:0 here (the
box has one GPU); their kernels never wait on one another.  bench.py's own N>1 path is
checked by a dry 2-rank run on the one device.
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


RUNS = [("winograd", 2), ("winograd", 4), ("winograd", 6), ("regular_fft", 6), ("regular_fft", 14),
        ("gauss_fft", 8), ("gauss_fft", 14), ("direct", 0)]


def _worker(rank, world, port, shape, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import synth
    import paper_1809_07851_b200 as fc
    from paper_1809_07851_b200 import parallel
    try:
        parallel.init("gloo")
        torch.cuda.set_device(0)
        fc.load()
        cfg = synth.custom(*shape, seed=111, dist="normal")
        I, W = synth.make_inputs(cfg)  # the global draw, identical on every rank
        lo, hi = parallel.shard_range(cfg.B, rank, world)
        x, w = I[lo:hi].contiguous().cuda(), W.cuda()
        res = {}
        for gemm in ("auto", "tcgen05", "ffma"):
            for method, m in RUNS:
                if method == "direct" and gemm != "auto":
                    continue
                p = fc.Plan(hi - lo, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm)
                y = p.forward(x, w).cpu()
                full = parallel.gather_batch(y, cfg.B, world)
                if rank == 0:
                    ref = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm).forward(
                        I.cuda(), w).cpu()
                    res["%s/%s/m=%d" % (gemm, method, m)] = bool(torch.equal(full, ref))
        parallel.barrier()
        if rank == 0:
            q.put(res)
    except Exception as exc:  # surface the failure in the parent
        q.put({"error": repr(exc)})
        raise
    finally:
        if torch.distributed.is_initialized():
            torch.distributed.destroy_process_group()


@pytest.mark.parametrize("shape", [(6, 32, 64, 30, 30, 3), (5, 24, 40, 21, 26, 3)])
def test_world2_sharded_equals_unsharded(shape):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert "error" not in res, res
    bad = [k for k, ok in res.items() if not ok]
    assert not bad, bad
    assert all(p.exitcode == 0 for p in procs)


def test_bench_two_ranks_dry_run():
    """bench.py --gpus 2 without torchrun relaunches itself as 2 ranks; on a one-GPU box the
    ranks share the device (oversubscribed) and rank 0 prints one line with n_gpus 2 and the
    strong-scaling shard sizes."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                          "--method", "winograd", "--m", "4", "--sweep-steps", "1", "--e2e-steps", "1",
                          "--no-extras", "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 64 and d["config"]["B_per_gpu"] == 32
    assert d["config"]["oversubscribed"] == (torch.cuda.device_count() < 2)
    assert len(d["ms_per_step_stats"]["per_rank_ms"]) == 2
    assert d["ms_per_step"] == pytest.approx(max(d["ms_per_step_stats"]["per_rank_ms"]))


ES_RUNS = [("winograd", 4, {}), ("regular_fft", 6, {}), ("regular_fft", 6, {"complex_mode": 0}),
           ("gauss_fft", 8, {"gauss_combine": 0}), ("gauss_fft", 8, {"gauss_combine": 1})]


def _es_worker(rank, world, port, shape, batch, q, p2p=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import synth
    import paper_1809_07851_b200 as fc
    from paper_1809_07851_b200 import parallel
    try:
        if world > 1:
            parallel.init("gloo")
        torch.cuda.set_device(0)
        fc.load()
        cfg = synth.custom(*shape, seed=131, dist="normal")
        I, W = synth.make_inputs(cfg)
        lo = sum(batch[:rank])
        x, w = I[lo:lo + batch[rank]].contiguous().cuda(), W.cuda()
        res = {}
        for gemm in ("auto", "tcgen05", "ffma"):
            for method, m, opts in ES_RUNS:
                es = fc.EShard(world, rank, batch, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm, **opts)
                ws = es.alloc_workspace()
                y = torch.empty(es.out_shape, device="cuda")
                if p2p:  # exchange through IPC-shared receive buffers (conv_eshard_forward_*_peer)
                    bufs = parallel.eshard_forward_p2p(es, x, w, y, ws, host_staging=True)
                    parallel.eshard_forward_p2p(es, x, w, y, ws, bufs=bufs, host_staging=True)  # buffers reused
                    torch.cuda.synchronize()
                    parallel.barrier()
                    parallel.eshard_release(bufs)
                else:
                    parallel.eshard_forward(es, x, w, y, ws, host_staging=True)
                torch.cuda.synchronize()
                ref = fc.Plan(batch[rank], cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm,
                              **opts).forward(x, w)
                # the whole batch on one plan, this rank's images
                full = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm, **opts).forward(
                    I.cuda(), w)[lo:lo + batch[rank]]
                res["%s/%s/m=%d/%s" % (gemm, method, m, opts)] = (bool(torch.equal(y, full)),
                                                                  bool(torch.equal(ref, full)))
        q.put((rank, res))
    except Exception as exc:
        q.put((rank, {"error": repr(exc)}))
        raise
    finally:
        if torch.distributed.is_initialized():
            torch.distributed.destroy_process_group()


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("shape,batch", [((5, 32, 256, 18, 18, 3), (3, 2)), ((4, 24, 64, 20, 17, 3), (1, 3)),
                                         ((3, 16, 32, 14, 14, 3), (3,))])
def test_element_sharded_equals_unsharded(shape, batch, p2p):
    """element-sharded forwards (rank j: elements [e0_j, e1_j) of every image,
    the transforms of its own images; all-to-alls of U and X) give each rank's images exactly
    the unsharded forward's output -- every contraction mode and method, complex mode on
    and off, Gauss three-plane and combined.  p2p: the exchange writes straight into the
    peers' IPC-mapped receive buffers instead of a collective (two processes on one device
    here; peer copies over NVLink across devices)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = len(batch)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_es_worker, args=(r, world, port, shape, batch, q, p2p)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, res in results:
        assert "error" not in res, (rank, res)
        bad = [k for k, (ok, _) in res.items() if not ok]
        assert not bad, (rank, bad)
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.parametrize("gpus,exchange", [(1, "collective"), (2, "collective"), (2, "p2p")])
def test_bench_eshard_mode(gpus, exchange):
    """bench.py --mode eshard prints one line per run: deep layer, FFT m = 14,
    element shards of E = 144 over the ranks."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, "bench.py", "--gpus", str(gpus), "--steps", "3", "--warmup", "3",
                          "--workload", "deep", "--mode", "eshard", "--method", "regular_fft", "--m", "14",
                          "--exchange", exchange, "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["value"] > 0 and d["config"]["parallelism"].startswith("es%d" % gpus)
    assert d["config"]["E"] == 144 and d["config"]["elements_per_rank"] == 144 // gpus
    assert d["config"]["exchange"] == exchange
