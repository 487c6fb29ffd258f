"""Multi-process host logic on CPU: world_size-2 gloo process group (no GPU)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_06223_b200 import dist as L


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, lr = L.env_ranks()
        mx = L.max_over_ranks([rank * 10.0 + 1.0, -rank])
        sm = L.sum_over_ranks([1.0, rank])
        ga = L.gather_over_ranks(100.0 + rank)
        start, stop = L.shard(256, r, w)
        n_local = torch.tensor([stop - start])
        dist.all_reduce(n_local)
        q.put((rank, r, w, lr, mx, sm, (start, stop), int(n_local.item()), ga))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, r, w, lr, mx, sm, rng, n_all, ga in out:
        assert (r, w, lr) == (rank, 2, rank)
        assert mx == [11.0, 0.0]          # max over ranks
        assert sm == [2.0, 1.0]           # sum over ranks
        assert n_all == 256               # shards cover the global batch
        assert ga == [100.0, 101.0]       # per-rank values, rank order
    assert out[0][6] == (0, 128) and out[1][6] == (128, 256)


@pytest.mark.parametrize("n,world", [(256, 1), (256, 8), (10, 3), (3, 8), (0, 4)])
def test_shard_partitions(n, world):
    ranges = [L.shard(n, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_single_process_reductions_are_identity():
    assert L.max_over_ranks([3.0, 4.0]) == [3.0, 4.0]
    assert L.gather_over_ranks(5.0) == [5.0]
    assert L.throughput(128, 8, 10, 1000.0) == 128 * 8 * 10


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = L.shard(10, rank, world)
        full = torch.arange(10 * 7, dtype=torch.float32).reshape(10, 7)
        if hi - lo == 10 // world:  # equal shards (all_gather needs equal sizes)
            got = L.exchange_logits(full[lo:hi].contiguous())
        else:
            got = None
        counts = L.active_counts([rank + 1, 10 * rank])
        mx = L.max_over_ranks([float(rank)])
        q.put((rank, None if got is None else got.tolist(), counts, mx))
    finally:
        dist.destroy_process_group()


def test_gloo_exchange_step():
    """The network's exchange step on 2 gloo ranks: the logits all-gather returns the
    whole batch in rank order on every rank; active counts sum; times take the max."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = torch.arange(70, dtype=torch.float32).reshape(10, 7).tolist()
    for rank, got, counts, mx in out:
        assert got == full
        assert counts == [3, 10]
        assert mx == [1.0]


def test_bench_relaunches_under_torchrun(monkeypatch):
    """bench.py --gpus N outside torchrun re-executes itself under
    torch.distributed.run with N processes (one per GPU) and 127.0.0.1 rendezvous."""
    import importlib.util
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    args = bench.parse()
    bench.relaunch(args)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
