"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

The path shards the batch of independent signals over ranks with no data-path collective
(SURVEY.md §8(e)); these tests check the partition, the MAX/SUM reductions used for the
device timing, and the validation gather, with the CPU oracle standing in for each rank's
transform (the per-rank CUDA transform is covered by the single-GPU parity tests).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1307_4569_b200 import dist as pd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_partition():
    for W in (0, 1, 2, 7, 16, 1024):
        for ws in (1, 2, 3, 4, 8):
            parts = [pd.shard(W, ws, r) for r in range(ws)]
            assert parts[0][0] == 0 and parts[-1][1] == W
            for (a0, b0), (a1, b1) in zip(parts, parts[1:]):
                assert b0 == a1
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        pd.shard(8, 2, 2)


def _worker(rank, ws, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    import oracle
    from synthetic import random_pair
    import torch.distributed as dist
    pd.init(backend="gloo")
    try:
        L, a, M, l1, l2, W = 96, 8, 12, 1, 2, 5
        fs = np.stack([random_pair(L, 100 + w)[0] for w in range(W)])
        _, g = random_pair(L, 7)
        w0, w1 = pd.shard(W, ws, rank)
        local = torch.from_numpy(oracle.dgt(fs[w0:w1], g, a, M, l1, l2))
        full = pd.gather_to_rank0(local, W)
        tmax = pd.allreduce(float(rank + 1), "max")
        tsum = pd.allreduce(float(w1 - w0), "sum")
        pd.barrier()
        if rank == 0:
            ref = oracle.dgt(fs, g, a, M, l1, l2)
            out_q.put((float(np.abs(full.numpy() - ref).max()), tmax, tsum))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_gather_reduce():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    err, tmax, tsum = q.get(timeout=10)
    assert err == 0.0          # sharded results gathered in order equal the single-process result
    assert tmax == 2.0         # MAX over ranks (device time is the max over ranks)
    assert tsum == 5.0         # every signal processed exactly once


def _bench_dry_run(*extra):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", *extra],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout   # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_spawns_ranks_weak():
    """`python bench.py --gpus 2` without torchrun re-executes itself with 2 ranks (gloo on CPU);
    weak scaling: every rank its own W signals, disjoint."""
    d = _bench_dry_run()
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    shards = sorted((r, a, b) for r, a, b in d["shards"])
    assert [r for r, _, _ in shards] == [0, 1]
    assert shards[0][1:] == (0, 1024) and shards[1][1:] == (1024, 2048)


def test_bench_spawns_ranks_strong():
    d = _bench_dry_run("--scaling", "strong")
    shards = sorted((r, a, b) for r, a, b in d["shards"])
    assert shards[0][1:] == (0, 512) and shards[1][1:] == (512, 1024)
