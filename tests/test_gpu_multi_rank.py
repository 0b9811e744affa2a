"""Two ranks driving the CUDA path (GPU box; both ranks share its one GPU).

Each rank plans from the same window, transforms its contiguous shard of a batch with the
fused hot-path kernel, and rank 0 gathers the shards (gloo: NCCL refuses two ranks on one
device).  The gathered coefficients must equal a single-process transform of the whole batch
bit for bit (same kernels, same per-signal work, no data-path collective).
The ranks' kernels never wait on one another, so sharing one GPU is only a functional check.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws), RANK=str(rank),
                      LOCAL_RANK=str(rank), NSDGT_DIST_BACKEND="gloo")
    import torch
    import torch.distributed as dist

    import paper_1307_4569_b200 as nsdgt
    from paper_1307_4569_b200 import dist as pd
    from synthetic import CONFIGS, batch, window
    pd.init()
    try:
        wl = CONFIGS[2]   # config 3's lattice (fused path), a small batch
        W = 7
        w0, w1 = pd.shard(W, ws, rank)
        plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype="c64")
        c = plan.execute(torch.from_numpy(batch(wl, w0, w1)).cuda()).cpu()
        full = pd.gather_to_rank0(c, W)
        pd.barrier()
        if rank == 0:
            out_q.put((full.numpy(), plan.info["kernel_path"]))
    finally:
        dist.destroy_process_group()


def test_two_ranks_cuda_shards_equal_single_process():
    import torch
    import torch.multiprocessing as mp

    import paper_1307_4569_b200 as nsdgt
    from synthetic import CONFIGS, batch, window
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    got, path = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    wl = CONFIGS[2]
    plan = nsdgt.Plan(wl.L, wl.a, wl.M, wl.lam1, wl.lam2, window(wl), dtype="c64")
    ref = plan.execute(torch.from_numpy(batch(wl, 0, 7)).cuda()).cpu().numpy()
    assert path == 2
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)
