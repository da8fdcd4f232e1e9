"""Data-parallel decomposition over shapes (world_size 2, gloo, CPU): sharding covers
every shape once, and the all-reduced per-rank weight gradients equal the
whole-batch gradient (cnn_ops.cpp:228 matmul_trans_b) computed by the CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_11385_b200.dist import allreduce_gradients, max_over_ranks, shard_range, sum_over_ranks


@pytest.mark.parametrize("n,world", [(8, 1), (8, 2), (64, 8), (7, 3), (3, 4), (0, 2)])
def test_shard_range_partitions(n, world):
    got = []
    sizes = []
    for r in range(world):
        rr = shard_range(n, world, r)
        got += list(rr)
        sizes.append(len(rr))
    assert got == list(range(n))
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from helpers import levels_to_arrays, random_pair
        from oracle.oracle import Restated
        R = Restated()
        n_shapes, cin, cout = 6, 3, 4
        spec = (3, 1, 0, cin, cout)
        fine, _ = random_pair(16, n_shapes, seed=77)
        rng = np.random.default_rng(3)
        w = rng.uniform(-1, 1, (cout, cin * 27)).astype(np.float32)
        full = levels_to_arrays(fine)
        x_all = rng.uniform(-1, 1, (cin, full.total_columns())).astype(np.float32)
        dy_all = rng.uniform(-1, 1, (cout, full.total_columns())).astype(np.float32)
        # this rank's shapes -> its own super-PSH (local prefix arrays)
        mine = shard_range(n_shapes, world, rank)
        local = levels_to_arrays([fine[i] for i in mine])
        lo, hi = int(full.data_acc[mine.start]), int(full.data_acc[mine.stop])
        cols = R.hash2col(local, x_all[:, lo:hi], local, spec)
        dw_local = R.matmul_trans_b(dy_all[:, lo:hi], cols)
        g = torch.from_numpy(dw_local.copy())
        allreduce_gradients([g])
        t = max_over_ranks(float(rank))
        # the sync-BN hook: per-channel double sums of this rank's rows (channel-major x) ->
        # global sums, equal to the sums over the whole batch
        bn = torch.from_numpy(x_all[:, lo:hi].astype(np.float64).sum(1))
        sum_over_ranks(bn)
        if rank == 0:
            cols_all = R.hash2col(full, x_all, full, spec)
            dw_full = R.matmul_trans_b(dy_all, cols_all)
            err = float(np.abs(g.numpy() - dw_full).max() / np.abs(dw_full).max())
            # the forward is shard-local: rank 0's output columns equal the full batch's
            y_local = R.matmul(w, cols)
            y_full = R.matmul(w, cols_all)
            bn_err = float(np.abs(bn.numpy() - x_all.astype(np.float64).sum(1)).max())
            q.put((err, bool(np.array_equal(y_local, y_full[:, lo:hi])), t, len(mine), bn_err))
    finally:
        dist.destroy_process_group()


def test_two_rank_gradient_allreduce_matches_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, y_equal, tmax, nmine, bn_err = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-6, err
    assert y_equal
    assert tmax == 1.0 and nmine == 3
    assert bn_err < 1e-9, bn_err
