"""Data-parallel native net with synchronised batch norm: two ranks on the
one visible GPU (gloo carries the CUDA tensors), each with half of the shapes, all-reducing
the batch-norm statistics (hc_native_bn_stat / _finalize / _apply phases) and the weight
gradients, must reproduce the single-process whole-batch step: BN normalises over the
global batch exactly as the reference does for one process (cnn_ops.cpp:456-470).
Differences are summation order only (per-rank dW splits, double BN sums)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _setup(b_total, shapes):
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from paper_1803_11385_b200 import net as nnet
    from paper_1803_11385_b200.psh import SuperPsh
    pyr = bench.shell_pyramid(16)
    levels = [SuperPsh.from_levels([lv] * len(shapes)) for lv in pyr]
    n1 = pyr[0].n
    g = torch.Generator(device="cuda").manual_seed(5)
    feats = torch.rand((3, n1 * b_total), device="cuda", generator=g) * 2 - 1
    cols = torch.cat([feats[:, s * n1:(s + 1) * n1] for s in shapes], dim=1)
    labels = torch.tensor([s % 4 for s in shapes], device="cuda")
    return nnet, levels, cols, labels


def _run(nnet, levels, cols, labels, b_total, sync_bn, epilogue_stats=True):
    net = nnet.NativeHashNet(4, 4, seed=1, dropout=0.0, sync_bn=sync_bn)
    net.epilogue_stats = epilogue_stats
    nb = nnet.NetBatch.build(levels)
    x = net.input_features(cols)
    loss, conv_g, head_g = net.loss_and_gradients(nb, x, labels, b_total)
    return net, float(loss), list(conv_g), [g.contiguous() for g in head_g]


def test_phased_bn_equals_fused_bn_single_rank(cuda):
    """One rank, identity 'all-reduce': the phase API reproduces the fused two-pass calls bit for
    bit (the single-process default takes its statistics from the conv epilogue instead)."""
    nnet, levels, cols, labels = _setup(4, [0, 1, 2, 3])
    a = _run(nnet, levels, cols, labels, 4, None, epilogue_stats=False)
    b = _run(nnet, levels, cols, labels, 4, lambda t: None)
    assert a[1] == b[1]
    for x, y in zip(a[2] + a[3], b[2] + b[3]):
        assert torch.equal(x, y)
    for ba, bb in zip(a[0].blocks, b[0].blocks):
        assert torch.equal(ba["run_mean"], bb["run_mean"]) and torch.equal(ba["run_var"], bb["run_var"])


def _worker(rank, world, port, q, shardings):
    """shardings: per step, each rank's list of shape indices of a b_total batch (ranks may own
    different numbers of shapes, and the split may change from step to step)."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        from paper_1803_11385_b200.dist import allreduce_gradients, sum_over_ranks
        all_errs = []
        for step in shardings:
            b_total = sum(len(m) for m in step)
            mine = step[rank]
            nnet, levels, cols, labels = _setup(b_total, mine)
            net, loss, conv_g, head_g = _run(nnet, levels, cols, labels, b_total, sum_over_ranks)
            allreduce_gradients(conv_g + head_g)
            lt = torch.tensor([loss], dtype=torch.float64)  # each rank's share of the global mean
            dist.all_reduce(lt)
            if rank == 0:
                nnet1, levels1, cols1, labels1 = _setup(b_total, list(range(b_total)))
                net1, loss1, conv1, head1 = _run(nnet1, levels1, cols1, labels1, b_total, None)
                errs = {"loss": abs(float(lt) - loss1) / abs(loss1)}
                for i, (a, b) in enumerate(zip(conv_g + head_g, conv1 + head1)):
                    errs[f"grad{i}"] = _rel(a.cpu().numpy(), b.cpu().numpy())
                for i, (ba, bb) in enumerate(zip(net.blocks, net1.blocks)):
                    errs[f"run_mean{i}"] = _rel(ba["run_mean"].cpu().numpy(), bb["run_mean"].cpu().numpy())
                    errs[f"run_var{i}"] = _rel(ba["run_var"].cpu().numpy(), bb["run_var"].cpu().numpy())
                all_errs.append(errs)
        if rank == 0:
            q.put(all_errs)
        dist.barrier()
    except Exception as e:  # surface the failure instead of hanging the parent
        q.put({"error": repr(e)})
        raise
    finally:
        dist.destroy_process_group()


def _spawn(shardings):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, shardings)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(res, dict), res  # {"error": ...}
    return res


def _check(errs):
    # BN statistics: double sums, order-only differences; gradients: bf16 conv operands with
    # identical values, fp32 split-K dW partials summed in a different grouping
    assert errs["loss"] < 1e-5, errs
    for k, v in errs.items():
        bar = 1e-6 if k.startswith("run_") else 1e-3
        assert v < bar, (k, v, errs)


def test_two_rank_sync_bn_equals_whole_batch(cuda):
    for errs in _spawn([[[0, 1], [2, 3]]]):
        _check(errs)


def test_two_rank_sync_bn_uneven_changing_shards(cuda):
    """Shard sizes differ between the ranks AND change from step to step (2+1 shapes, then
    1+2, then 1+3): the global row count rides in the statistics' all-reduce every step, so
    the collectives stay matched and the statistics use that step's global batch."""
    for errs in _spawn([[[0, 1], [2]], [[0], [1, 2]], [[0], [1, 2, 3]]]):
        _check(errs)
