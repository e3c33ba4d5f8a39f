"""World-size-2 CPU (gloo) tests of the multi-GPU host logic:
shard arithmetic, the tree-shard partial reduce + finalize (with oracle
partials standing in for hb_predict_raw, which needs a GPU), and the
max-over-ranks timing reduction the bench uses. The GPU side of the same
pipeline is tests/test_gpu_parity.py::test_tree_shard_partials_reduce_to_unsharded."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2010_04804_b200.dist import max_over_ranks, reduce_partials, row_shard, tree_shard


def test_row_shard_covers_rows():
    for n in (0, 1, 7, 10_000_000, 10_000_001):
        for w in (1, 2, 3, 8):
            blocks = [row_shard(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0
            for (s0, c0), (s1, _) in zip(blocks, blocks[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in blocks) == n
            assert max(c for _, c in blocks) - min(c for _, c in blocks) <= 1


def test_tree_shard_whole_rounds():
    for T, K, w in ((3500, 7, 1), (10_000, 1, 1), (500, 7, 7), (13, 1, 1), (21, 7, 1)):
        for world in (1, 2, 4, 8):
            rngs = [tree_shard(T, r, world, K, w) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == T
            for (a0, a1), (b0, _) in zip(rngs, rngs[1:]):
                assert a1 == b0
            if w == 1 and K > 1:
                assert all(a % K == 0 for a, _ in rngs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        e = synth.gen_forest(42, 6, 9, seed=3, family="mixed", n_outputs=3,
                             post=synth.POST_SOFTMAX, task=synth.TASK_CLASSIFICATION,
                             agg=synth.AGG_MEAN, base_score=[0.5, -0.25, 0.0])
        X = synth.gen_X(8, 400, 9, special_q24=1 << 19)
        t0, t1 = tree_shard(e.n_trees, rank, world, e.n_outputs, e.leaf_width)
        part = torch.from_numpy(oracle.raw(e, X, t0, t1))       # stands in for hb_predict_raw
        reduce_partials(part, dst=0)
        slow = max_over_ranks(1.0 + rank)
        if rank == 0:
            full = oracle.raw(e, X)
            m = oracle.margin(e, part.numpy())
            ok = np.allclose(part.numpy(), full, rtol=1e-12, atol=1e-12) and \
                np.allclose(m, oracle.margin(e, full), rtol=1e-12, atol=1e-12)
            q.put(("ok" if ok and slow == float(world) else "mismatch", slow))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tree_shard_reduce_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    status, slow = q.get(timeout=10)
    assert status == "ok", (status, slow)
