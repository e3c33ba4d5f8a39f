"""Multi-GPU scoring on one node; one process per GPU.

* Row sharding: rows are independent, so rank r scores a contiguous block of
  rows with a full model replica — no collective on the data path.
* Tree sharding (very large ensembles, e.g. C5): trees are additive, so rank r
  compiles a contiguous tree range (hb_compile_range), computes fp64 raw
  partial sums (HB_OUT_RAW64: the scorers accumulate in fp64), ONE
  reduce(SUM) in fp64 brings them to the root (NCCL over NVLink with backend
  "nccl"), and the root runs hb_finalize64 with the global per-output tree
  counts and base score — no fp32 rounding before the margin is formed
  (R23).

The paper itself is single-GPU ("distributed inference is future work",
PAPER.md P:129); this is the natural extension of its batch (row) and ensemble
(tree) dimensions. Plumbing only: every arithmetic step runs in libhb.so.
"""
from __future__ import annotations


def row_shard(n_rows: int, rank: int, world: int):
    """Contiguous, balanced block of rows for `rank`: (start, count)."""
    base, rem = divmod(n_rows, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def tree_shard(n_trees: int, rank: int, world: int, n_outputs: int = 1, leaf_width: int = 1):
    """Contiguous tree range [t0, t1) for `rank`. For per-class scalar trees
    (leaf_width == 1, K > 1, tree t feeds t % K) the cut points are multiples
    of K so each shard holds whole boosting rounds (balanced per class)."""
    unit = n_outputs if (leaf_width == 1 and n_outputs > 1 and n_trees % n_outputs == 0) else 1
    groups = n_trees // unit
    g0, gn = row_shard(groups, rank, world)
    t0 = g0 * unit
    t1 = (g0 + gn) * unit
    if rank == world - 1:
        t1 = n_trees
    return t0, t1


def reduce_partials(partial, dst: int = 0, group=None):
    """Sum the [n, K] raw partials of all ranks into `partial` on rank `dst`
    (one torch.distributed.reduce; NCCL for CUDA tensors, gloo for CPU)."""
    import torch.distributed as dist
    if partial.is_cuda and dist.get_backend(group) == "gloo":   # 1-GPU multi-rank tests
        host = partial.cpu()
        dist.reduce(host, dst=dst, op=dist.ReduceOp.SUM, group=group)
        partial.copy_(host)
        return partial
    dist.reduce(partial, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return partial


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (the timing rule: max over ranks)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "gloo":
        device = None
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class TreeShardedModel:
    """A tree shard of an ensemble on this rank's GPU; `predict` returns the
    finalized output on rank `root` (None elsewhere)."""

    def __init__(self, ensemble, rank: int, world: int, device: int, strategy="auto", root=0):
        from .hb import Model
        self.t0, self.t1 = tree_shard(ensemble.n_trees, rank, world, ensemble.n_outputs,
                                      ensemble.leaf_width)
        self.model = Model(ensemble, strategy=strategy, device=device,
                           tree_range=(self.t0, self.t1))
        self.rank, self.world, self.root = rank, world, root

    def predict(self, X, kind="proba", group=None):
        raw = self.model.predict_raw64(X)
        if self.world > 1:
            reduce_partials(raw, dst=self.root, group=group)
        if self.rank != self.root:
            return None
        return self.model.finalize(raw, kind)
