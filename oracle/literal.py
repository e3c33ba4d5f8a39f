"""Literal numpy transcriptions of the paper's three strategies (fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). These follow Alg. 1-3 of
PAPER.md step by step in the paper's notation, with the readings listed in
DESIGN.md §2 where the extraction is garbled. Their only job is the strategy
invariant (SURVEY.md §8(c) P-d): all three must reach the same leaf as the
plain walk in oracle.c for every (row, tree). They are small-input tools
(dense A is |F| x |I| per tree, PTT is 2^D per tree).
"""
from __future__ import annotations

import numpy as np


def _tree_lists(tr):
    """Ordered lists I (internal) and L (leaves) of one tree, node-id order
    (Table 3: "ordered lists with all nodes, internal nodes, leaf
    nodes")."""
    left = np.asarray(tr["left"])
    I = np.nonzero(left != -1)[0]
    L = np.nonzero(left == -1)[0]
    return I, L


def _subtree_leaves(tr, i):
    left, right = tr["left"], tr["right"]
    out, stack = [], [i]
    while stack:
        k = stack.pop()
        if left[k] == -1:
            out.append(k)
        else:
            stack += [left[k], right[k]]
    return out


def gemm_tensors(tr, n_features):
    """A, B, C, D, E of Table 3 for one tree.

    A[F_i, j] = 1 iff internal node I_j evaluates feature F_i.
    B[j]      = ThresholdValue(I_j).
    C[i, j]   = +1 if L_j in LeftSubTree(I_i), -1 if in RightSubTree(I_i), else 0.
    D[j]      = number of left edges on the root->L_j path (reading R5 of the
                garbled P:153 formula: "#{i : C_ij = +1}", prose P:164).
    E[j, :]   = leaf value(s) of L_j ("For regression tasks, we
                initialize E with label values").
    """
    I, L = _tree_lists(tr)
    lpos = {int(l): j for j, l in enumerate(L)}
    A = np.zeros((n_features, len(I)))
    B = np.zeros(len(I))
    C = np.zeros((len(I), len(L)))
    for j, i in enumerate(I):
        A[tr["feature"][i], j] = 1.0
        B[j] = tr["threshold"][i]
        for l in _subtree_leaves(tr, tr["left"][i]):
            C[j, lpos[l]] = 1.0
        for l in _subtree_leaves(tr, tr["right"][i]):
            C[j, lpos[l]] = -1.0
    D = (C == 1.0).sum(0).astype(np.float64)
    E = np.asarray(tr["leaf_value"], np.float64)[L]
    return I, L, A, B, C, D, E


def gemm_tree(tr, X, n_features, cmp):
    """Alg. 1 for one tree on finite X. Returns (leaf ids, R).

    T <- GEMM(X, A); T <- T < B; T <- GEMM(T, C); T <- T == D; R <- GEMM(T, E).
    The dense X·A is literal: it is only exact for finite X (0 * Inf = NaN;
    SURVEY.md V4), so callers pass finite rows. The kernel gathers instead.
    """
    I, L, A, B, C, D, E = gemm_tensors(tr, n_features)
    X = np.asarray(X, np.float64)
    if len(I) == 0:                       # single-leaf tree: always leaf 0
        return np.zeros(X.shape[0], np.int64), np.repeat(E, X.shape[0], 0)
    T = X @ A
    T = (T < B) if cmp == 0 else (T <= B)
    T = T.astype(np.float64) @ C
    T = (T == D).astype(np.float64)
    R = T @ E
    hits = T.sum(1)
    assert np.all(hits == 1), "GEMM strategy must select exactly one leaf"
    return L[np.argmax(T, 1)], R


def gemm_ensemble_padded(e, X, mask_pads=True):
    """Alg. 1 batched over trees with P:192's zero padding to max |I|, |L|.

    With literal zero padding a padded leaf column (C = 0, D = 0) matches every
    row (reading R7); ``mask_pads`` sets D of padded
    columns to an unreachable sentinel (1 with a zero C column). Returns the
    number of matching columns per (row, tree) and the leaf ids."""
    trees = [e.tree(t) for t in range(e.n_trees)]
    tens = [gemm_tensors(tr, e.n_features) for tr in trees]
    mI = max(len(t[0]) for t in tens)
    mL = max(len(t[1]) for t in tens)
    X = np.asarray(X, np.float64)
    n = X.shape[0]
    hits = np.zeros((n, e.n_trees), np.int64)
    leaves = np.zeros((n, e.n_trees), np.int64)
    for t, (I, L, A, B, C, D, E) in enumerate(tens):
        Ap = np.zeros((e.n_features, mI)); Ap[:, :len(I)] = A
        Bp = np.zeros(mI); Bp[:len(I)] = B
        Cp = np.zeros((mI, mL)); Cp[:len(I), :len(L)] = C
        Dp = np.zeros(mL); Dp[:len(L)] = D
        if mask_pads:
            Dp[len(L):] = 1.0
        T = X @ Ap
        T = ((T < Bp) if e.cmp == 0 else (T <= Bp)).astype(np.float64)
        S = T @ Cp
        M = S == Dp
        hits[:, t] = M.sum(1)
        leaves[:, t] = np.where(M[:, :len(L)].any(1), L[np.argmax(M[:, :len(L)], 1)] if len(L) else 0, -1)
    return hits, leaves


def tt_tensors(tr):
    """N_L, N_R, N_F, N_T, N_C of Table 5 for one tree.
    Leaves self-loop (N_L = N_R = i); N_F = 0 at leaves
    (reading R15: the paper's "1" is out of range when |F| = 1 with 0-based
    ids; the self-loop makes the value irrelevant); N_T = 0 at leaves."""
    left = np.asarray(tr["left"]); right = np.asarray(tr["right"])
    n = left.size
    idx = np.arange(n)
    leaf = left == -1
    NL = np.where(leaf, idx, left)
    NR = np.where(leaf, idx, right)
    NF = np.where(leaf, 0, np.asarray(tr["feature"]))
    NT = np.where(leaf, 0.0, np.asarray(tr["threshold"], np.float64))
    NC = np.asarray(tr["leaf_value"], np.float64)
    return NL, NR, NF, NT, NC


def tt_ensemble(e, X, tree_depth):
    """Alg. 2, per tree, TREE_DEPTH fixed iterations.

    T_I <- {root}^n; repeat TREE_DEPTH: T_F <- Gather(N_F, T_I);
    T_V <- Gather(X, T_F) (per-row gather, reading R16); T_T, T_L, T_R <-
    Gather(N_T | N_L | N_R, T_I); T_I <- Where(T_V < T_T, T_L, T_R).
    R <- Gather(N_C, T_I). Returns leaf ids [n, T] and values [n, T, w].
    The comparison is fp32 (both operands are fp32 values; reading R4)."""
    X32 = np.asarray(X, np.float32)
    n = X32.shape[0]
    rows = np.arange(n)
    leaves = np.zeros((n, e.n_trees), np.int64)
    vals = np.zeros((n, e.n_trees, e.leaf_width))
    for t in range(e.n_trees):
        NL, NR, NF, NT, NC = tt_tensors(e.tree(t))
        NT32 = NT.astype(np.float32)
        TI = np.zeros(n, np.int64)
        for _ in range(tree_depth):
            TF = NF[TI]
            TV = X32[rows, TF]
            TT = NT32[TI]
            TL = NL[TI]
            TR = NR[TI]
            TI = np.where((TV < TT) if e.cmp == 0 else (TV <= TT), TL, TR)
        leaves[:, t] = TI
        vals[:, t] = NC[TI]
    return leaves, vals


def ptt_tensors(e, D, rng=None):
    """Perfect-tree padding (readings R10-R13) and the level-interleaved
    N'_F, N'_T of P:286, plus N'_C [T, 2^D, w] and the slot -> original-leaf map.

    A leaf at depth D_k < D is replaced by a perfect subtree of depth D - D_k
    whose leaves all copy it; the inserted decision nodes "are free to perform
    arbitrary comparisons" — with ``rng`` they get random features/thresholds
    to show that, otherwise feature 0 / threshold +Inf.
    Interleave: level l (0-based), tree t, in-level position j at flat index
    T*(2^l - 1) + t*2^l + j (reading R14)."""
    T = e.n_trees
    NF = np.zeros(T * ((1 << D) - 1), np.int64)
    NT = np.zeros(T * ((1 << D) - 1), np.float32)
    NC = np.zeros((T, 1 << D, e.leaf_width))
    leaf_map = np.zeros((T, 1 << D), np.int64)
    for t in range(T):
        tr = e.tree(t)
        left, right = tr["left"], tr["right"]
        # heap position p (1-based) -> original node
        cur = {1: 0}
        for lvl in range(D):
            nxt = {}
            for p, o in cur.items():
                j = p - (1 << lvl)
                flat = T * ((1 << lvl) - 1) + t * (1 << lvl) + j
                if left[o] != -1:
                    NF[flat] = tr["feature"][o]
                    NT[flat] = tr["threshold"][o]
                    nxt[2 * p], nxt[2 * p + 1] = left[o], right[o]
                else:
                    if rng is not None:
                        NF[flat] = rng.integers(0, e.n_features)
                        NT[flat] = np.float32(rng.normal())
                    else:
                        NF[flat] = 0
                        NT[flat] = np.float32(np.inf)
                    nxt[2 * p], nxt[2 * p + 1] = o, o
            cur = nxt
        for p, o in cur.items():
            slot = p - (1 << D)
            NC[t, slot] = tr["leaf_value"][o]
            leaf_map[t, slot] = o
    return NF, NT, NC, leaf_map


def ptt_ensemble(e, X, D, rng=None):
    """Alg. 3 batched over trees.

    T_I <- {1}^n; repeat D: T_F <- Gather(N'_F, T_I); T_V <- Gather(X, T_F);
    T_T <- Gather(N'_T, T_I); T_I <- 2 T_I + Where(T_V < T_T, 0, 1).
    R <- Gather(N'_C, T_I) with the implicit offset T_I - 2^D (reading R11).
    Returns original leaf ids [n, T] and values [n, T, w]."""
    NF, NT, NC, leaf_map = ptt_tensors(e, D, rng)
    X32 = np.asarray(X, np.float32)
    n, T = X32.shape[0], e.n_trees
    rows = np.arange(n)[:, None]
    trees = np.arange(T)[None, :]
    TI = np.ones((n, T), np.int64)
    for lvl in range(D):
        flat = T * ((1 << lvl) - 1) + trees * (1 << lvl) + (TI - (1 << lvl))
        TF = NF[flat]
        TV = X32[rows, TF]
        TT = NT[flat]
        pred = (TV < TT) if e.cmp == 0 else (TV <= TT)
        TI = 2 * TI + np.where(pred, 0, 1)
    slot = TI - (1 << D)
    return leaf_map[trees, slot], NC[trees, slot]
