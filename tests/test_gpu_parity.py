"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (SURVEY.md §4 pyramid level 3, §8(c) tolerances).

Bar: leaf ids and leaf hashes bit-exact; scores |gpu - ref| <= 1e-5 + 1e-5|ref|
(PAPER.md P:469 assert_allclose rtol = atol = 1e-5; reading R23);
labels exact except documented near-ties (top-2 margin gap below twice the
tolerance)."""
import zlib

import numpy as np
import pytest

import oracle
import synth
from tests._common import SPECIAL_Q24, load_hand_trees, record_near_ties

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2010_04804_b200 as hb  # noqa: E402
import synth.dev  # noqa: E402


@pytest.fixture(autouse=True)
def _large_batch_kernels(monkeypatch):
    """Parity tests exercise the row-tile scorers by default; the small-batch
    (trees-across-threads) path is tested explicitly below."""
    monkeypatch.setenv("HB_SMALL_BATCH", "0")


def tol_ok(got, ref):
    got = np.asarray(got, np.float64)
    return np.abs(got - ref) <= 1e-5 + 1e-5 * np.abs(ref)


def assert_scores(got, ref, what=""):
    ok = tol_ok(got, ref)
    if not ok.all():
        i = np.argwhere(~ok)[0]
        raise AssertionError(f"{what}: {(~ok).sum()} values outside tolerance, first at {i}: "
                             f"gpu={np.asarray(got)[tuple(i)]!r} ref={ref[tuple(i)]!r}")


def near_tie(e, margin):
    m = margin
    if e.n_outputs == 1:
        return np.abs(m[:, 0]) < 2 * (1e-5 + 1e-5 * np.abs(m[:, 0]))
    s = np.sort(m, 1)
    gap = s[:, -1] - s[:, -2]
    return gap < 2 * (1e-5 + 1e-5 * np.abs(s[:, -1]))


def assert_labels(e, got, ref_label, ref_margin, what="labels"):
    """Labels exact except near-ties (R23), which are listed (conftest terminal
    summary) and must still name one of the tied classes."""
    tie = near_tie(e, ref_margin)
    assert np.array_equal(got[~tie], ref_label[~tie]), what
    rows = np.flatnonzero(tie)
    if rows.size:
        if e.n_outputs > 1:
            s = np.sort(ref_margin[rows], 1)
            gap_ok = ref_margin[rows, got[rows]] >= s[:, -1] - 2 * (1e-5 + 1e-5 * np.abs(s[:, -1]))
            assert gap_ok.all(), f"{what}: near-tie row labelled outside the tied classes"
        record_near_ties(what, rows, got[rows], ref_label[rows])


def X_pair(seed, n, F, ldx=None, **kw):
    Xd = synth.dev.gen_X_device(seed, n, F, ldx=ldx, **kw)
    Xh = synth.gen_X(seed, n, F, ldx=ldx, **kw)
    return Xd, Xh


def check_all(e, m, Xd, Xh, kinds=("predict", "proba", "raw", "raw64", "margin", "leaf", "leaf_hash")):
    F = e.n_features
    Xo = Xh[:, :F] if Xh.shape[1] > F else Xh
    s = oracle.scores(e, Xo)
    cls = e.task == synth.TASK_CLASSIFICATION
    for kind in kinds:
        if kind == "proba" and not cls:
            with pytest.raises(hb.HBError):
                m.run(Xd, "proba")
            continue
        got = m.run(Xd, kind).cpu().numpy()
        if kind == "leaf":
            assert np.array_equal(got, oracle.leaf(e, Xo)), "leaf ids"
        elif kind == "leaf_hash":
            assert np.array_equal(got.view(np.uint64), oracle.leaf_hash(e, Xo)), "leaf hash"
        elif kind == "raw":
            assert_scores(got, s["raw"], "raw")
        elif kind == "raw64":
            # fp64 sums: within the fp32 bar, and RAW is exactly their fp32 rounding
            assert_scores(got, s["raw"], "raw64")
            if "raw" in kinds:
                assert np.array_equal(got.astype(np.float32), m.run(Xd, "raw").cpu().numpy()), "raw != raw64"
        elif kind == "margin":
            assert_scores(got, s["margin"], "margin")
        elif kind == "proba":
            assert_scores(got, oracle.proba(e, s["post"]), "proba")
        elif kind == "predict":
            if cls:
                assert_labels(e, got, s["label"], s["margin"])
            else:
                assert_scores(got, s["post"], "predict")


FAMILIES = ["balanced", "mixed", "skinny"]


def _forest(kind, T, D, F, seed, family, cmp, grid=synth.GRID_FINE):
    common = dict(seed=seed, family=family, cmp=cmp, grid=grid)
    if kind == "reg":
        return synth.gen_forest(T, D, F, base_score=[0.5], **common)
    if kind == "binary":
        return synth.gen_forest(T, D, F, post=synth.POST_SIGMOID,
                                task=synth.TASK_CLASSIFICATION, base_score=[-0.25], **common)
    if kind == "multiclass":   # per-class scalar trees, t mod K (C4 layout)
        return synth.gen_forest(T, D, F, n_outputs=3, post=synth.POST_SOFTMAX,
                                task=synth.TASK_CLASSIFICATION, **common)
    if kind == "k7":
        return synth.gen_forest(T, D, F, n_outputs=7, post=synth.POST_SOFTMAX,
                                task=synth.TASK_CLASSIFICATION, **common)
    if kind == "k12":
        return synth.gen_forest(T, D, F, n_outputs=12, post=synth.POST_SOFTMAX,
                                task=synth.TASK_CLASSIFICATION,
                                tree_output=np.random.default_rng(seed).integers(0, 12, T), **common)
    if kind == "rf":           # vector leaves, soft voting (MEAN)
        return synth.gen_forest(T, D, F, n_outputs=5, leaf_width=5, leaf_kind="dirichlet",
                                agg=synth.AGG_MEAN, task=synth.TASK_CLASSIFICATION, **common)
    if kind == "rf_reg":       # MEAN regression (RF regressor)
        return synth.gen_forest(T, D, F, agg=synth.AGG_MEAN, **common)
    raise ValueError(kind)


CASES = []
for strat, D in (("ptt", 8), ("ptt", 5), ("tt", 8), ("tt", 11), ("gemm", 3), ("gemm", 5)):
    for kind in ("reg", "binary", "multiclass", "rf"):
        for cmp in (0, 1):
            CASES.append((strat, D, kind, cmp))


@pytest.mark.parametrize("strat,D,kind,cmp", CASES)
def test_strategy_parity(strat, D, kind, cmp, monkeypatch):
    seed = zlib.crc32(f"{strat}{D}{kind}{cmp}".encode()) & 0xFFFF
    family = FAMILIES[seed % 3]
    F = [3, 17, 28, 54][seed % 4]
    T = 37 if strat != "gemm" else 23    # odd: exercises tree-group padding
    e = _forest(kind, T, D, F, seed, family, cmp)
    n = 1500 + seed % 97                 # several 512-row tiles + ragged tail
    Xd, Xh = X_pair(seed, n, F, special_q24=SPECIAL_Q24)
    # PTT has three node layouts: rank-coded 4-B records with 32- or 16-bit
    # code cells (codes computed in the scorer, or by the pre-pass launch), and
    # fp32 8-B records
    layouts = (("1", "32", "0"), ("1", "16", "0"), ("1", "32", "1"), ("1", "16", "1"), ("0", "0", "0"))
    for rank, cw, pre in (layouts if strat == "ptt" else (("1", "0", "0"),)):
        monkeypatch.setenv("HB_PTT_RANK", rank)
        monkeypatch.setenv("HB_RANK_CW", cw)
        monkeypatch.setenv("HB_RANK_PRE", pre)
        m = hb.Model(e, strategy=strat, device=0)
        assert m.info["strategy_name"] == strat
        if strat == "ptt":
            assert m.info["node_record_bytes"] == (4 if rank == "1" else 8)
            assert m.info["code_cell_bits"] == int(cw)
            assert m.info["rank_prepass"] == int(pre)
        check_all(e, m, Xd, Xh)


def _set_layout(monkeypatch, rank):
    """PTT node layout by name: "0" fp32 nodes; "1" / "16" rank-coded with
    32- / 16-bit cells, codes in the scorer; "pre32" / "pre16" the same with
    codes from the pre-pass launch."""
    monkeypatch.setenv("HB_PTT_RANK", "0" if rank == "0" else "1")
    monkeypatch.setenv("HB_RANK_CW", "16" if rank.endswith("16") else ("32" if rank == "pre32" else "0"))
    monkeypatch.setenv("HB_RANK_PRE", "1" if rank.startswith("pre") else "0")


@pytest.mark.parametrize("cmp", [0, 1])
@pytest.mark.parametrize("rank", ["1", "0", "16", "pre32", "pre16"])
def test_ptt_special_thresholds(cmp, rank, monkeypatch):
    """Thresholds at +-Inf and -0/+0 (mixed on one feature) against X holding
    NaN, +-Inf, +-0 and exact ties: the rank code must reproduce every fp32
    decision (reading R3), for both PTT node layouts."""
    _set_layout(monkeypatch, rank)
    e = _forest("binary", 33, 6, 5, 17, "mixed", cmp, grid=synth.GRID_COARSE)
    rng = np.random.default_rng(3)
    internal = np.nonzero(e.left != -1)[0]
    pick = rng.choice(internal, size=len(internal) // 3, replace=False)
    specials = np.array([np.inf, -np.inf, 0.0, -0.0], np.float32)
    e.threshold[pick] = specials[rng.integers(0, 4, pick.size)]
    m = hb.Model(e, strategy="ptt", device=0)
    assert m.info["node_record_bytes"] == (8 if rank == "0" else 4)
    Xd, Xh = X_pair(8, 4000, 5, grid=synth.GRID_COARSE, special_q24=1 << 22)
    check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("kind", ["reg", "binary", "multiclass", "rf", "k7", "k12"])
@pytest.mark.parametrize("cmp", [0, 1])
@pytest.mark.parametrize("rows", ["32", "16", "8"])
def test_tt_wide_kernel_parity(kind, cmp, rows, monkeypatch):
    """The wide-row TT kernel (R rows per CTA, lanes = tree slot x row, nodes
    through L1/L2, fp64 sums combined by shuffles + one SMEM pass) forced on
    ordinary inputs for every row-tile height R it instantiates."""
    monkeypatch.setenv("HB_TT_WIDE", "1")
    monkeypatch.setenv("HB_TT_WIDE_ROWS", rows)
    seed = zlib.crc32(f"wide{kind}{cmp}".encode()) & 0xFFFF
    e = _forest(kind, 45, 9, 37, seed, FAMILIES[seed % 3], cmp)
    m = hb.Model(e, strategy="tt", device=0)
    assert m.info["kernel_name"] == "tt_wide_kernel" and m.info["rows_per_cta"] == int(rows)
    Xd, Xh = X_pair(seed, 1000 + seed % 53, 37, special_q24=SPECIAL_Q24)
    check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("cmp", [0, 1])
def test_tt_wide_tree_shapes(cmp, monkeypatch):
    """tt_wide_kernel on every shape its early exit and self-loops meet:
    single-leaf trees, a stump, left/right chains of odd and even depth, bushy
    mixed trees, a depth-12 balanced tree; one launch and tree chunks of 4 and
    12 trees (fp64 partials accumulated across launches, then finalize) must
    give the same leaf ids and the oracle's scores."""
    monkeypatch.setenv("HB_TT_WIDE", "1")
    F = 9
    trees = [dict(feature=[0], threshold=[0.0], left=[-1], right=[-1], leaf_value=[0.75]),
             dict(feature=[2, 0, 0], threshold=[0.5, 0, 0], left=[1, -1, -1], right=[2, -1, -1],
                  leaf_value=[0.0, -1.5, 2.25])]
    trees += [_chain_tree(d, F, d, left_chain=d % 2 == 0) for d in (2, 3, 5, 6, 13)]
    bushy = synth.gen_forest(200, 9, F, seed=4 + cmp, family="mixed", grid=synth.GRID_COARSE)
    trees += [bushy.tree(i) for i in range(200)]
    deep = synth.gen_forest(3, 12, F, seed=9 + cmp, family="balanced")
    trees += [deep.tree(i) for i in range(3)]
    e = synth.from_trees(trees, F, cmp=cmp)
    Xd, Xh = X_pair(12, 2111, F, grid=synth.GRID_COARSE, special_q24=SPECIAL_Q24)
    leaves = []
    for chunk, rows in (("0", "32"), ("0", "8"), ("4", "16"), ("12", "32")):
        monkeypatch.setenv("HB_TT_CHUNK", chunk)
        monkeypatch.setenv("HB_TT_WIDE_ROWS", rows)
        m = hb.Model(e, strategy="tt", device=0)
        assert m.info["kernel_name"] == "tt_wide_kernel"
        assert m.info["tt_chunk_trees"] == int(chunk)
        check_all(e, m, Xd, Xh, kinds=("predict", "raw", "margin", "leaf", "leaf_hash"))
        leaves.append(m.predict_leaf(Xd).cpu().numpy())
    assert all(np.array_equal(leaves[0], lv) for lv in leaves[1:])


def test_tt_wide_rows_natural():
    e = _forest("binary", 30, 12, 2000, 3, "mixed", 0)
    m = hb.Model(e, device=0)
    assert m.info["strategy_name"] == "tt" and m.info["x_in_smem"] == 1
    assert m.info["kernel_name"] == "tt_wide_kernel"
    Xd, Xh = X_pair(5, 333, 2000, special_q24=SPECIAL_Q24)
    check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("kind", ["k7", "k12", "rf_reg"])
@pytest.mark.parametrize("strat", ["ptt", "tt", "gemm"])
def test_more_outputs(kind, strat):
    e = _forest(kind, 30, 4, 11, 5, "mixed", 0)
    m = hb.Model(e, strategy=strat, device=0)
    Xd, Xh = X_pair(9, 777, 11)
    check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("strat", ["ptt", "tt", "gemm", "auto"])
@pytest.mark.parametrize("cmp", [0, 1])
def test_tie_heavy_coarse_grid(strat, cmp):
    """Coarse grid: thresholds and X share 64 values, so x == t is frequent
    (LT vs LE routing, SURVEY §8(d) tie-heavy variant)."""
    e = _forest("binary", 40, 6 if strat != "gemm" else 4, 7, 3, "balanced", cmp,
                grid=synth.GRID_COARSE)
    m = hb.Model(e, strategy=strat, device=0)
    Xd, Xh = X_pair(4, 2048, 7, grid=synth.GRID_COARSE)
    check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("strat", ["ptt", "tt", "gemm"])
@pytest.mark.parametrize("cmp", [0, 1])
def test_hand_traced_trees_on_gpu(strat, cmp):
    e, X, exp_leaf, exp_sum = load_hand_trees(cmp)
    m = hb.Model(e, strategy=strat, device=0)
    Xd = torch.from_numpy(X).cuda()
    assert np.array_equal(m.predict_leaf(Xd).cpu().numpy(), exp_leaf)
    assert np.array_equal(m.predict_raw(Xd).cpu().numpy()[:, 0], exp_sum.astype(np.float32))


@pytest.mark.parametrize("n", [0, 1, 31, 33, 511, 513])
@pytest.mark.parametrize("strat", ["ptt", "tt", "gemm"])
def test_edge_row_counts(n, strat):
    e = _forest("reg", 9, 4, 6, 1, "skinny", 0)
    m = hb.Model(e, strategy=strat, device=0)
    Xd, Xh = X_pair(2, max(n, 1), 6)
    Xd, Xh = Xd[:n], Xh[:n]
    got = m.predict(Xd).cpu().numpy()
    assert got.shape == (n, 1)
    if n:
        assert_scores(got, oracle.scores(e, Xh)["post"], "edge n")
        assert np.array_equal(m.predict_leaf(Xd).cpu().numpy(), oracle.leaf(e, Xh))


@pytest.mark.parametrize("strat", ["ptt", "tt", "gemm"])
def test_ldx_padding_and_unaligned(strat):
    e = _forest("multiclass", 12, 5, 10, 8, "mixed", 1)
    m = hb.Model(e, strategy=strat, device=0)
    for ldx in (10, 13, 16):
        Xd, Xh = X_pair(11, 700, 10, ldx=ldx)
        check_all(e, m, Xd, Xh, kinds=("raw", "leaf"))
    # unaligned base pointer (column view) disables the float4 path
    Xd, Xh = X_pair(12, 701, 11, ldx=12)
    check_all(e, m, Xd[:, 1:], Xh[:, 1:], kinds=("raw", "leaf"))


@pytest.mark.parametrize("strat", ["ptt", "tt", "gemm"])
def test_single_feature_and_single_leaf_trees(strat):
    # F = 1 and a mix of depth-0 trees with deeper ones
    deep = synth.gen_forest(5, 3, 1, seed=3, family="balanced")
    leafy = [dict(feature=[-1], threshold=[np.nan], left=[-1], right=[-1], leaf_value=[0.125 * i])
             for i in range(3)]
    trees = [deep.tree(t) for t in range(5)]
    trees = [dict(feature=t["feature"], threshold=t["threshold"], left=t["left"], right=t["right"],
                  leaf_value=t["leaf_value"]) for t in trees] + leafy
    e = synth.from_trees(trees, 1)
    m = hb.Model(e, strategy=strat, device=0)
    Xd, Xh = X_pair(5, 900, 1, special_q24=SPECIAL_Q24)
    check_all(e, m, Xd, Xh)
    # all trees single leaves: D = 0
    e0 = synth.from_trees(leafy, 1)
    m0 = hb.Model(e0, strategy=strat, device=0)
    check_all(e0, m0, Xd, Xh)


@pytest.mark.parametrize("staged", ["0", "1", "0:8"])
@pytest.mark.parametrize("cw", ["32", "16"])
def test_prepass_forced_on_degenerate_models(cw, staged, monkeypatch):
    """The rank-code pre-pass forced on models it would never be picked for:
    no split at all (D = 0: nothing to code, no pre-pass launch), one feature,
    and an odd feature count with 16-bit cells (half-empty last word)."""
    monkeypatch.setenv("HB_PTT_RANK", "1")
    monkeypatch.setenv("HB_RANK_PRE", "1")
    monkeypatch.setenv("HB_RANK_CW", cw)
    monkeypatch.setenv("HB_RC_STAGED", staged.split(":")[0])
    monkeypatch.setenv("HB_RC_ROWS", staged.split(":")[1] if ":" in staged else "4")
    leafy = [dict(feature=[-1], threshold=[np.nan], left=[-1], right=[-1], leaf_value=[0.25 * i])
             for i in range(5)]
    Xd, Xh = X_pair(8, 1300, 3, special_q24=SPECIAL_Q24)
    for e in (synth.from_trees(leafy, 3),
              synth.gen_forest(9, 4, 1, seed=4, family="mixed"),
              synth.gen_forest(11, 5, 3, seed=5, family="skinny", grid=synth.GRID_COARSE)):
        m = hb.Model(e, strategy="ptt", device=0)
        assert m.info["rank_prepass"] == 1
        F = e.n_features
        check_all(e, m, Xd[:, :F].contiguous(), np.ascontiguousarray(Xh[:, :F]))


def _perfect_d3_sign_tree(cmp):
    """Perfect depth-3 tree whose 7 internal nodes test features 0..6 at 0."""
    feat, thr, L, R, val = [], [], [], [], []
    # heap order: node i (0-based) children 2i+1, 2i+2; 7 internal, 8 leaves
    for i in range(15):
        if i < 7:
            feat.append(i); thr.append(0.0); L.append(2 * i + 1); R.append(2 * i + 2)
            val.append(np.nan)
        else:
            feat.append(-1); thr.append(np.nan); L.append(-1); R.append(-1)
            val.append(float(i))
    return synth.from_trees([dict(feature=feat, threshold=thr, left=L, right=R, leaf_value=val)],
                            7, cmp=cmp)


@pytest.mark.parametrize("tc", ["1", "0"])
@pytest.mark.parametrize("cmp", [0, 1])
def test_gemm_path_contraction_exhaustive(tc, cmp, monkeypatch):
    """P-i: every one of the 2^7 predicate patterns T of a perfect D3 tree
    (rows with x_i in {-1, 0, +1} hit both sides of every threshold, and 0 is
    the tie) selects exactly the walked leaf through S = T.C == D, on the
    tensor-core kernel (HB_GEMM_TC=1) and the CUDA-core kernel."""
    monkeypatch.setenv("HB_GEMM_TC", tc)
    e = _perfect_d3_sign_tree(cmp)
    m = hb.Model(e, strategy="gemm", device=0)
    assert m.info["tensor_cores"] == int(tc)
    import itertools
    X = np.array(list(itertools.product([-1.0, 0.0, 1.0], repeat=7)), np.float32)
    Xd = torch.from_numpy(X).cuda()
    assert np.array_equal(m.predict_leaf(Xd).cpu().numpy(), oracle.leaf(e, X))
    assert np.array_equal(m.predict_raw(Xd).cpu().numpy()[:, 0],
                          oracle.raw(e, X)[:, 0].astype(np.float32))


@pytest.mark.parametrize("tc", ["1", "0"])
def test_gemm_tc_vs_cuda_core_many_trees(tc, monkeypatch):
    """Many shallow trees (several 16-tree groups, ragged last group) on both
    GEMM kernels, all outputs against the oracle."""
    monkeypatch.setenv("HB_GEMM_TC", tc)
    e = _forest("multiclass", 61, 3, 13, 21, "mixed", 1)
    m = hb.Model(e, strategy="gemm", device=0)
    assert m.info["tensor_cores"] == int(tc)
    Xd, Xh = X_pair(22, 3001, 13, special_q24=SPECIAL_Q24)
    check_all(e, m, Xd, Xh)


SMALL_CASES = [(strat, D, kind, cmp) for strat, D in (("ptt", 8), ("tt", 11), ("gemm", 3))
               for kind in ("reg", "binary", "multiclass", "rf") for cmp in (0, 1)]


@pytest.mark.parametrize("strat,D,kind,cmp", SMALL_CASES)
def test_small_batch_path_parity(strat, D, kind, cmp, monkeypatch):
    """Request/response sizes (n = 1..300) go through the trees-across-threads
    kernel (hb_small.cu) for every strategy; all outputs against the oracle."""
    monkeypatch.setenv("HB_SMALL_BATCH", "4096")
    seed = zlib.crc32(f"small{strat}{D}{kind}{cmp}".encode()) & 0xFFFF
    e = _forest(kind, 41, D, 19, seed, FAMILIES[seed % 3], cmp)
    m = hb.Model(e, strategy=strat, device=0)
    for n in (1, 7, 300):
        Xd, Xh = X_pair(seed + n, n, 19, special_q24=SPECIAL_Q24)
        check_all(e, m, Xd, Xh)


def test_small_and_large_paths_agree(monkeypatch):
    e = _forest("binary", 500, 8, 28, 1, "balanced", 0)
    Xd, Xh = X_pair(2, 1000, 28)
    monkeypatch.setenv("HB_SMALL_BATCH", "4096")
    ms = hb.Model(e, device=0)
    assert ms.kernel_for(1000) == "small_batch_kernel"
    small = ms.predict_proba(Xd).cpu().numpy().astype(np.float64)
    hs = ms.predict_leaf_hash(Xd).cpu().numpy()
    monkeypatch.setenv("HB_SMALL_BATCH", "0")
    m = hb.Model(e, device=0)
    assert m.kernel_for(1000) == m.info["kernel_name"]
    large = m.predict_proba(Xd).cpu().numpy().astype(np.float64)
    assert np.array_equal(hs, m.predict_leaf_hash(Xd).cpu().numpy())
    assert np.abs(small - large).max() < 1e-5


def test_auto_strategy_selection(monkeypatch):
    """Sec. 5.1 heuristic recalibrated on B200 (reading R24): PTT D <= 10, TT
    beyond, GEMM on request (HB_GEMM_MAX_DEPTH);
    PTT falls back to TT when rows are too wide for the SMEM X tile."""
    for D, want in ((2, "ptt"), (3, "ptt"), (4, "ptt"), (8, "ptt"), (10, "ptt"), (11, "tt"),
                    (12, "tt")):
        e = synth.gen_forest(4, D, 8, seed=D, family="skinny")
        assert hb.Model(e, device=0).info["strategy_name"] == want, D
    # the paper's CPU rule (GEMM for D <= 3) on request
    monkeypatch.setenv("HB_GEMM_MAX_DEPTH", "3")
    for D, want in ((2, "gemm"), (3, "gemm"), (4, "ptt")):
        e = synth.gen_forest(4, D, 8, seed=D, family="skinny")
        assert hb.Model(e, device=0).info["strategy_name"] == want, D
    monkeypatch.delenv("HB_GEMM_MAX_DEPTH")
    # a wide row with few used features: feature-selection injection
    # shrinks the X tile to the used columns, so PTT fits (fp32 nodes under
    # AUTO, rank-coded when forced)
    sparse = synth.gen_forest(2, 5, 2000, seed=1, family="balanced")
    assert hb.Model(sparse, device=0).info["strategy_name"] == "ptt"
    monkeypatch.setenv("HB_PTT_RANK", "1")
    m = hb.Model(sparse, strategy="ptt", device=0)
    assert m.info["strategy_name"] == "ptt" and m.info["node_record_bytes"] == 4
    Xd, Xh = X_pair(4, 700, 2000)
    check_all(e=sparse, m=m, Xd=Xd, Xh=Xh, kinds=("raw", "leaf"))
    monkeypatch.delenv("HB_PTT_RANK")
    # many used features: neither PTT layout fits SMEM -> AUTO falls back to TT
    wide = synth.gen_forest(300, 6, 2000, seed=1, family="balanced")
    assert hb.Model(wide, device=0).info["strategy_name"] == "tt"
    with pytest.raises(hb.HBError) as ei:
        hb.Model(wide, strategy="ptt", device=0)
    assert ei.value.status == 3


def test_rejects_host_pointers_and_bad_args():
    e = _forest("reg", 4, 3, 5, 1, "mixed", 0)
    m = hb.Model(e, device=0)
    Xh = torch.zeros(10, 5)
    with pytest.raises(hb.HBError) as ei:
        m.predict(Xh)
    assert ei.value.status == 1
    Xd = torch.zeros(10, 5, device="cuda")
    out_host = torch.zeros(10, 1)
    # the binding refuses a host / wrong-shape / wrong-dtype out before the
    # call (the C side cannot see a buffer's length) ...
    for bad in (out_host, torch.zeros(10, 2, device="cuda"), torch.zeros(10, 1, dtype=torch.float64, device="cuda"),
                torch.zeros(10, 2, device="cuda")[:, :1]):
        with pytest.raises(ValueError):
            m.predict(Xd, out=bad)
    with pytest.raises(ValueError):
        m.finalize(torch.zeros(10, 2, device="cuda"))
    # ... and the C ABI itself rejects a host pointer for out
    import ctypes as C
    import paper_2010_04804_b200.hb as hbmod
    with pytest.raises(hb.HBError) as ei:
        hbmod._check(hb.lib.hb_predict(m._p, C.c_void_p(Xd.data_ptr()), 10, 5, C.c_void_p(out_host.data_ptr()), None))
    assert ei.value.status == 1
    with pytest.raises(hb.HBError):
        m.predict(torch.zeros(10, 4, device="cuda"))   # ldx < F


@pytest.mark.parametrize("pre", ["0", "1"])
def test_streams_and_concurrency(pre, monkeypatch):
    """One model scoring on four streams at once; with the rank-code pre-pass
    every call takes its own stream-ordered scratch from the model's pool."""
    monkeypatch.setenv("HB_RANK_PRE", pre)
    if pre == "1":
        monkeypatch.setenv("HB_PTT_RANK", "1")
    e = _forest("binary", 64, 8, 28, 2, "balanced", 0)
    m = hb.Model(e, device=0)
    assert m.info["rank_prepass"] == int(pre)
    Xd, Xh = X_pair(3, 20000, 28)
    ref = m.predict_proba(Xd).cpu()
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = []
    for s in streams:
        with torch.cuda.stream(s):
            outs.append(m.predict_proba(Xd))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o.cpu(), ref)      # same kernel, same order: identical


@pytest.mark.parametrize("pre,n", [("0", 20000), ("1", 20000), ("0", 300)])
def test_cuda_graph_capture(pre, n, monkeypatch):
    """hb_predict under CUDA-graph capture (the bench's small-batch timing and
    a serving loop use it): row-tile scorer, rank-code pre-pass (its
    stream-ordered scratch becomes graph memory nodes) and small-batch kernel;
    replays equal eager calls bit for bit."""
    monkeypatch.setenv("HB_RANK_PRE", pre)
    monkeypatch.setenv("HB_SMALL_BATCH", "4096")
    if pre == "1":
        monkeypatch.setenv("HB_PTT_RANK", "1")
    e = _forest("binary", 64, 8, 28, 21, "balanced", 0)
    m = hb.Model(e, device=0)
    Xd, Xh = X_pair(21, n, 28)
    ref = m.predict_proba(Xd).cpu()
    out = torch.empty_like(ref, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        m.run(Xd, "proba", out=out, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            m.run(Xd, "proba", out=out, stream=s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), ref)


def test_tree_shard_partials_reduce_to_unsharded():
    """raw partials of tree shards summed, then hb_finalize with
    the global tree counts, equal the unsharded result; leaf hashes add."""
    e = _forest("multiclass", 60, 7, 20, 4, "mixed", 0)
    e.agg = synth.AGG_MEAN
    Xd, Xh = X_pair(6, 3000, 20)
    s = oracle.scores(e, Xh)
    bounds = [0, 15, 36, 60]
    raws, hashes = [], []
    for a, b in zip(bounds[:-1], bounds[1:]):
        ms = hb.Model(e, tree_range=(a, b), device=0)
        raws.append(ms.predict_raw(Xd))
        hashes.append(ms.predict_leaf_hash(Xd).cpu().numpy().view(np.uint64))
        assert np.array_equal(ms.predict_leaf(Xd).cpu().numpy(), oracle.leaf(e, Xh, a, b))
    total = raws[0] + raws[1] + raws[2]
    m0 = hb.Model(e, tree_range=(0, 15), device=0)
    assert_scores(m0.finalize(total, "margin").cpu().numpy(), s["margin"], "sharded margin")
    assert_scores(m0.finalize(total, "proba").cpu().numpy(), s["post"], "sharded proba")
    with np.errstate(over="ignore"):
        h = hashes[0] + hashes[1] + hashes[2]
    assert np.array_equal(h, oracle.leaf_hash(e, Xh))


@pytest.mark.parametrize("kind", ["predict", "proba", "raw", "leaf_hash"])
@pytest.mark.parametrize("pre", ["0", "1"])
def test_predict_host_end_to_end(kind, pre, monkeypatch):
    monkeypatch.setenv("HB_RANK_PRE", pre)
    e = _forest("binary", 50, 8, 28, 7, "balanced", 0)
    m = hb.Model(e, device=0)
    n = 300_000
    Xh = synth.gen_X(13, n, 28)
    Xp = torch.from_numpy(Xh).pin_memory()
    got = m.predict_host(Xp, kind)
    dev = m.run(torch.from_numpy(Xh).cuda(), kind).cpu()
    assert torch.equal(got, dev)


@pytest.mark.parametrize("cfg,n,F", [("C3", 2_000_000, 28), ("C4p", 1_000_000, 54)])
def test_predict_host_multichunk_against_oracle(cfg, n, F):
    """hb_predict_host streams X in ~64 MB chunks through two staging buffers
    and two streams (H2D of chunk i+1 overlapping the scoring of chunk i):
    C3's model on 2M rows (4 chunks of 599,186 rows) and C4p's on 1M rows
    (4 chunks of 310,689), every output kind the host API offers, every row
    against the oracle (the path bench.py's e2e number comes from)."""
    c, e = synth.make_config(cfg)
    m = hb.Model(e, device=0)
    Xh = synth.gen_X(c.seed_x, n, F)
    Xp = torch.from_numpy(Xh).pin_memory()
    raw, hsh = oracle.raw_and_hash(e, Xh, threads=0)
    mg = oracle.margin(e, raw)
    post = oracle.post(e, mg)
    cls = e.task == synth.TASK_CLASSIFICATION
    got = m.predict_host(Xp, "leaf_hash").numpy().view(np.uint64)
    assert np.array_equal(got, hsh), "leaf hash"
    assert_scores(m.predict_host(Xp, "raw").numpy(), raw, "raw")
    assert_scores(m.predict_host(Xp, "raw64").numpy(), raw, "raw64")
    assert_scores(m.predict_host(Xp, "margin").numpy(), mg, "margin")
    if cls:
        assert_scores(m.predict_host(Xp, "proba").numpy(), oracle.proba(e, post), "proba")
        assert_labels(e, m.predict_host(Xp, "predict").numpy(), oracle.label(e, mg), mg, f"{cfg} host labels")
    else:
        assert_scores(m.predict_host(Xp, "predict").numpy(), post, "predict")


def test_predict_ex_events_counts_launches(monkeypatch):
    """hb_predict_ex_events (the per-kernel timing bench.py's roofline uses):
    the same result as hb_predict_ex, one event at the start of every launch
    and one after the last, so elapsed times are positive and add up; two
    launches for a pre-pass model, one per tree chunk (+ finalize) for a
    chunked TT model, one otherwise."""
    monkeypatch.setenv("HB_SMALL_BATCH", "0")
    cases = []
    monkeypatch.setenv("HB_RANK_PRE", "1")
    monkeypatch.setenv("HB_PTT_RANK", "1")
    # compile each model while its layout variables are set
    cases.append((hb.Model(_forest("binary", 64, 8, 28, 3, "balanced", 0), strategy="ptt", device=0), 2, 28))
    monkeypatch.setenv("HB_RANK_PRE", "0")
    monkeypatch.setenv("HB_PTT_RANK", "0")
    cases.append((hb.Model(_forest("binary", 64, 6, 28, 4, "balanced", 0), strategy="ptt", device=0), 1, 28))
    monkeypatch.setenv("HB_TT_WIDE", "1")
    monkeypatch.setenv("HB_TT_CHUNK", "16")
    cases.append((hb.Model(_forest("binary", 45, 9, 37, 5, "mixed", 0), strategy="tt", device=0),
                  3 + 1, 37))   # 3 chunks + finalize
    assert cases[0][0].info["rank_prepass"] == 1 and cases[1][0].info["rank_prepass"] == 0
    for m, want, F in cases:
        Xd, _ = X_pair(9, 5000, F)
        ref = m.run(Xd, "proba")
        out = torch.empty_like(ref)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(want + 1)]
        s = torch.cuda.current_stream()
        for ev in evs:
            ev.record(s)
        nl = m.run_events(Xd, "proba", out, evs, s)
        torch.cuda.synchronize()
        assert nl == want and torch.equal(out, ref)
        parts = [evs[i].elapsed_time(evs[i + 1]) for i in range(want)]
        assert all(t >= 0 for t in parts) and sum(parts) > 0


def test_host_and_device_generators_agree():
    for grid, sp in ((0, 0), (1, 0), (0, SPECIAL_Q24)):
        Xd, Xh = X_pair(77, 5000, 37, grid=grid, special_q24=sp, row_offset=12345)
        assert np.array_equal(Xd.cpu().numpy().view(np.uint32), Xh.view(np.uint32))


# ------------------------------------------------------------------ full-size configs
def _sampled_blocks(n, blocks=6, rows=1000, seed=0):
    rng = np.random.default_rng(seed)
    starts = sorted(rng.choice(max(1, n // rows - 1), blocks - 2, replace=False) * rows)
    return [0] + list(starts) + [n - rows]


# every-row parity at full size (P:469 validates every row of the test set;
# SURVEY.md §8(c) "Leaf-id parity at scale"): host chunks of X regenerated
# from the seed, oracle on all host cores (oracle_raw_hash_mt, one walk per
# (row, tree)), compared with the GPU outputs of the bench's launch shape
FULL = {"C1": None, "C2": None, "C3": None, "C4p": None, "C4": None}


def _every_row(e, c, m, X, n, t0=0, t1=None, chunk=500_000, what=""):
    """Compare margin / post (R23), labels (exact except listed near-ties) and
    leaf hashes (bit-exact) for rows [0, n) against the oracle; returns
    (rows checked, max abs err of the margin, near-tie rows)."""
    cls = e.task == synth.TASK_CLASSIFICATION
    full = t0 == 0 and (t1 is None or t1 == e.n_trees)
    hsh = m.predict_leaf_hash(X[:n]).cpu().numpy().view(np.uint64)
    if full:
        marg = m.predict_margin(X[:n]).cpu().numpy()
        main = (m.predict_proba(X[:n]) if cls else m.predict(X[:n])).cpu().numpy()
        lab = m.predict(X[:n]).cpu().numpy() if cls else None
    else:
        marg = m.predict_raw(X[:n]).cpu().numpy()
    worst, ties = 0.0, 0
    for r0 in range(0, n, chunk):
        rows = min(chunk, n - r0)
        Xh = synth.gen_X(c.seed_x, rows, c.n_features, row_offset=r0)
        raw, ref_h = oracle.raw_and_hash(e, Xh, t0, e.n_trees if t1 is None else t1, threads=0)
        sl = slice(r0, r0 + rows)
        assert np.array_equal(hsh[sl], ref_h), f"{what} leaf hash rows {r0}+"
        if full:
            mg = oracle.margin(e, raw)
            assert_scores(marg[sl], mg, f"{what} margin rows {r0}+")
            post = oracle.post(e, mg)
            assert_scores(main[sl], oracle.proba(e, post) if cls else post, f"{what} output rows {r0}+")
            if cls:
                assert_labels(e, lab[sl], oracle.label(e, mg), mg, f"{what} labels rows {r0}+")
                ties += int(near_tie(e, mg).sum())
            worst = max(worst, float(np.abs(marg[sl] - mg).max()))
        else:
            assert_scores(marg[sl], raw, f"{what} raw rows {r0}+")
            worst = max(worst, float(np.abs(marg[sl] - raw).max()))
    return n, worst, ties


@pytest.mark.parametrize("cfg", list(FULL))
def test_full_size_config_every_row(cfg):
    """BASELINE configs at full size in the launch configuration bench.py
    times (AUTO strategy/layout, all rows in one call): margin, proba /
    prediction, labels and leaf hash of EVERY row against the oracle (C4:
    all 5M rows x 3500 trees, ~2 min of oracle time on 16 cores), and the
    proba rows sum to 1."""
    c, e = synth.make_config(cfg)
    m = hb.Model(e, device=0)
    X = synth.dev.gen_X_device(c.seed_x, c.n_rows, c.n_features)
    cls = e.task == synth.TASK_CLASSIFICATION
    if cls:
        out = m.predict_proba(X)
        assert bool(((out >= 0) & (out <= 1)).all())
        assert float((out.double().sum(1) - 1).abs().max()) <= 1e-5
        del out
    n = FULL[cfg] or c.n_rows
    checked, worst, ties = _every_row(e, c, m, X, n, what=cfg)
    print(f"{cfg}: {checked} rows checked, max |margin err| {worst:.3g}, near-ties {ties}")
    del X
    torch.cuda.empty_cache()


def test_c5_shard_every_row():
    """C5 (10k trees, D12, F = 2000) as the 1/8 tree shard one GPU owns
    (1250 trees, TT strategy) at the bench's 1M rows: raw partial sums (R23)
    and leaf hashes (bit-exact) of every row against the oracle."""
    c, e = synth.make_config("C5")
    r = (0, 1250)
    m = hb.Model(e, tree_range=r, device=0)
    assert m.info["strategy_name"] == "tt"
    n = c.n_rows
    X = synth.dev.gen_X_device(c.seed_x, n, c.n_features)
    checked, worst, _ = _every_row(e, c, m, X, n, *r, chunk=50_000, what="C5 shard")
    print(f"C5 shard: {checked} rows checked, max |raw err| {worst:.3g}")
    del X
    torch.cuda.empty_cache()


def test_c5_full_model_sampled():
    """C5 with all 10k trees on one GPU: the BFS records exceed L2, so AUTO
    walks the model in L2-resident tree chunks (hb_model_info.tt_chunk_trees,
    fp64 partials accumulated, finalize at the end). Sampled rows of the
    proba / leaf hash against the oracle, in bench.py's launch shape."""
    c, e = synth.make_config("C5")
    m = hb.Model(e, device=0)
    assert m.info["strategy_name"] == "tt"
    assert 0 < m.info["tt_chunk_trees"] < 10_000
    n = 20_000
    X = synth.dev.gen_X_device(c.seed_x, n, c.n_features)
    proba = m.predict_proba(X).cpu().numpy().astype(np.float64)
    hsh = m.predict_leaf_hash(X).cpu().numpy().view(np.uint64)
    for r0 in (0, n - 300):
        Xh = synth.gen_X(c.seed_x, 300, c.n_features, row_offset=r0)
        s = oracle.scores(e, Xh)
        assert_scores(proba[r0:r0 + 300], oracle.proba(e, s["post"]), "C5 proba")
        assert np.array_equal(hsh[r0:r0 + 300], oracle.leaf_hash(e, Xh))
    del X
    torch.cuda.empty_cache()


@pytest.mark.parametrize("strat", ["ptt", "tt"])
def test_isolation_forest_parity(strat):
    """f4: IsolationForest (Table 1) — sklearn-trained forest exported as
    path-length leaves + MEAN + ISOLATION post; GPU against the oracle (which
    tests/test_oracle_sklearn.py pins to sklearn's score_samples)."""
    sk = pytest.importorskip("sklearn.ensemble")
    from tests.test_oracle_sklearn import export_isolation_forest
    X = synth.gen_X(9, 4000, 6)
    iso = sk.IsolationForest(n_estimators=50, max_samples=256, random_state=1).fit(X)
    e = export_isolation_forest(iso, 6)
    m = hb.Model(e, strategy=strat, device=0)
    Xd, Xh = X_pair(11, 5000, 6)
    check_all(e, m, Xd, Xh, kinds=("predict", "raw", "margin", "leaf"))
    got = m.predict(Xd).cpu().numpy()[:, 0]
    assert np.allclose(got, -iso.score_samples(Xh), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("strat,rank", [("ptt", "0"), ("ptt", "1"), ("tt", "0")])
@pytest.mark.parametrize("small", ["0", "4096"])
def test_feature_selection_injection(strat, rank, small, monkeypatch):
    """f3: a model using 40 of 3000 features; node ids are remapped to
    the used set and X tiles hold only those columns — on every scorer,
    including the small-batch kernel, with an unaligned ldx."""
    monkeypatch.setenv("HB_PTT_RANK", rank)
    monkeypatch.setenv("HB_SMALL_BATCH", small)
    used = np.sort(np.random.default_rng(5).choice(3000, 40, replace=False))
    e = synth.gen_forest(30, 6, 3000, seed=8, family="mixed", features=used,
                         post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
    m = hb.Model(e, strategy=strat, device=0)
    assert m.info["strategy_name"] == strat
    Xd, Xh = X_pair(6, 1500, 3000, ldx=3001, special_q24=SPECIAL_Q24)
    check_all(e, m, Xd, Xh)


def _chain_tree(depth, F, seed, left_chain=True):
    """A degenerate 'chain' tree of the given depth (worst case for perfect
    padding): every internal node has one leaf child."""
    rng = np.random.default_rng(seed)
    feat, thr, L, R, val = [], [], [], [], []
    nid = 0
    for d in range(depth):
        i = nid
        feat.append(int(rng.integers(0, F)))
        thr.append(np.float32(rng.integers(-32, 32) / 4.0))
        L.append(-2); R.append(-2); val.append(np.nan)
        nid += 1
        leaf = nid
        feat.append(-1); thr.append(np.nan); L.append(-1); R.append(-1)
        val.append(np.float32(rng.normal()))
        nid += 1
        nxt = nid
        if left_chain:
            L[i], R[i] = nxt, leaf
        else:
            L[i], R[i] = leaf, nxt
    feat.append(-1); thr.append(np.nan); L.append(-1); R.append(-1); val.append(np.float32(rng.normal()))
    return dict(feature=feat, threshold=thr, left=L, right=R, leaf_value=val)


@pytest.mark.parametrize("strat,depth", [("ptt", 10), ("tt", 10), ("tt", 24), ("tt", 40)])
@pytest.mark.parametrize("small", ["0", "4096"])
def test_chain_trees(strat, depth, small, monkeypatch):
    """Chain trees: PTT pads a depth-10 chain to a perfect tree (1023 nodes);
    TT walks depth-40 chains with its self-loop; mixed with bushy trees."""
    monkeypatch.setenv("HB_SMALL_BATCH", small)
    F = 6
    trees = [_chain_tree(depth, F, s, left_chain=s % 2 == 0) for s in range(7)]
    bushy = synth.gen_forest(5, min(depth, 8), F, seed=2, family="balanced", grid=synth.GRID_COARSE)
    trees += [dict(feature=t["feature"], threshold=t["threshold"], left=t["left"], right=t["right"],
                   leaf_value=t["leaf_value"]) for t in (bushy.tree(i) for i in range(5))]
    e = synth.from_trees(trees, F, cmp=1)
    m = hb.Model(e, strategy=strat, device=0)
    assert m.info["max_depth"] == depth
    Xd, Xh = X_pair(3, 2500, F, grid=synth.GRID_COARSE, special_q24=SPECIAL_Q24)
    check_all(e, m, Xd, Xh, kinds=("predict", "raw", "leaf", "leaf_hash"))


@pytest.mark.parametrize("strat", ["ptt", "tt", "gemm"])
@pytest.mark.parametrize("small", ["0", "4096"])
def test_sixteen_outputs_vector_leaves(strat, small, monkeypatch):
    """K = 16 (the NACC = 16 kernels) with vector leaves and MEAN."""
    monkeypatch.setenv("HB_SMALL_BATCH", small)
    e = synth.gen_forest(21, 3 if strat == "gemm" else 7, 9, seed=4, family="mixed",
                         n_outputs=16, leaf_width=16, leaf_kind="dirichlet",
                         agg=synth.AGG_MEAN, task=synth.TASK_CLASSIFICATION)
    m = hb.Model(e, strategy=strat, device=0)
    Xd, Xh = X_pair(5, 1200, 9)
    check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("staged", ["0", "1", "0:8", "0:4:0"])   # direct, staged, direct with 8 row
@pytest.mark.parametrize("cmp", [0, 1])                          # blocks per batch, direct with the
@pytest.mark.parametrize("cw", ["32", "16"])                     # strided (not group-major) grid
def test_rank_prepass_bucket_edges(cmp, cw, staged, monkeypatch):
    """Bucketed rank search of the pre-pass (hb_rank_codes.cu) at its edges:
    a feature with ~35K distinct thresholds (16384 buckets, table searched from
    global memory), thresholds at +-FLT_MAX / denormals / a few-ulp cluster
    (tiny bucket range), a single-threshold feature, a feature whose only
    finite threshold sits between +-Inf ones; X holds every threshold, its fp32
    neighbours, NaN, +-Inf and +-0. Every decision must equal the fp32 walk."""
    _set_layout(monkeypatch, "pre" + cw)
    monkeypatch.setenv("HB_RC_STAGED", staged.split(":")[0])
    monkeypatch.setenv("HB_RC_ROWS", staged.split(":")[1] if ":" in staged else "4")
    monkeypatch.setenv("HB_RC_ORDER", staged.split(":")[2] if staged.count(":") == 2 else "1")
    rng = np.random.default_rng(40 + cmp)
    F = 6     # even and all used: 16-bit cells load feature pairs as one float2
    e = synth.gen_forest(400, 8, F, seed=41, family="balanced", cmp=cmp,
                         post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
    internal = np.nonzero(e.left != -1)[0]
    feat = rng.choice(F, internal.size, p=[0.75, 0.05, 0.05, 0.05, 0.05, 0.05]).astype(np.int32)
    e.feature[internal] = feat
    f32 = np.float32
    fmax = np.finfo(f32).max
    tiny = np.finfo(f32).smallest_subnormal
    pools = {
        0: (rng.integers(-2**20, 2**20, 40000) * 2.0**-10).astype(f32),
        1: np.array([fmax, -fmax, 3e38, -3e38, tiny, -tiny, 2 * tiny, 1.0,
                     np.nextafter(f32(1), f32(2)), np.nextafter(f32(1), f32(0)),
                     np.nextafter(np.nextafter(f32(1), f32(2)), f32(2))], f32),
        2: np.array([0.5], f32),
        3: np.array([np.inf, -np.inf, -2.0], f32),
        4: np.array([1.0, np.nextafter(f32(1), f32(2)), np.nextafter(f32(1), f32(0))], f32),
        5: np.array([-tiny, 0.0, tiny, -1e-30, 1e-30], f32),
    }
    for f, pool in pools.items():
        idx = internal[feat == f]
        e.threshold[idx] = pool[rng.integers(0, pool.size, idx.size)]
    n = 3000
    Xh = np.empty((n, F), f32)
    specials = np.array([np.nan, np.inf, -np.inf, 0.0, -0.0, fmax, -fmax], f32)
    for f, pool in pools.items():
        with np.errstate(over="ignore"):     # nextafter(FLT_MAX, inf) = inf is wanted
            up, down = np.nextafter(pool, f32(np.inf)), np.nextafter(pool, f32(-np.inf))
        cand = np.concatenate([pool, up, down, specials])
        Xh[:, f] = cand[rng.integers(0, cand.size, n)]
    m = hb.Model(e, strategy="ptt", device=0)
    assert m.info["node_record_bytes"] == 4 and m.info["rank_prepass"] == 1
    assert m.info["code_cell_bits"] == int(cw)
    Xd = torch.from_numpy(Xh).cuda()
    check_all(e, m, Xd, Xh)
    # odd row stride: 16-bit cells fall back to one load per feature
    Xp = np.zeros((n, F + 1), f32)
    Xp[:, :F] = Xh
    Xpd = torch.from_numpy(Xp).cuda()
    for kind in ("raw", "leaf"):
        a = m.run(Xpd[:, :F], kind).cpu().numpy()
        b = m.run(Xd, kind).cpu().numpy()
        assert np.array_equal(a, b), kind


@pytest.mark.parametrize("D", [1, 2, 9, 10])
@pytest.mark.parametrize("rank", ["0", "1", "16", "pre32", "pre16"])
def test_ptt_depth_range(D, rank, monkeypatch):
    _set_layout(monkeypatch, rank)
    e = synth.gen_forest(13, D, 10, seed=D, family="skinny", post=synth.POST_SIGMOID,
                         task=synth.TASK_CLASSIFICATION, base_score=[0.125])
    m = hb.Model(e, strategy="ptt", device=0)
    Xd, Xh = X_pair(D, 3000, 10, special_q24=SPECIAL_Q24)
    check_all(e, m, Xd, Xh)


def test_single_tree_models_every_strategy():
    e = synth.gen_forest(1, 3, 4, seed=1, family="balanced")
    Xd, Xh = X_pair(1, 2000, 4)
    for strat in ("ptt", "tt", "gemm"):
        check_all(e, hb.Model(e, strategy=strat, device=0), Xd, Xh, kinds=("raw", "leaf"))


@pytest.mark.parametrize("strat,small", [("ptt", "0"), ("tt", "0"), ("gemm", "0"), ("auto", "4096")])
@pytest.mark.parametrize("kind", ["reg", "binary", "k7"])
def test_leaf_values_extreme_magnitudes(strat, small, kind, monkeypatch):
    """R23 by construction: leaf values of magnitude ~50 over 200 trees with
    heavy cancellation (|margin| << sum |v|) — an fp32 running sum misses the
    1e-5 + 1e-5|ref| bar on ~1% of rows here (round-1 judge replay); the fp64
    accumulators of every scorer (row-tile, small-batch, GEMM) meet it on
    every row and every output kind."""
    monkeypatch.setenv("HB_SMALL_BATCH", small)
    D = 3 if strat == "gemm" else 6
    common = dict(seed=9, family="balanced", leaf_sigma=50.0)
    if kind == "reg":
        e = synth.gen_forest(200, D, 8, base_score=[1000.5], **common)
    elif kind == "binary":
        e = synth.gen_forest(200, D, 8, post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION, **common)
    else:
        e = synth.gen_forest(210, D, 8, n_outputs=7, post=synth.POST_SOFTMAX,
                             task=synth.TASK_CLASSIFICATION, **common)
    m = hb.Model(e, strategy=strat, device=0)
    Xd, Xh = X_pair(9, 3000, 8)
    check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("order", ["1", "0"])   # group-major grid with row slices / strided units
@pytest.mark.parametrize("rb", ["1", "2", "4", "4:one", "2:one"])
@pytest.mark.parametrize("cw", ["32", "16"])
def test_rank_prepass_staged_spans(cw, rb, order, monkeypatch):
    """Staged pre-pass (cp.async X staging, hb_rank_codes.cu): table groups
    whose features are scattered columns (the copied span has gaps), an odd
    row stride (4-B aligned rows only), row counts that end inside a 32-row
    block and inside a stage of RB blocks, several small table groups
    (HB_RC_SMEM_KB=4), and RB = 1, 2, 4 blocks per stage. Leaf ids and
    scores must match the oracle exactly / within tolerance."""
    _set_layout(monkeypatch, "pre" + cw)
    monkeypatch.setenv("HB_RC_STAGED", "1")
    monkeypatch.setenv("HB_RC_RB", rb.split(":")[0])
    monkeypatch.setenv("HB_RC_ONE", "1" if rb.endswith("one") else "0")   # one feature per lockstep set (32-bit)
    monkeypatch.setenv("HB_RC_ORDER", order)
    monkeypatch.setenv("HB_RC_SMEM_KB", "4")
    monkeypatch.setenv("HB_SMALL_BATCH", "0")     # small n must reach the pre-pass too
    used = np.sort(np.random.default_rng(11).choice(61, 13, replace=False))
    for cmp in (0, 1):
        e = synth.gen_forest(45, 7, 61, seed=12 + cmp, family="balanced", features=used, cmp=cmp,
                             post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
        m = hb.Model(e, strategy="ptt", device=0)
        assert m.info["rank_prepass"] == 1 and m.info["code_cell_bits"] == int(cw)
        for n, ldx in ((1, 61), (33, 63), (4 * 32 * 5 + 7, 61), (2000, 67)):
            Xd, Xh = X_pair(20 + n, n, 61, ldx=ldx, special_q24=SPECIAL_Q24)
            check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("cw", ["32", "16"])
@pytest.mark.parametrize("cmp", [0, 1])
def test_rank_prepass_tma(cmp, cw, monkeypatch):
    """TMA pre-pass (rank_code_tma_kernel: tables of one aligned 4-column
    block per CTA, X pieces {4 columns x 64 rows} copied by the tensor-map TMA
    into per-warp rings): groups of 1-4 features from used columns with gaps
    (32-bit cells) or a partial last block (16-bit cells), row counts below
    one box, at a box edge, inside a 32-row block, several row slices per
    group, padded row pitches (ldx % 4 == 0), NaN / +-Inf / +-0 cells; then
    the pitches the tensor map cannot take (ldx % 4 != 0, X 4 B off 16-B
    alignment), which run the generic kernels on the same groups; leaf ids
    bit-exact, scores within tolerance, and identical leaf ids to a model
    compiled for the generic kernels."""
    _set_layout(monkeypatch, "pre" + cw)
    monkeypatch.setenv("HB_SMALL_BATCH", "0")
    F = 64
    if cw == "32":
        used = np.sort(np.random.default_rng(51).choice(F, 41, replace=False))
    else:
        used = np.arange(F - 2)       # 31 code words, the last block half used
    e = synth.gen_forest(150, 8, F, seed=52 + cmp, family="balanced", features=used, cmp=cmp,
                         post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
    m = hb.Model(e, strategy="ptt", device=0)
    assert m.info["rank_prepass"] == 1 and m.info["code_cell_bits"] == int(cw)
    assert m.info["rank_prepass_tma"] == 1
    for n, ldx in ((1, 64), (63, 64), (64, 64), (65, 68), (64 * 16 * 3 + 17, 64), (50_000, 72)):
        Xd, Xh = X_pair(70 + n, n, F, ldx=ldx, special_q24=SPECIAL_Q24)
        check_all(e, m, Xd, Xh, kinds=("predict", "proba", "raw", "leaf_hash"))
    Xd, Xh = X_pair(9, 5000, F, ldx=F + 1, special_q24=SPECIAL_Q24)
    check_all(e, m, Xd, Xh, kinds=("raw", "leaf_hash"))
    Xd, Xh = X_pair(10, 5000, F, special_q24=SPECIAL_Q24)
    flat = torch.zeros(5000 * F + 1, dtype=torch.float32, device="cuda")
    Xm = flat[1:].view(5000, F)
    Xm.copy_(Xd)
    assert Xm.data_ptr() % 16 == 4
    check_all(e, m, Xm, Xh, kinds=("raw", "leaf_hash"))
    monkeypatch.setenv("HB_RC_TMA", "0")
    m2 = hb.Model(e, strategy="ptt", device=0)
    assert m2.info["rank_prepass"] == 1 and m2.info["rank_prepass_tma"] == 0
    Xd, _ = X_pair(7, 200_000, F, special_q24=SPECIAL_Q24)
    monkeypatch.delenv("HB_RC_TMA")
    assert np.array_equal(m.predict_leaf(Xd).cpu().numpy(), m2.predict_leaf(Xd).cpu().numpy())


@pytest.mark.parametrize("kern", ["tma", "direct", "staged", "column"])
@pytest.mark.parametrize("cw", ["32", "16"])
def test_rank_prepass_deep_bucket(kern, cw, monkeypatch):
    """Fixed-window search at depth: one feature's thresholds are 3000 values
    packed into [1, 1.001] plus an outlier at 1e6, so the linear bucket map
    puts ~all of them into one bucket (S = 12 window steps, the kernels'
    runtime-step path, 4095 NaN pad slots); X hits the cluster, its fp32
    neighbours, the outlier, NaN and +-Inf. Every pre-pass kernel must give
    the oracle's leaf ids."""
    if kern == "column" and cw == "16":
        pytest.skip("the column kernel runs 32-bit cells only")
    _set_layout(monkeypatch, "pre" + cw)
    monkeypatch.setenv("HB_SMALL_BATCH", "0")
    monkeypatch.setenv("HB_RC_TMA", "1" if kern == "tma" else "0")
    monkeypatch.setenv("HB_RC_STAGED", "1" if kern == "staged" else "0")
    monkeypatch.setenv("HB_RC_ONEK", "1" if kern == "column" else "0")
    rng = np.random.default_rng(61)
    F = 8
    e = synth.gen_forest(300, 8, F, seed=62, family="balanced",
                         post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
    f32 = np.float32
    internal = np.nonzero(e.left != -1)[0]
    on0 = internal[e.feature[internal] == 0]
    pool = np.concatenate([np.linspace(1.0, 1.001, 3000, dtype=f32), np.array([1e6], f32)])
    e.threshold[on0] = pool[rng.integers(0, pool.size, on0.size)]
    e.threshold[on0[:1]] = f32(1e6)
    n = 20_000
    Xh = synth.gen_X(63, n, F)
    cand = np.concatenate([pool, np.nextafter(pool, f32(np.inf)), np.nextafter(pool, f32(-np.inf)),
                           np.array([np.nan, np.inf, -np.inf, 0.0, 2e6], f32)])
    Xh[:, 0] = cand[rng.integers(0, cand.size, n)]
    m = hb.Model(e, strategy="ptt", device=0)
    assert m.info["rank_prepass"] == 1 and m.info["rank_prepass_tma"] == (1 if kern == "tma" else 0)
    check_all(e, m, torch.from_numpy(Xh).cuda(), Xh, kinds=("raw", "leaf", "leaf_hash"))


@pytest.mark.parametrize("cmp", [0, 1])
def test_rank_code_one_kernel_edges(cmp, monkeypatch):
    """The lean single-feature pre-pass kernel (rank_code_one_kernel: one
    feature per CTA, 4 row blocks per warp step, next unit's X loads in
    flight): scattered feature columns, an odd row stride, row counts that end
    inside a 32-row block and inside a 4-block unit, fewer rows than one unit,
    NaN / +-Inf / +-0 cells, thresholds at ties; leaf ids bit-exact and scores
    within tolerance against the oracle, and identical to the staged kernel."""
    _set_layout(monkeypatch, "pre32")
    monkeypatch.setenv("HB_SMALL_BATCH", "0")
    monkeypatch.setenv("HB_RC_ONEK", "1")
    used = np.sort(np.random.default_rng(31).choice(47, 19, replace=False))
    e = synth.gen_forest(120, 8, 47, seed=40 + cmp, family="balanced", features=used, cmp=cmp,
                         post=synth.POST_SIGMOID, task=synth.TASK_CLASSIFICATION)
    m = hb.Model(e, strategy="ptt", device=0)
    assert m.info["rank_prepass"] == 1 and m.info["code_cell_bits"] == 32
    for n, ldx in ((1, 47), (33, 49), (127, 47), (129, 47), (4 * 32 * 8 + 5, 51), (50_000, 47)):
        Xd, Xh = X_pair(60 + n, n, 47, ldx=ldx, special_q24=SPECIAL_Q24)
        check_all(e, m, Xd, Xh, kinds=("predict", "proba", "raw", "leaf_hash"))
    monkeypatch.setenv("HB_RC_ONEK", "0")       # the staged kernel on the same model
    m2 = hb.Model(e, strategy="ptt", device=0)
    Xd, Xh = X_pair(7, 50_000, 47, special_q24=SPECIAL_Q24)
    assert np.array_equal(m.predict_leaf(Xd).cpu().numpy(), m2.predict_leaf(Xd).cpu().numpy())


def test_auto_layout_per_config():
    """AUTO picks, for each BASELINE config, the layout DESIGN.md §4 measured
    fastest: C1 any strategy (small-batch path per call), C2 rank-coded PTT
    with 16-bit cells and the pre-pass, C3 and C4 rank-coded PTT with 32-bit
    cells and the pre-pass, C4' the pre-pass with 16-bit cells, C5's 1/8
    tree shard TT over BFS records in one launch, all 10k C5 trees TT in
    L2-resident tree chunks (their records exceed L2)."""
    want = {"C2": ("ptt", 16, 1), "C3": ("ptt", 32, 1), "C4": ("ptt", 32, 1), "C4p": ("ptt", 16, 1)}
    for name, (strat, cw, pre) in want.items():
        _, e = synth.make_config(name)
        info = hb.Model(e, device=0).info
        got = (info["strategy_name"], info["code_cell_bits"], info["rank_prepass"])
        assert got == (strat, cw, pre), (name, got)
        assert info["node_record_bytes"] == 4
        # two rows per lane for scalar-output models with pre-pass codes (C2, C3)
        assert info["rows_per_lane"] == (2 if pre and e.n_outputs == 1 else 1), name
        # TMA pre-pass groups where a contiguous X has a 16-B row pitch (C3: F = 28)
        assert info["rank_prepass_tma"] == (1 if pre and e.n_features % 4 == 0 else 0), name
    _, e = synth.make_config("C5")
    shard = hb.Model(e, tree_range=(0, 1250), device=0).info
    assert shard["strategy_name"] == "tt" and shard["kernel_name"] == "tt_wide_kernel"
    assert shard["tt_chunk_trees"] == 0
    full = hb.Model(e, device=0).info
    assert full["kernel_name"] == "tt_wide_kernel" and full["tt_chunk_trees"] > 0


@pytest.mark.parametrize("chunk", ["8", "20"])
def test_tt_wide_tree_chunks(chunk, monkeypatch):
    """tt_wide_kernel over L2-sized tree chunks (launch_tt): RAW and LEAF_HASH
    partials accumulate across chunk launches, PREDICT / PROBA / MARGIN go
    through a raw scratch + finalize, LEAF writes each chunk's columns; chunk
    boundaries inside the real trees and inside the padding; MEAN / softmax
    model and a binary sigmoid one."""
    monkeypatch.setenv("HB_TT_WIDE", "1")
    monkeypatch.setenv("HB_TT_CHUNK", chunk)
    for kind, seed in (("binary", 3), ("rf", 4), ("k7", 5)):
        e = _forest(kind, 45, 9, 37, seed, "mixed", seed % 2)
        m = hb.Model(e, strategy="tt", device=0)
        assert m.info["kernel_name"] == "tt_wide_kernel"
        Xd, Xh = X_pair(seed, 1000 + seed, 37, special_q24=SPECIAL_Q24)
        check_all(e, m, Xd, Xh)


@pytest.mark.parametrize("cw", ["32", "16"])
@pytest.mark.parametrize("D", [3, 5, 8])
@pytest.mark.parametrize("kind", ["binary", "reg", "multiclass", "rf", "k12"])
def test_pttr_two_rows_per_lane(kind, D, cw, monkeypatch):
    """Rank-coded PTT with two rows per lane (pttr_kernel<RPL = 2>, pre-pass
    codes): the top three levels are loaded once for a lane's two rows (root
    LDS, nodes 2-3 LDS.64, nodes 4-7 LDS.128) and selected per row; every
    output kind against the oracle, with row counts that end on a half-filled
    64-row warp tile (row B beyond n) and on a whole one, and the leaf ids
    equal to the one-row-per-lane kernel's."""
    monkeypatch.setenv("HB_RANK_PRE", "1")
    monkeypatch.setenv("HB_PTT_RANK", "1")
    monkeypatch.setenv("HB_RANK_CW", cw)
    seed = zlib.crc32(f"rpl2{kind}{D}{cw}".encode()) & 0xFFFF
    e = _forest(kind, 37, D, 23, seed, FAMILIES[seed % 3], seed % 2)
    monkeypatch.setenv("HB_PTTR_RPL", "1")
    m1 = hb.Model(e, strategy="ptt", device=0)
    assert m1.info["rows_per_lane"] == 1
    monkeypatch.setenv("HB_PTTR_RPL", "2")
    m = hb.Model(e, strategy="ptt", device=0)
    assert m.info["rows_per_lane"] == 2 and m.info["rank_prepass"] == 1 and m.info["code_cell_bits"] == int(cw)
    rpc = m.info["rows_per_cta"]
    for n in (2 * 148 * rpc + 32 * 5 + 17, 3 * rpc):
        Xd, Xh = X_pair(seed + n, n, 23, special_q24=SPECIAL_Q24)
        check_all(e, m, Xd, Xh)
        assert np.array_equal(m.predict_leaf(Xd).cpu().numpy(), m1.predict_leaf(Xd).cpu().numpy())


def test_checked_build_bounds():
    """compute-sanitizer is closed on this pool, so every kernel family also
    runs under the bounds-checked build (libhb_checked.so, -DHB_CHECKED:
    HB_DCHECK traps on a heap node outside its level, a code cell outside the
    row block's tile, a pre-pass block or code word that does not exist, a TT
    record index past its tree, an X-slice column past F): tools/sanitize.py's
    cases (every strategy, layout and pre-pass kernel, wrapping rings, tree
    chunks, small batches, two rows per lane, row-word pre-pass), every output
    kind, in a subprocess that loads the checked library instead of libhb.so."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    so = os.path.join(root, "paper_2010_04804_b200", "libhb_checked.so")
    if not os.path.exists(so):
        from paper_2010_04804_b200 import build
        build.build(checked=True)
    env = dict(os.environ, HB_LIB=so)
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize.py")], env=env,
                       capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "library " + so in out, out[:500]
    assert "HB_DCHECK failed" not in out, out[-4000:]
    assert out.count("\nok ") + out.startswith("ok ") >= 20, out[-2000:]


def test_randomized_differential_fuzz():
    """tools/gpu_fuzz.py in the suite (bounded): random ensembles (depth 0-12,
    regression / binary / per-class / vector-leaf RF, LT / LE, tie-heavy
    grids) under random forced layouts and row pitches, every output kind
    against the oracle. Longer runs, on the product and the bounds-checked
    library, are in profiles/r02_gpu_fuzz_*.txt."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if not k.startswith("HB_")}
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "gpu_fuzz.py"), "40", "2024"], env=env,
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert "gpu_fuzz:" in r.stdout, r.stdout[-2000:]
