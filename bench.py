#!/usr/bin/env python
"""Benchmark: rows/sec scored (500 trees, depth 8) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
                    [--scaling strong|weak] [--impl ours|reference] [--strategy auto]
                    [--no-e2e] [--no-cpu]

One "step" is one pass of the whole hot path over one batch: one hb_predict
(proba for classification, predict for regression) call over all rows of the
rank's shard — X tile staging, the strategy's traversal, ensemble accumulate,
epilogue, store; two launches when the model runs the rank-code pre-pass, one
per L2-resident tree chunk plus a finalize for chunked TT models.

Multi-GPU: row-sharded configs (C1-C4) split the config's
rows over the ranks with no data-path collective (strong scaling, the
BASELINE "10M rows, rows sharded over 1/2/4/8 GPUs"; --scaling weak gives
every rank the full row count instead); C5 shards trees: every rank scores all
rows with its tree range, fp64 partials go through one NCCL reduce to rank 0,
which finalizes. Timing: W untimed warm-up steps, then K steps bracketed by
barrier + cuda synchronize, CUDA events on the launching stream, max over
ranks. X (> L2) is resident in HBM before the timed region. ``e2e`` repeats the
metric through hb_predict_host from pinned host memory (H2D of X and D2H of
the result inside the timed region).

The roofline names the dominant kernel of the call: its duration is measured
live by CUDA events the library records between its launches
(hb_predict_ex_events) over the timed steps; its algorithmic bytes are
SURVEY.md §8(d)'s per-row figure times the rows. ``traffic`` is the DRAM bytes
of every launch of one call (ncu, profiles/ncu_traffic.json) with the split.
``parity`` compares the GPU outputs with the oracle on the rows the oracle
baseline timed (outside the timed region).

--impl reference times the CPU oracle (the only reference this tier has) on a
bounded sample per step, on the host cores; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "rows/sec scored (500 trees, depth 8) at 1/2/4/8 B200; % of HBM/tensor roofline"
TOL = "|gpu - oracle| <= 1e-5 + 1e-5 |oracle| (P:469; DESIGN.md R23)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--rows", type=int, default=0, help="override the config's total rows")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="row-sharded configs: strong = the config's rows split over the ranks "
                         "(default); weak = every rank scores the full row count")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--shard", default=None, choices=["rows", "trees"],
                    help="default: trees for C5, rows otherwise")
    ap.add_argument("--emulate-gpus", type=int, default=0,
                    help="trees mode on ONE GPU: score only rank 0's tree shard of an "
                         "N-GPU run (the per-GPU piece of C5 on 8 GPUs); no reduce")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: run every rank on one device (multi-rank code path on a 1-GPU box)
    if os.environ.get("HB_BENCH_ONE_DEVICE"):
        local = 0
    return rank, world, local


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), "--query-gpu=" + self.FIELDS,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
            return
        # wait for the first sample (nvidia-smi can take a second to start),
        # so the timed region is sampled from its first step
        t0 = time.time()
        while time.time() - t0 < 5.0 and os.path.getsize(self.f.name) == 0:
            time.sleep(0.05)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)   # one more sample after the timed region
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        load = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------- oracle (CPU baseline)
def truncated_mean(xs):
    """"run all the experiments 5 times and report the truncated mean
    (by averaging the middle values)"."""
    s = sorted(xs)
    mid = s[1:-1] if len(s) >= 3 else s
    return float(np.mean(mid))


def oracle_call(e, X, t0, t1, threads):
    """What the oracle baseline computes for the line's workload: full scoring
    (raw -> margin -> post) for a whole model, raw sums for a tree shard."""
    import oracle
    if t0 == 0 and t1 == e.n_trees:
        return oracle.predict_mt(e, X, threads=threads)[1]
    oracle.raw(e, X, t0, t1, threads=threads if threads else 0)
    return threads or os.cpu_count()


def time_oracle(e, cfg, t0, t1, run_s=2.5, runs=5, threads=0, max_rows=None):
    """Oracle throughput on a bounded prefix of the workload's rows: `runs`
    timed runs of ~run_s each (5 runs, truncated mean; the min is
    reported too). Returns a dict (rate from the truncated mean of the run
    times, rows, cores)."""
    import synth
    max_rows = max_rows or cfg.n_rows
    probe = min(1000, max_rows)
    Xp = synth.gen_X(cfg.seed_x, probe, cfg.n_features)
    t = time.perf_counter()
    oracle_call(e, Xp, t0, t1, threads)
    rate = probe / max(time.perf_counter() - t, 1e-4)
    rows = int(min(max_rows, max(probe, rate * run_s)))
    X = synth.gen_X(cfg.seed_x, rows, cfg.n_features)
    times, used = [], 1
    for _ in range(runs):
        t = time.perf_counter()
        used = oracle_call(e, X, t0, t1, threads)
        times.append(time.perf_counter() - t)
    tm = truncated_mean(times)
    return {"value": rows / tm, "unit": "rows/s", "cores": int(used), "rows": rows,
            "runs": runs, "seconds_truncated_mean": tm, "seconds_min": min(times),
            "value_at_min": rows / min(times), "seconds_all": times}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return ""


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    import oracle
    import synth
    cfg, e = synth.make_config(args.config)
    # size each step for ~4 s of CPU work (HB_REF_STEP_S overrides)
    step_s = float(os.environ.get("HB_REF_STEP_S", "4.0"))
    r0 = time_oracle(e, cfg, 0, e.n_trees, run_s=min(0.5, step_s), runs=1)
    rows = int(min(cfg.n_rows, max(100, r0["value"] * step_s)))
    X = synth.gen_X(cfg.seed_x, rows, cfg.n_features)
    for _ in range(args.warmup):
        oracle.predict_mt(e, X[: max(1, rows // 8)])
    times, used = [], 1
    for _ in range(args.steps):
        t = time.perf_counter()
        _, used = oracle.predict_mt(e, X)
        times.append(time.perf_counter() - t)
    ms = 1e3 * float(np.mean(times))
    value = rows / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(cfg, e, rows, args),
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": used, "kind": "oracle",
                         "sample": f"first {rows} rows of {cfg.name} per step", "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, e, rows, args, mode="rows", scaling="strong", world=1):
    if mode == "rows":
        par = (f"rows sharded over {world} GPU(s), no collective ({scaling} scaling: "
               + ("the config's rows split over the ranks)" if scaling == "strong"
                  else "every rank scores the full row count)"))
    else:
        par = f"trees sharded over {world} GPU(s), one NCCL reduce of fp64 partials + finalize"
    return {"workload": f"{cfg.name}: {cfg.note}", "rows_total": rows, "n_trees": e.n_trees,
            "max_depth": cfg.depth, "n_features": cfg.n_features, "n_outputs": e.n_outputs,
            "family": cfg.family, "parallelism": par,
            "l2": ("X larger than L2 (streamed once per step, no flush needed); model (<13 MB) "
                   "L2-resident by design" if cfg.depth <= 10 else
                   "X larger than L2 (streamed once per step, no flush needed); depth-12 node records: "
                   "a 1/8 tree shard (~60 MB) is L2-resident, all 10k trees (~480 MB) are not")}


def launch_names(info, n, kind):
    """Kernel names of one call's launches, in order (hb_predict_ex_events):
    rank-code pre-pass + scorer; one launch per L2-resident tree chunk plus a
    finalize unless the output is accumulated in place (raw64, leaf hash)."""
    if n <= info["small_batch_max_rows"]:
        return ["small_batch_kernel"]
    if info.get("rank_prepass"):
        # TMA pre-pass on the bench's X (16-B aligned rows of 4k floats: C2,
        # C3, C4), else one of the generic pre-pass kernels
        tma = info.get("rank_prepass_tma") and info["n_features"] % 4 == 0   # contiguous X: ldx = F
        return ["rank_code_tma_kernel" if tma else "rank_code_kernel", "pttr_kernel"]
    chunk = info.get("tt_chunk_trees", 0)
    if chunk:
        pad = (info["n_trees"] + 3) // 4 * 4
        fin = [] if kind in ("raw64", "leaf_hash", "leaf") else ["finalize_kernel"]
        return [info["kernel_name"]] * (-(-pad // chunk)) + fin
    return [info["kernel_name"]]


def load_traffic(config, layout, rows, trees):
    """DRAM traffic of one call (every launch) from profiles/ncu_traffic.json,
    recorded by tools/traffic.py from one ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
    except (OSError, ValueError):
        return None
    return d.get(f"{config}:{layout}:{rows}:{trees}")


# ----------------------------------------------------------------- ours
def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("HB_BENCH_BACKEND", "nccl")   # gloo: 1-GPU multi-rank test
        # communicator set-up (transports, NVLink / NVLS channels) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2010_04804_b200 as hb
    import synth
    import synth.dev
    from paper_2010_04804_b200.dist import max_over_ranks, reduce_partials, row_shard, tree_shard

    cfg, e = synth.make_config(args.config)
    n_total = args.rows or cfg.n_rows
    mode = args.shard or ("trees" if cfg.name == "C5" else "rows")
    if args.emulate_gpus and world > 1 and args.emulate_gpus != world:
        raise SystemExit("--emulate-gpus N with several ranks needs N == world size")
    cls = e.task == synth.TASK_CLASSIFICATION
    kind = "proba" if cls else "predict"
    stream = torch.cuda.current_stream(local)
    scaling = args.scaling
    if mode == "rows":
        # rows sharded, model replicated, no data-path collective
        if scaling == "strong":
            r0, n = row_shard(n_total, rank, world)
        else:
            r0, n = rank * n_total, n_total
        t0, t1 = 0, e.n_trees
        m = hb.Model(e, strategy=args.strategy, device=local)
        X = synth.dev.gen_X_device(cfg.seed_x, n, cfg.n_features, row_offset=r0, device=local)
        out = m._out(n, kind, None, X.device)
        call_kind, call_out = kind, out
        rows_all = n_total if scaling == "strong" else n_total * world
    else:
        # trees sharded, all rows on every rank; one NCCL reduce of fp64
        # partials to rank 0, which finalizes (strong scaling over trees)
        shards = max(world, args.emulate_gpus)
        t0, t1 = tree_shard(e.n_trees, rank, shards, e.n_outputs, e.leaf_width)
        m = hb.Model(e, strategy=args.strategy, device=local, tree_range=(t0, t1))
        r0, n = 0, n_total
        X = synth.dev.gen_X_device(cfg.seed_x, n, cfg.n_features, device=local)
        raw = torch.empty((n, e.n_outputs), dtype=torch.float64, device=X.device)
        out = m._out(n, kind, None, X.device)
        call_kind, call_out = "raw64", raw
        rows_all = n
        scaling = "strong"
    info = m.info
    names = launch_names(info, n, call_kind)
    small = n <= info["small_batch_max_rows"]

    def tail():
        """The rest of a trees-mode step after the scorer call."""
        if mode == "trees":
            if dist:
                reduce_partials(raw, dst=0)
            if rank == 0:
                m.finalize(raw, kind, out=out, stream=stream)

    # request/response batch sizes (small-batch kernel) are launch-bound from
    # Python: capture `calls` calls in one CUDA graph and replay it, so the
    # device time per call is measured instead of the host issue rate
    calls = 1
    graph = None
    if mode == "rows" and small:
        calls = int(os.environ.get("HB_BENCH_GRAPH_CALLS", "200"))
        gs = torch.cuda.Stream(local)
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            for _ in range(3):
                m.run(X, kind, out=out, stream=gs)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            for _ in range(calls):
                m.run(X, kind, out=out, stream=gs)
        torch.cuda.synchronize()

    # per-launch events recorded by the library (hb_predict_ex_events)
    nev = len(names) + 1
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(args.steps)]
    for row in evs:
        for ev in row:
            ev.record(stream)          # creates the CUDA events up front

    def step(i=None):
        if graph is not None:
            graph.replay()
            return 1
        if i is None:
            m.run(X, call_kind, out=call_out, stream=stream)
            nl = len(names)
        else:
            nl = m.run_events(X, call_kind, call_out, evs[i], stream)
            assert nl == len(names), f"call made {nl} launches, expected {names}"
        tail()
        return nl

    for _ in range(max(args.warmup, 3)):     # timing rule: >= 3 warm-up steps
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = ClockSampler(local)
    time.sleep(0.25)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    launches = 0
    for i in range(args.steps):
        launches += step(i)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    total_ms = t_start.elapsed_time(t_end)
    if dist:
        total_ms = max_over_ranks(total_ms, device=X.device)
        dist.barrier()
    ms_per_step = total_ms / args.steps / calls
    value = rows_all / (ms_per_step * 1e-3)
    if graph is not None:
        launches = args.steps * calls
        names = ["small_batch_kernel"]

    # ---- per-kernel durations (library events), dominant kernel
    per_kernel = {}
    if graph is None:
        for row in evs:
            for j, nm in enumerate(names):
                per_kernel.setdefault(nm, []).append(row[j].elapsed_time(row[j + 1]))
        kern_total = {nm: float(np.sum(v)) / args.steps for nm, v in per_kernel.items()}
        kern_launch = {nm: float(np.mean(v)) for nm, v in per_kernel.items()}
        dom = max(kern_total, key=kern_total.get)
        dom_ms = kern_total[dom]             # per call (all launches of that kernel)
        call_ms = sum(kern_total.values())
    else:
        kern_total = kern_launch = {"small_batch_kernel": ms_per_step}
        dom, dom_ms, call_ms = "small_batch_kernel", ms_per_step, ms_per_step

    # ---- roofline of the dominant kernel
    D = info["max_depth"]
    w = info["leaf_width"]
    # per (row, tree) and level one 8-B node record + one 4-B X
    # value; per tree one leaf of 4w B. PTT walks D levels by construction; TT
    # is credited only the levels it actually traverses (mean root->leaf path
    # length of the reached leaves, measured on a sample of rows).
    levels = float(D)
    if info["strategy_name"] == "tt":
        levels = mean_path_length(m, e, X[: min(n, 2048)], t0, t1)
    per_row = (t1 - t0) * (levels * 12 + 4 * w)
    tensor = None
    if dom == "gemm_tc_kernel":
        # GEMM (Alg. 1): every internal node is evaluated — |I| gathers of an
        # 8-B node + 4-B X value — and one leaf of 12 B is gathered (SURVEY
        # §8(d): 7 x 12 + 12 = 96 B per (row, tree) at D3); the path
        # contraction is |I| x |L| MACs per (row, tree) on the tensor cores
        n_int, n_leaf = 2 ** D - 1, 2 ** D
        per_row = (t1 - t0) * (n_int * 12 + 12)
        macs = n * (t1 - t0) * n_int * n_leaf
        tf = 2 * macs / (dom_ms * 1e-3) / 1e12
        try:
            bf16 = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
        except (OSError, KeyError, ValueError):
            bf16 = 1590.0
        tensor = {"achieved_tflops": tf, "peak_tflops": bf16, "frac": tf / bf16,
                  "macs_per_row_tree": n_int * n_leaf,
                  "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)",
                  "note": "the contraction is integer-exact bf16 (operands in {-1, 0, 1}); "
                          "the tensor pipe is not what binds (SURVEY §8(d))"}
    achieved = per_row * n / (dom_ms * 1e-3) / 1e9
    chase = None
    if dom == "tt_wide_kernel" and rank == 0:
        # the walk's records come from L2 and every load depends on the one
        # before: besides the streaming L2 roof, measure dependent random
        # 16-B gathers in the same launch shape (tools/peaks.cu l2_chase) over
        # a buffer the size of the records one launch walks
        try:
            import tools
            tools.build()
            chunk = info.get("tt_chunk_trees") or info["n_trees"]
            rb = int(info["tt_record_bytes"] * min(1.0, chunk / max(1, info["n_trees"])))
            g = info.get("tt_walks_per_lane") or 4
            rate = tools.l2_chase(local, max(rb, 1 << 20), g)
            loads = n * (t1 - t0) * max(levels, 1.0)
            krate = loads / (dom_ms * 1e-3)
            chase = {"kernel_node_loads_per_s": krate, "chase_loads_per_s": rate, "frac": krate / rate,
                     "buffer_bytes": max(rb, 1 << 20), "chains_per_thread": g,
                     "note": "node loads = rows x trees x mean levels (one 16-B record per internal "
                             "node on the path); chase = dependent random 16-B __ldg gathers, "
                             "1024 threads per SM, the same chains per thread (tools/peaks.cu)"}
        except Exception as ex:  # pragma: no cover
            chase = {"error": str(ex)}
    peaks = {}
    if rank == 0:
        try:
            import tools
            tools.build()
            peaks = tools.peaks(local)
        except Exception as ex:  # pragma: no cover
            peaks = {"error": str(ex)}
    smem_peak = peaks.get("smem_gbs") or 148 * 128 * 1.965
    layout = info["strategy_name"] + ("-rank" if info.get("node_record_bytes") == 4 else "") + \
        ("-pre" if info.get("rank_prepass") else "") + ("-chunk" if info.get("tt_chunk_trees") else "")
    if small:
        layout = "small-batch"
    traffic = load_traffic(args.config, layout, n, t1 - t0)
    hbm_bytes = n * (cfg.n_features * 4 + (8 if (cls and e.n_outputs == 1) else 4 * e.n_outputs))
    measured = {}
    try:
        measured = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = measured.get("hbm_gbs", 6650.0)
    # nodes staged in SMEM (PTT, narrow TT) -> SMEM roof; tt_wide_kernel reads
    # node records through L1/L2 -> the measured L2 read roof
    l2_wide = info["strategy_name"] == "tt" and dom == "tt_wide_kernel"
    bound, peak = ("l2", peaks.get("l2_gbs") or 12000.0) if l2_wide else ("smem", smem_peak)
    roofline = {
        "bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "kernel": dom, "layout": layout,
        "kernel_ms": dom_ms, "kernel_ms_per_launch": kern_launch.get(dom),
        "kernel_ms_source": "CUDA events recorded by libhb between its launches "
                            "(hb_predict_ex_events) over the timed steps",
        "kernels_ms_per_call": kern_total,
        "call_ms": call_ms,
        "frac_call": per_row * n / (ms_per_step * 1e-3) / 1e9 / peak,
        "mean_levels_per_tree": levels,
        "algorithmic_bytes_per_row": per_row,
        "algorithmic_bytes_per_call": per_row * n,
        "traffic": traffic["dram_bytes_per_call"] if traffic else None,
        "traffic_split": traffic["launches"] if traffic else None,
        "traffic_note": ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of EVERY launch "
                         "of one call, from one ncu --set full capture (tools/traffic.py); "
                         "traffic_split lists them per launch" if traffic else
                         "no ncu capture recorded for this config/layout/rows"),
        "traffic_source": traffic.get("source") if traffic else None,
        "peak_source": ("measured L2 read microbenchmark (tools/peaks.cu), this run" if l2_wide else
                        "measured LDS.128 microbenchmark (tools/peaks.cu), this run")
        if (peaks.get("l2_gbs") if l2_wide else peaks.get("smem_gbs"))
        else "spec 148 SM x 128 B/clk x 1.965 GHz",
        "smem_peak_spec_gbs": 148 * 128 * 1.965,
        "l2_peak_gbs": peaks.get("l2_gbs"),
        "tensor": tensor,
        "dependent_gather": chase,
        "hbm": {"achieved": hbm_bytes / (ms_per_step * 1e-3) / 1e9, "peak": hbm_peak,
                "frac": hbm_bytes / (ms_per_step * 1e-3) / 1e9 / hbm_peak,
                "bytes_per_call": hbm_bytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if measured else "fallback 6.65 TB/s"},
    }

    # ---- e2e through the public host API (pinned host buffers)
    e2e = None
    shape, dt = m.out_shape(n, kind)
    if not args.no_e2e and mode == "rows":
        del out
        Xh = torch.empty((n, cfg.n_features), dtype=torch.float32).pin_memory()
        Xh.copy_(X.cpu())
        oh = torch.empty(shape, dtype=getattr(torch, dt)).pin_memory()
        m.predict_host(Xh, kind, out=oh)  # warm (allocates staging)
        if dist:
            dist.barrier()
        ts = []
        for _ in range(args.e2e_steps):
            w0 = time.perf_counter()
            m.predict_host(Xh, kind, out=oh)
            ts.append(time.perf_counter() - w0)
        t_e2e = float(np.mean(ts))
        if dist:
            t_e2e = max_over_ranks(t_e2e, device=X.device)
        e2e = {"value": rows_all / t_e2e, "unit": "rows/s", "ms_per_step": t_e2e * 1e3,
               "h2d_bytes_per_step": int(n * cfg.n_features * 4),
               "d2h_bytes_per_step": int(oh.numel() * oh.element_size()), "steps": args.e2e_steps,
               "api": "hb_predict_host (chunked H2D / score / D2H on two streams)"}
        del Xh, oh
        out = m._out(n, kind, None, X.device)
    elif not args.no_e2e and mode == "trees":
        # every rank streams all rows from pinned host memory through
        # hb_predict_host and gets its shard's fp64 partials back; the partials
        # go to the device for the NCCL reduce, rank 0 finalizes and reads the
        # result back (the partial round trip is n*K*8 B each way)
        Xh = torch.empty((n, cfg.n_features), dtype=torch.float32).pin_memory()
        Xh.copy_(X)
        rawh = torch.empty((n, e.n_outputs), dtype=torch.float64).pin_memory()
        oh = torch.empty(shape, dtype=getattr(torch, dt)).pin_memory()

        def e2e_step():
            m.predict_host(Xh, "raw64", out=rawh)
            raw.copy_(rawh)
            if dist:
                reduce_partials(raw, dst=0)
            if rank == 0:
                m.finalize(raw, kind, out=out, stream=stream)
                stream.synchronize()
                oh.copy_(out)
        e2e_step()  # warm (allocates staging)
        if dist:
            dist.barrier()
        ts = []
        for _ in range(args.e2e_steps):
            w0 = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - w0)
        t_e2e = float(np.mean(ts))
        if dist:
            t_e2e = max_over_ranks(t_e2e, device=raw.device)
        part = int(rawh.numel() * 8)
        e2e = {"value": rows_all / t_e2e, "unit": "rows/s", "ms_per_step": t_e2e * 1e3,
               "h2d_bytes_per_step": int(n * cfg.n_features * 4) + part,
               "d2h_bytes_per_step": part + int(oh.numel() * oh.element_size()),
               "steps": args.e2e_steps,
               "api": "hb_predict_host(raw64) per tree shard -> NCCL reduce of the partials -> "
                      "hb_finalize64 on rank 0 -> D2H"}
        del Xh, oh, rawh

    # ---- CPU oracle baseline (P:324 timing) and parity on the same rows
    cpu = parity = None
    if rank == 0 and not args.no_cpu:
        whole = t0 == 0 and t1 == e.n_trees
        tm = time_oracle(e, cfg, t0, t1, run_s=2.5, runs=5, max_rows=n)
        cpu = {"value": tm["value"], "unit": "rows/s", "cores": tm["cores"], "kind": "oracle",
               "sample": f"first {tm['rows']} rows of {cfg.name} (seed {cfg.seed_x:#x}), "
                         + ("full model" if whole else f"trees [{t0}, {t1})"),
               "timing": "5 runs, truncated mean (P:324); min also given",
               "value_at_min": tm["value_at_min"], "seconds_truncated_mean": tm["seconds_truncated_mean"],
               "seconds_min": tm["seconds_min"], "cpu": cpu_model()}
        # the oracle on all host cores, plus one core
        t1c = time_oracle(e, cfg, t0, t1, run_s=0.6, runs=5, threads=1, max_rows=n)
        cpu["single_core"] = {"value": t1c["value"], "unit": "rows/s", "cores": 1,
                              "rows": t1c["rows"], "value_at_min": t1c["value_at_min"]}
        parity = parity_report(m, e, cfg, X, tm["rows"], t0, t1, kind, cls)
        if mode == "trees" and whole is False:
            parity["scope"] = f"tree shard [{t0}, {t1}) raw fp64 partials and leaf hashes"
            if dist and world == max(world, args.emulate_gpus):
                # the NCCL-reduced, finalized output of the whole ensemble on
                # rank 0 (last timed step) against the full-model oracle
                import oracle
                rf = min(10_000, n)
                Xf = synth.gen_X(cfg.seed_x, rf, cfg.n_features)
                rawf, _ = oracle.raw_and_hash(e, Xf, threads=0)
                postf = oracle.post(e, oracle.margin(e, rawf))
                ref = oracle.proba(e, postf) if cls else postf
                got = out[:rf].double().cpu().numpy()
                d = np.abs(got - ref)
                parity["final_output"] = {
                    "rows": rf, "kind": kind, "max_abs_err": float(d.max()),
                    "outside_tol": int((d > 1e-5 + 1e-5 * np.abs(ref)).sum()),
                    "scope": f"{kind} of all {e.n_trees} trees after the reduce over {world} ranks"}
                parity["pass"] = parity["pass"] and parity["final_output"]["outside_tol"] == 0

    if rank == 0:
        cfgd = dict(workload_config(cfg, e, rows_all, args, mode, scaling, world), strategy=info["strategy_name"],
                    output=kind, rows_per_gpu=n, trees_per_gpu=t1 - t0,
                    timing=("CUDA graph of %d calls per timed step, value per call" % calls)
                    if calls > 1 else "one call per timed step")
        # seeds of the synthetic inputs, the compiled layout and its device memory
        # (SURVEY §5 metrics: seeds, peak memory)
        cfgd["seeds"] = {"x": cfg.seed_x, "trees": cfg.seed_t}
        cfgd["layout"] = {k: info.get(k) for k in ("kernel_name", "node_record_bytes", "code_cell_bits",
                                                   "rank_prepass", "rank_prepass_tma", "rows_per_lane",
                                                   "rows_per_cta", "tt_chunk_trees", "small_batch_max_rows")}
        cfgd["model_device_bytes"] = info.get("device_bytes")
        cfgd["torch_peak_bytes"] = int(torch.cuda.max_memory_allocated(local))   # X, outputs (torch allocator)
        if mode == "trees" and args.emulate_gpus and world == 1:
            cfgd["emulated_shard_of"] = args.emulate_gpus
            cfgd["trees_scored"] = t1 - t0
            cfgd["parallelism"] = (f"ONE GPU scoring rank 0's 1/{args.emulate_gpus} tree shard "
                                   f"({t1 - t0} of {e.n_trees} trees), no reduce")
            cfgd["value_note"] = ("rate of one GPU's tree shard = the 8-GPU job rate if the reduce "
                                  "were free; NOT the full-model single-GPU rate")
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32",
            "dtype_note": "fp32 X and thresholds, IEEE fp32 compares, fp64 leaf-value accumulation",
            "data": f"synthetic (seeded splitmix64 grid X; random {cfg.family} depth-{cfg.depth} forest)",
            "config": cfgd,
            "roofline": roofline, "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches,
            "gpu_launches_per_call": names,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def parity_report(m, e, cfg, X, rows, t0, t1, kind, cls):
    """GPU outputs vs the oracle on the rows the oracle baseline timed
    (outside the timed region): leaf-hash mismatches (bit-exact bar), max abs
    / rel error of the margin and of the returned output (R23 bar), labels
    outside near-ties, near-tie count."""
    import oracle
    rows = min(rows, X.shape[0])
    Xs = X[:rows]
    import synth
    Xh = synth.gen_X(cfg.seed_x, rows, cfg.n_features)
    raw, hsh = oracle.raw_and_hash(e, Xh, t0, t1, threads=0)
    g_hash = m.predict_leaf_hash(Xs).cpu().numpy().view(np.uint64)
    rep = {"rows": rows, "tolerance": TOL,
           "leaf_hash_mismatches": int((g_hash != hsh).sum())}

    def errs(got, ref, tag):
        got = np.asarray(got, np.float64)
        d = np.abs(got - ref)
        rep[f"{tag}_max_abs_err"] = float(d.max())
        rep[f"{tag}_max_rel_err"] = float((d / np.maximum(np.abs(ref), 1e-30)).max())
        rep[f"{tag}_outside_tol"] = int((d > 1e-5 + 1e-5 * np.abs(ref)).sum())

    if t0 == 0 and t1 == e.n_trees:
        mg = oracle.margin(e, raw)
        errs(m.predict_margin(Xs).cpu().numpy(), mg, "margin")
        post = oracle.post(e, mg)
        ref = oracle.proba(e, post) if cls else post
        errs(m.run(Xs, kind).cpu().numpy(), ref, kind)
        if cls:
            lab = m.predict(Xs).cpu().numpy()
            ref_lab = oracle.label(e, mg)
            if e.n_outputs == 1:
                tie = np.abs(mg[:, 0]) < 2 * (1e-5 + 1e-5 * np.abs(mg[:, 0]))
            else:
                s = np.sort(mg, 1)
                tie = s[:, -1] - s[:, -2] < 2 * (1e-5 + 1e-5 * np.abs(s[:, -1]))
            rep["near_ties"] = int(tie.sum())
            rep["near_tie_rows"] = [int(r) for r in np.flatnonzero(tie)[:20]]
            rep["label_mismatches_outside_near_ties"] = int((lab[~tie] != ref_lab[~tie]).sum())
            rep["label_mismatches_at_near_ties"] = int((lab[tie] != ref_lab[tie]).sum())
        bad = rep["leaf_hash_mismatches"] + rep["margin_outside_tol"] + rep[f"{kind}_outside_tol"] + \
            rep.get("label_mismatches_outside_near_ties", 0)
    else:
        errs(m.predict_raw64(Xs).cpu().numpy(), raw, "raw")
        bad = rep["leaf_hash_mismatches"] + rep["raw_outside_tol"]
    rep["pass"] = bad == 0
    return rep


def mean_path_length(m, e, X, t0, t1):
    """Mean number of levels the walk traverses per (row, tree): leaf depth of
    the reached leaf (leaf ids from the device, depths from the tree arrays)."""
    leaf = m.predict_leaf(X).cpu().numpy()
    tot = 0.0
    for j, t in enumerate(range(t0, t1)):
        a, b = int(e.node_offset[t]), int(e.node_offset[t + 1])
        L, R = e.left[a:b], e.right[a:b]
        depth = np.zeros(b - a, np.int32)
        order = [0]
        for i in order:
            if L[i] >= 0:
                depth[L[i]] = depth[R[i]] = depth[i] + 1
                order += [int(L[i]), int(R[i])]
        tot += depth[leaf[:, j]].mean()
    return tot / max(1, t1 - t0)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
