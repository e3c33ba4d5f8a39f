#!/usr/bin/env python
"""Benchmark: rows/sec scored (500 trees, depth 8) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
                    [--impl ours|reference] [--strategy auto] [--no-e2e] [--no-cpu]

One "step" is one pass of the whole hot path over one batch: a single fused
hb_predict_proba (or hb_predict for regression) launch over all rows of the
rank's shard (X tile staging, the strategy's traversal, ensemble accumulate,
epilogue, store). Rows are sharded across ranks with no data-path collective
(weak scaling: every rank scores its own n_rows). Timing: W untimed warm-up
steps, then K steps bracketed by barrier + cuda synchronize, CUDA events on
the launching stream, max over ranks. X (> L2) is resident in HBM before the
timed region. ``e2e`` repeats the metric through hb_predict_host from pinned
host memory (H2D of X and D2H of the result inside the timed region).

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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--rows", type=int, default=0, help="override rows per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--shard", default=None, choices=["rows", "trees"],
                    help="default: trees for C5, rows otherwise")
    ap.add_argument("--emulate-gpus", type=int, default=0,
                    help="trees mode on 1 GPU: score only rank 0's tree shard of an "
                         "N-GPU run (the per-GPU piece of C5 on 8 GPUs)")
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
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
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
def time_oracle(e, cfg, budget_s=12.0, max_rows=None, threads=0):
    """Oracle throughput on a bounded prefix sample of the workload, all host
    cores (std pthreads over row blocks). Returns (rows/s, cores, sample)."""
    import oracle
    import synth
    max_rows = max_rows or cfg.n_rows
    probe = min(2000, max_rows)
    Xp = synth.gen_X(cfg.seed_x, probe, cfg.n_features)
    t = time.perf_counter()
    _, used = oracle.predict_mt(e, Xp, threads=threads)
    dt = max(time.perf_counter() - t, 1e-4)
    rate = probe / dt
    rows = int(min(max_rows, max(probe, rate * budget_s)))
    X = synth.gen_X(cfg.seed_x, rows, cfg.n_features)
    t = time.perf_counter()
    _, used = oracle.predict_mt(e, X, threads=threads)
    dt = time.perf_counter() - t
    return rows / dt, used, f"first {rows} rows of {cfg.name} (seed {cfg.seed_x:#x}), full model", dt


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
    import synth
    cfg, e = synth.make_config(args.config)
    # size each step for ~4 s of CPU work (HB_REF_STEP_S overrides)
    step_s = float(os.environ.get("HB_REF_STEP_S", "4.0"))
    rate0, used, _, _ = time_oracle(e, cfg, budget_s=min(1.0, step_s))
    rows = int(min(cfg.n_rows, max(100, rate0 * step_s)))
    import oracle
    X = synth.gen_X(cfg.seed_x, rows, cfg.n_features)
    for _ in range(args.warmup):
        oracle.predict_mt(e, X[: max(1, rows // 8)])
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        _, used = oracle.predict_mt(e, X)
        times.append(time.perf_counter() - t)
    ms = 1e3 * float(np.mean(times))
    value = rows / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(cfg, e, rows, args),
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": used, "kind": "oracle",
                         "sample": f"first {rows} rows of {cfg.name} per step", "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def launches_per_call(info, kind, small):
    """Kernels one hb_predict call launches: rank-code pre-pass models two
    (pre-pass + scorer) except on the small-batch path; a TT model walked in
    L2-resident tree chunks one per chunk, plus the finalize for outputs that
    need the post transform."""
    chunk = info.get("tt_chunk_trees", 0)
    if chunk and not small:
        pad = (info["n_trees"] + 3) // 4 * 4
        return -(-pad // chunk) + (1 if kind in ("predict", "proba", "margin") else 0)
    return 2 if info.get("rank_prepass") and not small else 1


def workload_config(cfg, e, rows, args, mode="rows"):
    par = (f"rows sharded over {args.gpus} GPU(s), no collective" if mode == "rows" else
           f"trees sharded over {args.gpus} GPU(s), one NCCL reduce of fp64 partials + finalize")
    return {"workload": f"{cfg.name}: {cfg.note}", "rows_per_gpu": rows, "n_trees": e.n_trees,
            "max_depth": cfg.depth, "n_features": cfg.n_features, "n_outputs": e.n_outputs,
            "family": cfg.family, "parallelism": par,
            "l2": ("X larger than L2 (streamed once per step, no flush needed); model (<13 MB) "
                   "L2-resident by design" if cfg.depth <= 10 else
                   "X larger than L2 (streamed once per step, no flush needed); depth-12 node records: "
                   "a 1/8 tree shard (~60 MB) is L2-resident, all 10k trees (~480 MB) are not")}


# ----------------------------------------------------------------- ours
def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("HB_BENCH_BACKEND", "nccl")   # gloo: 1-GPU multi-rank test
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_2010_04804_b200 as hb
    import synth
    import synth.dev
    from paper_2010_04804_b200.dist import max_over_ranks, reduce_partials, tree_shard

    cfg, e = synth.make_config(args.config)
    n = args.rows or cfg.n_rows
    mode = args.shard or ("trees" if cfg.name == "C5" else "rows")
    cls = e.task == synth.TASK_CLASSIFICATION
    kind = "proba" if cls else "predict"
    stream = torch.cuda.current_stream(local)
    if mode == "rows":
        # rows sharded, model replicated, no data-path collective (weak scaling)
        t0, t1 = 0, e.n_trees
        m = hb.Model(e, strategy=args.strategy, device=local)
        X = synth.dev.gen_X_device(cfg.seed_x, n, cfg.n_features, row_offset=rank * n,
                                   device=local)
        shape, dt = m.out_shape(n, kind)
        out = torch.empty(shape, dtype=getattr(torch, dt), device=X.device)

        def step():
            m.run(X, kind, out=out, stream=stream)
        small = n <= int(os.environ.get("HB_SMALL_BATCH", "4096"))
        launches_per_step = launches_per_call(m.info, kind, small)
    else:
        # trees sharded, all rows on every rank; one NCCL reduce of fp32
        # partials to rank 0, which finalizes (strong scaling)
        t0, t1 = tree_shard(e.n_trees, rank, max(world, args.emulate_gpus), e.n_outputs,
                            e.leaf_width)
        m = hb.Model(e, strategy=args.strategy, device=local, tree_range=(t0, t1))
        X = synth.dev.gen_X_device(cfg.seed_x, n, cfg.n_features, device=local)
        raw = torch.empty((n, e.n_outputs), dtype=torch.float64, device=X.device)
        shape, dt = m.out_shape(n, kind)
        out = torch.empty(shape, dtype=getattr(torch, dt), device=X.device)

        def step():
            m.run(X, "raw64", out=raw, stream=stream)
            if dist:
                reduce_partials(raw, dst=0)
            if rank == 0:
                m.finalize(raw, kind, out=out, stream=stream)
        launches_per_step = launches_per_call(m.info, "raw64", False) + 1
    info = m.info

    # request/response batch sizes (small-batch kernel) are launch-bound from
    # Python: capture REPS calls in one CUDA graph and replay it, so the
    # device time per call is measured instead of the host issue rate
    calls = 1
    if mode == "rows" and n <= int(os.environ.get("HB_SMALL_BATCH", "4096")):
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

        def step():
            graph.replay()

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
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        evs[i][0].record(stream)
        if mode == "rows":
            step()
            evs[i][1].record(stream)
        else:
            m.run(X, "raw64", out=raw, stream=stream)   # the scorer launch(es) alone
            evs[i][1].record(stream)
            if dist:
                reduce_partials(raw, dst=0)
            if rank == 0:
                m.finalize(raw, kind, out=out, stream=stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    total_ms = t_start.elapsed_time(t_end)
    per_launch = [a.elapsed_time(b) for a, b in evs]
    if dist:
        total_ms = max_over_ranks(total_ms, device=X.device)
        dist.barrier()
    ms_per_step = total_ms / args.steps / calls
    per_launch = [t / calls for t in per_launch]
    rows_all = n * world if mode == "rows" else n
    value = rows_all / (ms_per_step * 1e-3)

    # ---- roofline of the dominant (only) kernel of the step
    kern_ms = float(np.mean(per_launch))
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
    achieved = per_row * n / (kern_ms * 1e-3) / 1e9
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
        ("-pre" if info.get("rank_prepass") else "") + ("-sector" if info.get("tt_sector") else "") + \
        ("-chunk" if info.get("tt_chunk_trees") else "")
    prof = load_profile(args.config, layout)
    kname = info["kernel_name"]
    if n <= int(os.environ.get("HB_SMALL_BATCH", "4096")):
        kname = "small_batch_kernel"      # request/response sizes (hb_small.cu)
    hbm_bytes = n * (cfg.n_features * 4 + (8 if (cls and e.n_outputs == 1) else 4 * e.n_outputs))
    measured = {}
    try:
        measured = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = measured.get("hbm_gbs", 6650.0)
    same_launch = prof.get("rows") == n and prof.get("trees", t1 - t0) == t1 - t0
    # nodes staged in SMEM (PTT, narrow TT) -> SMEM roof; tt_wide_kernel and
    # ttb_kernel read node records through L1/L2 -> the measured L2 read roof
    l2_wide = info["strategy_name"] == "tt" and kname in ("tt_wide_kernel", "ttb_kernel")
    bound, peak = ("l2", peaks.get("l2_gbs") or 12000.0) if l2_wide else ("smem", smem_peak)
    roofline = {
        "bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "mean_levels_per_tree": levels,
        # contract: traffic = dram__bytes_read.sum + dram__bytes_write.sum per
        # launch (one ncu --set full capture); the kernel is bound on chip, so
        # the comparable figure for achieved/algorithmic bytes is the SMEM one
        "traffic": prof.get("dram_bytes_per_launch") if same_launch else None,
        "traffic_smem": prof.get("smem_ld_bytes_per_launch") if same_launch else None,
        "traffic_note": "traffic = DRAM bytes per launch (X + output when the model is L2-resident); "
                        "traffic_smem = SMEM load wavefronts x 128 B per launch, the on-chip "
                        "counterpart of the algorithmic bytes",
        "traffic_source": prof.get("source"),
        # cross-check in bytes the kernel really loads from SMEM (ncu), over the
        # whole timed call (the pre-pass launch included when there is one)
        "frac_ncu_smem_bytes": (prof["smem_ld_bytes_per_launch"] / (kern_ms * 1e-3) / 1e9 / smem_peak)
        if (same_launch and bound == "smem" and prof.get("smem_ld_bytes_per_launch")) else None,
        "kernel": kname, "layout": layout, "kernel_ms": kern_ms,
        "kernel_ms_covers": ("rank-code pre-pass + pttr_kernel (both launches of one hb_predict call; "
                             "their split is in the ncu launch list under profiles/)")
        if info.get("rank_prepass") and kname != "small_batch_kernel" else
        (f"{kname} over L2-resident chunks of {info['tt_chunk_trees']} trees (one launch per chunk) + finalize"
         if info.get("tt_chunk_trees") else kname),
        "algorithmic_bytes_per_row": per_row,
        "peak_source": ("measured L2 read microbenchmark (tools/peaks.cu), this run" if l2_wide else
                        "measured LDS.128 microbenchmark (tools/peaks.cu), this run")
        if (peaks.get("l2_gbs") if l2_wide else peaks.get("smem_gbs"))
        else "spec 148 SM x 128 B/clk x 1.965 GHz",
        "smem_peak_spec_gbs": 148 * 128 * 1.965,
        "l2_peak_gbs": peaks.get("l2_gbs"),
        "hbm": {"achieved": hbm_bytes / (kern_ms * 1e-3) / 1e9, "peak": hbm_peak,
                "frac": hbm_bytes / (kern_ms * 1e-3) / 1e9 / hbm_peak,
                "peak_source": "MEASURED_PEAKS.json" if measured else "fallback 6.65 TB/s"},
    }

    # ---- e2e through the public host API (pinned host buffers)
    e2e = None
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
    elif not args.no_e2e and mode == "trees":
        # every rank streams all rows from pinned host memory through
        # hb_predict_host and gets its shard's raw partials back; the partials
        # go to the device for the NCCL reduce, rank 0 finalizes and reads the
        # result back (the partial round trip is n*K*4 B each way)
        Xh = torch.empty((n, cfg.n_features), dtype=torch.float32).pin_memory()
        Xh.copy_(X)
        del X
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
               "api": "hb_predict_host(raw) per tree shard -> NCCL reduce of the partials -> "
                      "hb_finalize on rank 0 -> D2H"}
        del Xh, oh, rawh

    cpu = None
    if rank == 0 and not args.no_cpu:
        rate, used, sample, secs = time_oracle(e, cfg, budget_s=12.0)
        cpu = {"value": rate, "unit": "rows/s", "cores": used, "kind": "oracle", "sample": sample,
               "seconds": secs, "cpu": cpu_model()}
        # the oracle on all host cores, plus one core
        r1, u1, s1, t1_ = time_oracle(e, cfg, budget_s=3.0, threads=1)
        cpu["single_core"] = {"value": r1, "unit": "rows/s", "cores": u1, "sample": s1,
                              "seconds": t1_}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak" if mode == "rows" else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic (seeded splitmix64 grid X; random {cfg.family} depth-{cfg.depth} forest)",
            "config": dict(workload_config(cfg, e, n, args, mode), strategy=info["strategy_name"],
                           output=kind, trees_per_gpu=t1 - t0,
                           timing=("CUDA graph of %d calls per timed step, value per call" % calls)
                           if calls > 1 else "one call per timed step"),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": args.steps * calls * launches_per_step,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def mean_path_length(m, e, X, t0, t1):
    """Mean number of levels the walk traverses per (row, tree): leaf depth of
    the reached leaf (leaf ids from the device, depths from the tree arrays)."""
    import numpy as np
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


def load_profile(config, strat):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(f"{config}:{strat}", {})
    except (OSError, ValueError):
        return {}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
