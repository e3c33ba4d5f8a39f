"""Summarise an ncu --set full report (run here, no GPU needed):

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [label] > profiles/<round>_<label>.txt

Prints the metrics the roofline / traffic claims rest on and the warp stall
breakdown; also returns a dict (used to update profiles/ncu_traffic.json).
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "kernel time"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/SMEM throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "SMEM load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "SMEM load bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "SMEM store wavefronts"),
    ("lts__t_sectors_op_read.sum", "L2 read sectors"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]


def raw(path):
    """Records of an ncu report (.ncu-rep) or of its `--page raw --csv` export (.csv)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    return [dict(zip(h, r)) for r in rows[2:]], dict(zip(h, u))


def summarize(path, label=""):
    recs, units = raw(path)
    res = []
    for d in recs:
        print(f"== {label} kernel: {d.get('Kernel Name', '')[:100]}")
        out = {}
        for k, name in KEYS:
            if k in d:
                print(f"  {name:32s} {d[k]:>22s} {units.get(k, '')}")
                out[k] = d[k]
        stalls = {k: d[k] for k in d if k.startswith("smsp__average_warp_latency_issue_stalled_")
                  or (k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"))}
        tot = 0.0
        vals = []
        for k, v in stalls.items():
            try:
                fv = float(v.replace(",", ""))
            except ValueError:
                continue
            vals.append((fv, k))
            tot += fv
        if vals and tot > 0:
            print("  top stall reasons (pc sampling / latency):")
            for fv, k in sorted(vals, reverse=True)[:8]:
                print(f"    {k.split('stalled_')[-1]:28s} {100 * fv / tot:5.1f}%")
        res.append(out)
    return res


if __name__ == "__main__":
    summarize(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
