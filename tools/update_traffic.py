"""Record one kernel's per-launch traffic from an ncu report into
profiles/ncu_traffic.json (read by bench.py for the roofline `traffic` field).

    python tools/update_traffic.py CONFIG LAYOUT ROWS report.ncu-rep profiles/<summary>.txt [KERNEL_SUBSTR] [TREES]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import raw  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def num(x):
    return float(str(x).replace(",", ""))


def main(cfg, layout, rows, rep, summary, kernel="", trees=None):
    recs, units = raw(rep)
    d = next(r for r in recs if kernel in r.get("Kernel Name", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = sum(num(d[k]) * scale.get(units.get(k, "byte"), 1)
               for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    smem = num(d["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]) * 128
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    js = json.load(open(p))
    js[f"{cfg}:{layout}"] = {"round": 1, "dram_bytes_per_launch": int(dram),
                             "smem_ld_bytes_per_launch": int(smem), "rows": int(rows),
                             "source": summary, "kernel": d.get("Kernel Name", "")[:60]}
    if trees:
        js[f"{cfg}:{layout}"]["trees"] = int(trees)
    json.dump(js, open(p, "w"), indent=1)
    print(cfg, layout, int(dram), int(smem))


if __name__ == "__main__":
    main(*sys.argv[1:8])
