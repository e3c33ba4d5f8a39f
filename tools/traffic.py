"""Record the DRAM traffic of every launch of one call (an ncu --set full
report of tools/one_call.py) into profiles/ncu_traffic.json, which bench.py
reads for roofline.traffic / traffic_split.

    python tools/traffic.py KEY report.ncu-rep profiles/<round>_<label>_ncu.txt

KEY is the line tools/one_call.py printed ("C3:ptt-rank-pre:10000000:500").
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import raw  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TSCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def as_int(x):
    return None if x != x else int(x)   # ncu reports -nan for some counters of long replays


def main(key, rep, summary):
    recs, units = raw(rep)
    launches = []
    for d in recs:
        dram = sum(num(d[k]) * SCALE.get(units.get(k, "byte"), 1)
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        smem = num(d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "0")) * 128
        ms = num(d.get("gpu__time_duration.sum", "0")) * TSCALE.get(units.get("gpu__time_duration.sum", "nsecond"), 1e-6)
        launches.append({"kernel": d.get("Kernel Name", "")[:80], "dram_bytes": as_int(dram),
                         "smem_ld_bytes": as_int(smem), "ncu_ms": round(ms, 4)})
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        js = json.load(open(p))
    except (OSError, ValueError):
        js = {}
    js = {k: v for k, v in js.items() if k.count(":") == 3 or k == "_about"}
    js["_about"] = ("DRAM traffic of every launch of ONE hb_predict call in bench.py's launch shape, "
                    "from one `ncu --set full --clock-control none` capture of tools/one_call.py "
                    "(key config:layout:rows:trees). dram = dram__bytes_read.sum + dram__bytes_write.sum; "
                    "smem = l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum x 128 B; ncu_ms = "
                    "gpu__time_duration under the profiler (cold cache, serialised: shares, not absolutes).")
    known = [l["dram_bytes"] for l in launches]
    js[key] = {"round": 2, "launches": launches,
               "dram_bytes_per_call": None if None in known else int(sum(known)),
               "source": summary}
    json.dump(js, open(p, "w"), indent=1)
    print(key, js[key]["dram_bytes_per_call"], [(l["kernel"][:30], l["dram_bytes"]) for l in launches])


if __name__ == "__main__":
    main(*sys.argv[1:4])
