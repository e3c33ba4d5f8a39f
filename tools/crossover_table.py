"""Render profiles/r02_crossover.json (tools/crossover.py) as the DESIGN.md
§6.1 markdown table: device µs per call for every forced strategy / layout,
the small-batch kernel, and what AUTO ran, with AUTO / best."""
import json
import sys

COLS = [("gemm", "GEMM"), ("ptt", "PTT fp32"), ("ptt-rank", "PTT rank (in-kernel)"),
        ("ptt-rank-pre", "PTT rank + pre-pass"), ("tt", "TT"), ("small", "small-batch")]


def main(path):
    d = json.load(open(path))
    res = d["results"]
    summ = {(s["depth"], s["batch"]): s for s in d["auto_vs_best"]}
    print("| D | batch | " + " | ".join(c for _, c in COLS) + " | **AUTO** (ran) | AUTO / best |")
    print("|---|---|" + "---|" * len(COLS) + "---|---|")
    for (D, n), s in sorted(summ.items()):
        cell = {}
        for r in res:
            if r["depth"] == D and r["batch"] == n:
                cell[r["kernel"]] = r
        vals = [f"{cell[k]['us_per_call']:.1f}" if k in cell else "–" for k, _ in COLS]
        ran = cell["auto"]["ran"].replace("_kernel", "")
        print(f"| {D} | {n} | " + " | ".join(vals) +
              f" | {s['auto_us']:.1f} ({ran}) | {s['auto_over_best']:.3f} |")
    print()
    print(f"max AUTO / best: {max(s['auto_over_best'] for s in summ.values()):.3f}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_crossover.json")
