"""Warp-stall samples of one `ncu --set full --import-source on` capture, split into the code
regions between barriers (statistics, uncompute stages, transposes, store / tile wait).

    ncu -i top_bwd.ncu-rep --page source --csv --print-source sass > top_bwd_sass.csv
    python tools/ncu_phases.py top_bwd_sass.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    segs, cur = [], None

    def new():
        return {"n": 0, "samples": 0, "stall": collections.Counter(), "ops": collections.Counter()}

    cur = new()
    for r in data:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        parts = src.split()
        if not parts:
            continue
        op = parts[1] if parts[0].startswith("@") else parts[0]
        cur["n"] += 1
        cur["samples"] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        for h in stalls:
            cur["stall"][h[6:]] += int(r[ix[h]] or 0)
        cur["ops"][op.split(".")[0]] += 1
        if op.startswith("BAR") or op.startswith("SYNCS") or op == "EXIT":
            segs.append((src[:44], cur))
            cur = new()
    segs.append(("end", cur))
    total = sum(c["samples"] for _, c in segs) or 1
    print(f"{path}: {total} warp samples; regions with >= 1% (ending at the instruction shown)")
    for lab, c in segs:
        if c["samples"] < 0.01 * total:
            continue
        top = ", ".join(f"{k} {100 * v // max(1, c['samples'])}%" for k, v in c["stall"].most_common(5))
        ops = ", ".join(f"{k}:{v}" for k, v in c["ops"].most_common(6))
        print(f"{100 * c['samples'] / total:5.1f}%  {c['n']:5d} instr  until {lab:44s} | {top} | {ops}")


if __name__ == "__main__":
    main(sys.argv[1])
