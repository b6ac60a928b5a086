"""Summarise ncu outputs into profiles/.

    python tools/ncu_summarize.py launches <launches.csv>          # per-kernel share of device time
    python tools/ncu_summarize.py traffic <report.ncu-rep> <name>   # dram bytes per launch -> json
    python tools/ncu_summarize.py mix <sass.csv> <label>             # executed instructions per opcode
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]]
        if name.startswith("qbg_"):
            name = "qbg_<specialised tile pass>"
        if name.startswith("qbs_"):
            name = "qbs_<specialised seed pass>"
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = v / 1000 if unit in ("ns", "nsecond") else v * 1000 if unit in ("ms", "msecond") else v
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {n:8d} {us:12.1f} {us / tot * 100:6.1f}%")


def traffic(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * units.get(rows[1][hdr.index("dram__bytes_read.sum")], 1)
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * units.get(rows[1][hdr.index("dram__bytes_write.sum")], 1)
        res = {name: rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
               "duration": d.get("gpu__time_duration.sum"), "kernel": d.get("Kernel Name", "")[:80]}
    print(json.dumps(res))


def mix(path, label):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ie = hdr.index("Instructions Executed")
    cnt = collections.Counter()
    for r in rows:
        if len(r) <= ie or not r[0].startswith("0x"):
            continue
        toks = r[1].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        cnt[op.split(".")[0]] += int(float(r[ie] or 0))
    tot = sum(cnt.values())
    print(f"{label}: {tot} warp instructions executed")
    for op, v in cnt.most_common(16):
        print(f"{op:12s} {v:12d} {100 * v / tot:5.1f}%")
    fp64 = sum(cnt[o] for o in ("DFMA", "DMUL", "DADD"))
    print(f"FP64 (DFMA + DMUL + DADD): {100 * fp64 / tot:.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "mix":
        mix(sys.argv[2], sys.argv[3])
    else:
        traffic(sys.argv[2], sys.argv[3])
