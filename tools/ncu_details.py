"""Key metrics + warp-stall breakdown of one `ncu --set full` report (text, for profiles/).

    python tools/ncu_details.py <report.ncu-rep>
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "L2 Hit Rate", "Achieved Occupancy"]
RAW = ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
STALLS = ['stall_barrier', 'stall_branch_resolving', 'stall_dispatch', 'stall_lg', 'stall_long_sb', 'stall_math',
          'stall_mio', 'stall_no_inst', 'stall_not_selected', 'stall_selected', 'stall_short_sb', 'stall_wait',
          'stall_membar', 'stall_misc', 'stall_sleep']


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    for r in csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))):
        if len(r) > 14 and r[12] in KEYS:
            print(f"{r[12]:36s} {r[14]:>14s} {r[13]}")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    if len(rows) > 2:
        for k, v in zip(rows[0], rows[2]):
            if k in RAW or k == "Kernel Name":
                print(f"{k:60s} {v}")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(rows) > 2:
        h, data = rows[1], rows[2:]
        idx = {n: h.index(n) for n in STALLS if n in h}
        tot = collections.Counter()
        byop = collections.defaultdict(collections.Counter)
        for r in data:
            t = r[1].strip().split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            for n, i in idx.items():
                v = int(r[i] or 0)
                tot[n] += v
                byop[op][n] += v
        s = sum(tot.values()) or 1
        print("warp-state samples (all):", ", ".join(f"{k[6:]} {100 * v / s:.1f}%" for k, v in tot.most_common()))
        for op, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:10]:
            print(f"  {op:8s} {100 * sum(c.values()) / s:5.1f}%  " + ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(4)))


if __name__ == "__main__":
    main(sys.argv[1])
