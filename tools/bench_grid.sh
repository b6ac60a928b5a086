#!/bin/bash
# Sweep of env-selected kernel geometries through bench.py (one line per setting):
#   tools/bench_grid.sh "QBG_PIPE=0" "QBG_PIPE=2 QBG_BWD_RB=3" ...
#   (BENCH_ARGS="--dtype c64" adds bench.py arguments)
for cfg in "$@"; do
  out=$(env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sharded $BENCH_ARGS 2>/dev/null | tail -1)
  python - "$cfg" "$out" <<'PY'
import json, sys
cfg, out = sys.argv[1], sys.argv[2]
try:
    d = json.loads(out)
except Exception:
    print(f"{cfg:40s} FAILED {out[:200]}"); sys.exit()
ks = " ".join(f"{k['name']}:{k['launches']}x{k['total_ms']/k['launches']:.3f}" for k in d["roofline"]["kernels"][:4])
print(f"{cfg:40s} {d['ms_per_step']:7.2f} ms  {ks}")
PY
done
