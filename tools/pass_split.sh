# Per-pass-type times of the bench step (QBG_PROF_KERNELS=1) under the QBG_EXP diagnostics of the
# checkpointed reverse pass: default, 3 = statistics without warp reduction, 4 = no transposes,
# 7 = no statistics, 8 = no uncompute ops.  Results of the diagnostic modes are wrong by design.
out=gpurun_out/${1:-split}
mkdir -p $out
for m in ${MODES:-0 3 4 7 8}; do
  QBG_PROF_KERNELS=1 QBG_EXP=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sharded > $out/exp$m.json 2> $out/exp$m.err
  echo "== QBG_EXP=$m rc=$?"
  python - $out/exp$m.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("ms/step", round(d["ms_per_step"], 3), "clk", d["clocks"]["sm_mhz"])
for k in d["roofline"]["kernels"]:
    print(f'  {k["name"]:40s} {k["launches"]:4d} {k["total_ms"] / k["launches"]:.4f}')
PY
done
