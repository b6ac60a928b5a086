# A/B of an engine switch on one box: parity suites of the checkpointed path with the candidate
# setting, then the per-pass split (QBG_PROF_KERNELS=1) for each setting.
#   VAR=QBG_CK_TAIL A=0 B=1 bash tools/ab_env.sh outdir
out=gpurun_out/${1:-abenv}
mkdir -p $out
env $VAR=$B timeout 1200 python -m pytest tests/test_gpu_ckpt.py tests/test_gpu_bench_parity.py tests/test_gpu_random_circuits.py tests/test_gpu_edge_cases.py -m gpu -q -x > $out/pytest.log 2>&1; echo "pytest($VAR=$B) $?"; tail -2 $out/pytest.log
for rep in 1 2; do for v in $A $B; do
  env $VAR=$v QBG_PROF_KERNELS=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sharded > $out/b_${v}_$rep.json 2> $out/b_${v}_$rep.err
  echo "== $VAR=$v rep $rep rc=$?"
  python - $out/b_${v}_$rep.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("ms/step", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["value"]), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k in d["roofline"]["kernels"][:10]:
    print(f'  {k["name"]:40s} {k["launches"]:4d} {k["total_ms"] / k["launches"]:.4f}')
PY
done; done
