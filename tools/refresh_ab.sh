# A/B of the values-only plan refresh (QBG_PLAN_REFRESH) on one box, plus the GPU suite
export QBG_JIT_CACHE=/tmp/jc_$RANDOM
mkdir -p gpurun_out/rf
timeout 600 python -m pytest tests/test_gpu_edge_cases.py -x -q > gpurun_out/rf/edge.log 2>&1; tail -2 gpurun_out/rf/edge.log
for i in 1 2; do
  for r in 1 0; do
    QBG_PLAN_REFRESH=$r timeout 600 python bench.py --no-cpu-baseline > gpurun_out/rf/bench_r${r}_$i.json 2> gpurun_out/rf/bench_r${r}_$i.err
    python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],round(d['value']),round(d['e2e']['value']),d['ms_per_step'],d['clocks']['sm_mhz'])" gpurun_out/rf/bench_r${r}_$i.json
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/rf/pytest_gpu.log 2>&1; tail -2 gpurun_out/rf/pytest_gpu.log
