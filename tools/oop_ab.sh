# A/B of the out-of-place first forward pass (QBG_FWD_OOP) on one box, then the GPU suite
export QBG_JIT_CACHE=/tmp/jc_$RANDOM
mkdir -p gpurun_out/oop
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q > gpurun_out/oop/quick.log 2>&1; tail -2 gpurun_out/oop/quick.log
for i in 1 2; do
  for r in 1 0; do
    QBG_FWD_OOP=$r timeout 600 python bench.py --no-cpu-baseline > gpurun_out/oop/bench_o${r}_$i.json 2> gpurun_out/oop/bench_o${r}_$i.err
    python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1],round(d['value']),round(d['e2e']['value']),d['ms_per_step'],d['clocks']['sm_mhz'])" gpurun_out/oop/bench_o${r}_$i.json
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/oop/pytest_gpu.log 2>&1; tail -2 gpurun_out/oop/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/oop/smoke.log 2>&1; tail -1 gpurun_out/oop/smoke.log
