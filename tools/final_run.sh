# round-end style check on one box: GPU suite, smoke, bench (c128 metric line), reference arm (short)
export QBG_JIT_CACHE=/tmp/jc_$RANDOM
mkdir -p gpurun_out/fin4
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin4/pytest_gpu.log 2>&1; tail -2 gpurun_out/fin4/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin4/smoke.log 2>&1; tail -1 gpurun_out/fin4/smoke.log
timeout 900 python bench.py > gpurun_out/fin4/bench.json 2> gpurun_out/fin4/bench.err
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(round(d['value']),round(d['e2e']['value']),d['ms_per_step'],d['clocks'],d['roofline']['frac'],d['roofline']['step'])" gpurun_out/fin4/bench.json
