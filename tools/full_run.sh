# round-end set on one B200 (run by gpurun from the repo root): the GPU suite, smoke(), bench.py
# (metric line + sharded_state), the reference arm (short), the c64 line, cfg-4 dense A/B.
# Uses the in-tree ahead-of-time kernel cache (jit_cache/) like the driver does.
out=gpurun_out/${1:-full}
mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > $out/pytest_gpu.log 2>&1; echo pytest $?; tail -2 $out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo smoke $?; tail -1 $out/smoke.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo bench $?
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(round(d['value']),round(d['e2e']['value']),d['ms_per_step'],d['clocks'],d['roofline']['frac'],d.get('sharded_state'))" $out/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2>&1; echo ref $?
timeout 600 python bench.py --dtype c64 --no-cpu-baseline > $out/bench_c64.json 2> $out/bench_c64.err; echo c64 $?
