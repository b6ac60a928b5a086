mkdir -p gpurun_out/r2g
timeout 600 python -m pytest tests/test_gpu_dense.py tests/test_gpu_random_circuits.py tests/test_gpu_parity.py -m gpu -q -rs -x > gpurun_out/r2g/pytest.log 2>&1; echo pytest $?; tail -5 gpurun_out/r2g/pytest.log
timeout 600 python tools/cfg4_dense.py --n 30 --depth 10 --modes tile,dense,tf32,cuda --dtype c64 --reps 2 > gpurun_out/r2g/cfg4_c64.jsonl 2> gpurun_out/r2g/cfg4_c64.err; echo cfg4 $?; tail -3 gpurun_out/r2g/cfg4_c64.err
cut -c1-300 gpurun_out/r2g/cfg4_c64.jsonl
timeout 600 python bench.py --no-cpu-baseline --no-sharded > gpurun_out/r2g/bench.json 2> gpurun_out/r2g/bench.err; echo bench $?
python -c "
import json; d=json.loads(open('gpurun_out/r2g/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['ms_per_launch'], d['roofline']['frac'], d['clocks'])"
