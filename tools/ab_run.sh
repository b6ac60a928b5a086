# quick A/B + parity check of the current tree on one box
out=gpurun_out/${1:-ab}
mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_random_circuits.py tests/test_gpu_engine_modes.py tests/test_gpu_edge_cases.py -m gpu -q -x > $out/pytest.log 2>&1; echo pytest $?; tail -2 $out/pytest.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-sharded > $out/bench$i.json 2> $out/bench$i.err; echo bench $?
python -c "
import json; d=json.loads(open('$out/bench$i.json').read().strip().splitlines()[-1])
r=d['roofline']
print(round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), [(k['name'], k['launches'], round(k['total_ms']/k['launches'],4)) for k in r['kernels'][:4]], round(r['frac'],3), d['clocks'])"
done
