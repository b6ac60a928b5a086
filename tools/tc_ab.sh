mkdir -p gpurun_out/r2tc
timeout 300 python -m pytest tests/test_gpu_dense.py -m gpu -q -rs -x > gpurun_out/r2tc/pytest.log 2>&1; echo pytest $?; tail -3 gpurun_out/r2tc/pytest.log
timeout 600 python tools/cfg4_dense.py --n 30 --depth 10 --modes tile,tf32,dense --dtype c64 --reps 2 > gpurun_out/r2tc/cfg4_c64.jsonl 2> gpurun_out/r2tc/cfg4_c64.err; echo cfg4 $?; tail -3 gpurun_out/r2tc/cfg4_c64.err
python -c "
import json
for l in open('gpurun_out/r2tc/cfg4_c64.jsonl'):
    d=json.loads(l); k=[v for n,v in d['kernels'].items() if n!='set_basis']
    print(d['mode'], round(d['forward_ms'],1), k[0] if k else None, d.get('check_vs_tile'))"
