mkdir -p gpurun_out/r2f
timeout 300 python -m pytest tests/test_gpu_dense.py -m gpu -q -rs -x > gpurun_out/r2f/pytest.log 2>&1; echo pytest $?; tail -5 gpurun_out/r2f/pytest.log
timeout 600 python tools/cfg4_dense.py --n 30 --depth 10 --modes tile,dense --dtype c64 > gpurun_out/r2f/cfg4_c64.jsonl 2> gpurun_out/r2f/cfg4_c64.err; echo cfg4 $?; tail -3 gpurun_out/r2f/cfg4_c64.err
cut -c1-900 gpurun_out/r2f/cfg4_c64.jsonl
