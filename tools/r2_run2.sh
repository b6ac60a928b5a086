mkdir -p gpurun_out/r2b
timeout 1500 python -m pytest tests/test_sharded.py tests/test_gpu_hygiene.py tests/test_gpu_shim.py tests/test_gpu_parity.py -m gpu -x -q -rs > gpurun_out/r2b/pytest.log 2>&1; echo pytest $?; tail -3 gpurun_out/r2b/pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err; echo bench $?; tail -c 1500 gpurun_out/r2b/bench.json; tail -5 gpurun_out/r2b/bench.err
