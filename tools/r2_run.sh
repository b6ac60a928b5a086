# round-2 GPU run: the GPU suite, smoke, bench (default cache = the in-tree AOT cache)
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/r2/pytest_gpu.log 2>&1; echo pytest $?; tail -3 gpurun_out/r2/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/r2/smoke.log
timeout 900 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo bench $?; tail -c 400 gpurun_out/r2/bench.json
