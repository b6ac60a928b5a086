export QBG_JIT_CACHE=/tmp/jc_$RANDOM
mkdir -p gpurun_out/h
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/h/pytest_gpu.log 2>&1; tail -2 gpurun_out/h/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/h/smoke.log 2>&1; tail -1 gpurun_out/h/smoke.log
timeout 900 python bench.py > gpurun_out/h/bench.json 2> gpurun_out/h/bench.err; tail -c 1500 gpurun_out/h/bench.json
