mkdir -p gpurun_out/r2e
timeout 300 python -m pytest tests/test_gpu_dense.py -m gpu -q -rs -x > gpurun_out/r2e/pytest.log 2>&1; echo pytest $?; tail -15 gpurun_out/r2e/pytest.log
timeout 600 python tools/cfg4_dense.py --n 30 --depth 10 --modes tile,dmma --dtype c64 > gpurun_out/r2e/cfg4_c64.jsonl 2> gpurun_out/r2e/cfg4_c64.err; echo cfg4 $?; tail -3 gpurun_out/r2e/cfg4_c64.err
QBG_DENSE_MMA=0 timeout 600 python tools/cfg4_dense.py --n 30 --depth 10 --modes dfma --reps 1 --dtype c64 >> gpurun_out/r2e/cfg4_c64.jsonl 2>> gpurun_out/r2e/cfg4_c64.err; echo dfma $?
cut -c1-700 gpurun_out/r2e/cfg4_c64.jsonl
