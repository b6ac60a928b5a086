export QBG_JIT_CACHE=/tmp/jc_$RANDOM
mkdir -p gpurun_out/modes
timeout 1200 python -m pytest tests/test_gpu_engine_modes.py -x -q -k refresh > gpurun_out/modes/refresh.log 2>&1; tail -2 gpurun_out/modes/refresh.log
