mkdir -p gpurun_out/san
export QBG_JIT_CACHE=/tmp/jc_$RANDOM
python tools/sanitize_smoke.py > gpurun_out/san/plain.log 2>&1; echo plain $?
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py > gpurun_out/san/memcheck.log 2>&1; echo memcheck $?; tail -5 gpurun_out/san/memcheck.log
