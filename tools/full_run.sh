set -x
export QBG_JIT_CACHE=/tmp/jc_$RANDOM
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 600 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qbg_ -s 45 -c 1 -f -o gpurun_out/top_bwd python tools/profile_step.py --steps 1 > gpurun_out/ncu_bwd.log 2>&1; echo ncu2 $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qbg_ -s 10 -c 1 -f -o gpurun_out/top_fwd python tools/profile_step.py --steps 1 > gpurun_out/ncu_fwd.log 2>&1; echo ncu3 $?
