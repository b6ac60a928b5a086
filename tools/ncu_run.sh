# ncu evidence on one box (each command only after the plain run exited 0): launch list of the
# bench command, then one --set full capture of a reverse and a forward pass
export QBG_JIT_CACHE=/tmp/jc_$RANDOM
mkdir -p gpurun_out/ncu
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu/plain.json 2>&1; echo plain $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu/ncu_launch.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qbg_ -s 45 -c 1 -f -o gpurun_out/ncu/top_bwd python tools/profile_step.py --steps 1 > gpurun_out/ncu/ncu_bwd.log 2>&1; echo ncu2 $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qbg_ -s 10 -c 1 -f -o gpurun_out/ncu/top_fwd python tools/profile_step.py --steps 1 > gpurun_out/ncu/ncu_fwd.log 2>&1; echo ncu3 $?
