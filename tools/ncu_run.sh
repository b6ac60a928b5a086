# ncu evidence (each command only after the plain run exited 0): launch list of the bench command,
# one --set full capture of a reverse and a forward pass, SASS source pages exported as CSV
out=gpurun_out/${1:-ncu}
mkdir -p $out
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sharded > $out/plain.json 2>&1; echo plain $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sharded > $out/ncu_launch.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qbg_ -s 45 -c 1 -f -o $out/top_bwd python tools/profile_step.py --steps 1 > $out/ncu_bwd.log 2>&1; echo ncu2 $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qbg_ -s 10 -c 1 -f -o $out/top_fwd python tools/profile_step.py --steps 1 > $out/ncu_fwd.log 2>&1; echo ncu3 $?
for r in top_bwd top_fwd; do
  ncu -i $out/$r.ncu-rep --page source --csv --print-source sass > $out/${r}_sass.csv 2>/dev/null
  ncu -i $out/$r.ncu-rep --page raw --csv > $out/${r}_raw.csv 2>/dev/null
  python tools/ncu_details.py $out/$r.ncu-rep > $out/${r}_details.txt 2>&1
done
ls -la $out
