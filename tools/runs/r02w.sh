# round-2 evidence: bench line, launch list of the bench command, ncu --set full of every hot kernel
T=r02w
mkdir -p gpurun_out/$T
timeout 900 python bench.py > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err
echo "bench rc $?"; head -c 300 gpurun_out/$T/bench.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$T/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-c3 \
  > gpurun_out/$T/launches_bench.log 2>&1
echo "launches rc $?"
PROF_KERNELS=tv,fwd,matched,fdk timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"fwd_mlayer|fill_|staged|march2|rof_march" -s 10 -c 10 -o gpurun_out/$T/full python tools/prof_c2.py \
  > gpurun_out/$T/ncu_full.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/$T/ncu_full.log
