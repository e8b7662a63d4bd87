timeout 1500 python tools/bench_scale.py c4 > gpurun_out/r02ao_c4.jsonl 2> gpurun_out/r02ao_c4.err
echo "c4 rc $?"; cat gpurun_out/r02ao_c4.jsonl; tail -2 gpurun_out/r02ao_c4.err
T=r02ao; mkdir -p gpurun_out/$T
PROF_KERNELS=tv,fwd,matched,fdk timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"fwd_mlayer|fill_|staged|march2|rof_march|transpose_add" -s 11 -c 11 -o gpurun_out/$T/full python tools/prof_c2.py \
  > gpurun_out/$T/ncu_full.log 2>&1
echo "ncu rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$T/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-c3 \
  > gpurun_out/$T/launches_bench.log 2>&1
echo "launches rc $?"
