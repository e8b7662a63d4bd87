# Round evidence on one B200: bench line, launch list of the same bench
# command, ncu --set full of the hot kernels (tools/prof_c2.py).
#   bash tools/profile_round.sh TAG
cd $GRAFT_REPO_ROOT
T=$1
mkdir -p gpurun_out/$T
timeout 600 python bench.py > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$T/launches.csv python bench.py --steps 2 --warmup 3 --no-extras \
  > gpurun_out/$T/launches_bench.log 2>&1
PROF_KERNELS=fwd,matched,fdk timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"fwd_mlayer|fill_|staged" -s 7 -c 7 -o gpurun_out/$T/full python tools/prof_c2.py \
  > gpurun_out/$T/ncu_full.log 2>&1
