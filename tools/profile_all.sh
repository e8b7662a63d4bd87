# ncu --set full of every hot kernel at config 2 (one process per group so
# each capture is the second launch of its kernel), for profiles/.
#   bash tools/profile_all.sh TAG
cd $GRAFT_REPO_ROOT
T=$1
mkdir -p gpurun_out/$T
PROF_KERNELS=fwd,matched,fdk,siddon timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"fwd_mlayer|fill_|staged|siddon" -s 8 -c 8 -o gpurun_out/$T/rays python tools/prof_c2.py \
  > gpurun_out/$T/ncu_rays.log 2>&1
PROF_KERNELS=tv timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"tv_gd|tv_step_g|rof_iter" -s 3 -c 3 -o gpurun_out/$T/tv python tools/prof_c2.py \
  > gpurun_out/$T/ncu_tv.log 2>&1
