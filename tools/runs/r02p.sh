export PROF_ONLY=matched_dense PROF_R=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:staged_kernel -c 2 \
  -o gpurun_out/ncu_matched_dense_r02p python tools/time_kernels.py > gpurun_out/ncu_matched_r02p.log 2>&1
echo "ncu rc $?"
export PROF_ONLY=tv_fused
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tv_march2 -c 1 \
  -o gpurun_out/ncu_tv_fused_r02p python tools/time_kernels.py > gpurun_out/ncu_tv_fused_r02p.log 2>&1
echo "ncu2 rc $?"
