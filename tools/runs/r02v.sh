CS_FWD_STAGED=1 PROF_ONLY=fwd TAG=staged_fwd python tools/time_kernels.py > gpurun_out/r02v_time.jsonl 2>&1
PROF_ONLY=fwd TAG=tex_fwd python tools/time_kernels.py >> gpurun_out/r02v_time.jsonl 2>&1
cat gpurun_out/r02v_time.jsonl
CS_FWD_STAGED=1 PROF_ONLY=fwd PROF_R=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:staged_kernel -c 1 \
  -o gpurun_out/ncu_staged_fwd_r02v python tools/time_kernels.py > gpurun_out/ncu_staged_fwd_r02v.log 2>&1
echo "ncu rc $?"
