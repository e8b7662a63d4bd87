# TV-GD marching kernel: parity, timing, ncu
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tv or split" > gpurun_out/r02j_pytest.log 2>&1
echo "pytest rc $?"; tail -15 gpurun_out/r02j_pytest.log
PROF_ONLY=tv_gd_iter,tv_grad,tv_fused,tv_step,tv_run10,rof_iter TAG=march python tools/time_kernels.py > gpurun_out/r02j_time.jsonl 2>&1
CS_TV_TILED=1 PROF_ONLY=tv_grad TAG=tiled python tools/time_kernels.py >> gpurun_out/r02j_time.jsonl 2>&1
cat gpurun_out/r02j_time.jsonl
PROF_ONLY=tv_fused,tv_grad PROF_R=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tv_march -c 2 \
  -o gpurun_out/ncu_tv_march_r02j python tools/time_kernels.py > gpurun_out/ncu_tv_r02j.log 2>&1
echo "ncu rc $?"
