timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tv or split" > gpurun_out/r02n_pytest.log 2>&1
echo "pytest rc $?"; tail -15 gpurun_out/r02n_pytest.log
PROF_ONLY=tv_grad,tv_fused,tv_step,tv_run10 TAG=pairs python tools/time_kernels.py > gpurun_out/r02n_time.jsonl 2>&1
cat gpurun_out/r02n_time.jsonl
PROF_ONLY=tv_fused,tv_grad PROF_R=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tv_march -c 6 \
  -o gpurun_out/ncu_tv_march_r02n python tools/time_kernels.py > gpurun_out/ncu_tv_r02n.log 2>&1
echo "ncu rc $?"
CS_TV_PAIRS=0 PROF_ONLY=tv_grad,tv_fused TAG=single python tools/time_kernels.py >> gpurun_out/r02n_time.jsonl 2>&1; tail -1 gpurun_out/r02n_time.jsonl
