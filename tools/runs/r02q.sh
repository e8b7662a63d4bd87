python tools/dbg/tv_variants.py 2>&1 | grep ndiff
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tv or split or rof" > gpurun_out/r02q_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02q_pytest.log
PROF_ONLY=tv_grad,tv_fused,tv_run10,rof_iter TAG=d8_guard python tools/time_kernels.py > gpurun_out/r02q_time.jsonl 2>&1
CS_ROF_MARCH=0 PROF_ONLY=rof_iter TAG=rof_r01 python tools/time_kernels.py >> gpurun_out/r02q_time.jsonl 2>&1
cat gpurun_out/r02q_time.jsonl
