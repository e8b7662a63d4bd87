timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loops.py -x -q > gpurun_out/r02u_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02u_pytest.log
PROF_ONLY=matched,matched_dense TAG=default_r02u python tools/time_kernels.py > gpurun_out/r02u_time.jsonl 2>&1
PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG=default_r02u_1024 python tools/time_kernels.py >> gpurun_out/r02u_time.jsonl 2>&1
cat gpurun_out/r02u_time.jsonl
