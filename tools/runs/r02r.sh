# matched flush rewrite: parity + timing
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "backward or matched or adjoint or randomised or c1 or slab or window or dense" > gpurun_out/r02r_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02r_pytest.log
PROF_ONLY=matched,matched_dense TAG=flush_ptr python tools/time_kernels.py > gpurun_out/r02r_time.jsonl 2>&1
PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG=flush_ptr_1024 python tools/time_kernels.py >> gpurun_out/r02r_time.jsonl 2>&1
cat gpurun_out/r02r_time.jsonl
