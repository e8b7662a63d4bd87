timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ooc.py -x -q -k "out_of_core or ooc or transposed or backward or matched or adjoint or randomised or c1 or slab or window or dense" > gpurun_out/r02ab_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02ab_pytest.log
PROF_ONLY=matched,matched_dense TAG=transposed python tools/time_kernels.py > gpurun_out/r02ab_time.jsonl 2>&1
CS_ST_TRANSPOSE=0 PROF_ONLY=matched_dense TAG=direct python tools/time_kernels.py >> gpurun_out/r02ab_time.jsonl 2>&1
PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG=transposed_1024 python tools/time_kernels.py >> gpurun_out/r02ab_time.jsonl 2>&1
cat gpurun_out/r02ab_time.jsonl
timeout 900 python -m pytest tests/test_gpu_loops.py -x -q > gpurun_out/r02ab_loops.log 2>&1
echo "loops rc $?"; tail -2 gpurun_out/r02ab_loops.log
