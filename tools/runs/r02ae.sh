timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "transposed or backward or matched or adjoint or randomised or c1 or slab or window or dense or tiny or odd or fullsize" > gpurun_out/r02ae_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02ae_pytest.log
PROF_ONLY=matched,matched_dense TAG=default_r02ae python tools/time_kernels.py > gpurun_out/r02ae_time.jsonl 2>&1
PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG=default_r02ae_1024 python tools/time_kernels.py >> gpurun_out/r02ae_time.jsonl 2>&1
PROF_N=2048 PROF_A=32 PROF_ONLY=matched_dense TAG=default_r02ae_2048 python tools/time_kernels.py >> gpurun_out/r02ae_time.jsonl 2>&1
cat gpurun_out/r02ae_time.jsonl
