timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "transposed or backward or matched or adjoint or randomised or c1 or slab or window or dense or tiny or odd or fullsize" > gpurun_out/r02ak_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02ak_pytest.log
for rep in 1 2; do
PROF_R=5 PROF_ONLY=matched,matched_dense TAG=default_r02ak python tools/time_kernels.py >> gpurun_out/r02ak_time.jsonl 2>&1
done
PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG=default_1024 python tools/time_kernels.py >> gpurun_out/r02ak_time.jsonl 2>&1
PROF_N=256 PROF_A=90 PROF_ONLY=matched_dense TAG=default_256 python tools/time_kernels.py >> gpurun_out/r02ak_time.jsonl 2>&1
cat gpurun_out/r02ak_time.jsonl
timeout 900 python -m pytest tests/test_gpu_loops.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02ak_loops.log 2>&1
echo "loops rc $?"; tail -2 gpurun_out/r02ak_loops.log
