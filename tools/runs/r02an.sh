timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "transposed or backward or matched or adjoint or randomised or c1 or slab or window or dense or tiny or odd" > gpurun_out/r02an_pytest.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/r02an_pytest.log
for rep in 1 2 3; do PROF_R=5 PROF_ONLY=matched_dense TAG="sdiv r$rep" python tools/time_kernels.py >> gpurun_out/r02an_time.jsonl 2>&1; done
PROF_N=256 PROF_A=90 PROF_ONLY=matched_dense TAG="sdiv 256" python tools/time_kernels.py >> gpurun_out/r02an_time.jsonl 2>&1
PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG="sdiv 1024" python tools/time_kernels.py >> gpurun_out/r02an_time.jsonl 2>&1
cat gpurun_out/r02an_time.jsonl
