timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loops.py -x -q -k "transposed or backward or matched or adjoint or randomised or c1 or slab or window or dense or tiny or odd or forward or sweep or config" > gpurun_out/r02aq_pytest.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/r02aq_pytest.log
for rep in 1 2 3; do for v in head .; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_R=5 PROF_ONLY=matched_dense TAG="$v r$rep" python tools/time_kernels.py >> gpurun_out/r02aq_time.jsonl 2>&1
done; done
for v in head .; do for n in 256 1024; do CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_N=$n PROF_A=64 PROF_ONLY=matched_dense TAG="$v $n" python tools/time_kernels.py >> gpurun_out/r02aq_time.jsonl 2>&1; done; done
cat gpurun_out/r02aq_time.jsonl
