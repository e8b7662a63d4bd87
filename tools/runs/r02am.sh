for rep in 1 2 3; do
 for v in . zof; do
  L=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so
  CS_LIB_PATH=$L PROF_R=5 PROF_ONLY=matched_dense TAG="$v r$rep" python tools/time_kernels.py >> gpurun_out/r02am_time.jsonl 2>&1
 done
done
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/zof/libconesplit_b200.so PROF_N=256 PROF_A=90 PROF_ONLY=matched_dense TAG="zof 256" python tools/time_kernels.py >> gpurun_out/r02am_time.jsonl 2>&1
PROF_N=256 PROF_A=90 PROF_ONLY=matched_dense TAG=". 256" python tools/time_kernels.py >> gpurun_out/r02am_time.jsonl 2>&1
cat gpurun_out/r02am_time.jsonl
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/zof/libconesplit_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "backward or matched or adjoint or randomised or c1 or slab or window or dense or tiny or odd" > gpurun_out/r02am_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02am_pytest.log
