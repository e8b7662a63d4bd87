for rep in 1 2 3; do for v in . vf; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_R=5 PROF_ONLY=matched_dense TAG="$v r$rep" python tools/time_kernels.py >> gpurun_out/r02ar_time.jsonl 2>&1
done; done
for v in . vf; do for n in 1024 2048; do CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_N=$n PROF_A=32 PROF_ONLY=matched_dense TAG="$v $n" python tools/time_kernels.py >> gpurun_out/r02ar_time.jsonl 2>&1; done; done
cat gpurun_out/r02ar_time.jsonl
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/vf/libconesplit_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "transposed or backward or matched or adjoint or randomised or c1 or slab or dense or odd" > gpurun_out/r02ar_pytest.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/r02ar_pytest.log
