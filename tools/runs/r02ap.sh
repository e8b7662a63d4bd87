timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "transposed or backward or matched or adjoint or randomised or c1 or slab or window or dense or tiny or odd or forward" > gpurun_out/r02ap_pytest.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/r02ap_pytest.log
for rep in 1 2 3; do for v in head .; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_R=5 PROF_ONLY=matched_dense TAG="$v r$rep" python tools/time_kernels.py >> gpurun_out/r02ap_time.jsonl 2>&1
done; done
for v in head .; do CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_N=256 PROF_A=90 PROF_ONLY=matched_dense TAG="$v 256" python tools/time_kernels.py >> gpurun_out/r02ap_time.jsonl 2>&1; done
cat gpurun_out/r02ap_time.jsonl
timeout 1500 python tools/bench_scale.py c4 > gpurun_out/r02ap_c4.jsonl 2> gpurun_out/r02ap_c4.err; echo "c4 rc $?"; cat gpurun_out/r02ap_c4.jsonl
