for rep in 1 2 3; do for v in head .; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_R=5 PROF_ONLY=fdk TAG="$v r$rep" python tools/time_kernels.py >> gpurun_out/r02ay_time.jsonl 2>&1
done; done
cat gpurun_out/r02ay_time.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fdk or backward or c1 or randomised or odd or tiny" > gpurun_out/r02ay_pytest.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/r02ay_pytest.log
