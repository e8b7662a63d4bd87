export PROF_ONLY=matched,matched_dense
TAG=default python tools/time_kernels.py > gpurun_out/r02e_time.jsonl
TAG=always CS_ST_PRECISE=1 python tools/time_kernels.py >> gpurun_out/r02e_time.jsonl
echo "coarse edge-only" > gpurun_out/r02e_fuzz.txt
FUZZ_COARSE=1 CS_ST_PRECISE_FP=1e9 python tools/fuzz_loops.py 10 5 >> gpurun_out/r02e_fuzz.txt 2>&1
echo "coarse default" >> gpurun_out/r02e_fuzz.txt
FUZZ_COARSE=1 python tools/fuzz_loops.py 10 5 >> gpurun_out/r02e_fuzz.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02e_pytest.log 2>&1
tail -15 gpurun_out/r02e_pytest.log
cat gpurun_out/r02e_time.jsonl gpurun_out/r02e_fuzz.txt
