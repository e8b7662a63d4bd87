export PROF_ONLY=matched,matched_dense
TAG=flushcol python tools/time_kernels.py > gpurun_out/r02h_time.jsonl
PROF_N=1024 PROF_A=64 TAG=flushcol_1024 python tools/time_kernels.py >> gpurun_out/r02h_time.jsonl
cat gpurun_out/r02h_time.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loops.py -x -q -k "not distributed and not bench_self" > gpurun_out/r02h_pytest.log 2>&1
tail -3 gpurun_out/r02h_pytest.log
