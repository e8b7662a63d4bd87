# precise matched boxes: precision sweep + cost
export PROF_ONLY=matched,matched_dense
TAG=auto python tools/time_kernels.py > gpurun_out/r02c_time.jsonl
TAG=never CS_ST_PRECISE=0 python tools/time_kernels.py >> gpurun_out/r02c_time.jsonl
TAG=always CS_ST_PRECISE=1 python tools/time_kernels.py >> gpurun_out/r02c_time.jsonl
TAG=fp2 CS_ST_PRECISE_FP=2.0 python tools/time_kernels.py >> gpurun_out/r02c_time.jsonl
python tools/fuzz_loops.py 25 3 > gpurun_out/r02c_fuzz_loops_auto.txt 2>&1
CS_ST_PRECISE=1 python tools/fuzz_loops.py 25 3 > gpurun_out/r02c_fuzz_loops_always.txt 2>&1
python tools/diag_loop_case.py 3 1 2 4 21 > gpurun_out/r02c_diag.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_pytest.log 2>&1
tail -3 gpurun_out/r02c_pytest.log
cat gpurun_out/r02c_time.jsonl gpurun_out/r02c_fuzz_loops_auto.txt | tail -20
