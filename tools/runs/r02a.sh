set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/diag_loop_case.py 3 1 2 3 4 11 13 16 17 21 > gpurun_out/diag_r02a.jsonl 2>&1
CS_STAGED_SMEM_KB=1 python tools/diag_loop_case.py 3 2 21 4 > gpurun_out/diag_r02a_global.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02a.log 2>&1
tail -3 gpurun_out/pytest_r02a.log
timeout 300 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
cat gpurun_out/bench_r02a.json
