python tools/diag_col_ray.py 3 21 > gpurun_out/diag_col_21.jsonl 2>&1
python tools/diag_col_ray.py 3 2 > gpurun_out/diag_col_2.jsonl 2>&1
CS_STAGED_SMEM_KB=1 python tools/diag_col_ray.py 3 21 > gpurun_out/diag_col_21_global.jsonl 2>&1
python tools/diag_col_ray.py 3 4 > gpurun_out/diag_col_4.jsonl 2>&1
