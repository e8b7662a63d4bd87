for kb in 48 52 54 56; do CS_ST_FOUR=1 CS_STAGED_SMEM_KB=$kb PROF_ONLY=matched_dense TAG=four_kb$kb python tools/time_kernels.py >> gpurun_out/r02ad_time.jsonl 2>&1; done
for kb in 64 72; do CS_STAGED_SMEM_KB=$kb PROF_ONLY=matched_dense TAG=three_kb$kb python tools/time_kernels.py >> gpurun_out/r02ad_time.jsonl 2>&1; done
CS_ST_FOUR=1 CS_STAGED_SMEM_KB=54 PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG=four_kb54_1024 python tools/time_kernels.py >> gpurun_out/r02ad_time.jsonl 2>&1
cat gpurun_out/r02ad_time.jsonl
