# matched A/B: T-pitch pad (0 / 31 / 15) x box smem (54 / 64 / 72 KB)
for tp in 0 31 15; do for kb in 54 64 72; do
CS_ST_TPAD=$tp CS_STAGED_SMEM_KB=$kb PROF_ONLY=matched_dense TAG=tp${tp}_kb${kb} python tools/time_kernels.py >> gpurun_out/r02t_time.jsonl 2>&1
done; done
for tp in 0 31; do CS_ST_TPAD=$tp PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG=tp${tp}_1024 python tools/time_kernels.py >> gpurun_out/r02t_time.jsonl 2>&1; done
cat gpurun_out/r02t_time.jsonl
