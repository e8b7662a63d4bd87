for v in s10 s12 s14; do
 L=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so
 for kb in 64 68 72; do
 CS_LIB_PATH=$L CS_ST_FOUR=0 CS_STAGED_SMEM_KB=$kb PROF_ONLY=matched_dense TAG="$v three$kb" python tools/time_kernels.py >> gpurun_out/r02ah_time.jsonl 2>&1
 done
done
L=$PWD/paper_1905_03748_b200/_lib/s12/libconesplit_b200.so
CS_LIB_PATH=$L CS_ST_FOUR=0 CS_STAGED_SMEM_KB=72 PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG="s12 three72 1024" python tools/time_kernels.py >> gpurun_out/r02ah_time.jsonl 2>&1
CS_LIB_PATH=$L CS_ST_FOUR=0 CS_STAGED_SMEM_KB=72 PROF_N=2048 PROF_A=32 PROF_ONLY=matched_dense TAG="s12 three72 2048" python tools/time_kernels.py >> gpurun_out/r02ah_time.jsonl 2>&1
PROF_N=2048 PROF_A=32 PROF_ONLY=matched_dense TAG=". four54 2048" python tools/time_kernels.py >> gpurun_out/r02ah_time.jsonl 2>&1
cat gpurun_out/r02ah_time.jsonl
