for v in . s12 s16; do
 L=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so
 CS_LIB_PATH=$L PROF_ONLY=matched_dense TAG="$v four54" python tools/time_kernels.py >> gpurun_out/r02ag_time.jsonl 2>&1
 CS_LIB_PATH=$L CS_ST_FOUR=0 CS_STAGED_SMEM_KB=72 PROF_ONLY=matched_dense TAG="$v three72" python tools/time_kernels.py >> gpurun_out/r02ag_time.jsonl 2>&1
done
cat gpurun_out/r02ag_time.jsonl
