for rep in 1 2 3; do
 for v in s14 s16 s20; do
  L=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so
  CS_LIB_PATH=$L CS_ST_FOUR=0 CS_STAGED_SMEM_KB=72 PROF_R=5 PROF_ONLY=matched_dense TAG="$v r$rep" python tools/time_kernels.py >> gpurun_out/r02aj_time.jsonl 2>&1
 done
done
for v in . s14; do
  L=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so
  four=0; [ "$v" = "." ] && four=1; kb=72; [ "$v" = "." ] && kb=54
  CS_LIB_PATH=$L CS_ST_FOUR=$four CS_STAGED_SMEM_KB=$kb PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG="$v 1024" python tools/time_kernels.py >> gpurun_out/r02aj_time.jsonl 2>&1
  CS_LIB_PATH=$L CS_ST_FOUR=$four CS_STAGED_SMEM_KB=$kb PROF_N=2048 PROF_A=32 PROF_ONLY=matched_dense TAG="$v 2048" python tools/time_kernels.py >> gpurun_out/r02aj_time.jsonl 2>&1
  CS_LIB_PATH=$L CS_ST_FOUR=$four CS_STAGED_SMEM_KB=$kb PROF_N=256 PROF_A=90 PROF_ONLY=matched_dense TAG="$v 256" python tools/time_kernels.py >> gpurun_out/r02aj_time.jsonl 2>&1
done
cat gpurun_out/r02aj_time.jsonl
