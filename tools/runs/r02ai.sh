for rep in 1 2 3; do
 for cfg in ".:1:54" "s12:0:72" "s14:0:72" "s12:0:64" "s10:0:68"; do
  v=${cfg%%:*}; rest=${cfg#*:}; four=${rest%%:*}; kb=${rest#*:}
  L=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so
  CS_LIB_PATH=$L CS_ST_FOUR=$four CS_STAGED_SMEM_KB=$kb PROF_R=5 PROF_ONLY=matched_dense TAG="$v f$four kb$kb r$rep" python tools/time_kernels.py >> gpurun_out/r02ai_time.jsonl 2>&1
 done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
cat gpurun_out/r02ai_time.jsonl
