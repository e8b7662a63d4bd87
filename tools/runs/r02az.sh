for rep in 1 2 3; do for v in . fpk; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_R=5 PROF_ONLY=fwd TAG="$v r$rep" python tools/time_kernels.py >> gpurun_out/r02az_time.jsonl 2>&1
done; done
cat gpurun_out/r02az_time.jsonl
