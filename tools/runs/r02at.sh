for rep in 1 2; do for v in . novf; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_R=3 PROF_ONLY=matched,matched_dense TAG="$v r$rep" python tools/time_kernels.py >> gpurun_out/r02at_time.jsonl 2>&1
done; done
cat gpurun_out/r02at_time.jsonl
