export PROF_ONLY=matched,matched_dense
TAG=auto python tools/time_kernels.py > gpurun_out/r02d_time.jsonl
TAG=edge CS_ST_PRECISE_FP=1e9 python tools/time_kernels.py >> gpurun_out/r02d_time.jsonl
TAG=never CS_ST_PRECISE=0 python tools/time_kernels.py >> gpurun_out/r02d_time.jsonl
TAG=fp2 CS_ST_PRECISE_FP=2.0 python tools/time_kernels.py >> gpurun_out/r02d_time.jsonl
for seed in 3 0 1; do
  echo "seed $seed edge" >> gpurun_out/r02d_fuzz.txt
  CS_ST_PRECISE_FP=1e9 python tools/fuzz_loops.py 25 $seed >> gpurun_out/r02d_fuzz.txt 2>&1
  echo "seed $seed fp2" >> gpurun_out/r02d_fuzz.txt
  CS_ST_PRECISE_FP=2.0 python tools/fuzz_loops.py 25 $seed >> gpurun_out/r02d_fuzz.txt 2>&1
  echo "seed $seed auto" >> gpurun_out/r02d_fuzz.txt
  python tools/fuzz_loops.py 25 $seed >> gpurun_out/r02d_fuzz.txt 2>&1
done
cat gpurun_out/r02d_time.jsonl gpurun_out/r02d_fuzz.txt
