# matched Atb at several volume sizes with the production occupancy rule
for n in 512 768 1024 2048; do
  PROF_N=$n PROF_A=32 PROF_ONLY=matched,matched_dense TAG="n$n A32" timeout 600 python tools/time_kernels.py
done
PROF_ONLY=matched,matched_dense TAG="n512 A360" timeout 600 python tools/time_kernels.py
