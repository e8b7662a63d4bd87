for kb in 64 72 80; do
  PROF_N=2048 PROF_A=32 CS_STAGED_SMEM_KB=$kb PROF_ONLY=matched,matched_dense TAG="n2048 A32 3cta kb$kb" timeout 600 python tools/time_kernels.py
  PROF_N=1024 PROF_A=32 CS_STAGED_SMEM_KB=$kb PROF_ONLY=matched,matched_dense TAG="n1024 A32 3cta kb$kb" timeout 600 python tools/time_kernels.py
done
