# ncu --set full of one dense matched launch (512^3, 36 views) with the
# per-thread RED flush (CS_ST_BULK=0) and the TMA bulk-reduce flush (=1).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bulk
for b in 0 1; do
  CS_ST_BULK=$b PROF_N=512 PROF_A=36 PROF_R=1 PROF_ONLY=matched_dense \
    timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:staged_kernel -s 1 -c 1 -o gpurun_out/bulk/full_b$b \
    python tools/time_kernels.py > gpurun_out/bulk/ncu_b$b.log 2>&1
done
