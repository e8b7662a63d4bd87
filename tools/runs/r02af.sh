T=r02af; mkdir -p gpurun_out/$T
PROF_KERNELS=matched timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"staged|transpose_add" -s 3 -c 3 -o gpurun_out/$T/full python tools/prof_c2.py > gpurun_out/$T/ncu_full.log 2>&1
echo "ncu rc $?"
