# matched chunk depth variants (dirs under _lib) at 512^3/360 views and 2048^3/32 views
for v in "$@"; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=matched,matched_dense TAG="n512 A360 $v" timeout 600 python tools/time_kernels.py
  PROF_N=2048 PROF_A=32 CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=matched,matched_dense TAG="n2048 A32 $v" timeout 600 python tools/time_kernels.py
done
