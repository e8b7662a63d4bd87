# matched Atb occupancy / box budget A/B at 1024^3 and 2048^3 (32 views)
#   bash tools/ab_matched_2048.sh   (needs _lib/m3 = ST_MINB=3 build)
for n in 1024 2048; do
for vk in ".:54" "m3:64" "m3:54" ".:48"; do
  v=${vk%%:*}; kb=${vk##*:}
  PROF_N=$n PROF_A=32 CS_STAGED_SMEM_KB=$kb CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=matched,matched_dense TAG="n$n $v:$kb" timeout 600 python tools/time_kernels.py
done
done
