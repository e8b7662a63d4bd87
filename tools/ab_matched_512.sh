for n in 512 768; do
for vk in ".:54" "m3:64"; do
  v=${vk%%:*}; kb=${vk##*:}
  PROF_N=$n PROF_A=32 CS_STAGED_SMEM_KB=$kb CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=matched,matched_dense TAG="n$n A32 $v:$kb" timeout 600 python tools/time_kernels.py
done
done
