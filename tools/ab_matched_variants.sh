# matched Atb timings of library variants x shared-box budgets:
#   bash tools/ab_matched_variants.sh OUT.jsonl "variant:kb" ...
out=$1; shift
for vk in "$@"; do
  v=${vk%%:*}; kb=${vk##*:}
  CS_STAGED_SMEM_KB=$kb CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=matched,matched_dense TAG="$v:$kb" timeout 300 python tools/time_kernels.py >> $out 2>> $out.err
done
