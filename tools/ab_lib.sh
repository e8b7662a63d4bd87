# A/B of library variants on the config-2 kernel timings:
#   bash tools/ab_lib.sh OUT.jsonl PROF_ONLY variant1 [variant2 ...]
# (variant = a dir under paper_1905_03748_b200/_lib, "." = production)
cd $GRAFT_REPO_ROOT
out=$1; only=$2; shift 2
mkdir -p $(dirname $out)
for v in "$@"; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=$only TAG=$v timeout 300 python tools/time_kernels.py >> $out 2>> $out.err
done
