# A/B of the matched flush: per-thread REDs (CS_ST_BULK=0, default) vs the
# TMA bulk reduce (CS_ST_BULK=1), dense and phantom stacks, then the
# matched parity tests under the bulk flush.
#   bash tools/ab_matched_bulk.sh OUT.jsonl
cd $GRAFT_REPO_ROOT
out=$1
mkdir -p $(dirname $out)
for b in 0 1; do
  for na in "256 180" "512 360" "1024 64"; do
    set -- $na
    CS_ST_BULK=$b PROF_N=$1 PROF_A=$2 PROF_ONLY=matched,matched_dense \
      TAG="bulk=$b n$1 A$2" timeout 600 python tools/time_kernels.py >> $out 2>> $out.err
  done
done
CS_ST_BULK=1 timeout 900 python -m pytest tests -m gpu -x -q -k "matched or adjoint or loop or sirt or cgls" >> $out.tests 2>&1
echo "tests_rc=$?" >> $out.tests
