# FDK: floor by a round-down magic add (FADD.RM) instead of FRND, A/B vs HEAD
for v in head .; do
  for i in 1 2; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=fdk TAG="fdk $v" timeout 300 python tools/time_kernels.py
  done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "fdk" 2>&1 | tail -2
