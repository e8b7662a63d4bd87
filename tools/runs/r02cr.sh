# matched: sample loop unrolled by two, A/B vs HEAD
for i in 1 2; do
for v in head .; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=matched_dense,matched TAG="matched $v n512" timeout 300 python tools/time_kernels.py
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG="matched $v n1024" timeout 300 python tools/time_kernels.py
done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "matched or adjoint or backward or loop" 2>&1 | tail -2
