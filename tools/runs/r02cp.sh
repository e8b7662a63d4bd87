# TV-GD fused marching kernel: plane loop unrolled by two, A/B vs HEAD
for i in 1 2; do
for v in head .; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=tv_fused,tv_run10,tv_grad TAG="tv $v" timeout 300 python tools/time_kernels.py
done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "tv or TV or rof or split or march" 2>&1 | tail -2
