# FDK: footprint staged as column pairs (one LDS.64 per bilinear row), A/B vs HEAD
for i in 1 2; do
for v in head .; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=fdk TAG="fdk $v" timeout 300 python tools/time_kernels.py
done
done
for v in head .; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_N=256 PROF_A=180 PROF_ONLY=fdk TAG="fdk $v n256" timeout 300 python tools/time_kernels.py
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_N=1024 PROF_A=64 PROF_ONLY=fdk TAG="fdk $v n1024" timeout 300 python tools/time_kernels.py
done
timeout 900 python -m pytest tests -m gpu -x -q -k "fdk or FDK or golden or fine" 2>&1 | tail -2
