# A/B: matched register accumulation on cell change (CS_ST_ACC=1 build in _lib/acc)
for v in . acc; do
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_ONLY=matched,matched_dense TAG=$v python tools/time_kernels.py >> gpurun_out/r02x_time.jsonl 2>&1
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so PROF_N=1024 PROF_A=64 PROF_ONLY=matched_dense TAG=${v}_1024 python tools/time_kernels.py >> gpurun_out/r02x_time.jsonl 2>&1
done
cat gpurun_out/r02x_time.jsonl
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/acc/libconesplit_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "backward or matched or adjoint or randomised or c1 or slab or window or dense" > gpurun_out/r02x_pytest.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/r02x_pytest.log
export PROF_ONLY=matched_dense PROF_R=1
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/acc/libconesplit_b200.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:staged_kernel -c 2 \
  -o gpurun_out/ncu_matched_acc_r02x python tools/time_kernels.py > gpurun_out/ncu_matched_acc_r02x.log 2>&1
echo "ncu rc $?"
