timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tv or split or rof" > gpurun_out/r02bc_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02bc_pytest.log
python tools/dbg/tv_variants.py 2>&1 | grep ndiff
for rep in 1 2 3; do for k in 1 0; do
CS_TV_TMA=$k PROF_ONLY=tv_grad,tv_fused,tv_run10 TAG="tma$k r$rep" python tools/time_kernels.py >> gpurun_out/r02bc_time.jsonl 2>&1
done; done
cat gpurun_out/r02bc_time.jsonl
PROF_ONLY=tv_fused PROF_R=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tv_march2 -c 1 \
  -o gpurun_out/ncu_tv_tma_r02bc python tools/time_kernels.py > gpurun_out/ncu_tv_tma_r02bc.log 2>&1
echo "ncu rc $?"
