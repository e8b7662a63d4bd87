# ncu: matched Atb on the dense stack (full set + source), launch list of the bench
export PROF_ONLY=matched_dense PROF_R=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:staged_kernel -c 2 \
  -o gpurun_out/ncu_matched_dense_r02g python tools/time_kernels.py > gpurun_out/ncu_matched_r02g.log 2>&1
echo "ncu rc $?"
unset PROF_ONLY PROF_R
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r02g.csv python bench.py --steps 2 --warmup 1 --no-extras --no-c3 > gpurun_out/launches_r02g.log 2>&1
echo "ncu2 rc $?"
ls -la gpurun_out/
timeout 900 python -m pytest tests/test_gpu_loops.py -x -q -k "distributed" > gpurun_out/r02g_pytest.log 2>&1
tail -15 gpurun_out/r02g_pytest.log
