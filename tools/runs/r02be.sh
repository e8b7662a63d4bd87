timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tv or split or rof" > gpurun_out/r02be_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02be_pytest.log
for rep in 1 2 3; do for k in 1 0; do
CS_TV_TMA=$k PROF_ONLY=rof_iter TAG="tma$k r$rep" python tools/time_kernels.py >> gpurun_out/r02be_time.jsonl 2>&1
done; done
cat gpurun_out/r02be_time.jsonl
