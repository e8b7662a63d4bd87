for p in 0 1; do for n in 256 512 1024; do
CS_ST_PAIR=$p PROF_N=$n PROF_A=180 PROF_ONLY=matched_dense,matched timeout 600 python tools/time_kernels.py > gpurun_out/r02bp_${p}_${n}.json 2>&1
echo "pair=$p n=$n: $(tail -1 gpurun_out/r02bp_${p}_${n}.json)"
done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_loops.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02bp_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02bp_pytest.log
