python tools/dbg/tv_variants.py 2>&1 | grep ndiff
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tv or split" > gpurun_out/r02o_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02o_pytest.log
PROF_ONLY=tv_grad,tv_fused,tv_run10 TAG=pairs_pinned python tools/time_kernels.py > gpurun_out/r02o_time.jsonl 2>&1
cat gpurun_out/r02o_time.jsonl
