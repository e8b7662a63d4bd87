timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loops.py -x -q -k "tv or split or rof or sart or loops or sweep or config" > gpurun_out/r02av_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02av_pytest.log
PROF_ONLY=tv_grad,tv_fused,tv_step,tv_run10,rof_iter TAG=f32step python tools/time_kernels.py > gpurun_out/r02av_time.jsonl 2>&1
cat gpurun_out/r02av_time.jsonl
