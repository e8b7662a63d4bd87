timeout 600 python -m pytest tests/test_gpu_refhook.py -x -q > gpurun_out/r02ax_pytest.log 2>&1
echo "pytest rc $?"; tail -15 gpurun_out/r02ax_pytest.log
