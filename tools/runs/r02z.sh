timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ooc.py -x -q -k "out_of_core or ooc or loops" > gpurun_out/r02z_pytest.log 2>&1
echo "pytest rc $?"; tail -15 gpurun_out/r02z_pytest.log
