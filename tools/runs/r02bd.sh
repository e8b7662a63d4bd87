timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tv or split or rof" > gpurun_out/r02bd_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02bd_pytest.log
