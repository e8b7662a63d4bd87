timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ooc.py -x -q -k "tv or split or out_of_core or ooc or rof" > gpurun_out/r02bg_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02bg_pytest.log
timeout 2400 python tools/bench_scale.py oocloops 1536 64 6 3 > gpurun_out/r02bg_big.jsonl 2> gpurun_out/r02bg_big.err
echo "big rc $?"; cat gpurun_out/r02bg_big.jsonl; tail -3 gpurun_out/r02bg_big.err
