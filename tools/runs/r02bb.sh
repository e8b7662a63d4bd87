timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loops.py -x -q -k "tv or split or rof or sart or loops or sweep or config or out_of_core" > gpurun_out/r02bb_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02bb_pytest.log
timeout 2400 python tools/bench_scale.py oocloops 1536 64 6 3 > gpurun_out/r02bb_big.jsonl 2> gpurun_out/r02bb_big.err
echo "big rc $?"; cat gpurun_out/r02bb_big.jsonl; tail -3 gpurun_out/r02bb_big.err
