timeout 900 python -m pytest tests/test_gpu_ooc.py tests/test_gpu_parity.py -x -q -k "streamed_tv or out_of_core or split" > gpurun_out/r02bs_pytest.log 2>&1
echo "pytest rc $?"; tail -5 gpurun_out/r02bs_pytest.log
timeout 900 python tools/dbg/ooc_profile.py 1024 1.5 > gpurun_out/r02bs_prof.txt 2>&1; echo "prof rc $?"; head -1 gpurun_out/r02bs_prof.txt; sed -n 8,30p gpurun_out/r02bs_prof.txt | cut -c1-150
timeout 2400 python tools/bench_scale.py oocloops 1536 64 6 3 > gpurun_out/r02bs_big.jsonl 2> gpurun_out/r02bs_big.err
echo "big rc $?"; cat gpurun_out/r02bs_big.jsonl; tail -3 gpurun_out/r02bs_big.err
