timeout 2400 python tools/bench_scale.py oocloops 1536 64 6 3 > gpurun_out/r02ba_big.jsonl 2> gpurun_out/r02ba_big.err
echo "big rc $?"; cat gpurun_out/r02ba_big.jsonl; tail -3 gpurun_out/r02ba_big.err
