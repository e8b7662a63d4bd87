free -g | head -2; nproc
timeout 600 python tools/bench_scale.py oocloops 384 32 0.1 2 > gpurun_out/r02aa_small.jsonl 2> gpurun_out/r02aa_small.err
echo "small rc $?"; cat gpurun_out/r02aa_small.jsonl; tail -3 gpurun_out/r02aa_small.err
timeout 1500 python tools/bench_scale.py oocloops 1536 64 6 3 > gpurun_out/r02aa_big.jsonl 2> gpurun_out/r02aa_big.err
echo "big rc $?"; cat gpurun_out/r02aa_big.jsonl; tail -3 gpurun_out/r02aa_big.err
