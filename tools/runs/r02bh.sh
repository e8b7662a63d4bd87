timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02bh_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02bh_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02bh_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r02bh_smoke.log
timeout 600 python bench.py > gpurun_out/r02bh_bench.json 2> gpurun_out/r02bh_bench.err; echo "bench rc $?"; cat gpurun_out/r02bh_bench.json | head -c 600
timeout 2400 python tools/bench_scale.py oocloops 1536 64 6 3 > gpurun_out/r02bh_big.jsonl 2> gpurun_out/r02bh_big.err
echo "big rc $?"; cat gpurun_out/r02bh_big.jsonl; tail -3 gpurun_out/r02bh_big.err
