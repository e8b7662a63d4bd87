timeout 900 python bench.py > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err
echo "bench rc $?"
cat gpurun_out/bench_r02f.json
tail -5 gpurun_out/bench_r02f.err
timeout 900 python -m pytest tests/test_gpu_loops.py -x -q -k "distributed or bench_self" > gpurun_out/r02f_pytest.log 2>&1
tail -15 gpurun_out/r02f_pytest.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02f.json 2>&1
cat gpurun_out/bench_ref_r02f.json
