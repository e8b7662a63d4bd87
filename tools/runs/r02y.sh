timeout 600 python bench.py > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err
echo "bench rc $?"; tail -3 gpurun_out/r02y_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02y_bench_ref.json 2> gpurun_out/r02y_bench_ref.err
echo "ref rc $?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02y_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02y_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02y_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r02y_smoke.log
