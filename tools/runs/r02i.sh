# baseline of the restored tree: full GPU suite + bench
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_pytest.log 2>&1
echo "pytest rc $?"; tail -5 gpurun_out/r02i_pytest.log
timeout 600 python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
echo "bench rc $?"; cat gpurun_out/r02i_bench.json | head -c 600
