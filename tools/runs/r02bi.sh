timeout 900 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/r02bi_peer.log 2>&1
echo "peer rc $?"; tail -30 gpurun_out/r02bi_peer.log
timeout 900 python -m pytest tests/test_gpu_loops.py -x -q -k "distributed or two_ranks" > gpurun_out/r02bi_loops.log 2>&1
echo "loops rc $?"; tail -5 gpurun_out/r02bi_loops.log
