timeout 900 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/r02bl_peer.log 2>&1
echo "peer rc $?"; tail -5 gpurun_out/r02bl_peer.log; grep -i "warn" gpurun_out/r02bl_peer.log | head
timeout 900 python -m pytest tests/test_gpu_loops.py -x -q -k "distributed or two_ranks" > gpurun_out/r02bl_loops.log 2>&1
echo "loops rc $?"; tail -3 gpurun_out/r02bl_loops.log
