timeout 900 python -m pytest tests/test_gpu_determinism.py -x -q > gpurun_out/r02bo_det.log 2>&1
echo "det rc $?"; tail -2 gpurun_out/r02bo_det.log
timeout 600 python bench.py --no-extras --no-c3 > gpurun_out/r02bo_bench.json 2> gpurun_out/r02bo_bench.err; echo "bench rc $?"; python -c "
import json;d=json.loads(open('gpurun_out/r02bo_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ax_gups'], d['atb_matched_gups'], d['clocks'])"
for d in 0 1; do CS_ST_DETERMINISTIC=$d PROF_N=512 PROF_A=180 PROF_ONLY=matched_dense timeout 600 python tools/time_kernels.py 2>&1 | tail -1; done
