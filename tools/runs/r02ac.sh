timeout 600 python bench.py > gpurun_out/r02ac_bench.json 2> gpurun_out/r02ac_bench.err
echo "bench rc $?"; tail -2 gpurun_out/r02ac_bench.err
python -c "
import json;d=json.load(open('gpurun_out/r02ac_bench.json'))
print({k:d.get(k) for k in ['value','ax_gups','atb_matched_gups','atb_matched_sparse_gups','gpu_launches']}, d['e2e']['value'], d['roofline']['frac'], d['config3_step']['value'])"
T=r02ac; mkdir -p gpurun_out/$T
PROF_KERNELS=matched timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"staged|transpose_add" -s 2 -c 2 -o gpurun_out/$T/full python tools/prof_c2.py > gpurun_out/$T/ncu_full.log 2>&1
echo "ncu rc $?"
