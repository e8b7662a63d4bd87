timeout 600 python bench.py > gpurun_out/r02bf_bench.json 2> gpurun_out/r02bf_bench.err
echo "bench rc $?"; tail -2 gpurun_out/r02bf_bench.err
python -c "
import json;d=json.load(open('gpurun_out/r02bf_bench.json'))
print({k:d.get(k) for k in ['value','ax_gups','atb_matched_gups','atb_matched_sparse_gups','atb_fdk_gups','gpu_launches','tv_gd_gvox_iter_per_s','tv_gd_hbm_frac','tv_gd_run_gvox_iter_per_s','tv_rof_gvox_iter_per_s','tv_rof_hbm_frac','os_sart_s_per_iter','sart_tv_s_per_iter','cgls_s_per_iter','fdk_s']}, d['e2e']['value'], d['roofline']['frac'], d['config3_step']['value'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02bf_bench_ref.json 2> gpurun_out/r02bf_bench_ref.err
echo "ref rc $?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02bf_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02bf_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bf_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r02bf_smoke.log
T=r02bf; mkdir -p gpurun_out/$T
PROF_KERNELS=tv timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"march2|rof_march" -s 3 -c 3 -o gpurun_out/$T/tv python tools/prof_c2.py > gpurun_out/$T/ncu_tv.log 2>&1
echo "ncu rc $?"
