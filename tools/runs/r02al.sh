timeout 600 python bench.py > gpurun_out/r02al_bench.json 2> gpurun_out/r02al_bench.err
echo "bench rc $?"; tail -2 gpurun_out/r02al_bench.err
python -c "
import json;d=json.load(open('gpurun_out/r02al_bench.json'))
print({k:d.get(k) for k in ['value','ax_gups','atb_matched_gups','atb_matched_sparse_gups','gpu_launches','tv_gd_run_gvox_iter_per_s','tv_rof_gvox_iter_per_s','os_sart_s_per_iter','cgls_s_per_iter']}, d['e2e']['value'], d['roofline']['frac'], d['config3_step']['value'], d['config3_step']['atb_matched_gups'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02al_bench_ref.json 2> gpurun_out/r02al_bench_ref.err
echo "ref rc $?"
