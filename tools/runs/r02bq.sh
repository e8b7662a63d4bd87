timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02bq_pytest.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/r02bq_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02bq_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/r02bq_smoke.log
timeout 600 python bench.py > gpurun_out/r02bq_bench.json 2> gpurun_out/r02bq_bench.err; echo "bench rc $?"; python -c "
import json;d=json.loads(open('gpurun_out/r02bq_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ax_gups'], d['atb_matched_gups'], d['e2e']['value'], d['sart_tv_s_per_iter'], d['os_sart_s_per_iter'], d['cgls_s_per_iter'], d['config3_step']['value'], d['clocks'])"
timeout 600 python bench.py --impl reference > gpurun_out/r02bq_bench_ref.json 2> gpurun_out/r02bq_bench_ref.err; echo "ref rc $?"; head -c 400 gpurun_out/r02bq_bench_ref.json
