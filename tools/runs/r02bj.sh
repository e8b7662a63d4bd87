A="--steps 4 --warmup 3 --c3-size 1024 --c3-angles 256 --c3-block 64"
for m in peer nccl; do
CS_BENCH_BACKEND=gloo CS_EXCHANGE=$m timeout 900 python bench.py --gpus 2 $A > gpurun_out/r02bj_2r_$m.json 2> gpurun_out/r02bj_2r_$m.err
echo "2 ranks $m rc $?"; head -c 1500 gpurun_out/r02bj_2r_$m.json; echo
done
timeout 900 python bench.py --gpus 1 --no-extras $A > gpurun_out/r02bj_1r.json 2> gpurun_out/r02bj_1r.err
echo "1 rank rc $?"; python -c "
import json; d=json.loads(open('gpurun_out/r02bj_1r.json').read().strip().splitlines()[-1]); print(json.dumps(d.get('config3_step', {}))[:1200])"
