# deterministic matched with the transposed frame: tests + timing
timeout 900 python -m pytest tests/test_gpu_determinism.py -x -q > gpurun_out/r02cd_det.log 2>&1
echo "det rc $?"; tail -5 gpurun_out/r02cd_det.log
for t in 1 0; do
for n in 512 1024; do
CS_ST_DETERMINISTIC=1 CS_ST_TRANSPOSE=$t PROF_N=$n PROF_A=180 PROF_ONLY=matched_dense,matched TAG="det=1 transpose=$t n$n A180" timeout 600 python tools/time_kernels.py > gpurun_out/r02cd_t_${t}_${n}.json 2>&1
echo "$(tail -1 gpurun_out/r02cd_t_${t}_${n}.json)"
done; done
