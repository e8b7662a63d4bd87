timeout 900 python -m pytest tests/test_gpu_determinism.py -x -q > gpurun_out/r02bk_det.log 2>&1
echo "det rc $?"; tail -15 gpurun_out/r02bk_det.log
for d in 0 1; do
for n in 512 1024; do
CS_ST_DETERMINISTIC=$d PROF_N=$n PROF_A=180 PROF_ONLY=matched_dense,matched timeout 600 python tools/time_kernels.py > gpurun_out/r02bk_t_${d}_${n}.json 2>&1
echo "det=$d n=$n: $(tail -1 gpurun_out/r02bk_t_${d}_${n}.json)"
done; done
