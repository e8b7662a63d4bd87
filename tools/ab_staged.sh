# A/B of the staged matched kernel's chunk depth / box budget (variant
# libraries built by paper_1905_03748_b200.build with -DCS_ST_S=..)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
L=$PWD/paper_1905_03748_b200/_lib
run() { CS_LIB_PATH=$1 CS_STAGED_SMEM_KB=$2 PROF_ONLY=matched,matched_dense TAG=$3 timeout 300 python tools/time_kernels.py >> gpurun_out/ab/staged.jsonl 2>> gpurun_out/ab/staged.err; }
run $L/libconesplit_b200.so 64 s8_64k
run $L/libconesplit_b200.so 48 s8_48k
run $L/s12/libconesplit_b200.so 64 s12_64k
run $L/s16/libconesplit_b200.so 64 s16_64k
run $L/s16/libconesplit_b200.so 96 s16_96k
run $L/s12/libconesplit_b200.so 96 s12_96k
