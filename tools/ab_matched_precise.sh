bash tools/ab_lib.sh gpurun_out/ab/pw.jsonl matched,matched_dense . pw2 pw3
for v in pw2 pw3; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so timeout 700 python tools/fuzz_loops.py 25 3 > gpurun_out/ab/fzl_$v.log 2>/dev/null
done
