set -x
for d in 256 512 1024 2048; do
 for k in 1 auto; do
  if [ $k = auto ]; then unset CS_ST_LANE_STRIDE; else export CS_ST_LANE_STRIDE=$k; fi
  echo "stride=$k"; python tools/fine_detector.py $d
 done
done
unset CS_ST_LANE_STRIDE
for k in 2 4 8; do CS_ST_LANE_STRIDE=$k python tools/fine_detector.py 2048; done
