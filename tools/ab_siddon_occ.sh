for v in . sid8 sid12 sid16; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so python tools/ab_siddon_dda.py "dda $v" /tmp/s_$v.npy
done
