python tools/ab_siddon_dda.py base /tmp/sb.npy
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/dda/libconesplit_b200.so python tools/ab_siddon_dda.py dda /tmp/sd.npy
python -c "
import numpy as np
a=np.load('/tmp/sb.npy'); b=np.load('/tmp/sd.npy')
print('relL2 dda vs base', float(np.linalg.norm((a-b).ravel())/np.linalg.norm(a.ravel())), 'maxabs', float(np.abs(a-b).max()))
"
CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/dda/libconesplit_b200.so python -m pytest tests -m gpu -x -q 2>&1 | tail -3
