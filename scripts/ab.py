import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2206_01683_b200._abi as abi
abi.LIB_PATH = abi.LIB_PATH.replace('libfsg.so', sys.argv[1])
import cases as K
c = K.case_session_frame(); c['script'] = [("step", 0)]
o = K.run_oracle_session(c); g = K.run_gpu_session(c, "fp64")
d = np.abs(g['fw'] - o['fw']).reshape(-1, 3).max(1)
print(sys.argv[1], 'maxdiff', d.max(), 'bad', int((d > 0).sum()))
