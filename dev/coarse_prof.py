import ctypes, os, sys
os.environ['MMPR_LIB'] = '/root/repo/dev/libmmpr_cprof.so'
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2310_11365_b200 import _lib as L
lib = L.load()
lib.mmpr_dev_coarse_prof.argtypes = [ctypes.c_void_p]
sys.argv = ['x', '512']
exec(open('/root/repo/dev/coarse_probe.py').read())
buf = np.zeros(4, dtype=np.int64)
lib.mmpr_dev_coarse_prof(buf.ctypes.data)
lib.mmpr_dev_coarse_prof(buf.ctypes.data)  # reset after warm-ups, then one more row
import torch
kernels.coarse_row(ode_d, om_d, integ, times, 1, rho0, fine, cache, macro, cout, raw, st, skip_until=1)
lib.mmpr_dev_coarse_prof(buf.ctypes.data)
print('euler cycles per call', buf[0] / max(buf[1], 1), 'calls', buf[1], 'total cycles per slice', buf[2] / 512)
