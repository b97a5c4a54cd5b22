import os, sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2310_11365_b200 import _lib as L, kernels, noise
L.load()
N, S, P = 64, 100, 100000
xi = kernels.noise_buffer(N, S, P)
keys = noise.step_keys(0, False, 0, 0, N, S)
ts = []
for _ in range(4):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); noise.fill_normals(keys, P, xi, xi.stride(1)); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(os.environ.get('MMPR_LIB', 'default'), 'noise fill ms', [round(t, 3) for t in ts], f'{N*S*P/min(ts)/1e6:.1f} Gnormals/s')
# spot-check two streams vs numpy
for (n, j) in [(0, 0), (63, 99), (17, 42)]:
    ref = np.random.Generator(np.random.Philox(np.random.SeedSequence((0, 1, n, j)))).standard_normal(P)
    got = xi[n, j, :P].cpu().numpy()
    d = got != ref
    print(' stream', n, j, 'mismatch', int(d.sum()), 'all tails' if np.all(np.abs(ref[d]) > 3.654) else 'NON-TAIL MISMATCH')
