"""Noise-kernel wave quantisation: time vs number of streams (development aid)."""
import sys
import torch
sys.path.insert(0, '/root/repo')
from paper_2310_11365_b200.noise import slice_noise, row_pitch
from paper_2310_11365_b200 import kernels
S, P = 100, 100_000
buf = kernels.noise_buffer(80, S, P)
for n in (4, 8, 12, 16, 20, 23, 24, 32, 40, 47, 48, 56, 64, 71, 72, 80):
    slice_noise(0, 0, n, S, P, out=buf[:n]); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); slice_noise(0, 0, n, S, P, out=buf[:n]); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    print(f'streams {n * S:5d} ({n * S / 2368:.2f} waves): {t:.3f} ms  {n * S * P / t / 1e6:.1f} G normals/s', flush=True)
