"""Does noise generation overlap the fine sweep?  Config-4 shapes
(development aid): fine sweep of 64 slices, noise of 64 slices, alone,
concurrently, and pipelined in slice batches (noise batch b+1 || sweep b)."""
import sys
import torch
sys.path.insert(0, '/root/repo')
import paper_2310_11365_b200 as mm
from paper_2310_11365_b200 import kernels
from paper_2310_11365_b200.noise import slice_noise, step_keys, fill_normals, row_pitch

N, S, P, dt = 64, 100, 100_000, 1e-3
dev = torch.device('cuda')
xa = kernels.noise_buffer(N, S, P); xa.normal_()
xb = kernels.noise_buffer(N, S, P)
x = torch.randn((N, P), dtype=torch.float64, device=dev) * 0.1 + 1.0
out = torch.empty_like(x)
t0 = torch.zeros(N, dtype=torch.float64, device=dev)
bad = torch.empty(N, dtype=torch.int32, device=dev)
model = mm.make_perturbed_ou(mm.PerturbedOUSpec(a=-1.0, a_E=0.5, B=0.5)).descriptor
lo, hi = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
keys = step_keys(0, False, 0, 0, N, S)

def fine(a=0, b=N, xi=xa):
    kernels.fine_sweep(model, x[a:b], out[a:b], t0[a:b], S, dt, xi[a:b], bad[a:b])

def noise(a=0, b=N, stream=None):
    fill_normals(keys[a * S:b * S], P, xb[a:b], row_pitch(P), stream=stream)

def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)

def concurrent(fine_first, fs, ns):
    def go():
        main = torch.cuda.current_stream()
        fs.wait_stream(main); ns.wait_stream(main)
        order = [lambda: fine_on(fs), lambda: noise(stream=ns)] if fine_first else \
                [lambda: noise(stream=ns), lambda: fine_on(fs)]
        for f in order: f()
        main.wait_stream(fs); main.wait_stream(ns)
    return go

def fine_on(s, a=0, b=N):
    with torch.cuda.stream(s):
        fine(a, b)

def pipelined(B, fs, ns):
    def go():
        main = torch.cuda.current_stream()
        fs.wait_stream(main); ns.wait_stream(main)
        for a in range(0, N, B):
            b = min(N, a + B)
            noise(a, b, stream=ns)
            ev = torch.cuda.Event(); ev.record(ns)
            fs.wait_event(ev)
            with torch.cuda.stream(fs):
                kernels.fine_sweep(model, x[a:b], out[a:b], t0[a:b], S, dt, xb[a:b], bad[a:b])
        main.wait_stream(fs); main.wait_stream(ns)
    return go

fine(); noise(); torch.cuda.synchronize()
tf, tn = timed(fine), timed(noise)
print(f'fine alone {tf:.3f} ms, noise alone {tn:.3f} ms, sum {tf + tn:.3f}', flush=True)
for ff in (True, False):
    for name, fs, ns in (('equal prio', lo, torch.cuda.Stream()), ('fine high prio', hi, lo)):
        print(f'concurrent fine_first={ff} {name}: {timed(concurrent(ff, fs, ns)):.3f} ms', flush=True)
for B in (8, 14, 16, 28, 32, 64):
    for name, fs, ns in (('equal', torch.cuda.Stream(), torch.cuda.Stream()), ('fine hi', hi, lo)):
        print(f'pipelined B={B} {name}: {timed(pipelined(B, fs, ns)):.3f} ms', flush=True)
for B in (14, 16, 32):
    print(f'noise alone in batches of {B}: {timed(lambda: [noise(a, min(N, a + B)) for a in range(0, N, B)]):.3f} ms')
