"""Quick GPU probe of libmmpr kernels vs numpy (development aid)."""
import ctypes, math, sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2310_11365_b200 import _lib as L

lib = L.load()
print(lib.mmpr_version().decode())
dev = torch.device('cuda')
st = L.stream_handle()

def words_of(entropy):
    w = []
    for v in entropy:
        v = int(v)
        if v == 0: w.append(0)
        while v > 0: w.append(v & 0xffffffff); v >>= 32
    return np.array(w, dtype=np.uint32)

# ---- keys
seed = 20240601
keys = torch.zeros((3, 5, 2), dtype=torch.int64, device=dev)
L.call('mmpr_noise_keys', seed, 0, 0, 2, 3, 5, keys.data_ptr(), st)
kh = keys.cpu().numpy().view(np.uint64)
ok = True
for a in range(3):
    for j in range(5):
        ref = np.random.SeedSequence((seed, 1, 2 + a, j)).generate_state(2, np.uint64)
        ok &= np.array_equal(ref, kh[a, j])
print('keys frozen ok', ok)
L.call('mmpr_noise_keys', seed, 1, 7, 2, 3, 5, keys.data_ptr(), st)
kh = keys.cpu().numpy().view(np.uint64)
ok = all(np.array_equal(np.random.SeedSequence((seed, 2, 2 + a, j, 7)).generate_state(2, np.uint64), kh[a, j]) for a in range(3) for j in range(5))
print('keys fresh ok', ok)

# ---- normals
P = 100000
nst = 15
out = torch.zeros((nst, P), dtype=torch.float64, device=dev)
L.call('mmpr_noise_keys', seed, 0, 0, 0, 3, 5, keys.data_ptr(), st)
L.call('mmpr_normals_fill', keys.data_ptr(), nst, P, out.data_ptr(), P, 0, 0.0, 1.0, st)
o = out.cpu().numpy()
bad = 0; tails = 0; maxulp = 0
for a in range(3):
    for j in range(5):
        ref = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, 1, a, j)))).standard_normal(P)
        got = o[a * 5 + j]
        d = got != ref
        bad += d.sum(); tails += (np.abs(ref) > 3.6541528853610087).sum()
        if d.any():
            maxulp = max(maxulp, np.max(np.abs(got[d] - ref[d]) / np.spacing(np.abs(ref[d]))))
            print('  stream', a, j, 'mismatch idx', np.nonzero(d)[0][:5], got[d][:3], ref[d][:3])
print('normals mismatches', bad, 'of', nst * P, 'tails', tails, 'max ulp', maxulp)

# entropy key + affine (sample_initial normal(1.0, 0.01))
w = words_of((0, 0))
key1 = torch.zeros(2, dtype=torch.int64, device=dev)
L.call('mmpr_entropy_key', w.ctypes.data, len(w), key1.data_ptr(), st)
x0 = torch.zeros(10000, dtype=torch.float64, device=dev)
L.call('mmpr_normals_fill', key1.data_ptr(), 1, 10000, x0.data_ptr(), 10000, 1, 1.0, math.sqrt(0.01), st)
ref0 = np.random.Generator(np.random.Philox(np.random.SeedSequence((0, 0)))).normal(1.0, math.sqrt(0.01), 10000)
print('init sample equal', np.array_equal(x0.cpu().numpy(), ref0))

# ---- fine sweep (OU) with numpy-exact injected noise
def ref_fine(x, xi, a, aE, B, dt):
    sq = math.sqrt(dt)
    for j in range(xi.shape[0]):
        s = float(np.mean(x))
        x = x + (a * x + aE * s) * dt + np.full_like(x, B) * sq * xi[j]
    return x

for P, S, nsl in [(7, 5, 2), (100, 5, 2), (1000, 10, 3), (10000, 20, 3), (100000, 20, 2), (12345, 7, 2)]:
    pitch = P + (P & 1)
    rng = np.random.default_rng(P)
    xin = rng.normal(1.0, 0.1, (nsl, P))
    xi = rng.standard_normal((nsl, S, P))
    xi_d = torch.zeros((nsl, S, pitch), dtype=torch.float64, device=dev)
    xi_d[:, :, :P] = torch.from_numpy(xi)
    xin_d = torch.from_numpy(xin).to(dev)
    xout_d = torch.zeros_like(xin_d)
    bad = torch.zeros(nsl, dtype=torch.int32, device=dev)
    fm = torch.zeros(nsl, dtype=torch.float64, device=dev)
    t0 = torch.zeros(nsl, dtype=torch.float64, device=dev)
    model = L.Model(); model.kind = L.MODEL_OU; model.stat_kind = 0
    model.p[0] = -1.0; model.p[1] = 0.5; model.p[2] = 0.5
    dt = 1e-3
    L.call('mmpr_fine_sweep', ctypes.byref(model), nsl, P, S, dt, math.sqrt(dt), t0.data_ptr(), xin_d.data_ptr(), P,
           xout_d.data_ptr(), P, xi_d.data_ptr(), S * pitch, pitch, bad.data_ptr(), fm.data_ptr(), st)
    torch.cuda.synchronize()
    got = xout_d.cpu().numpy()
    eq = all(np.array_equal(got[s], ref_fine(xin[s], xi[s], -1.0, 0.5, 0.5, dt)) for s in range(nsl))
    fmeq = all(fm.cpu().numpy()[s] == np.mean(got[s]) for s in range(nsl))
    print('fine P', P, 'bitwise', eq, 'final mean', fmeq, 'bad', bad.cpu().numpy())

clusters = ctypes.c_int32(0); ctas = ctypes.c_int32(0)
for P in [10000, 100000]:
    L.call('mmpr_fine_sweep_occupancy', P, ctypes.byref(clusters), ctypes.byref(ctas))
    print('occupancy P', P, 'ctas/slice', ctas.value, 'max active clusters', clusters.value)

# ---- timings (C4-like)
N, S, P = 64, 100, 100000
pitch = P
keys = torch.zeros((N, S, 2), dtype=torch.int64, device=dev)
xi_d = torch.empty((N, S, pitch), dtype=torch.float64, device=dev)
L.call('mmpr_noise_keys', 0, 0, 0, 0, N, S, keys.data_ptr(), st)
for it in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    L.call('mmpr_normals_fill', keys.data_ptr(), N * S, P, xi_d.data_ptr(), pitch, 0, 0.0, 1.0, st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f'noise fill {N*S*P/1e6:.0f}M normals: {ms:.3f} ms -> {N*S*P/ms/1e9:.3f} Gnormals/s')
xin_d = torch.randn((N, P), dtype=torch.float64, device=dev)
xout_d = torch.empty_like(xin_d)
bad = torch.zeros(N, dtype=torch.int32, device=dev); t0 = torch.zeros(N, dtype=torch.float64, device=dev)
for it in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    L.call('mmpr_fine_sweep', ctypes.byref(model), N, P, S, 1e-3, math.sqrt(1e-3), t0.data_ptr(), xin_d.data_ptr(), P,
           xout_d.data_ptr(), P, xi_d.data_ptr(), S * pitch, pitch, bad.data_ptr(), None, st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    byts = N * S * P * 8 + 2 * N * P * 8
    print(f'fine sweep {N}x{P}x{S}: {ms:.3f} ms -> {N*S*P/ms/1e9:.1f} G p-steps/s, {byts/ms/1e6:.0f} GB/s')
# spot check the first slice vs numpy for the big case
xh = xin_d[0].cpu().numpy(); xih = xi_d[0].cpu().numpy()
print('C4 slice0 bitwise', np.array_equal(ref_fine(xh, xih, -1.0, 0.5, 0.5, 1e-3), xout_d[0].cpu().numpy()))
