"""Shared-memory bank model of the matched kernel's ATOMS:
for config-2 rays, the max bank load (wavefronts) of one corner deposit per
warp-sample for warp shapes 32x1 (production), 16x2, 8x4 and z-stride pads.

    python tools/sim_smem_banks.py
"""
import numpy as np, math
n=512; A=360; nu=nv=512
dso, dsd = 2.0*n, 4.0*n
pix = 2*math.sqrt(2)*n/nu
g0 = -n/2.0
rng = np.random.default_rng(0)
def ray_cells(th, u, v):
    src = np.array([dso*math.cos(th), dso*math.sin(th), 0.0])
    axis = np.array([math.cos(th), math.sin(th), 0.0]); uh = np.array([-math.sin(th), math.cos(th), 0.0]); vh = np.array([0,0,1.0])
    p = (dso-dsd)*axis + ((u-(nu-1)/2)*pix)*uh + ((v-(nv-1)/2)*pix)*vh
    d = p - src; d /= np.linalg.norm(d)
    t0, t1 = -1e300, 1e300
    for i in range(3):
        if d[i] != 0:
            ta, tb = (g0 - src[i])/d[i], (-g0 - src[i])/d[i]
            ta, tb = min(ta, tb), max(ta, tb)
            t0, t1 = max(t0, ta), min(t1, tb)
    if t0 >= t1: return None
    L = t1 - t0; ns = math.ceil(L/0.5); st = L/ns
    k = np.arange(ns)
    q = (src[None,:] + (t0 + (k[:,None]+0.5)*st)*d[None,:] - g0) - 0.5
    return np.floor(q).astype(int)
shapes = {"32x1": (32,1), "16x2": (16,2), "8x4": (8,4)}
res = {}
for trial in range(60):
    a = rng.integers(0, A); th = 2*math.pi*a/A
    M = 0 if abs(math.cos(th)) >= abs(math.sin(th)) else 1
    T = 1 - M
    u0 = rng.integers(100, nu - 140); v0 = rng.integers(100, nv - 140)
    for name, (wu, wv) in shapes.items():
        lanes = [ray_cells(th, u0 + du, v0 + dv) for dv in range(wv) for du in range(wu)]
        if any(c is None for c in lanes): continue
        K = min(len(c) for c in lanes)
        # box origin: min over the warp (approx.)
        allc = np.concatenate([c[:K] for c in lanes])
        lo = allc.min(0); ext = allc.max(0) - lo + 2
        for pad in range(0, 32, 4):
            if M == 1:   # [z][y][x]: x innermost, sy = ext_x padded, sz = sy*ext_y
                sx, sy = 1, ((ext[0] + 3) // 4) * 4
                sz = sy * ext[1] + pad
            else:        # [z][x][y]: y innermost, sx = ext_y | 1
                sy, sx = 1, ext[1] | 1
                sz = sx * ext[0] + pad
            wf = 0; cnt = 0
            for k in range(0, K, 3):
                addr = [ (c[k][2]-lo[2])*sz + (c[k][1]-lo[1])*sy + (c[k][0]-lo[0])*sx for c in lanes]
                # wavefronts = max over banks of distinct addresses in that bank (same-address atomics also serialize: count all)
                banks = {}
                for ad in addr: banks.setdefault(ad % 32, []).append(ad)
                wf += max(len(v) for v in banks.values()); cnt += 1
            res.setdefault((name, pad), []).append(wf / cnt)
for (name, pad), v in sorted(res.items()):
    print(name, "pad", pad, round(float(np.mean(v)), 2))
