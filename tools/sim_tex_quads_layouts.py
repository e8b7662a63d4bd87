"""Texture quad-slot model of the Ax layouts: per quad
(4 lanes) and tld4 instruction, the number of distinct layers among the
lanes that re-gather, for u- or v-adjacent quads on z- or main-axis layers
(cur = production r01h, m2_v = main-axis layers with v-adjacent quads,
ml_v = the same plus one-layer M-step reuse).

    python tools/sim_tex_quads_layouts.py [warps]
"""
import numpy as np, math, sys
n=512; A=360; nu=nv=512
dso, dsd = 2.0*n, 4.0*n
pix = 2*math.sqrt(2)*n/nu
g0 = -n/2.0
rng = np.random.default_rng(0)
tot = {"cur":0, "zl_v":0, "ml_u":0, "ml_v":0, "m2_v":0}; samp_tot=0
def rays(th, u0, v0):
    src = np.array([dso*math.cos(th), dso*math.sin(th), 0.0])
    axis = np.array([math.cos(th), math.sin(th), 0.0]); uh = np.array([-math.sin(th), math.cos(th), 0.0]); vh = np.array([0,0,1.0])
    out = {}
    for dv in range(4):
        for du in range(8):
            u, v = u0 + du, v0 + dv
            p = (dso-dsd)*axis + ((u-(nu-1)/2)*pix)*uh + ((v-(nv-1)/2)*pix)*vh
            d = p - src; d /= np.linalg.norm(d)
            t0, t1 = -1e300, 1e300
            for i in range(3):
                if d[i] != 0:
                    ta, tb = (g0 - src[i])/d[i], (-g0 - src[i])/d[i]
                    ta, tb = min(ta, tb), max(ta, tb)
                    t0, t1 = max(t0, ta), min(t1, tb)
            if t0 >= t1: out[(du,dv)] = None; continue
            L = t1 - t0; ns = math.ceil(L/0.5); st = L/ns
            k = np.arange(ns)
            q = (src[None,:] + (t0 + (k[:,None]+0.5)*st)*d[None,:] - g0) - 0.5
            out[(du,dv)] = np.floor(q).astype(int)
    return out
def cost(quads, M, K, mode):
    # mode 'z': z-layered, both tld4 when any cell change; layer = iz (and iz+1)
    # mode 'm': main-axis layered; G1 when any change (layer: new M layer), G2 when T/z change
    c = 0
    T = 1 - M
    for lanes in quads:
        for kk in range(K):
            g1 = set(); g2 = set()
            for cl in lanes:
                if cl is None or kk >= len(cl): continue
                cell = cl[kk]; prev = cl[kk-1] if kk > 0 else None
                if prev is None or np.any(cell != prev):
                    if mode == 'z':
                        g1.add(cell[2]); g2.add(cell[2]+1)
                    elif mode == 'm2':
                        g1.add(cell[M]); g2.add(cell[M]+1)
                    elif False:
                        g1.add(cell[2]); g2.add(cell[2]+1)
                    else:
                        full = prev is None or cell[T] != prev[T] or cell[2] != prev[2] or abs(cell[M]-prev[M]) > 1
                        if full:
                            g1.add(cell[M]); g2.add(cell[M]+1)
                        else:
                            g1.add(cell[M] + (1 if cell[M] > prev[M] else 0))
            c += len(g1) + len(g2)
    return c
for trial in range(int(sys.argv[1]) if len(sys.argv)>1 else 60):
    a = rng.integers(0, A); th = 2*math.pi*a/A
    M = 0 if abs(math.cos(th)) >= abs(math.sin(th)) else 1
    u0 = rng.integers(0, nu - 8); v0 = rng.integers(0, nv - 4)
    R = rays(th, u0, v0)
    if all(c is None for c in R.values()): continue
    K = max(len(c) for c in R.values() if c is not None)
    uq = [[R[(4*(qi%2)+j, qi//2)] for j in range(4)] for qi in range(8)]
    vq = [[R[(qi, j)] for j in range(4)] for qi in range(8)]
    samp_tot += sum(len(c) for c in R.values() if c is not None)
    tot["cur"] += cost(uq, M, K, 'z'); tot["zl_v"] += cost(vq, M, K, 'z')
    tot["ml_u"] += cost(uq, M, K, 'm'); tot["ml_v"] += cost(vq, M, K, 'm'); tot["m2_v"] += cost(vq, M, K, 'm2')
print({k: round(v/samp_tot, 4) for k, v in tot.items()}, "(layer-slots per ray-sample, counting distinct layers per quad)")
