"""Texture quad-slot model of the Ax kernel: for warps
of 8u x 4v rays on the config-2 geometry (fp64 sample cells), count per
quad (4 consecutive lanes) the tld4 instructions that have at least one
active lane -- the measured cost unit of the texture pipe
(tools/micro/fetch_rates.cu, modes 15-17) -- for the production z-layered
kernel and for a main-axis-layered variant.

    python tools/sim_tex_quads.py
"""
import numpy as np, math
n=512; A=360; nu=nv=512
dso, dsd = 2.0*n, 4.0*n
pix = 2*math.sqrt(2)*n/nu
g0 = -n/2.0
rng = np.random.default_rng(0)
cur_tot = 0; new_tot = 0; samp_tot = 0
for trial in range(200):
    a = rng.integers(0, A); th = 2*math.pi*a/A
    src = np.array([dso*math.cos(th), dso*math.sin(th), 0.0])
    axis = np.array([math.cos(th), math.sin(th), 0.0]); uh = np.array([-math.sin(th), math.cos(th), 0.0]); vh = np.array([0,0,1.0])
    M = 0 if abs(math.cos(th)) >= abs(math.sin(th)) else 1
    T = 1 - M
    # a warp: 8u x 4v tile; quads = 4 consecutive u in a row
    u0 = rng.integers(0, nu - 8); v0 = rng.integers(0, nv - 4)
    cells = []; lens = []
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
            if t0 >= t1:
                cells.append(None); continue
            L = t1 - t0; ns = math.ceil(L/0.5); st = L/ns
            k = np.arange(ns)
            q = (src[None,:] + (t0 + (k[:,None]+0.5)*st)*d[None,:] - g0) - 0.5
            cells.append(np.floor(q).astype(int))
    if all(c is None for c in cells): continue
    K = max(len(c) for c in cells if c is not None)
    # per lane per step: change flags
    cur = 0; new = 0; samples = 0
    for quad in range(8):
        lanes = [cells[(quad // 2) * 8 + (quad % 2) * 4 + j] for j in range(4)]
        anyc = np.zeros(K, bool); anyM = np.zeros(K, bool); anyTZ = np.zeros(K, bool)
        for c in lanes:
            if c is None: continue
            samples += len(c)
            ch = np.ones(len(c), bool); ch[1:] = np.any(c[1:] != c[:-1], axis=1)
            tz = np.ones(len(c), bool); tz[1:] = (c[1:, T] != c[:-1, T]) | (c[1:, 2] != c[:-1, 2])
            anyc[:len(c)] |= ch
            anyTZ[:len(c)] |= tz
            anyM[:len(c)] |= ch & ~tz
        cur += 2 * anyc.sum()
        new += (anyc).sum() + anyTZ.sum()
    cur_tot += cur; new_tot += new; samp_tot += samples
print("quad-slots per ray-sample: current", cur_tot / samp_tot * 4, " x-layered", new_tot / samp_tot * 4, " ratio", new_tot / cur_tot)
