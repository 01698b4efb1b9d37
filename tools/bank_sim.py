"""Offline shared-memory bank-conflict model for the dock kernel's grid gathers.
Lane map as in dock.cu: lane = j*K + k (4 atoms x 8 angles per pass).  For each pass,
each of the 8 corner LDS costs max over banks of #distinct addresses (active lanes)."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import vsgen
from scipy.spatial.transform import Rotation

lib = vsgen.ligands(300, 4)
pk = vsgen.pocket(101)
rot, _ = vsgen.pose_table(8)
K = 8
cs = vsgen.angle_table(K)
th = np.arctan2(cs[:, 1], cs[:, 0])

def passes():
    out = []
    for i in range(lib.n):
        x, fr = lib.ligand(i)
        xc = x - x.mean(0)
        for p in range(0, 8, 3):
            y = xc @ rot[p].T.astype(np.float64) + 15.5
            for f in fr:
                a, b, lo, hi = f
                u = (y[b] - y[a]); u /= np.linalg.norm(u)
                R = [Rotation.from_rotvec(t * u) for t in th]
                for base in range(lo, hi, 4):
                    lanes = []
                    for jl in range(4):
                        j = base + jl
                        if j >= hi: continue
                        for k in range(K):
                            lanes.append(R[k].apply(y[j] - y[b]) + y[b])
                    out.append(np.array(lanes))
    return out

P = passes()
print("passes", len(P), "mean active lanes", np.mean([len(l) for l in P]))

def cost(rs, ps, swz=None):
    tot = 0
    for L in P:
        c = np.clip(L, 0, 31)
        i0 = np.minimum(np.floor(c), 30).astype(int)
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    x, yy, z = i0[:, 0] + dx, i0[:, 1] + dy, i0[:, 2] + dz
                    addr = z * ps + yy * rs + x if swz is None else swz(x, yy, z)
                    bank = addr % 32
                    mx = 0
                    for bk in np.unique(bank):
                        mx = max(mx, len(np.unique(addr[bank == bk])))
                    tot += mx
    return tot / (8 * len(P))

for rs, ps in [(32, 1024), (33, 33 * 32), (33, 33 * 32 + 8), (32, 1024 + 4), (32, 1024 + 8), (36, 36 * 32 + 16), (40, 40*32+8), (33, 33*32+16), (34, 34*32+4), (37, 37*32+3)]:
    print(rs, ps, round(cost(rs, ps), 3), "KB", ps * 32 * 4 / 1024)

if len(sys.argv) > 1:
    sub = P[::4]
    P[:] = sub
    best = []
    for rs in range(32, 38):
        for d in range(0, 33):
            ps = rs * 32 + d
            best.append((cost(rs, ps), rs, ps))
    best.sort()
    for b in best[:12]:
        print("search", b, ps * 32 * 4 / 1024)
