"""Bank-conflict model for the PPW=4 lane map: lanes = 4 poses x 8 angles of one moving atom."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import vsgen
from scipy.spatial.transform import Rotation
lib = vsgen.ligands(200, 4, (20, 64))
rot, _ = vsgen.pose_table(64)
K = 8
th = 2 * np.pi * np.arange(K) / K
passes = []
for i in range(lib.n):
    x, fr = lib.ligand(i)
    xc = x - x.mean(0)
    for p0 in range(0, 64, 16):
        ys = [xc @ rot[p0 + q].T.astype(np.float64) + 15.5 for q in range(4)]
        for f in fr:
            a, b, lo, hi = f
            for j in range(lo, hi):
                lanes = []
                for y in ys:
                    u = (y[b] - y[a]); u /= np.linalg.norm(u)
                    for t in th:
                        lanes.append(Rotation.from_rotvec(t * u).apply(y[j] - y[b]) + y[b])
                passes.append(np.array(lanes))
print("passes", len(passes))
def cost(rs, ps):
    tot = 0
    for L in passes[::3]:
        i0 = np.minimum(np.floor(np.clip(L, 0, 31)), 30).astype(int)
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    addr = (i0[:, 2] + dz) * ps + (i0[:, 1] + dy) * rs + i0[:, 0] + dx
                    bank = addr % 32
                    tot += max(len(np.unique(addr[bank == b])) for b in np.unique(bank))
    return tot / (8 * len(passes[::3]))
res = []
for rs in (32, 33, 34, 35, 36):
    for d in range(0, 33):
        res.append((round(cost(rs, rs * 32 + d), 3), rs, rs * 32 + d))
res.sort()
print(res[:8])
print("current", cost(33, 1063), "unpadded", cost(32, 1024))
