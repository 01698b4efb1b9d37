"""Bank-conflict model of the dock kernel's corner gathers for the current lane map
(one warp = 4 poses x 8 angle steps of one moving atom) and a search over padded grid
strides (row rs, plane ps in floats).  Conflict degree of one LDS = max over the 32 banks
of the number of DISTINCT words requested (broadcasts are free); averaged over the 8
corner loads of every sweep evaluation of a sample of C4-shaped ligands.

Result (40 ligands, 20-120 atoms): (33, 1063) 3.21, (34, 1097) 3.06, unpadded 7.5,
uniform random words 3.5.  (34, 1097) costs 4.5 KB more than (33, 1063)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from scipy.spatial.transform import Rotation

import vsgen


def passes(n=40, seed=4):
    lib = vsgen.ligands(n, seed, (20, 120))
    rot, _ = vsgen.pose_table(64)
    th = 2 * np.pi * np.arange(8) / 8
    out = []
    for i in range(lib.n):
        x, fr = lib.ligand_ranges(i)
        xc = x - x.mean(0)
        for p0 in range(0, 64, 32):
            ys = [xc @ rot[p0 + q].T.astype(np.float64) + 15.5 for q in range(4)]
            for a, b, lo, hi in fr:
                for j in range(lo, hi):
                    L = []
                    for y in ys:
                        u = (y[b] - y[a]) / np.linalg.norm(y[b] - y[a])
                        for t in th:
                            L.append(Rotation.from_rotvec(t * u).apply(y[j] - y[b]) + y[b])
                    out.append(np.floor(np.clip(np.array(L), 0, 31)).astype(np.int64))
    return np.array(out)


def cost(P, rs, ps):
    tot = 0.0
    rows = np.repeat(np.arange(len(P)), 32).reshape(len(P), 32)
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                addr = (P[:, :, 2] + dz) * ps + (P[:, :, 1] + dy) * rs + P[:, :, 0] + dx
                srt = np.sort(addr, axis=1)
                uniq = np.concatenate([np.ones((len(addr), 1), bool), srt[:, 1:] != srt[:, :-1]], axis=1)
                cnt = np.zeros((len(addr), 32), int)
                np.add.at(cnt, (rows[uniq], (srt % 32)[uniq]), 1)
                tot += cnt.max(1).mean()
    return tot / 8


if __name__ == "__main__":
    P = passes()[::2]
    print("current (34, 1097):", round(cost(P, 34, 1097), 3), " (33, 1063):", round(cost(P, 33, 1063), 3),
          " unpadded:", round(cost(P, 32, 1024), 3))
    if len(sys.argv) > 1:
        res = sorted((round(cost(P, rs, ps), 3), rs, ps) for rs in (32, 33, 34, 35, 36) for ps in range(32 * rs, 32 * rs + 40))
        print(res[:12])
