import sys; sys.path.insert(0, "/root/repo")
import vsgen, numpy as np
from paper_2303_06150_b200 import Engine
lib = vsgen.ligands(200000, 4, (20, 120), (0, 20))
for S in (2, 3, 4, 8):
    pks = [vsgen.pocket(101 + q) for q in range(S)]
    for fused in (True, False):
        e = Engine(fused_sites=fused)
        rot, tr = vsgen.pose_table(64); e.set_poses(rot, tr); e.set_angles(vsgen.angle_table(8))
        ids = [e.load_pocket(p) for p in pks]
        ms = []
        for it in range(3):
            e.submit_library(lib, ids); e.wait(); ms.append(e.stats()["dock_ms"])
        st = e.stats()
        print(S, "fused" if fused else "per-pocket", "dock_ms", round(np.median(ms[1:]), 2), "launches", st["dock_launches"], "fused", st["fused_launches"], "lig-pockets/s %.3e" % (lib.n * S / np.median(ms[1:]) * 1e3))
        e.close()
