"""Dock-phase time of a C5-shaped campaign (N ligands x 4 pockets), per-pocket or fused
 launches (prints one line; not a bench value).  python tools/fused_time.py N fused"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import vsgen
from paper_2303_06150_b200 import Engine
n, fused = int(sys.argv[1]), bool(int(sys.argv[2]))
lib = vsgen.ligands(n, 4)
e = Engine(fused_sites=fused, bucket_multiple=16, n_streams=4)
e.set_poses(*vsgen.pose_table(64)); e.set_angles(vsgen.angle_table(8))
ids = [e.load_pocket(vsgen.pocket(s)) for s in (101, 102, 103, 104)]
d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
ms = []
for it in range(4):
    e.submit(*d, ids, on_device=True); e.wait()
    ms.append(e.stats()["dock_ms"])
st = e.stats()
print(f"fused={fused} cluster={os.environ.get('VSDOCK_CLUSTER', 'auto')} n={n} dock_ms={np.median(ms[1:]):.2f} "
      f"Geval/s={st['evals_alg'] / np.median(ms[1:]) / 1e6:.1f} fused_launches={st['fused_launches']} "
      f"classes={[(c['kernel_atoms'], c['warps_per_cta']) for c in e.classes()]}")
