"""Time the dock phase for an N-ligand C4-shaped library (prints one line; not a bench value)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import vsgen
from paper_2303_06150_b200 import Engine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
na, nr = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (6, 23)
ATOMS = tuple(int(x) for x in os.environ.get("ATOMS", "20,120").split(","))
lib = vsgen.ligands(n, 4, ATOMS)
e = Engine(atom_clusters=na, rot_clusters=nr, launch_per_bucket=bool(int(os.environ.get("LPB", "0"))), bucket_multiple=int(os.environ.get("BM", "16")), n_streams=int(os.environ.get("NS", "4")))
T = int(os.environ.get("TYPED", "0"))   # > 0: typed submit with T atom types (Q24)
e.set_poses(*vsgen.pose_table(64)); e.set_angles(vsgen.angle_table(8))
pid = e.load_pocket(vsgen.typed_pocket(101, n_types=T) if T else vsgen.pocket(101))
import torch
d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
ty = torch.from_numpy(vsgen.atom_types(lib, n_types=T)).cuda() if T else None
ms = []
for it in range(4):
    e.submit(*d, [pid], on_device=True, atom_type=ty); e.wait()
    ms.append(e.stats()["dock_ms"])
st = e.stats()
print(f"{os.environ.get('TAG','')} n={n} grid={na}x{nr} dock_ms={np.median(ms[1:]):.2f} prep_ms={st['prep_ms']:.2f} "
      f"Geval/s={st['evals_alg']/np.median(ms[1:])/1e6:.1f} lig/s={n/np.median(ms[1:])*1e3:.3e} launches={st['dock_launches']} "
      f"classes={[(c['kernel_atoms'], c['warps_per_cta'], c['ligands_per_cta']) for c in e.classes()]}")
r = e.results(0)
np.save(f"gpurun_out/scores_{os.environ.get('TAG','x')}.npy", r.best_score)
