"""Small driver for ncu: one bucketed submit of an N-ligand C4-shaped library (not a bench value)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import vsgen
from paper_2303_06150_b200 import Engine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
na, nr = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (6, 23)
lib = vsgen.ligands(n, 4)
e = Engine(atom_clusters=na, rot_clusters=nr)
e.set_poses(*vsgen.pose_table(64)); e.set_angles(vsgen.angle_table(8)); pid = e.load_pocket(vsgen.pocket(101))
for _ in range(2):
    e.submit_library(lib, [pid]); e.wait()
print(e.stats())
