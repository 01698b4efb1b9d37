"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck); SURVEY.md 5 race
detection row, VERDICT r1 "missing" 7.  Usage: python tools/sanitize_case.py <case>

  c1      C1 (16 ligands, 32^3 FIX grid, P = 8, K = 8): every prep / dock / finalize / top-k kernel
  edge    a 14^3 grid (atoms on and beyond the faces: the top-face corner handling) + K = 6
  ring    launch_per_bucket with bucket capacity 1 on 8 streams: many tiny launches of the round ring
  win     a 48^3 grid at 0.5 A (WIN mode: window + global corners)
Exits non-zero if the results are not finite (the sanitizer's own report is the evidence)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import vsgen
from paper_2303_06150_b200 import Engine


def run(lib, pk, P=8, K=8, **kw):
    e = Engine(**kw)
    rot, tr = vsgen.pose_table(P, tau=1.0)
    e.set_poses(rot, tr)
    e.set_angles(vsgen.angle_table(K))
    pid = e.load_pocket(pk)
    e.submit_library(lib, [pid])
    e.wait()
    r = e.results(0)
    xyz = e.coords(0)
    keys, nv = e.local_topk(0, 8)
    idx, sc = e.merge_topk(keys[:nv], 8)
    assert np.isfinite(r.best_score).all() and np.isfinite(xyz).all() and len(idx) == min(8, lib.n)
    e.close()


case = sys.argv[1] if len(sys.argv) > 1 else "c1"
if case == "c1":
    run(vsgen.ligands(16, 1, (20, 40), (0, 4)), vsgen.pocket(101))
elif case == "edge":
    run(vsgen.ligands(12, 17, (40, 90), (2, 10)), vsgen.pocket(106, n=14), K=6)
elif case == "ring":
    run(vsgen.ligands(40, 9, (20, 60), (0, 6)), vsgen.pocket(101), P=30, launch_per_bucket=True, bucket_capacity=1,
        n_streams=8)
elif case == "win":
    run(vsgen.ligands(12, 5, (20, 90), (0, 8)), vsgen.pocket(108, n=48, spacing=0.5))
else:
    raise SystemExit(f"unknown case {case}")
print("case", case, "ok")
