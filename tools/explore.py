"""Scratch exploration on the GPU box: smoke, C2 parity stats, timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__ as g
g.smoke()
import vsgen, oracle
from oracle import parity
from paper_2303_06150_b200 import Engine
c = vsgen.CONFIGS["C2"]
t = time.time(); lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"]); print("gen C2", time.time() - t, "cpus", os.cpu_count())
pk = vsgen.pocket(101); rot, tr = vsgen.pose_table(64); cs = vsgen.angle_table(8)
res = {}
for name, (na, nr) in {"bucketed": (6, 23), "unsorted": (1, 1)}.items():
    eng = Engine(atom_clusters=na, rot_clusters=nr, debug_poses=(name == "bucketed"))
    eng.set_poses(rot, tr); eng.set_angles(cs); pid = eng.load_pocket(pk)
    for it in range(3):
        t = time.time(); eng.submit_library(lib, [pid]); eng.wait(); dt = time.time() - t
        st = eng.stats()
        print(name, "wall", dt, "prep_ms", st["prep_ms"], "dock_ms", st["dock_ms"], "launches", st["kernel_launches"], "buckets", st["n_buckets"], "evals", st["evals_alg"], "Geval/s", st["evals_alg"] / st["dock_ms"] / 1e6)
    r = eng.results(0)
    res[name] = r
    print(eng.classes())
    if name == "bucketed":
        xyz = eng.coords(0)
        ps, pa = eng.pose_debug(0)
        rng = np.random.default_rng(0)
        idx = rng.choice(lib.n, 60, replace=False)
        t = time.time()
        rep = parity.check(lib, idx, pk, rot, tr, cs, r.best_score, r.best_pose, r.angles, xyz, ps, pa)
        print("parity", rep.summary(), time.time() - t)
        for f in rep.failures[:10]: print("  ", f)
print("bucketed==unsorted scores", np.array_equal(res["bucketed"].best_score, res["unsorted"].best_score),
      np.array_equal(res["bucketed"].angles, res["unsorted"].angles))
# throughput at larger scale
t = time.time(); big = vsgen.ligands(200_000, 4); print("gen 200k", time.time() - t)
eng = Engine()
eng.set_poses(rot, tr); eng.set_angles(cs); pid = eng.load_pocket(pk)
for it in range(3):
    t = time.time(); eng.submit_library(big, [pid]); eng.wait(); dt = time.time() - t
    st = eng.stats()
    print("200k wall", dt, "prep_ms", st["prep_ms"], "dock_ms", st["dock_ms"], "lig/s", 200000 / st["dock_ms"] * 1e3, "Geval/s", st["evals_alg"] / st["dock_ms"] / 1e6, "launches", st["dock_launches"])
