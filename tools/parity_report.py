"""Parity at scale (not a bench value): the CUDA path through the C-ABI against the fp64
oracle (oracle/parity.py) on every BASELINE config, far beyond the pytest samples.

  C1: all 16 ligands, every pose replayed         C2: all 10,000 ligands, every pose replayed
  C3: all 8,192 ligands (best pose + independent) C4: every 100th of 1M (10,000 ligands)
  C5: every 500th of 1M for each of the 4 pockets
  (DENSE=1: C3 every pose replayed, C4 every 10th ligand, C5 every 100th per pocket)
  variants: C2 typed (4 atom types, typed pocket, Q24) every ligand and pose replayed; C2 with rigid
  refinement (Q23, 2 rounds of the 13-move table) every 5th ligand, every pose replayed

Writes gpurun_out/parity_report.json (one summary per config)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import vsgen
from oracle import parity
from paper_2303_06150_b200 import Engine

BAND, TOL_S, TOL_X = 1e-5, 1e-4, 1e-3


def run(name, every, debug, typed=0, refine=False):
    c = vsgen.CONFIGS[name]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    if typed:
        lib.atom_type = vsgen.atom_types(lib, n_types=typed)
        pks = [vsgen.typed_pocket(s, n_types=typed) for s in c["pockets"]]
    else:
        pks = [vsgen.pocket(s) for s in c["pockets"]]
    rot, tr = vsgen.pose_table(c["P"])
    cs = vsgen.angle_table(c["K"])
    e = Engine(debug_poses=debug, bucket_multiple=16, n_streams=4)
    e.set_poses(rot, tr)
    e.set_angles(cs)
    ref = None
    if refine:
        q, dd = vsgen.refine_table()
        ref = (2, q, dd)
        e.set_refine(*ref)
    ids = [e.load_pocket(p) for p in pks]
    d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
    ty = torch.from_numpy(lib.atom_type).cuda() if typed else None
    e.submit(*d, ids, on_device=True, atom_type=ty)
    e.wait()
    out = []
    for slot, pk in enumerate(pks):
        r = e.results(slot)
        xyz = e.coords(slot)
        ps, pa = e.pose_debug(slot) if debug else (None, None)
        idx = np.arange(0, lib.n, every)
        t = time.time()
        kw = {}
        if refine:
            kw = dict(refine=ref, gpu_refine=e.refine(slot), gpu_pose_refine=e.pose_refine_debug(slot) if debug else None)
        rep = parity.check(lib, idx, pk, rot, tr, cs, r.best_score, r.best_pose, r.angles, xyz, ps, pa,
                           band=BAND, tol_score=TOL_S, tol_xyz=TOL_X, **kw)
        tag = name + (f" typed T={typed}" if typed else "") + (" + refinement (2 rounds, 13 moves)" if refine else "")
        row = {"config": tag, "pocket": int(c["pockets"][slot]), "ligands_checked": int(len(idx)),
               "of": int(lib.n), "every_pose_replayed": bool(debug), "steps_replayed": rep.n_steps,
               "near_ties": rep.near_ties, "independent_equal": rep.independent_equal,
               "independent_checked": rep.independent_checked, "max_score_rel_err": rep.max_score_err,
               "max_xyz_err_A": rep.max_xyz_err, "max_step_gap": rep.max_step_gap,
               "failures": len(rep.failures), "first_failures": [str(f) for f in rep.failures[:5]],
               "check_s": round(time.time() - t, 1)}
        print(json.dumps(row), flush=True)
        out.append(row)
    e.close()
    return out


if __name__ == "__main__":
    # DENSE=1: C3 with every pose replayed, C4 every 10th ligand, C5 every 100th per pocket
    dense = os.environ.get("DENSE") == "1"
    rows = []
    rows += run("C1", 1, True)
    rows += run("C2", 1, True)
    rows += run("C3", 1, dense)
    rows += run("C4", 10 if dense else 100, False)
    rows += run("C5", 100 if dense else 500, False)
    rows += run("C2", 1, True, typed=4)
    rows += run("C2", 5, True, refine=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump({"band": BAND, "tol_score": TOL_S, "tol_xyz": TOL_X, "rows": rows},
              open("gpurun_out/parity_report.json", "w"), indent=1)
