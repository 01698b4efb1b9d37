"""Projected strong scaling of C4 on one B200 (not a bench value): every rank r of W runs its
LPT share of the full 1M-ligand library (validate + bucket the whole library, pack + dock its
own buckets, local top-1000) on this GPU in turn; the step time of W GPUs is the max over ranks
(+ the NCCL all-gather of 8 KB per rank, not included)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import vsgen
from paper_2303_06150_b200 import Engine
c = vsgen.CONFIGS["C4"]
lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
rot, tr = vsgen.pose_table(c["P"]); cs = vsgen.angle_table(c["K"]); pk = vsgen.pocket(101)
mx = int(lib.n_atoms.max())
out = {}
for W in (1, 2, 4, 8):
    per = []
    for r in range(W):
        e = Engine(rank=r, world_size=W)
        e.set_poses(rot, tr); e.set_angles(cs); ids = [e.load_pocket(pk)]
        ts = []
        for it in range(4):
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            e.submit(*d, ids, on_device=True, max_atoms=mx); e.wait()
            e.local_topk(0, 1000)
            ev1.record(); torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        st = e.stats()
        per.append({"rank": r, "ms": float(np.median(ts[1:])), "dock_ms": st["dock_ms"], "prep_ms": st["prep_ms"],
                    "owned": st["n_owned"]})
        e.close()
    tmax = max(p["ms"] for p in per)
    out[W] = {"step_ms_max_over_ranks": tmax, "ligands_per_s": c["n"] / tmax * 1e3, "ranks": per}
    print(W, f"{tmax:.2f} ms  {c['n'] / tmax * 1e3:.3e} lig/s  speedup {out[1]['step_ms_max_over_ranks'] / tmax:.2f}",
          [round(p["ms"], 2) for p in per], flush=True)
json.dump(out, open("gpurun_out/scaling_proj.json", "w"), indent=1)
