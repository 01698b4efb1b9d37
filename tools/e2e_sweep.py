"""e2e pipeline diagnostics (not a bench value): PipelinedDocker wall time vs chunk schedule on C4,
with the host timeline of every chunk (wait for its upload, submit = prep incl. host syncs,
read-back queueing).  python tools/e2e_sweep.py [n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import vsgen
from paper_2303_06150_b200.pipeline import PipelinedDocker, chunk_bounds
c = vsgen.CONFIGS["C4"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else c["n"]
lib = vsgen.ligands(n, c["seed"], c["atoms"], c["rot"])
pk = [vsgen.pocket(s) for s in c["pockets"]]
rot, tr = vsgen.pose_table(c["P"]); cs = vsgen.angle_table(c["K"])
h = [torch.from_numpy(a).pin_memory() for a in lib.arrays()]
pd = PipelinedDocker(); pd.setup(rot, tr, cs, pk)
mx = int(lib.n_atoms.max())
for chunks, coords, zc, lc in ((0, True, False, False), (0, True, False, True), (4, True, False, True),
                               (8, True, False, True), (4, True, False, False), (8, True, False, False),
                               (0, True, True, False)):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        pd.run(*h, k=1000, chunks=chunks, max_atoms=mx, coords=coords, zero_copy=zc, library_copy=lc)
        ts.append(time.perf_counter() - t)
    dt = float(np.median(ts[1:]))
    print(f"chunks={chunks} coords={coords} zero_copy={zc} library_copy={lc} {chunk_bounds(n, chunks)[1:]}: {dt*1e3:.1f} ms "
          f"{n/dt:.3e} lig/s", flush=True)
    T0 = pd.trace[0][3]
    for r in pd.trace:
        print(f"   chunk {r[0]} [{r[1]},{r[2]}) start {1e3*(r[3]-T0):7.2f}  upload-wait {1e3*(r[4]-r[3]):6.2f}  "
              f"submit {1e3*(r[5]-r[4]):6.2f}  queue-readback {1e3*(r[6]-r[5]):6.2f} ms")
pd.close()
