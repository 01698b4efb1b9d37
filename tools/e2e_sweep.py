"""e2e pipeline experiment (not a bench value): PipelinedDocker wall time vs chunk schedule on C4."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import vsgen
from paper_2303_06150_b200 import Engine
from paper_2303_06150_b200.pipeline import PipelinedDocker, chunk_bounds
c = vsgen.CONFIGS["C4"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else c["n"]
lib = vsgen.ligands(n, c["seed"], c["atoms"], c["rot"])
pk = [vsgen.pocket(s) for s in c["pockets"]]
rot, tr = vsgen.pose_table(c["P"]); cs = vsgen.angle_table(c["K"])
h = [torch.from_numpy(a).pin_memory() for a in lib.arrays()]
pd = PipelinedDocker(); pd.setup(rot, tr, cs, pk)
mx = int(lib.n_atoms.max())
for first, growth in ((32, 4), (32, 6), (64, 6), (32, 8), (16, 4)):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        pd.run(*h, k=1000, chunks=0, max_atoms=mx, first=first, growth=growth)
        ts.append(time.perf_counter() - t)
    dt = float(np.median(ts[1:]))
    print(f"first=n/{first} growth={growth} {chunk_bounds(n, 0, first, growth)[1:]}: {dt*1e3:.1f} ms  {n/dt:.3e} lig/s", flush=True)
    for r in pd.trace:
        print(f"   chunk {r[0]} wait-copy {1e3*(r[2]-r[1]):.2f} ms  compute {1e3*(r[3]-r[2]):.2f} ms  prep {r[4]:.2f} dock {r[5]:.2f}")
pd.close()
