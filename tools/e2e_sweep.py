"""e2e pipeline experiment (not a bench value): PipelinedDocker wall time vs chunk count on C4."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import vsgen
from paper_2303_06150_b200 import Engine
from paper_2303_06150_b200.pipeline import PipelinedDocker
c = vsgen.CONFIGS["C4"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else c["n"]
lib = vsgen.ligands(n, c["seed"], c["atoms"], c["rot"])
pk = [vsgen.pocket(s) for s in c["pockets"]]
rot, tr = vsgen.pose_table(c["P"]); cs = vsgen.angle_table(c["K"])
h = [torch.from_numpy(a).pin_memory() for a in (lib.atom_off, lib.xyz, lib.frag_off, lib.frags)]
e = Engine(); e.set_poses(rot, tr); e.set_angles(cs); ids = [e.load_pocket(p) for p in pk]
for on_dev in (True, False):
    b = [x.cuda() for x in h] if on_dev else h
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        e.submit(*b, ids, on_device=on_dev, max_atoms=int(lib.n_atoms.max())); e.wait(); r = e.results(0)
        dt = time.perf_counter() - t
    st = e.stats()
    print(f"single engine on_device={on_dev}: {dt*1e3:.1f} ms wall, prep {st['prep_ms']:.2f} dock {st['dock_ms']:.2f}")
e.close()
pd = PipelinedDocker(n_buffers=2); pd.setup(rot, tr, cs, pk)
for chunks in (2, 4, 8, 16):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        pd.run(*h, k=1000, chunks=chunks, max_atoms=int(lib.n_atoms.max()))
        dt = time.perf_counter() - t
    print(f"pipelined chunks={chunks}: {dt*1e3:.1f} ms wall  {n/dt:.3e} lig/s")
    if chunks == 4:
        for r in pd.trace:
            print(f"  chunk {r[0]} wait-copy {1e3*(r[2]-r[1]):.2f} ms  compute {1e3*(r[3]-r[2]):.1f} ms  prep {r[4]:.2f} dock {r[5]:.2f}")
pd.close()
