"""The paper's experiments re-run on B200.  Writes CSVs to gpurun_out/.

  heatmap N     Fig. 4: throughput speed-up vs the 1x1 cluster grid, by the
                number of atom x rotamer clusters, for an N-ligand paper-shaped library; both launch
                structures (fused per class, and one launch per bucket as the paper).
  sweep  N      Fig. 2: three ligands (17/53/99 atoms) replicated N times,
                one launch per bucket, bucket size k/3 * l for k = 1..12 plus "All".
  tail   N      tail effect: 6 x 23 over 1 x 1 for libraries of 3k .. N ligands.
Timing: CUDA events of the library (dock phase) and wall time of the whole submit (step);
device-resident library; median of 3 after 1 warm-up.  Not bench values.
"""
import csv
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import vsgen
from paper_2303_06150_b200 import Engine


def timed(e, d, ids, reps=3):
    e.submit(*d, ids, on_device=True)
    e.wait()
    st, dock = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        e.submit(*d, ids, on_device=True)
        e.wait()
        st.append(time.perf_counter() - t)
        dock.append(e.stats()["dock_ms"])
    s = e.stats()
    return float(np.median(st)) * 1e3, float(np.median(dock)), s


def setup(e, pockets):
    e.set_poses(*vsgen.pose_table(64))
    e.set_angles(vsgen.angle_table(8))
    return [e.load_pocket(p) for p in pockets]


def heatmap(n):
    lib = vsgen.ligands(n, 4)
    d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
    pk = [vsgen.pocket(101)]
    out = open(f"gpurun_out/heatmap_{n}.csv", "w", newline="")
    w = csv.writer(out)
    w.writerow(["mode", "atom_clusters", "rotamer_clusters", "cells_populated", "buckets", "dock_launches",
                "step_ms", "dock_ms", "ligands_per_s", "speedup_vs_1x1"])
    for mode in ("fused", "per_bucket"):
        base = None
        for na in range(1, 7):
            for nr in (1, 2, 3, 4, 6, 8, 12, 16, 23):
                e = Engine(atom_clusters=na, rot_clusters=nr, launch_per_bucket=(mode == "per_bucket"),
                           bucket_multiple=1 if mode == "per_bucket" else 16, n_streams=4)
                ids = setup(e, pk)
                step, dock, s = timed(e, d, ids)
                bk, _ = e.manifest(want_perm=False)
                cells = len({b["cell"] for b in bk})
                thr = n / (step / 1e3)
                if base is None:
                    base = thr
                w.writerow([mode, na, nr, cells, s["n_buckets"], s["dock_launches"], f"{step:.3f}", f"{dock:.3f}",
                            f"{thr:.1f}", f"{thr / base:.4f}"])
                out.flush()
                print(mode, na, nr, cells, s["n_buckets"], f"{step:.2f} ms", f"{thr / base:.3f}x", flush=True)
                e.close()
    out.close()


def sweep(n):
    pk = [vsgen.pocket(101)]
    out = open(f"gpurun_out/bucket_sweep_{n}.csv", "w", newline="")
    w = csv.writer(out)
    w.writerow(["atoms", "rot_bonds", "streams", "k_thirds", "bucket_size", "l_eq1", "dock_launches", "step_ms",
                "dock_ms", "ligands_per_s"])
    for A, R in ((17, 3), (53, 8), (99, 14)):
        one = vsgen.ligands(1, 50 + A, (A, A), (R, R))
        lib = vsgen.replicate(one, 0, n)
        d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
        probe = Engine(atom_clusters=1, rot_clusters=1)
        ids = setup(probe, pk)
        probe.submit(*d, ids, on_device=True)
        probe.wait()
        l = probe.classes()[0]["l"]
        probe.close()
        for streams in (1, 4):
            sizes = [(k, max(1, k * l // 3)) for k in range(1, 13)] + [("All", n)]
            for k, size in sizes:
                e = Engine(atom_clusters=1, rot_clusters=1, launch_per_bucket=True, bucket_capacity=size,
                           n_streams=streams)
                ids = setup(e, pk)
                step, dock, s = timed(e, d, ids)
                thr = n / (step / 1e3)
                w.writerow([A, int(one.n_frags[0]), streams, k, size, l, s["dock_launches"], f"{step:.3f}",
                            f"{dock:.3f}", f"{thr:.1f}"])
                out.flush()
                print(A, streams, k, size, s["dock_launches"], f"{step:.2f} ms", f"{thr:.3e}", flush=True)
                e.close()
    out.close()


def tail(n_max):
    """Tail-effect study: bucketed (6 x 23) over unsorted (1 x 1) as
    the library grows, for both launch structures."""
    pk = [vsgen.pocket(101)]
    out = open("gpurun_out/tail_effect.csv", "w", newline="")
    w = csv.writer(out)
    w.writerow(["ligands", "mode", "buckets_6x23", "step_ms_1x1", "step_ms_6x23", "ligands_per_s_6x23", "speedup"])
    full = vsgen.ligands(n_max, 4)
    for n in (3000, 10000, 30000, 100000, 300000, 1000000):
        if n > n_max:
            break
        lib = full.subset(np.arange(n)) if n < n_max else full
        d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
        for mode in ("fused", "per_bucket"):
            res = {}
            for na, nr in ((1, 1), (6, 23)):
                e = Engine(atom_clusters=na, rot_clusters=nr, launch_per_bucket=(mode == "per_bucket"),
                           bucket_multiple=1 if mode == "per_bucket" else 16, n_streams=4)
                ids = setup(e, pk)
                step, dock, s = timed(e, d, ids)
                res[(na, nr)] = (step, s["n_buckets"])
                e.close()
            s11, s623 = res[(1, 1)][0], res[(6, 23)][0]
            w.writerow([n, mode, res[(6, 23)][1], f"{s11:.3f}", f"{s623:.3f}", f"{n / (s623 / 1e3):.1f}", f"{s11 / s623:.4f}"])
            out.flush()
            print(n, mode, f"{s11:.2f} ms vs {s623:.2f} ms", f"{s11 / s623:.3f}x", flush=True)
    out.close()


if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    what, n = sys.argv[1], int(sys.argv[2])
    {"heatmap": heatmap, "sweep": sweep, "tail": tail}[what](n)
