"""Parity contract and replay checker -- TEST INFRASTRUCTURE.

Greedy trajectories fork after a near-tie, so angle indices are compared in two ways:

1. **Replay.** For each ligand (and, with the per-pose debug output, each pose) the
   GPU's own angle sequence is replayed in fp64 by the oracle
   (:func:`oracle.replay_pose`).  Every GPU choice must be within the near-tie band of
   the fp64 minimum at that step; the final score and coordinates must match the
   replayed state within the tolerances (Q12).
2. **Independent run.** The oracle docks the ligand on its own.  For every ligand whose
   oracle trajectory has no near-tie (all step margins and the best-pose margin above the
   band), the GPU's best pose and angle indices must be bit-identical.

Bands and tolerances are arguments so tests state them explicitly.  A library carrying
``atom_type`` is replayed on its typed pocket's channels (Q24).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

import oracle


@dataclass
class ParityReport:
    n_ligands: int = 0
    n_steps: int = 0
    near_ties: int = 0            # GPU choice != fp64 argmin but inside the band
    independent_checked: int = 0  # ligands with no oracle near-tie
    independent_equal: int = 0
    max_score_err: float = 0.0    # relative, max(1,|S|)
    max_xyz_err: float = 0.0      # Angstrom
    max_step_gap: float = 0.0     # relative gap of a GPU choice above the fp64 min
    failures: list = field(default_factory=list)

    @property
    def ok(self):
        return not self.failures

    def summary(self):
        return (f"ligands={self.n_ligands} steps={self.n_steps} near_ties={self.near_ties} "
                f"independent={self.independent_equal}/{self.independent_checked} "
                f"max_score_err={self.max_score_err:.3g} max_xyz_err={self.max_xyz_err:.3g} "
                f"max_step_gap={self.max_step_gap:.3g} failures={len(self.failures)}")


def _rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


def check(lib, idx, pocket, rot, trans, cs, gpu_score, gpu_pose, gpu_angles, gpu_xyz=None,
          gpu_pose_score=None, gpu_pose_angles=None, S_w=1, band=1e-5, tol_score=1e-4, tol_xyz=1e-3,
          nthreads=None, refine=None, gpu_refine=None, gpu_pose_refine=None) -> ParityReport:
    """Check ligands ``idx`` of ``lib`` (GPU arrays indexed like the full library).  ``refine`` =
    (n_ref, rot, trans) when the rigid refinement ran (Q23): its moves (``gpu_refine`` [n, n_ref],
    ``gpu_pose_refine`` [n, P, n_ref]) are replayed and banded like the angle steps."""
    rep = ParityReport()
    idx = [int(i) for i in idx]
    P = rot.shape[0]
    n_ref = int(refine[0]) if refine is not None else 0
    sub = lib.subset(idx)
    ref = oracle.dock_batch(sub, pocket, rot, trans, cs, S_w, want_xyz=False, want_debug=True, nthreads=nthreads,
                            refine=refine if n_ref else None)
    for j, i in enumerate(idx):
        rep.n_ligands += 1
        x, fr = lib.ligand(i)
        R = len(fr)
        f0 = int(lib.frag_off[i])
        a0 = int(lib.atom_off[i])
        ty = None if getattr(lib, "atom_type", None) is None else lib.atom_type[a0:a0 + len(x)]   # Q24
        p = int(gpu_pose[i])
        if not (0 <= p < P):
            rep.failures.append((i, f"best pose {p} out of range"))
            continue
        poses = range(P) if gpu_pose_score is not None else [p]
        rep_scores = {}
        for q in poses:
            if gpu_pose_angles is not None:
                kseq = gpu_pose_angles[P * S_w * f0 + q * S_w * R: P * S_w * f0 + (q + 1) * S_w * R]
            else:
                kseq = gpu_angles[S_w * f0: S_w * f0 + S_w * R]
            if n_ref:
                mseq = gpu_pose_refine[i, q] if gpu_pose_refine is not None else gpu_refine[i]
                s, y, steps, rsc = oracle.replay_pose(pocket, x, fr, rot[q], trans[q], cs, kseq, S_w, refine=refine,
                                                      mseq=mseq, want_refine=True, types=ty)
                for st, m in zip(rsc, mseq):
                    rep.n_steps += 1
                    mn = float(st.min())
                    gap = (float(st[int(m)]) - mn) / max(1.0, abs(mn))
                    rep.max_step_gap = max(rep.max_step_gap, gap)
                    if gap > band:
                        rep.failures.append((i, f"pose {q}: refinement move {int(m)} {gap:.3g} above the fp64 min"))
                    elif int(m) != int(np.argmin(st)):
                        rep.near_ties += 1
            else:
                s, y, steps = oracle.replay_pose(pocket, x, fr, rot[q], trans[q], cs, kseq, S_w, types=ty)
            rep_scores[q] = s
            for st, k in zip(steps, kseq):
                rep.n_steps += 1
                m = float(st.min())
                gap = (float(st[int(k)]) - m) / max(1.0, abs(m))
                rep.max_step_gap = max(rep.max_step_gap, gap)
                if gap > band:
                    rep.failures.append((i, f"pose {q}: chose k={int(k)} {gap:.3g} above the fp64 min (band {band})"))
                elif int(k) != int(np.argmin(st)):
                    rep.near_ties += 1
            gs = float(gpu_pose_score[i, q]) if gpu_pose_score is not None else float(gpu_score[i])
            e = _rel(gs, s)
            rep.max_score_err = max(rep.max_score_err, e)
            if e > tol_score:
                rep.failures.append((i, f"pose {q}: score {gs} vs replay {s} (rel {e:.3g})"))
            if q == p:
                e = _rel(float(gpu_score[i]), s)
                rep.max_score_err = max(rep.max_score_err, e)
                if e > tol_score:
                    rep.failures.append((i, f"best score {gpu_score[i]} vs replay {s}"))
                if gpu_xyz is not None:
                    d = float(np.max(np.abs(np.asarray(gpu_xyz[a0:a0 + len(x)], np.float64) - y))) if len(x) else 0.0
                    rep.max_xyz_err = max(rep.max_xyz_err, d)
                    if d > tol_xyz:
                        rep.failures.append((i, f"coordinates differ by {d:.3g} A"))
        if gpu_pose_score is not None:
            mn = min(rep_scores.values())
            if (rep_scores[p] - mn) / max(1.0, abs(mn)) > band:
                rep.failures.append((i, f"best pose {p} is {rep_scores[p] - mn:.3g} above the replayed minimum"))
        # independent run: bit-exact indices where the oracle has no near-tie
        sm = float(np.min(ref.step_margin[j])) if P else np.inf
        pm = float(ref.pose_margin[j])
        if sm > band and pm > band:
            rep.independent_checked += 1
            ok = int(ref.best_pose[j]) == p
            ra = ref.angles[S_w * int(sub.frag_off[j]): S_w * int(sub.frag_off[j]) + S_w * R]
            ga = gpu_angles[S_w * f0: S_w * f0 + S_w * R]
            ok = ok and np.array_equal(np.asarray(ra), np.asarray(ga))
            if n_ref:
                ok = ok and np.array_equal(np.asarray(ref.refine[j]), np.asarray(gpu_refine[i]))
            e = _rel(float(gpu_score[i]), float(ref.best_score[j]))
            ok = ok and e <= tol_score
            if ok:
                rep.independent_equal += 1
            else:
                rep.failures.append((i, f"independent run differs without a near-tie: pose {p} vs {int(ref.best_pose[j])},"
                                        f" angles {list(ga)} vs {list(ra)}, score rel err {e:.3g}"))
    return rep
