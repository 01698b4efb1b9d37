"""oracle -- plain CPU oracle of the LiGen dock-and-score hot path (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2303_06150_b200``) never imports it and shares no code with it.

Contents, each citing the passage it follows (P:n = PAPER.md line n,
S:n = SPEC.md line n, Qn = DESIGN.md reading n, a1..a11 = SURVEY.md 8(a) rows):

* docking (a6-a9): ``oracle.c`` in fp64 via ctypes -- :func:`dock_batch`,
  :func:`replay_pose`, :func:`grid_score`, :func:`place`, :func:`rotate`.
* bucketing (a2-a3): :func:`atom_boundaries`, :func:`rotamer_boundaries`
  (S:215-223), :func:`assign`, :class:`StreamingBucketizer`
  (S:235-253), :func:`bucketize` (stable sort by cell + chunking, Q18).
* launch sizing: :func:`active_blocks_per_sm`, :func:`bucket_capacity_native`
  (Eq. 1), :func:`ligand_footprint` / :func:`max_bucket_multiple`
  (S:137-155).
* sharding (a4): :func:`lpt_shards`.
* ranking (a10-a11): :func:`topk` (first k of the (score, index) sort), :func:`merge_topk`.

Pins: tests/test_oracle_pins.py, tests/test_bucketing_oracle.py (golden
fixtures from SPEC's worked examples under tests/golden/).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        # -ffp-contract=off: no fused multiply-add, plain fp64 as written
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _SO, src, "-lm", "-lpthread"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        p, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        lib.oracle_dock_batch.argtypes = [i64, p, p, p, p, p, p, p, p, p, p, i32, p, p, i32, p, i32, p, p, p, p, p, p, p,
                                          p, i32, i32, p, p, p, p, i32]
        lib.oracle_dock_batch.restype = i32
        lib.oracle_replay_pose.argtypes = [p, p, p, i32, p, p, i32, p, p, p, p, p, i32, p, i32, p, p, p, i32, i32, p, p, p,
                                           p]
        lib.oracle_replay_pose.restype = f64
        lib.oracle_grid_score_points.argtypes = [p, p, p, i64, p, p, p]
        lib.oracle_grid_score_points.restype = i32
        lib.oracle_place.argtypes = [p, p, i32, p, p, p, p]
        lib.oracle_place.restype = i32
        lib.oracle_rotate.argtypes = [i32, p, i32, i32, p, i32, f64, f64]
        lib.oracle_rotate.restype = i32
        lib.oracle_rigid_move.argtypes = [p, i32, p, p]
        lib.oracle_rigid_move.restype = None
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _pocket_args(pocket):
    """(dims {nx, ny, nz, T}, prm, grid [T*nz*ny*nx]) -- a pocket with a 4-D grid [T, nz, ny, nx] is
    typed (Q24)."""
    nx, ny, nz = pocket.dims
    T = 1 if pocket.grid.ndim == 3 else int(pocket.grid.shape[0])
    dims = np.array([nx, ny, nz, T], np.int32)
    prm = np.array(list(pocket.origin) + [pocket.spacing] + list(pocket.center) + [pocket.out_slope], np.float64)
    return dims, prm, _c(pocket.grid, np.float32)


# ----------------------------------------------------------------------------- docking (a6-a9)

@dataclass
class DockResult:
    best_score: np.ndarray      # float64 [n]
    best_pose: np.ndarray       # int32 [n]
    angles: np.ndarray          # uint8 [S_w * sum R] (CSR by S_w*frag_off)
    xyz: np.ndarray | None      # float64 [sum A, 3] best-pose coordinates (Angstrom)
    pose_score: np.ndarray | None   # float64 [n, P]
    pose_angles: np.ndarray | None  # uint8 [P * S_w * sum R]
    step_margin: np.ndarray | None  # float64 [n, P]
    pose_margin: np.ndarray | None  # float64 [n]
    refine: np.ndarray | None = None       # uint8 [n, n_ref] refinement moves of the best pose (Q23)
    pose_refine: np.ndarray | None = None  # uint8 [n, P, n_ref]


def _refine_args(refine):
    """(n_ref, J, rotations [J,9] f32, translations [J,3] f32) of ``refine`` = (n_ref, rot, trans) or None."""
    if refine is None or int(refine[0]) == 0:
        return 0, 1, np.eye(3, dtype=np.float32).reshape(1, 9), np.zeros((1, 3), np.float32)
    n_ref, q, d = refine
    q = _c(np.asarray(q, np.float32).reshape(-1, 9), np.float32)
    d = _c(np.asarray(d, np.float32).reshape(-1, 3), np.float32)
    return int(n_ref), int(q.shape[0]), q, d


def _types(t):
    return None if t is None else _c(t, np.uint8).reshape(-1)


def dock_batch(lib, pocket, rot, trans, cs, S_w: int = 1, want_xyz=True, want_debug=True, nthreads=None,
               refine=None, atom_type=None) -> DockResult:
    """Dock every ligand of ``lib`` (a vsgen.Library-like CSR batch) into ``pocket``; fp64.
    ``refine`` = (n_ref, move rotations [J,3,3], move translations [J,3] in Angstrom): rigid
    refinement rounds after the sweeps (Q23).  ``atom_type`` (uint8
    per atom, default ``lib.atom_type``) selects each atom's grid channel of a typed pocket (Q24)."""
    L = _load()
    n = lib.n
    P, K = int(rot.shape[0]), int(cs.shape[0])
    dims, prm, G = _pocket_args(pocket)
    ao, fo = _c(lib.atom_off, np.int64), _c(lib.frag_off, np.int64)
    xyz = _c(lib.xyz, np.float32)
    fax, mo, ma = _c(lib.frag_axis, np.int32), _c(lib.move_off, np.int64), _c(lib.move_atoms, np.int32)
    if ma.size == 0:
        ma = np.zeros(1, np.int32)
    rot, trans, cs = _c(rot, np.float32), _c(trans, np.float32), _c(cs, np.float32)
    nA, nR = int(ao[-1]), int(fo[-1])
    ty = _types(atom_type if atom_type is not None else getattr(lib, "atom_type", None))
    if ty is not None and ty.size == 0:
        ty = np.zeros(1, np.uint8)
    bs = np.zeros(n, np.float64); bp = np.zeros(n, np.int32)
    ang = np.zeros(max(1, S_w * nR), np.uint8)
    xo = np.zeros((max(1, nA), 3), np.float64) if want_xyz else None
    ps = np.zeros((n, P), np.float64) if want_debug else None
    pa = np.zeros(max(1, P * S_w * nR), np.uint8) if want_debug else None
    sm = np.zeros((n, P), np.float64) if want_debug else None
    pm = np.zeros(n, np.float64) if want_debug else None
    nthreads = nthreads or (os.cpu_count() or 1)
    n_ref, J, q, d = _refine_args(refine)
    rf = np.zeros((max(1, n), max(1, n_ref)), np.uint8)
    prf = np.zeros((max(1, n), P, max(1, n_ref)), np.uint8) if want_debug else None
    rc = L.oracle_dock_batch(n, _p(ao), _p(xyz), _p(ty), _p(fo), _p(fax), _p(mo), _p(ma), _p(dims), _p(prm), _p(G), P, _p(rot), _p(trans),
                             K, _p(cs), S_w, _p(bs), _p(bp), _p(ang), _p(xo), _p(ps), _p(pa), _p(sm), _p(pm),
                             n_ref, J, _p(q), _p(d), _p(rf) if n_ref else None, _p(prf) if (n_ref and prf is not None) else None,
                             nthreads)
    if rc != 0:
        raise ValueError("oracle_dock_batch: invalid arguments")
    return DockResult(bs, bp, ang[:S_w * nR], None if xo is None else xo[:nA], ps,
                      None if pa is None else pa[:P * S_w * nR], sm, pm,
                      rf[:n, :n_ref], None if prf is None else prf[:n, :, :n_ref])


def _frags_csr(frags):
    """(frag_axis [R,2] int32, move_off [R+1] int64, move_atoms int32) of a ligand's fragments, given in
    the general form (vsgen.Frags, or a list of (a, b, moving atoms)) or the range form [R,4]."""
    if isinstance(frags, np.ndarray) and frags.ndim == 2 and frags.shape[1] == 4:
        items = [(int(a), int(b), np.arange(lo, hi)) for a, b, lo, hi in frags]
    else:
        items = [(int(a), int(b), np.asarray(m)) for a, b, m in frags]
    ax = np.array([[a, b] for a, b, _ in items], np.int32).reshape(-1, 2)
    mo = np.zeros(len(items) + 1, np.int64)
    mo[1:] = np.cumsum([len(m) for _, _, m in items])
    ma = np.concatenate([np.asarray(m, np.int32) for _, _, m in items]) if items else np.zeros(0, np.int32)
    return ax, mo, (ma if ma.size else np.zeros(1, np.int32)).astype(np.int32)


def replay_pose(pocket, xyz, frags, rot9, tr3, cs, kseq, S_w: int = 1, refine=None, mseq=None, want_refine=False,
                types=None):
    """Replay a given angle sequence from pose (rot9, tr3), then (``refine``, Q23) the given
    refinement moves ``mseq``.  ``frags``: general form (vsgen.Frags) or range form [R,4];
    ``types``: the ligand's atom types (grid channels, Q24) or None.

    Returns (final_score, final_xyz [A,3] fp64, step_scores [S_w*R, K] fp64), plus the refinement
    round scores [n_ref, J] when ``want_refine``."""
    L = _load()
    dims, prm, G = _pocket_args(pocket)
    xyz = _c(xyz, np.float32)
    ax, mo, ma = _frags_csr(frags)
    A, R, K = int(xyz.shape[0]), int(ax.shape[0]), int(cs.shape[0])
    kseq = _c(kseq, np.uint8)
    steps = np.zeros((max(1, S_w * R), K), np.float64)
    y = np.zeros((max(1, A), 3), np.float64)
    n_ref, J, q, d = _refine_args(refine)
    ms = _c(mseq if n_ref else np.zeros(1), np.uint8)
    rs = np.zeros((max(1, n_ref), J), np.float64)
    s = L.oracle_replay_pose(_p(dims), _p(prm), _p(G), A, _p(xyz), _p(_types(types)), R, _p(ax), _p(mo), _p(ma),
                             _p(_c(rot9, np.float32)), _p(_c(tr3, np.float32)), K, _p(_c(cs, np.float32)), S_w,
                             _p(kseq), _p(steps), _p(y), n_ref, J, _p(q), _p(d), _p(ms), _p(rs))
    if want_refine:
        return float(s), y[:A], steps[:S_w * R], rs[:n_ref]
    return float(s), y[:A], steps[:S_w * R]


def rigid_move(y, q9, d3) -> np.ndarray:
    """One rigid refinement move about the centroid (Q23), fp64; returns a copy."""
    L = _load()
    y = np.array(y, dtype=np.float64, order="C").reshape(-1, 3)
    L.oracle_rigid_move(_p(y), y.shape[0], _p(_c(np.asarray(q9).reshape(9), np.float32)),
                        _p(_c(np.asarray(d3).reshape(3), np.float32)))
    return y


def grid_score(pocket, pts, types=None) -> np.ndarray:
    """g(y) at arbitrary points [n,3] (Angstrom), fp64 (a8); ``types`` = the channel of every point
    (typed pocket, Q24), None = channel 0."""
    L = _load()
    dims, prm, G = _pocket_args(pocket)
    pts = _c(pts, np.float64).reshape(-1, 3)
    out = np.zeros(pts.shape[0], np.float64)
    ty = _types(types)
    if ty is not None and (ty.shape[0] != pts.shape[0] or (ty.size and int(ty.max()) >= dims[3])):
        raise ValueError("grid_score: one type per point, each < the pocket's channels")
    L.oracle_grid_score_points(_p(dims), _p(prm), _p(G), pts.shape[0], _p(pts), _p(ty), _p(out))
    return out


def place(pocket, xyz, rot9, tr3) -> np.ndarray:
    """y_i = R (x_i - xbar) + c + tau (a6), fp64."""
    L = _load()
    dims, prm, _ = _pocket_args(pocket)
    xyz = _c(xyz, np.float32)
    y = np.zeros((xyz.shape[0], 3), np.float64)
    L.oracle_place(_p(dims), _p(prm), xyz.shape[0], _p(xyz), _p(_c(rot9, np.float32)), _p(_c(tr3, np.float32)), _p(y))
    return y


def rotate(y, frag, ck, sk) -> np.ndarray:
    """Rotate one fragment of coordinates y by (cos, sin) (a7), fp64; returns a copy.  ``frag`` is
    (a, b, moving atoms) (general form) or (a, b, lo, hi) (range form, M = [lo, hi))."""
    L = _load()
    y = np.array(y, dtype=np.float64, order="C").reshape(-1, 3)
    if len(frag) == 4 and np.isscalar(frag[2]):
        a, b, lo, hi = (int(v) for v in frag)
        mv = np.arange(lo, hi, dtype=np.int32)
    else:
        a, b, mv = int(frag[0]), int(frag[1]), np.asarray(frag[2], np.int32)
    mv = np.ascontiguousarray(mv, np.int32)
    L.oracle_rotate(y.shape[0], _p(y), a, b, _p(mv if mv.size else np.zeros(1, np.int32)), int(mv.size), float(ck),
                    float(sk))
    return y


# ----------------------------------------------------------------------------- bucketing (a2-a3)

class BucketingError(ValueError):
    """Argument / overflow errors.  ``axis`` names the overflowing axis."""

    def __init__(self, msg, axis=None, index=None):
        super().__init__(msg)
        self.axis = axis
        self.index = index


def atom_boundaries(n_clusters: int, warp_size: int, max_atoms: int) -> List[int]:
    """[1*ws, 2*ws, ..., (n-1)*ws, max_atoms] ("up to 32 and 64 atoms").

    Reading Q16: when S:207's precondition max_atoms >= ws*(n-1)+1 fails, the last
    boundary is raised to ws*n (every boundary a warp multiple)."""
    if n_clusters < 1:
        raise BucketingError("n_clusters must be >= 1")
    last = max_atoms if max_atoms >= warp_size * (n_clusters - 1) + 1 else warp_size * n_clusters
    return [warp_size * i for i in range(1, n_clusters)] + [last]


def rotamer_boundaries(n_clusters: int, max_rotamers: int) -> List[int]:
    """unit clusters if n > max; else geometric, denser at low values.

    boundary_i = max(prev + 1, round(max * (2^i - 1) / (2^n - 1))), boundary_n = max,
    with prev_0 = -1 (Q17); round = half-up, evaluated exactly in integers."""
    if n_clusters < 1:
        raise BucketingError("n_clusters must be >= 1")
    if max_rotamers < 0:
        raise BucketingError("max_rotamers must be >= 0")
    if n_clusters > max_rotamers:
        return list(range(0, max_rotamers + 1))
    out, prev = [], -1
    den = (1 << n_clusters) - 1
    for i in range(1, n_clusters + 1):
        if i == n_clusters:
            b = max_rotamers
        else:
            num = max_rotamers * ((1 << i) - 1)
            b = (2 * num + den) // (2 * den)       # round half up of num/den
        b = max(prev + 1, b)
        out.append(b)
        prev = b
    return out


def assign(atom_b: Sequence[int], rot_b: Sequence[int], n_atoms: int, n_rot: int):
    """each index is the smallest i with value <= boundaries[i]; overflow names the axis."""
    ai = next((i for i, b in enumerate(atom_b) if n_atoms <= b), None)
    if ai is None:
        raise BucketingError(f"atoms {n_atoms} > {atom_b[-1]}", axis="atoms")
    ri = next((i for i, b in enumerate(rot_b) if n_rot <= b), None)
    if ri is None:
        raise BucketingError(f"rotamers {n_rot} > {rot_b[-1]}", axis="rotamers")
    return ai, ri


@dataclass
class Bucket:
    cell: tuple             # (atom_class, rot_class)
    capacity: int
    ligands: list           # input indices, input order


class StreamingBucketizer:
    """SPEC's streaming bucketizer: push emits a full bucket; flush returns partials."""

    def __init__(self, atom_b, rot_b, capacity_per_atom_class):
        self.atom_b, self.rot_b, self.cap = list(atom_b), list(rot_b), list(capacity_per_atom_class)
        self.open = {}

    def push(self, index: int, n_atoms: int, n_rot: int):
        cell = assign(self.atom_b, self.rot_b, n_atoms, n_rot)
        b = self.open.setdefault(cell, [])
        b.append(index)
        if len(b) == self.cap[cell[0]]:
            del self.open[cell]
            return Bucket(cell, self.cap[cell[0]], b)
        return None

    def flush(self):
        out = [Bucket(c, self.cap[c[0]], self.open[c]) for c in sorted(self.open)]   # row-major cell order
        self.open = {}
        return out


def bucketize(n_atoms, n_rot, atom_b, rot_b, capacity_per_atom_class, n_move=None, move_b=None) -> List[Bucket]:
    """Canonical manifest (Q18): cell-major (atom class, then rotamer class); within a cell,
    input order; each cell cut into consecutive buckets of its atom class's capacity
    (the last may be partial -- the tail).  With ``move_b`` the cell gets a third
    key, the moving-atom count class, assigned by the same rule."""
    cells = {}
    for i, (a, r) in enumerate(zip(n_atoms, n_rot)):
        try:
            cell = assign(atom_b, rot_b, int(a), int(r))
            if move_b is not None:
                mi = next((j for j, b in enumerate(move_b) if int(n_move[i]) <= b), None)
                if mi is None:
                    raise BucketingError(f"moving atoms {n_move[i]} > {move_b[-1]}", axis="moving atoms")
                cell = cell + (mi,)
        except BucketingError as e:
            e.index = i
            raise
        cells.setdefault(cell, []).append(i)
    out = []
    for cell in sorted(cells):
        cap = int(capacity_per_atom_class[cell[0]])
        idx = cells[cell]
        for s in range(0, len(idx), cap):
            out.append(Bucket(cell, cap, idx[s:s + cap]))
    return out


# ----------------------------------------------------------------------------- launch sizing

def active_blocks_per_sm(regs_per_sm, max_threads_per_sm, max_blocks_per_sm, shared_mem_per_sm, reg_alloc_granularity,
                         regs_per_thread, block_size, shared_per_block, measured_active_blocks=None, sm_count=None):
    """b = min(register, thread, block, shared-memory limits) (P:223 occupancy query)."""
    if block_size > max_threads_per_sm:
        raise BucketingError("block_size > max_threads_per_sm")
    if measured_active_blocks is not None:
        return measured_active_blocks // sm_count
    per_block_regs = -(-(regs_per_thread * block_size) // reg_alloc_granularity) * reg_alloc_granularity
    lim = [regs_per_sm // per_block_regs, max_threads_per_sm // block_size, max_blocks_per_sm]
    if shared_per_block > 0:
        lim.append(shared_mem_per_sm // shared_per_block)
    b = min(lim)
    if b == 0:
        raise BucketingError("kernel does not fit")
    return b


def bucket_capacity_native(b: int, sm_count: int, block_size: int, warp_size: int) -> int:
    """Eq. 1: l = b * SM * t / ws, exact integers."""
    if block_size % warp_size != 0:
        raise BucketingError("warp_size must divide block_size")
    return b * sm_count * (block_size // warp_size)


def ligand_footprint(n_sites: int, base_bytes: int, per_site_bytes: int) -> int:
    """S:137-145 (P:331-333 footprint grows linearly with docking sites)."""
    return base_bytes + n_sites * per_site_bytes


def max_bucket_multiple(global_mem_bytes: int, l: int, per_ligand_bytes: int, n_buffers: int) -> int:
    """largest k >= 0 with k * l * per_ligand_bytes * n_buffers <= global memory."""
    return global_mem_bytes // (l * per_ligand_bytes * n_buffers)


# ----------------------------------------------------------------------------- sharding (a4)

def ligand_work(n_atoms, n_moving, P: int, K: int, S_w: int = 1) -> np.ndarray:
    """E_alg,i = P * (A_i + S_w * (K - 1) * sum_r |M_ir|) evaluations (SURVEY 8 'E_alg')."""
    return P * (np.asarray(n_atoms, np.int64) + S_w * (K - 1) * np.asarray(n_moving, np.int64))


def lpt_shards(weights: Sequence[int], world: int) -> List[List[int]]:
    """a4: buckets by weight descending (ties: id ascending) to the least-loaded rank (ties: lowest rank)."""
    order = sorted(range(len(weights)), key=lambda b: (-int(weights[b]), b))
    load = [0] * world
    out = [[] for _ in range(world)]
    for b in order:
        r = min(range(world), key=lambda q: (load[q], q))
        out[r].append(b)
        load[r] += int(weights[b])
    return out


# ----------------------------------------------------------------------------- ranking (a10-a11)

def topk(scores, k: int, index=None) -> np.ndarray:
    """P:174 rank per docking site: the first k of the ascending (score, index) sort (Q2, Q11, Q20)."""
    scores = np.asarray(scores)
    index = np.arange(len(scores)) if index is None else np.asarray(index)
    order = sorted(range(len(scores)), key=lambda i: (float(scores[i]), int(index[i])))
    return np.array([int(index[i]) for i in order[:k]], dtype=np.int64)


def merge_topk(parts, k: int) -> np.ndarray:
    """Global top-k from per-rank (scores, index) lists: top-k of their union."""
    s = np.concatenate([np.asarray(p[0], np.float64) for p in parts]) if parts else np.zeros(0)
    i = np.concatenate([np.asarray(p[1], np.int64) for p in parts]) if parts else np.zeros(0, np.int64)
    return topk(s, k, i)
