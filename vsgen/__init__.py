"""vsgen -- seeded synthetic inputs shared by the oracle side and the CUDA side.

INPUT GENERATORS ONLY: this package draws ligands, pocket grids, pose tables
and angle tables.  It holds none of the method's arithmetic (no placement, no
rotation sweep, no interpolation, no bucketing); the oracle (``oracle/``) and
the product (``paper_2303_06150_b200``) each implement that independently.

The recipe (SURVEY.md 8(d) "Generators"):

* ligands: ``gen.c`` (C, multithreaded, prefix-stable: ligand i depends only
  on (seed, i)); atoms ~ U[alo, ahi], rotatable bonds ~ U[rlo, rhi]
  independent ("weak relationship", l.412 "between 20 and 120
  ... from 0 to 20 rotamers"; SPEC.md l.36-44 uniform).
* pocket grid: 32^3 fp32 lattice at 1.0 A; a pseudo-receptor of 96 atoms on a
  9-13 A shell around the centre with a 50 degree mouth; value
  sum_j [5 exp(-d^2/2) - exp(-d^2/8)] + 0.01 |x - c|^2 evaluated in fp64.
* pose table: p = 0 identity, p >= 1 Shoemake-uniform rotations from
  splitmix64(pose_seed, p), fp64 -> fp32 3x3; translations 0 (reading Q7).
* angle table: theta_k = 2 pi k / K, (cos, sin) fp64 -> fp32, entry 0 = (1, 0)
  exactly (reading Q3).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libvsgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c into libvsgen.so (gcc, -O2, pthreads)."""
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fPIC", "-shared",
                               "-o", _SO, src, "-lm", "-lpthread"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        p = ctypes.c_void_p
        lib.vsgen_ligand_shapes.argtypes = [i64, u64, i64, i32, i32, i32, i32, p, p, p, i32]
        lib.vsgen_ligand_shapes.restype = i32
        lib.vsgen_ligand_fill.argtypes = [i64, u64, i64, i32, i32, i32, i32, p, p, p, p, i32]
        lib.vsgen_ligand_fill.restype = i32
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Frags:
    """Fragments of ONE ligand in the C-ABI's general form (include/vsdock.h):
    axis[r] = (a, b) (rotation axis a -> b, b on the moving side) and moves[r] = the
    moving-atom set M_r (ligand-local indices, axis atoms excluded; "a
    subset of the molecule atoms that can rotate")."""

    def __init__(self, axis, moves):
        self.axis = np.asarray(axis, np.int32).reshape(-1, 2)
        self.moves = [np.asarray(m, np.int32).reshape(-1) for m in moves]

    def __len__(self):
        return int(self.axis.shape[0])

    def __iter__(self):
        for r in range(len(self)):
            yield int(self.axis[r, 0]), int(self.axis[r, 1]), self.moves[r]

    def __eq__(self, o):
        return (isinstance(o, Frags) and np.array_equal(self.axis, o.axis) and len(self.moves) == len(o.moves)
                and all(np.array_equal(a, b) for a, b in zip(self.moves, o.moves)))

    @staticmethod
    def from_ranges(fr):
        fr = np.asarray(fr, np.int32).reshape(-1, 4)
        return Frags(fr[:, :2], [np.arange(lo, hi, dtype=np.int32) for _, _, lo, hi in fr])


def _csr_from_ranges(frags):
    """General-form CSR (frag_axis, move_off, move_atoms) of range-form fragments {a, b, lo, hi}."""
    frags = np.asarray(frags, np.int32).reshape(-1, 4)
    cnt = (frags[:, 3] - frags[:, 2]).astype(np.int64)
    move_off = np.zeros(len(frags) + 1, np.int64)
    move_off[1:] = np.cumsum(cnt)
    # concatenated aranges lo..hi-1 of every fragment
    starts = np.repeat(frags[:, 2].astype(np.int64) - move_off[:-1], cnt)
    move_atoms = (np.arange(int(move_off[-1]), dtype=np.int64) + starts).astype(np.int32)
    return np.ascontiguousarray(frags[:, :2]), move_off, move_atoms


@dataclass
class Library:
    """A ligand batch in the C-ABI's CSR layout (include/vsdock.h vs_ligand_batch).

    Ligand i: atoms atom_off[i]..atom_off[i+1] (xyz, Angstrom), fragments
    f = frag_off[i]..frag_off[i+1] with axis frag_axis[f] = (a, b) and moving set
    move_atoms[move_off[f]..move_off[f+1]] (ligand-local indices).  ``frags`` keeps the
    generator's range form {a, b, lo, hi} when every M_r is a contiguous range (the
    generator numbers atoms in DFS preorder); it is None for a renumbered library."""
    ligand_id: np.ndarray   # uint64 [n]
    atom_off: np.ndarray    # int64 [n+1]
    xyz: np.ndarray         # float32 [sum A, 3], Angstrom, AoS
    frag_off: np.ndarray    # int64 [n+1]
    frag_axis: np.ndarray   # int32 [sum R, 2]
    move_off: np.ndarray    # int64 [sum R + 1]
    move_atoms: np.ndarray  # int32 [sum |M_r|]
    n_moving: np.ndarray = field(default=None)  # int32 [n]: sum_r |M_r| (generator metadata)
    frags: np.ndarray = field(default=None)     # int32 [sum R, 4] range form, or None
    atom_type: np.ndarray = field(default=None) # uint8 [sum A]: grid channel per atom (Q24), or None

    @staticmethod
    def from_ranges(ligand_id, atom_off, xyz, frag_off, frags, n_moving=None) -> "Library":
        ax, mo, ma = _csr_from_ranges(frags)
        return Library(np.asarray(ligand_id, np.uint64), np.asarray(atom_off, np.int64),
                       np.ascontiguousarray(xyz, np.float32), np.asarray(frag_off, np.int64), ax, mo, ma,
                       n_moving, np.ascontiguousarray(frags, np.int32).reshape(-1, 4))

    @staticmethod
    def from_ligands(ligs, ligand_id=None) -> "Library":
        """Build from a list of (xyz [A,3], Frags) in the general form."""
        n = len(ligs)
        A = [len(x) for x, _ in ligs]
        R = [len(f) for _, f in ligs]
        ao = np.zeros(n + 1, np.int64); ao[1:] = np.cumsum(A)
        fo = np.zeros(n + 1, np.int64); fo[1:] = np.cumsum(R)
        xyz = np.concatenate([np.asarray(x, np.float32).reshape(-1, 3) for x, _ in ligs]) if n else np.zeros((0, 3), np.float32)
        ax = np.concatenate([f.axis for _, f in ligs]) if n else np.zeros((0, 2), np.int32)
        mv = [m for _, f in ligs for m in f.moves]
        mo = np.zeros(len(mv) + 1, np.int64); mo[1:] = np.cumsum([len(m) for m in mv])
        ma = np.concatenate(mv).astype(np.int32) if mv else np.zeros(0, np.int32)
        nm = np.array([sum(len(m) for m in f.moves) for _, f in ligs], np.int32)
        ids = np.arange(n, dtype=np.uint64) if ligand_id is None else np.asarray(ligand_id, np.uint64)
        return Library(ids, ao, np.ascontiguousarray(xyz), fo, np.ascontiguousarray(ax, np.int32).reshape(-1, 2),
                       mo, np.ascontiguousarray(ma), nm, None)

    @property
    def n(self) -> int:
        return int(self.ligand_id.shape[0])

    @property
    def n_atoms(self) -> np.ndarray:
        return np.diff(self.atom_off).astype(np.int32)

    @property
    def n_frags(self) -> np.ndarray:
        return np.diff(self.frag_off).astype(np.int32)

    @property
    def moving_per_ligand(self) -> np.ndarray:
        """sum_r |M_r| per ligand (from the CSR itself)."""
        per_frag = np.diff(self.move_off)
        out = np.zeros(self.n, np.int64)
        if per_frag.size:
            np.add.at(out, np.repeat(np.arange(self.n), self.n_frags), per_frag)
        return out

    def arrays(self):
        """The C-ABI batch arrays, in vs_ligand_batch order."""
        return (self.ligand_id, self.atom_off, self.xyz, self.frag_off, self.frag_axis, self.move_off,
                self.move_atoms)

    def ligand(self, i: int):
        """(xyz [A,3] float32, Frags) of ligand i (general form)."""
        a0, a1 = int(self.atom_off[i]), int(self.atom_off[i + 1])
        f0, f1 = int(self.frag_off[i]), int(self.frag_off[i + 1])
        moves = [self.move_atoms[int(self.move_off[f]):int(self.move_off[f + 1])] for f in range(f0, f1)]
        return self.xyz[a0:a1], Frags(self.frag_axis[f0:f1], moves)

    def ligand_ranges(self, i: int):
        """(xyz, range-form frags [R,4]) of a preordered (generator-numbered) library."""
        assert self.frags is not None, "range form only exists for the generator's DFS-preordered libraries"
        a0, a1 = int(self.atom_off[i]), int(self.atom_off[i + 1])
        f0, f1 = int(self.frag_off[i]), int(self.frag_off[i + 1])
        return self.xyz[a0:a1], self.frags[f0:f1]

    def subset(self, idx) -> "Library":
        idx = np.asarray(idx, dtype=np.int64)
        ligs = [self.ligand(int(i)) for i in idx]
        out = Library.from_ligands(ligs, self.ligand_id[idx].copy())
        if self.atom_type is not None:
            out.atom_type = (np.concatenate([self.atom_type[int(self.atom_off[i]):int(self.atom_off[i + 1])] for i in idx])
                             if len(idx) else np.zeros(0, np.uint8)).astype(np.uint8)
        if self.frags is not None:
            out.frags = (np.concatenate([self.ligand_ranges(int(i))[1] for i in idx]) if len(idx)
                         else np.zeros((0, 4), np.int32)).astype(np.int32).reshape(-1, 4)
        return out

    def permuted(self, seed: int) -> "Library":
        """The same molecules with the atoms of every ligand renumbered by a seeded random
        permutation (coordinates, axes and moving sets remapped): the moving sets are then
        arbitrary atom subsets, not ranges.  Returns (library, perm): perm[g] = the global index
        in the new library of old global atom g (new.xyz[perm] == old.xyz)."""
        rng = np.random.Generator(np.random.PCG64(seed))
        ligs, perms = [], []
        for i in range(self.n):
            x, f = self.ligand(i)
            p = rng.permutation(len(x)).astype(np.int32)        # old index j -> new index p[j]
            nx = np.empty_like(x)
            nx[p] = x
            ligs.append((nx, Frags(p[f.axis] if len(f) else f.axis, [p[m] for m in f.moves])))
            perms.append(p.astype(np.int64) + int(self.atom_off[i]))
        out = Library.from_ligands(ligs, self.ligand_id.copy())
        perm = np.concatenate(perms) if perms else np.zeros(0, np.int64)
        if self.atom_type is not None:
            out.atom_type = np.empty_like(self.atom_type)
            out.atom_type[perm] = self.atom_type
        return out, perm


def ligands(n: int, seed: int, atoms=(20, 120), rot=(0, 20), first: int = 0, nthreads: int | None = None) -> Library:
    """Draw ligands first..first+n-1 of the seeded stream (prefix-stable)."""
    if n < 0 or atoms[0] < 1 or atoms[1] < atoms[0] or rot[0] < 0 or rot[1] < rot[0]:
        raise ValueError("inverted or invalid range")
    if atoms[1] > 256 or rot[1] > 32:
        raise ValueError("generator supports at most 256 atoms and 32 rotatable bonds")
    lib = _load()
    nthreads = nthreads or min(64, os.cpu_count() or 1)
    A = np.zeros(n, np.int32); R = np.zeros(n, np.int32); M = np.zeros(n, np.int32)
    rc = lib.vsgen_ligand_shapes(n, seed, first, atoms[0], atoms[1], rot[0], rot[1], _ptr(A), _ptr(R), _ptr(M), nthreads)
    if rc != 0:
        raise RuntimeError("vsgen_ligand_shapes failed")
    ao = np.zeros(n + 1, np.int64); ao[1:] = np.cumsum(A, dtype=np.int64)
    fo = np.zeros(n + 1, np.int64); fo[1:] = np.cumsum(R, dtype=np.int64)
    xyz = np.empty((int(ao[-1]), 3), np.float32)
    frags = np.empty((int(fo[-1]), 4), np.int32)
    rc = lib.vsgen_ligand_fill(n, seed, first, atoms[0], atoms[1], rot[0], rot[1], _ptr(ao), _ptr(fo), _ptr(xyz), _ptr(frags), nthreads)
    if rc != 0:
        raise RuntimeError("vsgen_ligand_fill failed")
    ids = np.arange(first, first + n, dtype=np.uint64)
    return Library.from_ranges(ids, ao, xyz, fo, frags, M)


def replicate(lib: Library, i: int, n: int) -> Library:
    """n copies of ligand i of `lib`, differing only in id."""
    if n < 0:
        raise ValueError("n must be >= 0")
    x, f = lib.ligand_ranges(i)
    A, R = len(x), len(f)
    ao = np.arange(n + 1, dtype=np.int64) * A
    fo = np.arange(n + 1, dtype=np.int64) * R
    xyz = np.tile(x, (n, 1)).astype(np.float32)
    fr = np.tile(f, (n, 1)).astype(np.int32).reshape(-1, 4)
    nm = None if lib.n_moving is None else np.full(n, lib.n_moving[i], np.int32)
    return Library.from_ranges(np.arange(n, dtype=np.uint64), ao, xyz, fo, fr, nm)


# ----------------------------------------------------------------------------- pocket

@dataclass
class Pocket:
    """A pocket grid: node (i,j,k) sits at origin + spacing*(i,j,k); values [nz,ny,nx] fp32, x fastest."""
    grid: np.ndarray        # float32 [nz, ny, nx]
    origin: tuple
    spacing: float
    center: tuple
    out_slope: float = 1.0  # kappa, energy per Angstrom of out-of-box excess (reading Q9)

    @property
    def dims(self):
        nz, ny, nx = self.grid.shape[-3:]
        return nx, ny, nz

    @property
    def n_channels(self) -> int:
        """Grid channels T: a 4-D grid [T, nz, ny, nx] is a typed pocket (Q24)."""
        return 1 if self.grid.ndim == 3 else int(self.grid.shape[0])


def pocket(seed: int, n=32, spacing: float = 1.0, n_receptor: int = 96,
           shell=(9.0, 13.0), mouth_deg: float = 50.0, out_slope: float = 1.0, center_offset=(0.0, 0.0, 0.0),
           origin=(0.0, 0.0, 0.0)) -> Pocket:
    """A synthetic pocket.  ``n`` = nx = ny = nz, or (nx, ny, nz).  The docking centre c is the
    grid centre moved by ``center_offset`` (Angstrom); the receptor shell surrounds c."""
    nx, ny, nz = (n, n, n) if np.isscalar(n) else tuple(int(v) for v in n)
    rng = np.random.Generator(np.random.PCG64(seed))
    origin = np.asarray(origin, np.float64)
    c = origin + spacing * (np.array([nx, ny, nz], np.float64) - 1) / 2.0 + np.asarray(center_offset, np.float64)
    pts = []
    cos_half = math.cos(math.radians(mouth_deg / 2.0))
    while len(pts) < n_receptor:
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        if v[2] > cos_half:          # the mouth: no receptor atoms inside the cone around +z
            continue
        r = rng.uniform(shell[0], shell[1])
        pts.append(c + r * v)
    P = np.array(pts)
    Z, Y, X = np.meshgrid(origin[2] + spacing * np.arange(nz), origin[1] + spacing * np.arange(ny),
                          origin[0] + spacing * np.arange(nx), indexing="ij")
    node = np.stack([X, Y, Z], axis=-1)                  # [nz, ny, nx, 3]
    G = 0.01 * np.sum((node - c) ** 2, axis=-1)
    for p in P:
        d2 = np.sum((node - p) ** 2, axis=-1)
        G += 5.0 * np.exp(-d2 / 2.0) - np.exp(-d2 / 8.0)
    return Pocket(G.astype(np.float32), tuple(float(v) for v in origin), float(spacing),
                  tuple(float(v) for v in c), float(out_slope))


# ----------------------------------------------------------------------------- atom types (Q24)

# Type t of a heavy atom (Q24 and section 4): 0 = C, 1 = N, 2 = O, 3 = S
# with drug-like frequencies; the pair table gives the attractive well depth of ligand type t
# against receptor type s (polar pairs bind more strongly, carbon-polar less).
TYPE_FREQ = (0.70, 0.13, 0.14, 0.03)
_WELL = np.array([[1.0, 0.6, 0.6, 1.1],
                  [0.6, 1.4, 1.8, 0.7],
                  [0.6, 1.8, 1.2, 0.7],
                  [1.1, 0.7, 0.7, 1.3]])


def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of uint64 counters, vectorised (the same mix as _splitmix64)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def atom_types(lib: Library, seed: int = 11, n_types: int = 4) -> np.ndarray:
    """uint8 type of every atom of ``lib`` (input order): a counter-based draw (splitmix64 of
    (seed, ligand id, atom index)) from TYPE_FREQ restricted to the first n_types types.  A
    function of the ligand id and atom index only, so slices and permutations keep their types."""
    if not 1 <= n_types <= len(TYPE_FREQ):
        raise ValueError("n_types must be in [1, 4]")
    A = lib.n_atoms.astype(np.int64)
    lid = np.repeat(lib.ligand_id.astype(np.uint64), A)
    j = (np.arange(int(lib.atom_off[-1]), dtype=np.int64) - np.repeat(lib.atom_off[:-1], A)).astype(np.uint64)
    with np.errstate(over="ignore"):
        key = (np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)) ^ (lid * np.uint64(0x9E3779B97F4A7C15)) ^ (
            j * np.uint64(0xBF58476D1CE4E5B9))
    u = (_splitmix64_np(key) >> np.uint64(11)).astype(np.float64) / 9007199254740992.0
    cdf = np.cumsum(np.array(TYPE_FREQ[:n_types]) / sum(TYPE_FREQ[:n_types]))
    return np.minimum(np.searchsorted(cdf, u, side="right"), n_types - 1).astype(np.uint8)


def typed_pocket(seed: int, n_types: int = 4, n=32, spacing: float = 1.0, n_receptor: int = 96,
                 shell=(9.0, 13.0), mouth_deg: float = 50.0, out_slope: float = 1.0,
                 center_offset=(0.0, 0.0, 0.0), origin=(0.0, 0.0, 0.0)) -> Pocket:
    """A typed pocket (Q24): the receptor of :func:`pocket` (same seed, same atoms) with a receptor
    type per atom (drawn from TYPE_FREQ); channel t holds, for a ligand atom of type t, the same
    confinement term plus per receptor atom s a repulsive core and an attractive well of depth
    _WELL[t, type(s)].  Grid [n_types, nz, ny, nx] float32."""
    base = pocket(seed, n, spacing, n_receptor, shell, mouth_deg, out_slope, center_offset, origin)
    nx, ny, nz = base.dims
    rng = np.random.Generator(np.random.PCG64(seed))
    cos_half = math.cos(math.radians(mouth_deg / 2.0))
    c = np.array(base.center)
    pts = []
    while len(pts) < n_receptor:   # the same draws as pocket(): the same receptor atoms
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        if v[2] > cos_half:
            continue
        pts.append(c + rng.uniform(shell[0], shell[1]) * v)
    rt = np.random.Generator(np.random.PCG64(seed + 7919)).choice(4, size=n_receptor, p=TYPE_FREQ)
    o = np.asarray(origin, np.float64)
    Z, Y, X = np.meshgrid(o[2] + spacing * np.arange(nz), o[1] + spacing * np.arange(ny),
                          o[0] + spacing * np.arange(nx), indexing="ij")
    node = np.stack([X, Y, Z], axis=-1)
    conf = 0.01 * np.sum((node - c) ** 2, axis=-1)
    G = np.empty((n_types, nz, ny, nx), np.float64)
    for t in range(n_types):
        g = conf.copy()
        for p, s in zip(pts, rt):
            d2 = np.sum((node - p) ** 2, axis=-1)
            g += 5.0 * np.exp(-d2 / 2.0) - _WELL[t, s] * np.exp(-d2 / 8.0)
        G[t] = g
    return Pocket(G.astype(np.float32), base.origin, base.spacing, base.center, base.out_slope)


# ----------------------------------------------------------------------------- tables

_M64 = (1 << 64) - 1


def _splitmix64(state: int):
    state = (state + 0x9E3779B97F4A7C15) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return state, z ^ (z >> 31)


def pose_table(P: int, seed: int = 7, tau: float = 0.0):
    """(rot [P,3,3] float32 row-major, trans [P,3] float32).  p = 0 is the identity.

    tau > 0: every pose p >= 1 also carries a translation tau_p drawn uniformly in the ball of
    radius tau (Angstrom) from the same splitmix64 stream (reading Q7 sets tau = 0 by default)."""
    rot = np.zeros((P, 3, 3), np.float64)
    for p in range(P):
        if p == 0:
            rot[p] = np.eye(3)
            continue
        s = (seed * 0xD1B54A32D192ED03 ^ (p * 0x9E3779B97F4A7C15)) & _M64
        s, a = _splitmix64(s)
        s, b = _splitmix64(s)
        s, d = _splitmix64(s)
        u1, u2, u3 = [(x >> 11) / 9007199254740992.0 for x in (a, b, d)]
        x = math.sqrt(1 - u1) * math.sin(2 * math.pi * u2)
        y = math.sqrt(1 - u1) * math.cos(2 * math.pi * u2)
        z = math.sqrt(u1) * math.sin(2 * math.pi * u3)
        w = math.sqrt(u1) * math.cos(2 * math.pi * u3)
        rot[p] = [[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                  [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                  [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]]
    trans = np.zeros((P, 3), np.float64)
    if tau > 0:
        for p in range(1, P):
            s = (seed * 0x9E3779B97F4A7C15 ^ (p * 0xD1B54A32D192ED03) ^ 0x5851F42D4C957F2D) & _M64
            while True:
                v = []
                for _ in range(3):
                    s, a = _splitmix64(s)
                    v.append(2.0 * ((a >> 11) / 9007199254740992.0) - 1.0)
                if v[0] * v[0] + v[1] * v[1] + v[2] * v[2] <= 1.0:
                    break
            trans[p] = tau * np.array(v)
    return rot.astype(np.float32), trans.astype(np.float32)


def refine_table(delta: float = 0.25, degrees: float = 10.0):
    """Rigid refinement move table (Q23): (rot [J,3,3] float32, trans
    [J,3] float32, Angstrom).  Move 0 is the identity (exactly); then +-delta translations along
    x, y, z and +-degrees rotations about x, y, z (about the pose centroid): J = 13."""
    rots = [np.eye(3)]
    trs = [np.zeros(3)]
    for a in range(3):
        for sg in (1.0, -1.0):
            t = np.zeros(3)
            t[a] = sg * delta
            rots.append(np.eye(3))
            trs.append(t)
    th = math.radians(degrees)
    for a in range(3):
        for sg in (1.0, -1.0):
            c, s_ = math.cos(sg * th), math.sin(sg * th)
            b, d = (a + 1) % 3, (a + 2) % 3
            m = np.eye(3)
            m[b, b] = c
            m[b, d] = -s_
            m[d, b] = s_
            m[d, d] = c
            rots.append(m)
            trs.append(np.zeros(3))
    return np.array(rots, np.float32), np.array(trs, np.float32)


def angle_table(K: int) -> np.ndarray:
    """[K,2] float32 (cos, sin) of theta_k = 2 pi k / K; entry 0 is exactly (1, 0)."""
    t = np.array([[math.cos(2 * math.pi * k / K), math.sin(2 * math.pi * k / K)] for k in range(K)])
    t[0] = (1.0, 0.0)
    return t.astype(np.float32)


# ----------------------------------------------------------------------------- configs

# BASELINE.json configs[i] -> concrete synthetic inputs
CONFIGS = {
    "C1": dict(n=16, atoms=(20, 40), rot=(0, 4), seed=1, P=8, K=8, pockets=(101,)),
    "C2": dict(n=10_000, atoms=(20, 120), rot=(0, 20), seed=2, P=64, K=8, pockets=(101,)),
    "C3": dict(n=8_192, atoms=(80, 150), rot=(15, 25), seed=3, P=64, K=8, pockets=(101,)),
    "C4": dict(n=1_000_000, atoms=(20, 120), rot=(0, 20), seed=4, P=64, K=8, pockets=(101,)),
    "C5": dict(n=1_000_000, atoms=(20, 120), rot=(0, 20), seed=4, P=64, K=8, pockets=(101, 102, 103, 104)),
}
