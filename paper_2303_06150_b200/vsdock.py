"""ctypes binding of include/vsdock.h (argument marshalling only).

Every step of the hot path runs in libvsdock.so's CUDA kernels; this module
only converts numpy / torch buffers to pointers, owns the device workspace (a
torch uint8 tensor) and hands the library torch's current CUDA stream.  There
is no CPU fallback: if the library or a CUDA device is missing, constructing an
:class:`Engine` raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libvsdock.so")

VS_OK, VS_E_ARG, VS_E_PARSE, VS_E_OVERFLOW_ATOMS, VS_E_OVERFLOW_ROTAMERS = 0, -1, -2, -3, -4
VS_E_NOFIT, VS_E_WORKSPACE, VS_E_CUDA, VS_E_STATE = -5, -6, -7, -9
_NAMES = {0: "VS_OK", -1: "VS_E_ARG", -2: "VS_E_PARSE", -3: "VS_E_OVERFLOW_ATOMS", -4: "VS_E_OVERFLOW_ROTAMERS",
          -5: "VS_E_NOFIT", -6: "VS_E_WORKSPACE", -7: "VS_E_CUDA", -9: "VS_E_STATE"}

SYMBOLS = ["vs_create", "vs_destroy", "vs_last_error", "vs_workspace_size", "vs_set_workspace", "vs_load_pocket",
           "vs_set_pose_table", "vs_set_angle_table", "vs_submit", "vs_wait", "vs_get_results", "vs_get_coords",
           "vs_get_pose_debug", "vs_local_topk", "vs_keys", "vs_select_keys", "vs_merge_topk", "vs_get_manifest", "vs_query_classes",
           "vs_score_points", "vs_get_stats", "vs_plan_boundaries", "vs_plan_lpt", "vs_set_refine_table", "vs_get_refine",
           "vs_get_pose_refine_debug", "vs_load_pocket_typed", "vs_submit_typed", "vs_score_points_typed"]


class VsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code
        import re
        m = re.search(r"ligand (\d+)", msg or "")
        self.ligand = int(m.group(1)) if m else None


class vs_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("n_sweeps", ctypes.c_int32), ("n_atom_clusters", ctypes.c_int32),
                ("n_rot_clusters", ctypes.c_int32), ("atom_upper_bound", ctypes.c_int32),
                ("rot_upper_bound", ctypes.c_int32), ("bucket_multiple", ctypes.c_int32),
                ("n_streams", ctypes.c_int32), ("rank", ctypes.c_int32), ("world_size", ctypes.c_int32),
                ("debug_poses", ctypes.c_int32), ("launch_per_bucket", ctypes.c_int32),
                ("bucket_capacity", ctypes.c_int32), ("n_move_clusters", ctypes.c_int32),
                ("move_upper_bound", ctypes.c_int32), ("fused_sites", ctypes.c_int32), ("stream", ctypes.c_void_p)]


class vs_pocket_desc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("origin", ctypes.c_float * 3), ("spacing", ctypes.c_float), ("center", ctypes.c_float * 3),
                ("out_slope", ctypes.c_float)]


class vs_ligand_batch(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("ligand_id", ctypes.c_void_p), ("atom_off", ctypes.c_void_p),
                ("xyz", ctypes.c_void_p), ("frag_off", ctypes.c_void_p), ("frag_axis", ctypes.c_void_p),
                ("move_off", ctypes.c_void_p), ("move_atoms", ctypes.c_void_p), ("on_device", ctypes.c_int32)]


class vs_bucket(ctypes.Structure):
    _fields_ = [("cell", ctypes.c_int32), ("atom_class", ctypes.c_int32), ("rot_class", ctypes.c_int32),
                ("atom_bound", ctypes.c_int32), ("kernel_atoms", ctypes.c_int32), ("capacity", ctypes.c_int32),
                ("size", ctypes.c_int32), ("owner", ctypes.c_int32), ("launch_order", ctypes.c_int32),
                ("move_class", ctypes.c_int32), ("start", ctypes.c_int64), ("weight", ctypes.c_uint64)]


class vs_class_info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("atom_bound", "kernel_atoms", "warps_per_cta", "threads_per_cta",
                                              "regs_per_thread", "static_smem", "dyn_smem", "blocks_per_sm",
                                              "sm_count", "ligands_per_cta", "l", "capacity")]


class vs_stats(ctypes.Structure):
    _fields_ = [("n_ligands", ctypes.c_int64), ("n_owned", ctypes.c_int64), ("n_buckets", ctypes.c_int64),
                ("n_owned_buckets", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("dock_launches", ctypes.c_int64), ("fused_launches", ctypes.c_int64), ("evals_alg", ctypes.c_double),
                ("h2d_bytes", ctypes.c_uint64),
                ("prep_ms", ctypes.c_float),
                ("dock_ms", ctypes.c_float), ("topk_ms", ctypes.c_float)]


_lib = None


def load_library():
    """Load libvsdock.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} is missing; run __graft_entry__.build() (nvcc, sm_100a)")
    lib = ctypes.CDLL(SO_PATH)
    P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    sig = {
        "vs_create": [ctypes.POINTER(vs_config), ctypes.POINTER(P)],
        "vs_destroy": [P],
        "vs_last_error": [P],
        "vs_workspace_size": [P, I64, I64, I64, I64, I32, I32, ctypes.POINTER(SZ)],
        "vs_set_workspace": [P, P, SZ],
        "vs_load_pocket": [P, ctypes.POINTER(vs_pocket_desc), P, I32, ctypes.POINTER(I32)],
        "vs_set_pose_table": [P, I32, P, P],
        "vs_set_angle_table": [P, I32, P],
        "vs_submit": [P, ctypes.POINTER(vs_ligand_batch), P, I32],
        "vs_wait": [P],
        "vs_get_results": [P, I32, P, P, P, P, I32],
        "vs_get_coords": [P, I32, P, I32],
        "vs_get_pose_debug": [P, I32, P, P],
        "vs_set_refine_table": [P, I32, I32, P, P],
        "vs_get_refine": [P, I32, P, I32],
        "vs_get_pose_refine_debug": [P, I32, P],
        "vs_local_topk": [P, I32, I32, P, ctypes.POINTER(I32)],
        "vs_keys": [P, I32, ctypes.c_uint32, P, ctypes.POINTER(I64)],
        "vs_select_keys": [P, P, I64, I32, P],
        "vs_merge_topk": [P, P, I64, I32, P, P, P, ctypes.POINTER(I32)],
        "vs_get_manifest": [P, I32, P, ctypes.POINTER(I32), P],
        "vs_query_classes": [P, I32, P, ctypes.POINTER(I32)],
        "vs_score_points": [P, I32, I64, P, P],
        "vs_get_stats": [P, ctypes.POINTER(vs_stats)],
        "vs_plan_boundaries": [I32, I32, I32, I32, P, ctypes.POINTER(I32), P, ctypes.POINTER(I32)],
        "vs_plan_lpt": [P, I32, I32, P, P],
        "vs_load_pocket_typed": [P, ctypes.POINTER(vs_pocket_desc), I32, P, I32, ctypes.POINTER(I32)],
        "vs_submit_typed": [P, ctypes.POINTER(vs_ligand_batch), P, P, I32],
        "vs_score_points_typed": [P, I32, I64, P, P, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = None if name == "vs_destroy" else (ctypes.c_char_p if name == "vs_last_error" else I32)
    _lib = lib
    return lib


def _ptr(x):
    """Pointer of a numpy array or torch tensor (None passes through)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return ctypes.c_void_p(x.ctypes.data)
    assert x.is_contiguous()
    return ctypes.c_void_p(x.data_ptr())


def plan_boundaries(n_atom_clusters, atom_ub, n_rot_clusters, rot_ub):
    """Host-only a2 class boundaries exactly as vs_submit computes them (no GPU needed)."""
    lib = load_library()
    ab = np.zeros(8, np.int32)
    rb = np.zeros(33, np.int32)
    na, nr = ctypes.c_int32(), ctypes.c_int32()
    rc = lib.vs_plan_boundaries(n_atom_clusters, atom_ub, n_rot_clusters, rot_ub, _ptr(ab), ctypes.byref(na),
                                _ptr(rb), ctypes.byref(nr))
    if rc != VS_OK:
        raise VsError(rc, "vs_plan_boundaries")
    return list(ab[: na.value]), list(rb[: nr.value])


def plan_lpt(weights, world):
    """Host-only a4 LPT plan exactly as vs_submit computes it: (owner[b], launch_order[b])."""
    lib = load_library()
    w = np.ascontiguousarray(weights, np.uint64)
    owner = np.zeros(max(1, len(w)), np.int32)
    order = np.zeros(max(1, len(w)), np.int32)
    rc = lib.vs_plan_lpt(_ptr(w), len(w), world, _ptr(owner), _ptr(order))
    if rc != VS_OK:
        raise VsError(rc, "vs_plan_lpt")
    return owner[: len(w)], order[: len(w)]


@dataclass
class Results:
    ligand_id: np.ndarray    # uint64 [n]
    best_score: np.ndarray   # float32 [n]
    best_pose: np.ndarray    # int32 [n]
    angles: np.ndarray       # uint8 [S_w * sum R]


class Engine:
    """One context per GPU (include/vsdock.h).  Device memory and the stream come from torch."""

    def __init__(self, device: int = 0, n_sweeps: int = 1, atom_clusters: int = 6, rot_clusters: int = 23,
                 atom_upper_bound: int = 0, rot_upper_bound: int = 0, bucket_multiple: int = 16, n_streams: int = 4,
                 rank: int = 0, world_size: int = 1, debug_poses: bool = False, launch_per_bucket: bool = False,
                 bucket_capacity: int = 0, move_clusters: int = 1, move_upper_bound: int = 0,
                 fused_sites: bool = False, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("vsdock needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        self._torch = torch
        self.lib = load_library()
        self.device = device
        self.n_sweeps = n_sweeps
        torch.cuda.set_device(device)
        st = stream if stream is not None else torch.cuda.current_stream(device)
        self._stream = st
        cfg = vs_config(device, n_sweeps, atom_clusters, rot_clusters, atom_upper_bound, rot_upper_bound,
                        bucket_multiple, n_streams, rank, world_size, int(debug_poses), int(launch_per_bucket),
                        int(bucket_capacity), int(move_clusters), int(move_upper_bound), int(bool(fused_sites)),
                        ctypes.c_void_p(st.cuda_stream))
        h = ctypes.c_void_p()
        self._check(self.lib.vs_create(ctypes.byref(cfg), ctypes.byref(h)), None)
        self.h = h
        self.ws = None
        self.P = self.K = None
        self.n_ref = 0
        self._n = 0
        self._batch_keep = None

    def _check(self, rc, h="self"):
        if rc != VS_OK:
            hh = self.h if h == "self" else None
            msg = self.lib.vs_last_error(hh).decode() if hh else ""
            raise VsError(rc, msg)

    def close(self):
        if getattr(self, "h", None):
            self.lib.vs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- tables and pockets
    def set_poses(self, rot, trans):
        rot = np.ascontiguousarray(rot, np.float32).reshape(-1, 9)
        trans = np.ascontiguousarray(trans, np.float32).reshape(-1, 3)
        self._check(self.lib.vs_set_pose_table(self.h, rot.shape[0], _ptr(rot), _ptr(trans)))
        self.P = rot.shape[0]

    def set_angles(self, cs):
        cs = np.ascontiguousarray(cs, np.float32).reshape(-1, 2)
        self._check(self.lib.vs_set_angle_table(self.h, cs.shape[0], _ptr(cs)))
        self.K = cs.shape[0]

    def set_refine(self, n_rounds, rot=None, trans=None):
        """Rigid refinement after the sweeps (Q23): ``n_rounds`` greedy
        rounds over the move table (rot [J,3,3], trans [J,3] Angstrom; move 0 = identity).  0 = off."""
        if not n_rounds:
            self._check(self.lib.vs_set_refine_table(self.h, 0, 0, None, None))
            self.n_ref = 0
            return
        rot = np.ascontiguousarray(rot, np.float32).reshape(-1, 9)
        trans = np.ascontiguousarray(trans, np.float32).reshape(-1, 3)
        self._check(self.lib.vs_set_refine_table(self.h, int(n_rounds), rot.shape[0], _ptr(rot), _ptr(trans)))
        self.n_ref = int(n_rounds)

    def refine(self, slot=0) -> np.ndarray:
        """Refinement moves of every ligand's best pose, uint8 [n, n_rounds] (0xFF: another rank's)."""
        out = np.zeros((max(1, self._n), max(1, self.n_ref)), np.uint8)
        if self.n_ref:
            self._check(self.lib.vs_get_refine(self.h, slot, _ptr(out), 0))
        return out[: self._n, : self.n_ref]

    def pose_refine_debug(self, slot=0) -> np.ndarray:
        """Every pose's refinement moves, uint8 [n, P, n_rounds] (requires debug_poses)."""
        out = np.zeros((max(1, self._n), self.P, max(1, self.n_ref)), np.uint8)
        if self.n_ref:
            self._check(self.lib.vs_get_pose_refine_debug(self.h, slot, _ptr(out)))
        return out[: self._n, :, : self.n_ref]

    def load_pocket(self, pocket) -> int:
        """Load a pocket grid [nz, ny, nx], or a typed pocket [T, nz, ny, nx] (Q24: vs_load_pocket_typed)."""
        g = np.ascontiguousarray(pocket.grid, np.float32)
        nz, ny, nx = g.shape[-3:]
        d = vs_pocket_desc(nx, ny, nz, (ctypes.c_float * 3)(*pocket.origin), pocket.spacing,
                           (ctypes.c_float * 3)(*pocket.center), pocket.out_slope)
        pid = ctypes.c_int32()
        if g.ndim == 4:
            self._check(self.lib.vs_load_pocket_typed(self.h, ctypes.byref(d), g.shape[0], _ptr(g), 0, ctypes.byref(pid)))
        else:
            self._check(self.lib.vs_load_pocket(self.h, ctypes.byref(d), _ptr(g), 0, ctypes.byref(pid)))
        return pid.value

    # ---- workspace
    def reserve(self, n_lig, n_atoms, n_frags, n_moving, max_atoms, n_pockets):
        nbytes = ctypes.c_size_t()
        self._check(self.lib.vs_workspace_size(self.h, n_lig, n_atoms, n_frags, n_moving, max_atoms, n_pockets,
                                               ctypes.byref(nbytes)))
        if self.ws is None or self.ws.numel() < nbytes.value:
            if self.ws is not None:
                # the library queues work on the engine's stream: the old block must not be
                # handed to another allocation while that work can still touch it
                self._stream.synchronize()
            self.ws = None
            self.ws = self._torch.empty(nbytes.value, dtype=self._torch.uint8, device=f"cuda:{self.device}")
            self._check(self.lib.vs_set_workspace(self.h, ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel()))
        return nbytes.value

    # ---- the hot path
    def submit(self, ligand_id, atom_off, xyz, frag_off, frag_axis, move_off, move_atoms, pockets, on_device=None,
               max_atoms=None, atom_type=None):
        """Submit a CSR ligand batch in the general form of include/vsdock.h (numpy host arrays,
        pinned torch CPU tensors, or CUDA tensors; ``ligand_id`` may be None).  on_device: 0 host
        (copied), 1 device, 2 pinned host read in place by the kernels (owned ligands only).
        ``atom_type`` (uint8 per atom, same memory kind): a typed submit (vs_submit_typed, Q24)."""
        n = int(atom_off.shape[0]) - 1
        if on_device is None:
            on_device = hasattr(xyz, "is_cuda") and xyz.is_cuda
        on_device = int(on_device)
        if max_atoms is None:
            if on_device == 1:
                max_atoms = int((atom_off[1:] - atom_off[:-1]).max().item()) if n > 0 else 1
            else:
                max_atoms = int(np.diff(np.asarray(atom_off)).max()) if n > 0 else 1
        nA = int(xyz.shape[0])
        nR = int(frag_axis.shape[0])
        nM = int(move_atoms.shape[0])
        pockets = np.ascontiguousarray(pockets, np.int32).reshape(-1)
        self.reserve(n, nA, nR, nM, max(1, min(256, max_atoms)), len(pockets))
        b = vs_ligand_batch(n, _ptr(ligand_id), _ptr(atom_off), _ptr(xyz), _ptr(frag_off), _ptr(frag_axis),
                            _ptr(move_off), _ptr(move_atoms), on_device)
        self._batch_keep = (ligand_id, atom_off, xyz, frag_off, frag_axis, move_off, move_atoms, atom_type)
        if atom_type is not None:
            if hasattr(atom_type, "data_ptr"):
                assert str(atom_type.dtype) == "torch.uint8", "atom_type must be uint8"
            else:
                atom_type = np.ascontiguousarray(atom_type, np.uint8)
                self._batch_keep = self._batch_keep[:-1] + (atom_type,)
            self._check(self.lib.vs_submit_typed(self.h, ctypes.byref(b), _ptr(atom_type), _ptr(pockets), len(pockets)))
        else:
            self._check(self.lib.vs_submit(self.h, ctypes.byref(b), _ptr(pockets), len(pockets)))
        self._n, self._nA, self._nR = n, nA, nR
        self._npk = len(pockets)

    def submit_library(self, lib, pockets, **kw):
        """Submit a vsgen.Library-like batch; its ``atom_type`` (if any) makes the submit typed (Q24)."""
        if kw.get("atom_type") is None and getattr(lib, "atom_type", None) is not None:
            kw["atom_type"] = lib.atom_type
        return self.submit(*lib.arrays(), pockets, **kw)

    def wait(self):
        self._check(self.lib.vs_wait(self.h))

    def results(self, slot=0) -> Results:
        i = np.empty(max(1, self._n), np.uint64)
        s = np.empty(self._n, np.float32)
        p = np.empty(self._n, np.int32)
        a = np.empty(max(1, self.n_sweeps * self._nR), np.uint8)
        self._check(self.lib.vs_get_results(self.h, slot, _ptr(i), _ptr(s), _ptr(p), _ptr(a), 0))
        return Results(i[: self._n], s, p, a[: self.n_sweeps * self._nR])

    def results_into(self, slot, best_score, best_pose, angles=None, ligand_id=None):
        """Copy the results into caller-owned HOST arrays (pinned for full-speed DMA)."""
        self._check(self.lib.vs_get_results(self.h, slot, _ptr(ligand_id), _ptr(best_score), _ptr(best_pose),
                                            _ptr(angles), 0))

    def results_device(self, slot, best_score, best_pose, angles=None, ligand_id=None):
        self._check(self.lib.vs_get_results(self.h, slot, _ptr(ligand_id), _ptr(best_score), _ptr(best_pose),
                                            _ptr(angles), 1))

    def coords(self, slot=0) -> np.ndarray:
        out = np.empty((max(1, self._nA), 3), np.float32)
        self._check(self.lib.vs_get_coords(self.h, slot, _ptr(out), 0))
        return out[: self._nA]

    def coords_into(self, slot, out, mode=2):
        """Best-pose coordinates into a caller-owned buffer [n_atoms, 3]: mode 2 = pinned host,
        asynchronous (complete after the next wait / submit on this engine), 0 = host, 1 = device."""
        self._check(self.lib.vs_get_coords(self.h, slot, _ptr(out), mode))

    def results_async(self, slot, best_score, best_pose, angles=None, ligand_id=None):
        """Results into pinned HOST arrays, asynchronously on the engine's stream."""
        self._check(self.lib.vs_get_results(self.h, slot, _ptr(ligand_id), _ptr(best_score), _ptr(best_pose),
                                            _ptr(angles), 2))

    def select_keys(self, keys_dev, k, out=None):
        """Device top-k (ascending, UINT64_MAX padded) of a device int64 key tensor."""
        if out is None:
            out = self._torch.empty(k, dtype=self._torch.int64, device=f"cuda:{self.device}")
        self._check(self.lib.vs_select_keys(self.h, _ptr(keys_dev), int(keys_dev.numel()), k, _ptr(out)))
        return out

    def synchronize(self):
        self._stream.synchronize()

    def pose_debug(self, slot=0):
        s = np.empty((self._n, self.P), np.float32)
        a = np.empty(max(1, self.P * self.n_sweeps * self._nR), np.uint8)
        self._check(self.lib.vs_get_pose_debug(self.h, slot, _ptr(s), _ptr(a)))
        return s, a[: self.P * self.n_sweeps * self._nR]

    def local_topk(self, slot, k):
        """Device tensor [k] of uint64 keys (as int64) and the number of valid entries."""
        t = self._torch.empty(k, dtype=self._torch.int64, device=f"cuda:{self.device}")
        nv = ctypes.c_int32()
        self._check(self.lib.vs_local_topk(self.h, slot, k, _ptr(t), ctypes.byref(nv)))
        return t, nv.value

    def keys_into(self, slot, out, index_offset=0):
        """Write this rank's (score, ligand index + index_offset) keys for ``slot`` into the
        DEVICE int64 tensor ``out`` (asynchronous); returns how many were written."""
        nk = ctypes.c_int64()
        self._check(self.lib.vs_keys(self.h, slot, int(index_offset), _ptr(out), ctypes.byref(nk)))
        return nk.value

    def merge_topk(self, keys_dev, k, with_ids=False):
        """Global top-k of gathered keys: (ligand index, score[, ligand id of the last batch])."""
        idx = np.empty(k, np.int64)
        sc = np.empty(k, np.float32)
        ids = np.empty(k, np.uint64) if with_ids else None
        m = ctypes.c_int32()
        self._check(self.lib.vs_merge_topk(self.h, _ptr(keys_dev), int(keys_dev.numel()), k, _ptr(idx), _ptr(sc),
                                           _ptr(ids), ctypes.byref(m)))
        if with_ids:
            return idx[: m.value], sc[: m.value], ids[: m.value]
        return idx[: m.value], sc[: m.value]

    def manifest(self, want_perm=True):
        nb = ctypes.c_int32()
        self._check(self.lib.vs_get_manifest(self.h, 0, None, ctypes.byref(nb), None))
        arr = (vs_bucket * max(1, nb.value))()
        perm = np.empty(max(1, self._n), np.uint32) if want_perm else None
        self._check(self.lib.vs_get_manifest(self.h, nb.value, arr, ctypes.byref(nb), _ptr(perm)))
        keys = [f[0] for f in vs_bucket._fields_]
        buckets = [{k: getattr(arr[i], k) for k in keys} for i in range(nb.value)]
        return buckets, (perm[: self._n] if want_perm else None)

    def classes(self):
        n = ctypes.c_int32()
        self._check(self.lib.vs_query_classes(self.h, 0, None, ctypes.byref(n)))
        arr = (vs_class_info * max(1, n.value))()
        self._check(self.lib.vs_query_classes(self.h, n.value, arr, ctypes.byref(n)))
        keys = [f[0] for f in vs_class_info._fields_]
        return [{k: getattr(arr[i], k) for k in keys} for i in range(n.value)]

    def stats(self):
        s = vs_stats()
        self._check(self.lib.vs_get_stats(self.h, ctypes.byref(s)))
        return {f[0]: getattr(s, f[0]) for f in vs_stats._fields_}

    def score_points(self, pocket_id, pts, types=None):
        """g at points (Angstrom) by the dock kernel's device function; ``types`` (Q24): the channel
        of every point of a typed pocket (the TYPED layout's path)."""
        pts = np.ascontiguousarray(pts, np.float32).reshape(-1, 3)
        out = np.empty(pts.shape[0], np.float32)
        if types is not None:
            t = np.ascontiguousarray(types, np.uint8).reshape(-1)
            self._check(self.lib.vs_score_points_typed(self.h, pocket_id, pts.shape[0], _ptr(pts), _ptr(t), _ptr(out)))
        else:
            self._check(self.lib.vs_score_points(self.h, pocket_id, pts.shape[0], _ptr(pts), _ptr(out)))
        return out
