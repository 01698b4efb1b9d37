"""Double-buffered host -> results pipeline.

LiGen overlaps transfers with compute by handing buckets to CPU "workers" that copy
into a free device buffer, run, and copy results back ("double buffering technique
for hiding data transfers").  On B200 the same overlap needs no worker pool: the
library is cut into chunks, and two contexts (engines, each with its own device
workspace and stream) alternate over them:

* chunk c + 1's host-to-device copy runs on a copy stream (the H2D copy engine) while
  chunk c is prepared and docked;
* chunk c's outputs -- best score, best pose, angle indices and the best-pose
  coordinates (a9, replayed by the finalize kernel) -- are read back ASYNCHRONOUSLY into
  pinned host buffers on chunk c's own stream (the D2H copy engine), so they overlap the
  docking of chunk c + 1 on the other engine;
* every chunk's ranking keys are written on the device (vs_keys, index = library index);
  at the end one device top-k selection (vs_select_keys) gives this rank's list, which is
  all-gathered across ranks (NCCL) and merged (vs_merge_topk) -- no host round trip of
  keys.

Compute phases still serialise on the SMs (the persistent dock kernel holds one CTA per
SM), which is the point: the copy engines work under it.
"""
from __future__ import annotations

import numpy as np

from .vsdock import Engine


def chunk_bounds(n: int, chunks: int = 0, first: int = 32, growth: int = 4):
    """Chunk boundaries of an n-ligand library.  chunks > 0: equal chunks.  chunks = 0: a
    geometric ramp at both ends -- first chunk n / first, each next one up to `growth` times
    the previous, mirrored at the end -- so only a small first upload and a small last
    read-back are exposed while every other copy hides under a neighbour's docking."""
    if n <= 0:
        return [0, 0]
    if chunks > 0:
        chunks = min(int(chunks), n)
        return [n * c // chunks for c in range(chunks + 1)]
    ramp, size = [], max(1, n // first)
    while 2 * (sum(ramp) + size) <= n and len(ramp) < 8:
        ramp.append(size)
        size *= growth
    mid = n - 2 * sum(ramp)
    cap = growth * ramp[-1] if ramp else mid       # middle pieces stay within `growth` of the ramp
    pieces = -(-mid // cap) if mid > 0 else 0
    midl = [mid * (j + 1) // pieces - mid * j // pieces for j in range(pieces)]
    sizes = ramp + midl + ramp[::-1]
    b = [0]
    for s in sizes:
        b.append(b[-1] + s)
    return b


class PipelinedDocker:
    """Dock a host-resident library in chunks over two alternating engines; copies in both
    directions overlap the docking."""

    def __init__(self, device: int = 0, n_engines: int = 2, **engine_kw):
        import torch
        self._torch = torch
        self.device = device
        self.dev = torch.device(f"cuda:{device}")
        self.copy = torch.cuda.Stream(device=device)
        self.streams = [torch.cuda.Stream(device=device) for _ in range(max(1, int(n_engines)))]
        self.engines = [Engine(device=device, stream=s, **engine_kw) for s in self.streams]
        self.engine = self.engines[0]
        self.n_sweeps = self.engine.n_sweeps
        self._pinned = {}
        self.trace = []

    def setup(self, rot, trans, cs, pockets):
        for e in self.engines:
            e.set_poses(rot, trans)
            e.set_angles(cs)
            ids = [e.load_pocket(p) for p in pockets]
        self.pocket_ids = ids
        return ids

    def _pin(self, name, shape, dtype):
        """Reusable pinned host output buffer (allocating page-locked memory per run would cost
        more than the copies)."""
        torch = self._torch
        key = (name, tuple(shape), dtype)
        if key not in self._pinned:
            self._pinned[key] = torch.empty(tuple(shape), dtype=dtype).pin_memory()
        return self._pinned[key].numpy()

    @staticmethod
    def _slices(arrays, lo, hi):
        """Chunk [lo, hi) as views of the caller's arrays: offsets keep their library values (the
        library rebases them on the device, vs_ligand_batch), data arrays start at the chunk's
        first element -- no host-side arithmetic on the critical path."""
        ids, atom_off, xyz, frag_off, frag_axis, move_off, move_atoms = arrays[:7]
        a0, a1 = int(atom_off[lo]), int(atom_off[hi])
        f0, f1 = int(frag_off[lo]), int(frag_off[hi])
        m0, m1 = int(move_off[f0]), int(move_off[f1])
        out = [ids[lo:hi], atom_off[lo:hi + 1], xyz[a0:a1], frag_off[lo:hi + 1], frag_axis[f0:f1],
               move_off[f0:f1 + 1], move_atoms[m0:m1]]
        if len(arrays) > 7:            # atom types of a typed run (Q24), sliced like xyz
            out.append(arrays[7][a0:a1])
        return out, (a0, a1, f0, f1)

    def _issue_copy(self, arrays, lo, hi):
        """Chunk [lo, hi) to the device on the copy stream (pinned sources: asynchronous)."""
        torch = self._torch
        host, box = self._slices(arrays, lo, hi)
        host = [h if isinstance(h, torch.Tensor) else torch.from_numpy(np.asarray(h)) for h in host]
        with torch.cuda.stream(self.copy):
            dev = []
            for h in host:
                # 8 MB pieces: one copy engine serves every stream's H2D one request at a time,
                # and the other engine's small preparation copies must not wait behind a whole
                # chunk upload
                d = torch.empty(h.shape, dtype=h.dtype, device=self.dev)
                fd, fh = d.reshape(-1), h.reshape(-1)
                step = max(1, (8 << 20) // max(1, h.element_size()))
                for i in range(0, fh.numel(), step):
                    fd[i:i + step].copy_(fh[i:i + step], non_blocking=True)
                dev.append(d)
            ev = torch.cuda.Event()
            ev.record(self.copy)
        return dev, ev, box

    def run(self, ligand_id, atom_off, xyz, frag_off, frag_axis, move_off, move_atoms, k: int = 1000,
            chunks: int = 0, max_atoms: int = 256, group=None, coords: bool = True, first: int = 32,
            growth: int = 4, zero_copy=None, atom_type=None, library_copy: bool = True):
        """Dock the library (the C-ABI's general-form CSR arrays; pinned torch CPU tensors for
        overlapped copies) into every pocket of ``setup``.  ``zero_copy`` (default: with more than
        one rank): the kernels read each rank's ligands straight from the pinned host arrays
        (on_device = 2) instead of every rank uploading the whole library.  Returns a dict of host
        arrays:

        ``ligand_id`` [n], ``best_score`` / ``best_pose`` [pockets, n], ``angles`` [pockets, S_w * sum R],
        ``xyz`` [pockets, sum A, 3] (best-pose coordinates, input atom order; with ``coords``), and
        ``topk`` = per pocket (library index [m], score [m], ligand id [m]), merged across ranks.
        The per-ligand arrays are reused buffers: copy them to keep them past the next run.
        ``atom_type`` (uint8 per atom, pinned like the rest): a typed run (vs_submit_typed, Q24).
        ``library_copy`` (default): hand each chunk's pinned host slices to the C-ABI (vs_submit
        with on_device = 0: the library issues the host-to-device copies on the engine's stream,
        so chunk i + 1's upload on one engine overlaps chunk i's docking on the other); False:
        stage them with torch copies on a separate copy stream (measured equal on B200:
        8.59 vs 8.61 M ligands/s, profiles/r02c_e2e_pipeline_sweep.txt)."""
        from . import parallel
        from .vsdock import VsError
        torch = self._torch
        import torch.distributed as dist
        if zero_copy is None:
            zero_copy = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
        n = int(atom_off.shape[0]) - 1
        nA, nR = int(xyz.shape[0]), int(frag_axis.shape[0])
        npk = len(self.pocket_ids)
        S_w = self.n_sweeps
        bounds = chunk_bounds(n, chunks, first, growth)
        nch = len(bounds) - 1
        best = self._pin("best", (npk, n), torch.float32)
        pose = self._pin("pose", (npk, n), torch.int32)
        ang = self._pin("ang", (npk, max(1, S_w * nR)), torch.uint8)
        xyz_out = self._pin("xyz", (npk, max(1, nA), 3), torch.float32) if coords else None
        all_keys = [torch.empty(max(1, n), dtype=torch.int64, device=self.dev) for _ in range(npk)]
        nkeys = [0] * npk
        arrays = (ligand_id, atom_off, xyz, frag_off, frag_axis, move_off, move_atoms)
        if atom_type is not None:
            arrays = arrays + (atom_type,)
        self.trace = []
        ne = len(self.engines)
        staged = not zero_copy and not library_copy     # torch copies on the copy stream
        inflight = {} if not staged else {c: self._issue_copy(arrays, bounds[c], bounds[c + 1])
                                          for c in range(min(ne, nch))}
        keep = {}
        failed = None
        pending = None

        def readback(e, lo, hi, a0, a1, f0, f1):
            """Asynchronous a9 read-back of one chunk into the pinned outputs (engine e's stream:
            after its docking)."""
            for s in range(npk):
                e.results_async(s, best[s, lo:hi], pose[s, lo:hi], ang[s, S_w * f0:S_w * f1] if f1 > f0 else None)
                if coords and a1 > a0:
                    e.coords_into(s, xyz_out[s, a0:a1], mode=2)

        import time
        for c in range(nch):
            lo, hi = bounds[c], bounds[c + 1]
            e = self.engines[c % ne]
            t0 = time.perf_counter()
            if not staged:
                # zero copy: read in place (on_device = 2); library copy: vs_submit copies (0)
                dev, (a0, a1, f0, f1) = self._slices(arrays, lo, hi)
                mode = 2 if zero_copy else 0
            else:
                dev, ev, (a0, a1, f0, f1) = inflight.pop(c)
                ev.synchronize()    # chunk c resident (submit reads its CSR totals)
                mode = 1
            t1 = time.perf_counter()
            t2 = t1
            if hi > lo and failed is None:     # (chunk_bounds never yields an empty chunk)
                # returns once the dock launches are queued; the read-backs below queue behind
                # them on the same stream and run on the D2H engine while the other engine docks
                try:
                    e.submit(*dev[:7], self.pocket_ids, on_device=mode, max_atoms=max_atoms,
                             atom_type=dev[7] if len(dev) > 7 else None)
                except VsError as err:       # rank-local a1 error: still join the collective below
                    failed = err
                    if err.ligand is not None:
                        failed.ligand = err.ligand + lo
                    keep[c % ne] = dev
                    continue
                t2 = time.perf_counter()
                for s in range(npk):
                    nkeys[s] += e.keys_into(s, all_keys[s][nkeys[s]:], lo)
                # the read-backs of the PREVIOUS chunk are queued only now, after this chunk's
                # preparation: the copy engine serves D2H requests in submission order, so a
                # read-back queued earlier would hold up this preparation's small status reads
                if pending is not None:
                    readback(*pending)
                pending = (e, lo, hi, a0, a1, f0, f1)
            keep[c % ne] = dev      # the engine borrows the chunk until its next submit
            if c + ne < nch and staged:
                # the buffer slot of chunk c + ne is engine c's: its copy may only overwrite
                # device memory the engine no longer reads -- new tensors, so no hazard
                inflight[c + ne] = self._issue_copy(arrays, bounds[c + ne], bounds[c + ne + 1])
            self.trace.append((c, lo, hi, t0, t1, t2, time.perf_counter()))   # host timeline (diagnostics)
        if pending is not None:
            readback(*pending)
        for st in self.streams:
            st.synchronize()
        e = self.engine
        tops = []
        ids_host = np.asarray(ligand_id)
        status = parallel.encode_status(failed)
        for s in range(npk):
            if failed is None:
                mine = e.select_keys(all_keys[s][:nkeys[s]], k)     # this rank's top-k, on the device
            else:
                mine = torch.full((k,), -1, dtype=torch.int64, device=self.dev)
            e.synchronize()                                    # (the collective runs on torch's stream)
            g, err = parallel.gather_keys_checked(mine, status, group)   # NCCL all-gather (W x (k + 1))
            if err is not None:
                parallel.raise_gathered(err)
            torch.cuda.current_stream(self.dev).synchronize()
            idx, sc = e.merge_topk(g, k)
            tops.append((idx, sc, ids_host[idx] if len(idx) else np.zeros(0, np.uint64)))
        e.synchronize()
        out = {"ligand_id": ids_host, "best_score": best, "best_pose": pose, "angles": ang[:, :S_w * nR],
               "topk": tops}
        if coords:
            out["xyz"] = xyz_out[:, :nA]
        return out

    def close(self):
        for e in self.engines:
            e.close()
