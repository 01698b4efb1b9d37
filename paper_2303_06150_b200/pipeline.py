"""Double-buffered host -> results pipeline.

LiGen overlaps transfers with compute by handing buckets to CPU "workers" that copy
into a free device buffer, run, and copy results back ("double buffering technique
for hiding data transfers").  On B200 one context is enough: the library is cut into
chunks, chunk i + 1's host-to-device copy runs on a copy stream (the copy engines)
while chunk i is prepared, docked and ranked on the context's compute stream, into
``n_buffers`` rotating device buffers.

Compute phases are deliberately serialised: the persistent dock kernel holds every SM
(one CTA per SM, ~227 KB of shared memory), so a second context's preparation kernels
could not start before the dock drains anyway -- and its local top-k would queue behind
the other context's dock.  What overlaps is the only thing that can: PCIe copies against
SM work.  Each chunk is a full hot-path submit (validate, bucket, pack, dock, local top-k);
every chunk's ranking keys are collected on the device (vs_keys) and ranked once at the end
(vs_merge_topk), then across ranks with one all-gather of k keys per pocket
(``parallel.gather_keys``).
"""
from __future__ import annotations

import numpy as np

from .vsdock import Engine


def _bounds(atom_off, frag_off, lo, hi):
    ao = np.asarray(atom_off[lo:hi + 1])
    fo = np.asarray(frag_off[lo:hi + 1])
    return ao, fo, int(ao[0]), int(ao[-1]), int(fo[0]), int(fo[-1])


def chunk_bounds(n: int, chunks: int = 0, first: int = 32, growth: int = 4):
    """Chunk boundaries of an n-ligand library.  chunks > 0: equal chunks.  chunks = 0: a
    geometric schedule -- first chunk n / first, each next one at most `growth` times the
    previous -- so only a small first copy is exposed while every later copy (~7x faster
    than docking the same ligands on B200) still hides under the previous chunk's dock."""
    if n <= 0:
        return [0, 0]
    if chunks > 0:
        chunks = min(int(chunks), n)
        return [n * c // chunks for c in range(chunks + 1)]
    b, size = [0], max(1, n // first)
    while b[-1] < n:
        b.append(min(n, b[-1] + size))
        size *= growth
    if len(b) > 2 and (b[-1] - b[-2]) < (b[-2] - b[-3]) // 4:   # fold a tiny tail into its predecessor
        b.pop(-2)
    return b


class PipelinedDocker:
    """Dock a host-resident library in chunks; H2D of the next chunk overlaps the current one."""

    def __init__(self, device: int = 0, n_buffers: int = 2, **engine_kw):
        import torch
        self._torch = torch
        self.device = device
        self.dev = torch.device(f"cuda:{device}")
        self.n_buffers = max(2, int(n_buffers))
        self.compute = torch.cuda.Stream(device=device)
        self.copy = torch.cuda.Stream(device=device)
        self.engine = Engine(device=device, stream=self.compute, **engine_kw)
        self.engines = [self.engine]
        self.trace = []

    def setup(self, rot, trans, cs, pockets):
        e = self.engine
        e.set_poses(rot, trans)
        e.set_angles(cs)
        self.pocket_ids = [e.load_pocket(p) for p in pockets]
        return self.pocket_ids

    def _issue_copy(self, arrays, lo, hi):
        """Chunk [lo, hi) to the device on the copy stream: rebased offsets + xyz / frags slices."""
        torch = self._torch
        atom_off, xyz, frag_off, frags = arrays
        ao, fo, a0, a1, f0, f1 = _bounds(atom_off, frag_off, lo, hi)
        host = [torch.from_numpy(np.ascontiguousarray(ao - a0)), xyz[a0:a1],
                torch.from_numpy(np.ascontiguousarray(fo - f0)), frags[f0:f1]]
        host = [h if isinstance(h, torch.Tensor) else torch.from_numpy(np.asarray(h)) for h in host]
        with torch.cuda.stream(self.copy):
            dev = [h.to(self.dev, non_blocking=True) for h in host]
            ev = torch.cuda.Event()
            ev.record(self.copy)
        return dev, ev, host

    def run(self, atom_off, xyz, frag_off, frags, k: int = 1000, chunks: int = 0, max_atoms: int = 256,
            group=None, first: int = 32, growth: int = 4):
        """Returns (best_score [P][n], best_pose [P][n], topk [(index, score)] per pocket) on the host.

        xyz / frags should be pinned host tensors (torch ``pin_memory``) for overlapped copies.
        ``chunks``: see ``chunk_bounds`` (0 = geometric schedule).  With ``rank`` / ``world_size`` engine options under an initialised process group, every
        rank docks its LPT share of each chunk and the per-pocket top-k is merged across ranks."""
        import time
        from . import parallel
        torch = self._torch
        e = self.engine
        n = int(atom_off.shape[0]) - 1
        npk = len(self.pocket_ids)
        bounds = chunk_bounds(n, chunks, first, growth)
        chunks = len(bounds) - 1
        # pinned host outputs: the per-chunk result reads are plain DMA, not staged copies
        best = torch.full((npk, n), float("nan"), dtype=torch.float32).pin_memory().numpy()
        pose = torch.full((npk, n), -1, dtype=torch.int32).pin_memory().numpy()
        # every chunk's keys land in one device array per pocket (index + chunk offset); the
        # ranking is one selection at the end (no per-chunk top-k round trip)
        all_keys = [torch.empty(max(1, n), dtype=torch.int64, device=self.dev) for _ in range(npk)]
        nkeys = [0] * npk
        arrays = (atom_off, xyz, frag_off, frags)
        self.trace = []
        inflight = {}
        for c in range(min(self.n_buffers - 1, chunks)):
            inflight[c] = self._issue_copy(arrays, bounds[c], bounds[c + 1])
        for c in range(chunks):
            lo, hi = bounds[c], bounds[c + 1]
            nxt = c + self.n_buffers - 1
            dev, ev, _host = inflight.pop(c)
            t0 = time.perf_counter()
            ev.synchronize()        # chunk c resident (the engine reads its CSR totals on submit)
            t1 = time.perf_counter()
            if hi > lo:
                # submit returns once the dock launches are queued; the preparation's small
                # host<->device exchanges are over by then, so the prefetch issued next shares
                # the copy engine with nothing and runs under the dock
                e.submit(*dev, self.pocket_ids, on_device=True, max_atoms=max_atoms)
            if nxt < chunks:
                inflight[nxt] = self._issue_copy(arrays, bounds[nxt], bounds[nxt + 1])
            if hi > lo:
                e.wait()
                for s in range(npk):
                    e.results_into(s, best[s, lo:hi], pose[s, lo:hi])
                    nkeys[s] += e.keys_into(s, all_keys[s][nkeys[s]:], lo)
            st = e.stats()
            self.trace.append((c, t0, t1, time.perf_counter(), st["prep_ms"], st["dock_ms"]))
            del dev                 # buffer free once the chunk's work completed (wait above)
        tops = []
        for s in range(npk):
            idx, sc = e.merge_topk(all_keys[s][:nkeys[s]], k)
            mine = torch.full((k,), -1, dtype=torch.int64)   # UINT64_MAX pads, as local_topk
            mine[: len(idx)] = parallel.encode_keys(sc, idx)
            g = parallel.gather_keys(mine.to(self.dev), group)
            if g.numel() > k:                  # more than one rank: merge the gathered rankings
                idx, sc = e.merge_topk(g, k)
            tops.append((idx, sc))
        return best, pose, tops

    def close(self):
        self.engine.close()
