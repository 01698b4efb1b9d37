"""World-size-2 CPU test of the multi-GPU host path with the gloo backend.

Every rank plans the same shard from the same library (product code: vs_plan_boundaries,
vs_plan_lpt), the shards partition the buckets, and the per-pocket ranking exchange
(paper_2303_06150_b200.parallel.gather_keys, the same call bench.py uses over NCCL)
gathers each rank's local top-k keys so that their merge equals the global top-k."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import vsgen
        from paper_2303_06150_b200 import parallel
        from paper_2303_06150_b200.vsdock import plan_boundaries, plan_lpt
        lib = vsgen.ligands(3000, 2, (20, 120), (0, 20))
        ab, rb = plan_boundaries(6, int(lib.n_atoms.max()), 23, int(lib.n_frags.max()))
        buckets = oracle.bucketize(lib.n_atoms, lib.n_frags, ab, rb, [148 * 2] * len(ab))
        E = oracle.ligand_work(lib.n_atoms, lib.n_moving, 64, 8)
        w = np.array([int(E[b.ligands].sum()) for b in buckets], np.uint64)
        owner, order = plan_lpt(w, world)
        t = torch.from_numpy(owner.astype(np.int64))
        allo = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allo, t)
        same = all(torch.equal(allo[0], x) for x in allo)
        mine = [b for i, b in enumerate(buckets) if owner[i] == rank]
        owned = np.concatenate([b.ligands for b in mine]) if mine else np.zeros(0, np.int64)
        # stand-in scores with many exact ties (the ranking must break them by ligand index)
        scores = np.round(np.random.default_rng(0).normal(size=lib.n), 2).astype(np.float32)
        k = 100
        local = oracle.topk(scores[owned], k, owned)
        keys = parallel.encode_keys(scores[local], local)
        if keys.numel() < k:
            keys = torch.cat([keys, torch.full((k - keys.numel(),), -1, dtype=torch.int64)])
        g = parallel.gather_keys(keys)
        idx, sc = parallel.decode_keys(g)
        merged = oracle.merge_topk([(sc, idx)], k)
        n_owned = torch.tensor([len(owned)])
        dist.all_reduce(n_owned)
        out[rank] = dict(same=same, merged=list(merged), want=list(oracle.topk(scores, k)),
                         n_owned=int(n_owned.item()), n=lib.n, gathered=int(g.numel()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_plan_and_merge():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        o = out[r]
        assert o["same"], "ranks disagree on the LPT shard"
        assert o["n_owned"] == o["n"], "shards do not partition the library"
        assert o["gathered"] == world * 100
        assert o["merged"] == o["want"]


def _worker_err(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_06150_b200 import parallel
        from paper_2303_06150_b200.vsdock import VsError, VS_E_PARSE
        k = 16
        keys = torch.arange(k, dtype=torch.int64) + 100 * rank
        # rank 1's a1 ingest rejected its ligand 4242 (rank-local error): it still joins the gather
        err = VsError(VS_E_PARSE, "ligand 4242: moving sets not laminar") if rank == 1 else None
        g, e = parallel.gather_keys_checked(keys if err is None else torch.full((k,), -1), parallel.encode_status(err))
        ok_g, ok_e = parallel.gather_keys_checked(keys, 0)        # a clean step afterwards
        out[rank] = dict(err=e, n=int(g.numel()), ok_err=ok_e, ok_keys=ok_g.tolist())
    finally:
        dist.destroy_process_group()


def test_two_ranks_rank_local_error_reaches_every_rank():
    """Errors of a1's per-atom checks are rank-local (each rank validates the ligands it docks):
    the failing rank's status rides in the same all-gather as the keys, so BOTH ranks see it and no
    rank blocks in a collective the other never reaches (parallel.gather_keys_checked)."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_err, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        o = out[r]
        assert o["err"] == (1, 4242, -2)           # (rank, ligand index, VS_E_PARSE) on every rank
        assert o["n"] == world * 16
        assert o["ok_err"] is None and o["ok_keys"] == list(range(16)) + list(range(100, 116))
