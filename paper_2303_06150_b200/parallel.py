"""Multi-GPU plumbing for the hot path (a4 shard, a11 gather + merge).

One process per GPU.  Every rank submits the SAME library to its own Engine
(``rank``/``world_size`` in the config): the manifest and the LPT shard are pure
functions of the library (vs_plan_lpt), so every rank agrees on who docks which
bucket without communicating.  The only exchange is the per-pocket ranking
("for each docking site, we can rank the input chemical
library"): each rank's k best keys are all-gathered (NCCL over NVLink on B200;
gloo in the CPU tests) and merged into the global top-k on the device.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def gather_keys(keys_local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's [k] key vector into one [world * k] tensor (rank-major)."""
    if not (dist.is_available() and dist.is_initialized()):
        return keys_local
    world = dist.get_world_size(group)
    if world == 1:
        return keys_local
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * keys_local.numel(), dtype=keys_local.dtype, device=keys_local.device)
        dist.all_gather_into_tensor(out, keys_local, group=group)   # NVLink / NVSwitch
        return out
    # gloo (CPU tests, single-GPU test hook): host staging
    host = keys_local.detach().cpu()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    return torch.cat(parts).to(keys_local.device)


def encode_status(err) -> int:
    """A rank's submit outcome as one int64: 0 = ok, else (ligand index << 8) | -code."""
    if err is None:
        return 0
    return (max(0, int(getattr(err, "ligand", 0) or 0)) << 8) | (-int(err.code) & 0xFF)


def gather_keys_checked(keys_local: torch.Tensor, status: int = 0, group=None):
    """gather_keys with every rank's submit status riding along in one extra slot, so a rank
    whose a1 ingest rejected one of ITS ligands (errors are rank-local: each rank validates the
    ligands it docks) still joins the collective and every rank learns of the error from the
    same single all-gather.  Returns (gathered keys [world * k], first error or None) where the
    first error is (rank, ligand index, VS_E_* code) of the lowest failing rank."""
    st = torch.tensor([int(status)], dtype=torch.int64, device=keys_local.device)
    g = gather_keys(torch.cat([keys_local.reshape(-1), st]), group)
    world = g.numel() // (keys_local.numel() + 1)
    g = g.view(world, keys_local.numel() + 1)
    stats = g[:, -1].cpu().tolist()
    err = None
    for r, v in enumerate(stats):
        if v:
            err = (r, int(v) >> 8, -(int(v) & 0xFF))
            break
    return g[:, :-1].reshape(-1), err


def raise_gathered(err):
    from .vsdock import VsError
    r, li, code = err
    raise VsError(code, f"rank {r}: ligand {li} (batch index) failed a1 ingest; see that rank's log")


def global_topk(engine, slot: int, k: int, group=None, failed=None):
    """a10 + a11: local top-k on this rank's buckets, all-gather, merge on the device.
    ``failed``: this rank's VsError from its submit (it still joins the collective).

    Returns (ligand index [m] int64, score [m] float32) on the host, identical on every rank
    and bit-identical to the single-GPU ranking (keys are unique and totally ordered)."""
    if failed is None:
        keys, _ = engine.local_topk(slot, k)      # synchronous on the engine's stream
    else:
        keys = torch.full((k,), -1, dtype=torch.int64, device=f"cuda:{engine.device}")
    g, err = gather_keys_checked(keys, encode_status(failed), group)
    if err is not None:
        raise_gathered(err)
    torch.cuda.current_stream(keys.device).synchronize()   # the merge runs on the engine's stream
    return engine.merge_topk(g, k)


def decode_keys(keys: torch.Tensor):
    """(ligand index, score) of uint64 keys ord(score) << 32 | index held in an int64 tensor (host)."""
    import numpy as np
    u = keys.detach().cpu().numpy().view(np.uint64)
    valid = u != np.uint64(0xFFFFFFFFFFFFFFFF)
    u = u[valid]
    idx = (u & np.uint64(0xFFFFFFFF)).astype(np.int64)
    ordv = (u >> np.uint64(32)).astype(np.uint32)
    bits = np.where(ordv & np.uint32(0x80000000), ordv & np.uint32(0x7FFFFFFF), ~ordv).astype(np.uint32)
    return idx, bits.view(np.float32)


def encode_keys(scores, index):
    """Inverse of decode_keys, for host-side TESTS only (the product path keeps keys on the device):
    int64 tensor of ord(score) << 32 | index."""
    import numpy as np
    s = np.asarray(scores, np.float32) + np.float32(0.0)
    b = s.view(np.uint32)
    o = np.where(b & np.uint32(0x80000000), ~b, b | np.uint32(0x80000000)).astype(np.uint64)
    k = (o << np.uint64(32)) | np.asarray(index, np.uint64)
    return torch.from_numpy(k.view(np.int64).copy())
