"""GPU parity: the CUDA path through the C-ABI (libvsdock.so) against the fp64 oracle.

Contract (BASELINE.json north_star): bucketing, ordering and
angle indices bit-exact outside near-ties (band 1e-5 * max(1, |S|)); final scores
within 1e-4 * max(1, |S|); best-pose coordinates within 1e-3 A.  Every GPU angle
choice is replayed in fp64 (oracle.parity).
"""
import numpy as np
import pytest

import oracle
import vsgen
from oracle import parity

pytestmark = pytest.mark.gpu

BAND, TOL_S, TOL_X = 1e-5, 1e-4, 1e-3


def engine(**kw):
    from paper_2303_06150_b200 import Engine
    return Engine(**kw)


def setup(e, pockets, P, K, seed=7):
    rot, tr = vsgen.pose_table(P, seed)
    cs = vsgen.angle_table(K)
    e.set_poses(rot, tr)
    e.set_angles(cs)
    ids = [e.load_pocket(p) for p in pockets]
    return rot, tr, cs, ids


def run(lib, pockets, P=8, K=8, debug=True, **kw):
    e = engine(debug_poses=debug, **kw)
    rot, tr, cs, ids = setup(e, pockets, P, K)
    e.submit_library(lib, ids)
    e.wait()
    return e, rot, tr, cs


def check(e, lib, idx, pk, rot, tr, cs, slot=0, debug=True, S_w=1):
    r = e.results(slot)
    xyz = e.coords(slot)
    ps, pa = e.pose_debug(slot) if debug else (None, None)
    rep = parity.check(lib, idx, pk, rot, tr, cs, r.best_score, r.best_pose, r.angles, xyz, ps, pa, S_w=S_w,
                       band=BAND, tol_score=TOL_S, tol_xyz=TOL_X)
    assert rep.ok, rep.summary() + "\n" + "\n".join(map(str, rep.failures[:10]))
    return rep, r


# ----------------------------------------------------------------------------- a8

def test_grid_score_hook_vs_oracle():
    pk = vsgen.pocket(101)
    e = engine()
    pid = e.load_pocket(pk)
    rng = np.random.default_rng(0)
    pts = rng.uniform(-5, 36, size=(20000, 3)).astype(np.float32)
    g = e.score_points(pid, pts)
    ref = oracle.grid_score(pk, pts.astype(np.float64))
    assert np.max(np.abs(g - ref) / np.maximum(1, np.abs(ref))) < 2e-6
    # node exactness: integer coordinates (h = 1, origin 0) hit nodes exactly
    nodes = rng.integers(0, 32, size=(2000, 3)).astype(np.float32)
    g = e.score_points(pid, nodes)
    want = pk.grid[nodes[:, 2].astype(int), nodes[:, 1].astype(int), nodes[:, 0].astype(int)]
    assert np.array_equal(g, want)


# ----------------------------------------------------------------------------- C1 full

def test_c1_full_parity_every_pose():
    c = vsgen.CONFIGS["C1"]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    pk = vsgen.pocket(101)
    e, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"])
    rep, r = check(e, lib, range(lib.n), pk, rot, tr, cs)
    assert rep.independent_checked >= lib.n // 2 and rep.independent_equal == rep.independent_checked


# ----------------------------------------------------------------------------- C2 / C3 samples

@pytest.fixture(scope="module")
def c2():
    c = vsgen.CONFIGS["C2"]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    return c, lib, vsgen.pocket(101)


def test_c2_sample_parity_and_bucketing_invariance(c2):
    c, lib, pk = c2
    e, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"])
    rng = np.random.default_rng(2)
    idx = rng.choice(lib.n, 1000, replace=False)
    rep, r = check(e, lib, idx, pk, rot, tr, cs)
    assert rep.independent_equal == rep.independent_checked > 300
    # Q22: bit-identical whatever the launch structure (one launch per bucket, bucket multiple, streams)
    # and whatever the cluster grid: every class of K = 8 runs the same 4-poses-per-warp lane map,
    # so the unsorted 1 x 1 grid (one class, A_c = 128) gives the same bits as 6 x 23
    for kw in (dict(launch_per_bucket=True, bucket_multiple=1), dict(bucket_multiple=3, n_streams=1),
               dict(atom_clusters=1, rot_clusters=1), dict(atom_clusters=3, rot_clusters=5)):
        e2, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False, **kw)
        r2 = e2.results(0)
        assert np.array_equal(r.best_score, r2.best_score) and np.array_equal(r.best_pose, r2.best_pose)
        assert np.array_equal(r.angles, r2.angles)
        assert np.array_equal(e.coords(0), e2.coords(0))


def test_round_ring_many_tiny_launches_bit_identical(c2):
    """The dock kernel's round ring: launches of 1..5 rounds on up to 148 CTAs
    (exhaustion at the first, second or a later sequence, CTAs with no round at all), P not a
    multiple of the poses per warp, several ligands per round, many streams -- all bit-identical
    to one fused launch per class."""
    c, lib, pk = c2
    sub = lib.subset(np.arange(1500))
    for P in (64, 30, 6):
        e, *_ = run(sub, [pk], P=P, K=c["K"], debug=False)
        ref, ref_xyz = e.results(0), e.coords(0)
        for cap in (1, 2, 5):
            e2, *_ = run(sub, [pk], P=P, K=c["K"], debug=False, launch_per_bucket=True, bucket_capacity=cap,
                         n_streams=8)
            r2 = e2.results(0)
            assert np.array_equal(ref.best_score, r2.best_score), (P, cap)
            assert np.array_equal(ref.best_pose, r2.best_pose) and np.array_equal(ref.angles, r2.angles)
            assert np.array_equal(ref_xyz, e2.coords(0))


def test_c3_large_ligand_sample_parity():
    c = vsgen.CONFIGS["C3"]
    lib = vsgen.ligands(2048, c["seed"], c["atoms"], c["rot"])
    pk = vsgen.pocket(101)
    e, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"])
    assert {cl["kernel_atoms"] for cl in e.classes()} >= {96, 128, 160}
    rng = np.random.default_rng(3)
    check(e, lib, rng.choice(lib.n, 200, replace=False), pk, rot, tr, cs)


# ----------------------------------------------------------------------------- a2-a4 bit-exact

@pytest.mark.parametrize("grid", [(6, 23), (1, 1), (3, 3), (4, 5)])
def test_manifest_bit_exact_vs_oracle(c2, grid):
    c, lib, pk = c2
    e, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False, atom_clusters=grid[0], rot_clusters=grid[1],
                bucket_multiple=1)
    buckets, perm = e.manifest()
    cls = e.classes()
    ab, rb = oracle.atom_boundaries(grid[0], 32, int(lib.n_atoms.max())), oracle.rotamer_boundaries(grid[1], int(lib.n_frags.max()))
    assert [cl["atom_bound"] for cl in cls] == ab
    ref = oracle.bucketize(lib.n_atoms, lib.n_frags, ab, rb, [cl["capacity"] for cl in cls])
    assert len(ref) == len(buckets)
    assert np.array_equal(perm, np.concatenate([b.ligands for b in ref]).astype(np.uint32))
    for b, rbk in zip(buckets, ref):
        assert (b["atom_class"], b["rot_class"]) == rbk.cell
        assert b["size"] == len(rbk.ligands) and b["capacity"] == rbk.capacity
    # exact work weights and the LPT shard
    E = oracle.ligand_work(lib.n_atoms, lib.n_moving, c["P"], c["K"])
    w = [int(E[rbk.ligands].sum()) for rbk in ref]
    assert [b["weight"] for b in buckets] == w
    for W in (2, 4, 8):
        sh = oracle.lpt_shards(w, W)
        owners = {bb: r for r, bl in enumerate(sh) for bb in bl}
        eW, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False, atom_clusters=grid[0], rot_clusters=grid[1],
                     bucket_multiple=1, rank=W - 1, world_size=W)
        bW, _ = eW.manifest(want_perm=False)
        assert [b["owner"] for b in bW] == [owners[i] for i in range(len(bW))]


def test_eq1_class_table_matches_occupancy_model(c2):
    c, lib, pk = c2
    e, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
    for cl in e.classes():
        # S:109 min-of-limits with B200 limits: 64K regs, 2048 threads, 32 CTAs, 228 KB smem (1 KB/CTA reserved)
        b = oracle.active_blocks_per_sm(65536, 2048, 32, 233472, 256, cl["regs_per_thread"], cl["threads_per_cta"],
                                        cl["dyn_smem"] + cl["static_smem"] + 1024)
        assert cl["blocks_per_sm"] == b
        assert cl["l"] == oracle.bucket_capacity_native(b, cl["sm_count"], 32 * cl["ligands_per_cta"], 32)
        assert cl["sm_count"] == 148


# ----------------------------------------------------------------------------- a10/a11 bit-exact

def test_topk_and_virtual_rank_merge_bit_exact(c2):
    import torch
    c, lib, pk = c2
    e, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
    r = e.results(0)
    for k in (1, 10, 1000, 4096):
        keys, nv = e.local_topk(0, k)
        idx, sc = e.merge_topk(keys[:nv], k)
        want = oracle.topk(r.best_score, k)
        assert list(idx) == list(want)
        assert np.array_equal(sc, r.best_score[want])
    # W virtual ranks on one GPU: each docks its LPT shard; gather + merge == single GPU
    for W in (2, 4):
        parts = []
        for rank in range(W):
            eR, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False, rank=rank, world_size=W)
            rr = eR.results(0)
            own = ~np.isnan(rr.best_score)
            assert np.array_equal(rr.best_score[own], r.best_score[own])
            keys, _ = eR.local_topk(0, 1000)
            parts.append(keys)
            merger = eR
        gathered = torch.cat(parts)
        idx, sc = merger.merge_topk(gathered, 1000)
        assert list(idx) == list(oracle.topk(r.best_score, 1000))


def test_topk_vs_oracle_scores_outside_ties(c2):
    """The GPU ranking equals the fp64 oracle's ranking except where scores are within the band."""
    c, lib, pk = c2
    sub = lib.subset(np.arange(400))
    e, rot, tr, cs = run(sub, [pk], P=c["P"], K=c["K"], debug=False)
    r = e.results(0)
    ref = oracle.dock_batch(sub, pk, rot, tr, cs, want_xyz=False, want_debug=False)
    g = oracle.topk(r.best_score, 50)
    o = oracle.topk(ref.best_score, 50)
    for a, b in zip(g, o):
        if a != b:
            assert abs(ref.best_score[a] - ref.best_score[b]) <= 2 * TOL_S * max(1, abs(ref.best_score[b]))


# ----------------------------------------------------------------------------- edge cases

def mk_lib(ligs):
    return vsgen.Library.from_ligands(ligs)


NOFRAG = vsgen.Frags(np.zeros((0, 2), np.int32), [])


def test_edge_cases_tiny_ligands_and_tables():
    """Tiny ligands (A = 1, 2) and every table shape, including angle counts that are not powers
    of two (theta_k = 2 pi k / K for K = 3, 6, 12: lane map of the next power of two)."""
    pk = vsgen.pocket(102)
    base = vsgen.ligands(40, 9, (20, 40), (0, 4))
    ligs = [base.ligand(i) for i in range(base.n)]
    ligs += [(np.array([[1.0, 2.0, 3.0]]), NOFRAG),                                  # A = 1
             (np.array([[0, 0, 0], [1.5, 0, 0]], np.float32), NOFRAG)]               # A = 2, R = 0
    lib = mk_lib(ligs)
    for P, K in [(1, 8), (7, 8), (8, 1), (8, 2), (4, 16), (4, 32), (33, 4), (8, 6), (8, 12), (5, 3), (4, 24)]:
        e, rot, tr, cs = run(lib, [pk], P=P, K=K)
        check(e, lib, range(lib.n), pk, rot, tr, cs)


def test_two_sweeps_and_two_pockets_with_different_grids():
    lib = vsgen.ligands(30, 12, (20, 60), (1, 6))
    pk1 = vsgen.pocket(103)
    pk2 = vsgen.pocket(104, n=28, spacing=1.25)
    e = engine(debug_poses=True, n_sweeps=2)
    rot, tr, cs, ids = setup(e, [pk1, pk2], 8, 8)
    e.submit_library(lib, ids)
    e.wait()
    for slot, pk in enumerate([pk1, pk2]):
        check(e, lib, range(lib.n), pk, rot, tr, cs, slot=slot, S_w=2)


def test_non_cubic_grid_runtime_strides():
    """A 36 x 30 x 26 grid (nx > 32: the runtime-stride layout, not the fixed 32 x 32-plane
    one), off-centre origin, h = 0.8 A: the score hook and full docking parity."""
    rng = np.random.default_rng(11)
    base = vsgen.pocket(105, n=36, spacing=0.8)
    G = np.ascontiguousarray(base.grid[:26, :30, :36]) + rng.normal(0, 0.05, (26, 30, 36)).astype(np.float32)
    origin = (-1.5, 0.25, 2.0)
    h = 0.8
    center = tuple(o + h * (n - 1) / 2 for o, n in zip(origin, (36, 30, 26)))
    pk = vsgen.Pocket(G.astype(np.float32), origin, h, center, 0.7)
    e = engine()
    pid = e.load_pocket(pk)
    pts = rng.uniform(-4, 32, size=(20000, 3)).astype(np.float32)
    g = e.score_points(pid, pts)
    ref = oracle.grid_score(pk, pts.astype(np.float64))
    # fp32 u = (x - o) * (1/h) with h = 0.8 (1/h inexact): |du| <~ 2 ulp(40) ~ 8e-6 grid units,
    # times |grad g| <~ 2 per grid unit -> 2e-5 (the h = 1 hook test above is exact to 2e-6)
    assert np.max(np.abs(g - ref) / np.maximum(1, np.abs(ref))) < 2e-5
    lib = vsgen.ligands(24, 13, (20, 60), (0, 6))
    e2, rot, tr, cs = run(lib, [pk], P=8, K=8)
    check(e2, lib, range(lib.n), pk, rot, tr, cs)


def test_small_grid_atoms_outside_the_box():
    """A 14^3 grid at 1 A around ligands of 40-90 atoms: many atoms sit on or beyond the
    faces (clamped, penalised), so the weight-0 top-edge corner reads that land past the last
    plane (into the zeroed pose buffers on the fixed-stride layout) are exercised; full parity
    against the oracle, every pose replayed."""
    base = vsgen.pocket(106, n=14, spacing=1.0)
    lib = vsgen.ligands(24, 17, (40, 90), (2, 10))
    e, rot, tr, cs = run(lib, [base], P=8, K=8)
    check(e, lib, range(lib.n), base, rot, tr, cs)
    # score hook on points all around and outside the box, including exact top-face points
    e2 = engine()
    pid = e2.load_pocket(base)
    rng = np.random.default_rng(6)
    pts = rng.uniform(-6, 20, size=(20000, 3)).astype(np.float32)
    pts[:2000, rng.integers(0, 3, 2000)] = 13.0          # exactly on the top faces
    g = e2.score_points(pid, pts)
    ref = oracle.grid_score(base, pts.astype(np.float64))
    assert np.max(np.abs(g - ref) / np.maximum(1, np.abs(ref))) < 2e-6


def test_empty_batch():
    e = engine()
    setup(e, [vsgen.pocket(101)], 8, 8)
    e.submit_library(mk_lib([]), [0])
    e.wait()
    assert e.results(0).best_score.size == 0


def test_validation_errors_name_the_ligand():
    from paper_2303_06150_b200 import VsError
    from paper_2303_06150_b200 import vsdock
    base = vsgen.ligands(10, 5, (20, 40), (1, 4))
    e = engine()
    setup(e, [vsgen.pocket(101)], 8, 8)

    def copy_lig(i):
        x, f = base.ligand(i)
        return np.array(x, copy=True), vsgen.Frags(np.array(f.axis, copy=True), [np.array(m, copy=True) for m in f.moves])

    def bad(mutate, what):
        ligs = [copy_lig(i) for i in range(base.n)]
        mutate(ligs)
        with pytest.raises(VsError) as ei:
            e.submit_library(mk_lib(ligs), [0])
        assert ei.value.code == vsdock.VS_E_PARSE
        assert "ligand 3" in str(ei.value) and what in str(ei.value), str(ei.value)

    def nan(l): l[3][0][2, 1] = np.nan
    def huge(l): l[3][0][1, 0] = 3e6
    def axis_eq(l): l[3][1].axis[0, 1] = l[3][1].axis[0, 0]
    def axis_oob(l): l[3][1].axis[0, 0] = 999
    def move_oob(l): l[3][1].moves[0][0] = 1000
    def axis_in(l): l[3][1].moves[0][0] = l[3][1].axis[0, 1]
    def dup(l): l[3][1].moves[0] = np.concatenate([l[3][1].moves[0], l[3][1].moves[0][:1]])
    def empty(l): l[3][1].moves[0] = np.zeros(0, np.int32)

    def crossing(l):        # two moving sets that overlap without nesting
        x, f = l[3]
        A = len(x)
        free = [i for i in range(A) if i not in set(f.axis[0].tolist())]
        a_set = np.array(free[: len(free) // 2 + 1], np.int32)
        b_set = np.array(free[len(free) // 2 - 1:], np.int32)
        f.moves[0] = a_set
        f2 = vsgen.Frags(np.concatenate([f.axis, f.axis[:1]]), f.moves + [b_set])
        l[3] = (x, f2)

    def too_big(l): l[3] = (np.zeros((300, 3), np.float32), NOFRAG)
    bad(nan, "non-finite coordinate")
    bad(huge, "magnitude")
    bad(axis_eq, "axis atoms are equal")
    bad(axis_oob, "axis atom index out of range")
    bad(move_oob, "moving atom index out of range")
    bad(axis_in, "axis atom inside its own moving set")
    bad(dup, "listed twice")
    bad(empty, "moving set empty")
    bad(crossing, "not laminar")
    bad(too_big, "atom count")
    # overflow names the axis: user upper bounds below the data
    e2 = engine(atom_upper_bound=30, rot_upper_bound=2, atom_clusters=1, rot_clusters=1)
    setup(e2, [vsgen.pocket(101)], 8, 8)
    with pytest.raises(VsError) as ei:
        e2.submit_library(base, [0])
    assert ei.value.code in (vsdock.VS_E_OVERFLOW_ATOMS, vsdock.VS_E_OVERFLOW_ROTAMERS)
    assert "axis" in str(ei.value)


# ----------------------------------------------------------------------------- full size (bench config)

def test_c4_full_size_sampled_parity():
    """BASELINE configs[3] at full size in bench.py's launch configuration; sampled ligands
    against the oracle one by one, plus properties over all 1M outputs."""
    import torch
    c = vsgen.CONFIGS["C4"]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    pk = vsgen.pocket(101)
    e = engine(bucket_multiple=16, n_streams=4)
    rot, tr, cs, ids = setup(e, [pk], c["P"], c["K"])
    d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
    e.submit(*d, ids, on_device=True)
    e.wait()
    r = e.results(0)
    assert np.array_equal(r.ligand_id, lib.ligand_id)
    assert np.isfinite(r.best_score).all()
    assert ((r.best_pose >= 0) & (r.best_pose < c["P"])).all()
    assert (r.angles < c["K"]).all()
    rng = np.random.default_rng(4)
    idx = rng.choice(lib.n, 400, replace=False)
    xyz = e.coords(0)
    rep = parity.check(lib, idx, pk, rot, tr, cs, r.best_score, r.best_pose, r.angles, xyz, band=BAND,
                       tol_score=TOL_S, tol_xyz=TOL_X)
    assert rep.ok, rep.summary() + str(rep.failures[:5])


def test_c5_full_size_campaign_sampled_parity_and_topk():
    """BASELINE configs[4]: the C4 library x 4 pockets in one submit (bench launch
    configuration); per pocket, sampled ligands against the oracle and the top-1000 equal to
    the sorted ranking of the GPU scores; pockets differ (scores are not copies)."""
    import torch
    c = vsgen.CONFIGS["C5"]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    pks = [vsgen.pocket(s) for s in c["pockets"]]
    e = engine(bucket_multiple=16, n_streams=4)
    rot, tr, cs, ids = setup(e, pks, c["P"], c["K"])
    d = [torch.from_numpy(a).cuda() for a in lib.arrays()]
    e.submit(*d, ids, on_device=True)
    e.wait()
    rng = np.random.default_rng(5)
    prev = None
    for slot, pk in enumerate(pks):
        r = e.results(slot)
        assert np.isfinite(r.best_score).all()
        if prev is not None:
            assert not np.array_equal(prev, r.best_score)
        prev = r.best_score
        idx = rng.choice(lib.n, 100, replace=False)
        rep = parity.check(lib, idx, pk, rot, tr, cs, r.best_score, r.best_pose, r.angles, e.coords(slot),
                           band=BAND, tol_score=TOL_S, tol_xyz=TOL_X)
        assert rep.ok, rep.summary() + str(rep.failures[:5])
        keys, _ = e.local_topk(slot, 1000)
        ti, ts = e.merge_topk(keys, 1000)
        assert list(ti) == list(oracle.topk(r.best_score, 1000))
        assert np.array_equal(ts, r.best_score[ti])


def test_keys_with_offset_rank_like_local_topk(c2):
    """vs_keys: every owned ligand's key with a ligand-index offset; ranking them with
    vs_merge_topk equals the local top-k shifted by the offset (streamed-library path)."""
    import torch
    c, lib, pk = c2
    sub = lib.subset(np.arange(3000))
    e, *_ = run(sub, [pk], P=c["P"], K=c["K"], debug=False)
    r = e.results(0)
    out = torch.empty(sub.n, dtype=torch.int64, device="cuda")
    n = e.keys_into(0, out, 123456)
    assert n == sub.n
    idx, sc = e.merge_topk(out[:n], 500)
    want = oracle.topk(r.best_score, 500)
    assert list(idx - 123456) == list(want)
    assert np.array_equal(sc, r.best_score[want])


def test_pipelined_docker_matches_single_submit_and_oracle(c2):
    """The double-buffered public host API: two engines alternating over chunks,
    asynchronous read-back of every a9 output.  Bit-identical to one submit (scores, poses, angle
    indices, coordinates), the same ranking with ligand ids, and the pipeline's own outputs pass
    the oracle parity contract on a sample."""
    import torch
    from paper_2303_06150_b200.pipeline import PipelinedDocker
    c, lib, pk = c2
    e, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
    r = e.results(0)
    xyz1 = e.coords(0)
    pd = PipelinedDocker()
    pd.setup(rot, tr, cs, [pk])
    h = [torch.from_numpy(a).pin_memory() for a in lib.arrays()]
    for chunks in (3, 0):
        out = pd.run(*h, k=100, chunks=chunks)
        assert np.array_equal(out["best_score"][0], r.best_score)
        assert np.array_equal(out["best_pose"][0], r.best_pose)
        assert np.array_equal(out["angles"][0], r.angles)
        assert np.array_equal(out["xyz"][0], xyz1)
        idx, sc, ids = out["topk"][0]
        assert list(idx) == list(oracle.topk(r.best_score, 100))
        assert np.array_equal(sc, r.best_score[idx]) and np.array_equal(ids, lib.ligand_id[idx])
    rng = np.random.default_rng(7)
    sample = rng.choice(lib.n, 60, replace=False)
    rep = parity.check(lib, sample, pk, rot, tr, cs, out["best_score"][0], out["best_pose"][0], out["angles"][0],
                       out["xyz"][0], band=BAND, tol_score=TOL_S, tol_xyz=TOL_X)
    assert rep.ok, rep.summary() + str(rep.failures[:5])
    pd.close()


# ----------------------------------------------------------------------------- round 2: inputs the
# round-1 suite never exercised (VERDICT r1 "what's weak" 1, 2; "missing" 4)

def test_translated_poses_and_offcentre_pocket_every_pose():
    """a6 y = R_p (x - xbar) + c + tau_p with tau_p != 0 and c off the grid centre: every pose of
    every ligand replayed in fp64 (C1 shape, plus a C2-shaped sample)."""
    pk = vsgen.pocket(101, center_offset=(1.75, -2.5, 1.0))
    c = vsgen.CONFIGS["C1"]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    e = engine(debug_poses=True)
    rot, tr = vsgen.pose_table(c["P"], tau=2.0)
    cs = vsgen.angle_table(c["K"])
    e.set_poses(rot, tr)
    e.set_angles(cs)
    pid = e.load_pocket(pk)
    e.submit_library(lib, [pid])
    e.wait()
    rep, r = check(e, lib, range(lib.n), pk, rot, tr, cs)
    assert rep.independent_checked >= lib.n // 2 and rep.independent_equal == rep.independent_checked
    assert len(set(r.best_pose.tolist())) > 1        # translations change which pose wins
    lib2 = vsgen.ligands(300, 21, (20, 120), (0, 20))
    rot2, tr2 = vsgen.pose_table(64, tau=1.5)
    e2 = engine(debug_poses=True)
    e2.set_poses(rot2, tr2)
    e2.set_angles(cs)
    e2.load_pocket(pk)
    e2.submit_library(lib2, [0])
    e2.wait()
    check(e2, lib2, range(0, 300, 10), pk, rot2, tr2, cs)


def test_large_ligands_classes_192_224_256_and_32_fragments():
    """161-256 atoms and 26-32 rotatable bonds: the 192 / 224 / 256 atom classes, their (poses per
    warp, warps) policy fallbacks and shared-memory layouts near 227 KB; sampled full parity."""
    lib = vsgen.ligands(600, 31, (161, 256), (26, 32))
    assert lib.n_atoms.max() > 224 and lib.n_frags.max() == 32 and lib.n_frags.min() >= 26
    pk = vsgen.pocket(101)
    e, rot, tr, cs = run(lib, [pk], P=16, K=8, atom_clusters=8)      # boundaries 32, 64, ..., 224, 256
    cls = {cl["kernel_atoms"]: cl for cl in e.classes()}
    assert {192, 224, 256} <= set(cls), cls
    for ac in (192, 224, 256):
        assert cls[ac]["dyn_smem"] + cls[ac]["static_smem"] <= 232448 and cls[ac]["blocks_per_sm"] == 1
    by_class = {ac: [i for i in range(lib.n) if ac - 32 < lib.n_atoms[i] <= ac] for ac in (192, 224, 256)}
    idx = sorted(i for ac in by_class for i in by_class[ac][:6])
    check(e, lib, idx, pk, rot, tr, cs)
    # the default (production) path at P = 64 for the same classes: best pose / score / coordinates
    e64, rot64, tr64, cs64 = run(lib.subset(idx), [pk], P=64, K=8, debug=False, atom_clusters=8)
    r64 = e64.results(0)
    sub = lib.subset(idx)
    rep = parity.check(sub, range(sub.n), pk, rot64, tr64, cs64, r64.best_score, r64.best_pose, r64.angles,
                       e64.coords(0), band=BAND, tol_score=TOL_S, tol_xyz=TOL_X)
    assert rep.ok, rep.summary() + str(rep.failures[:5])


def test_permuted_atoms_dock_bit_identically_and_match_the_oracle():
    """General moving sets: the same molecules with randomly renumbered atoms (moving
    sets become arbitrary subsets) go through a1's laminar check and canonical renumbering and dock
    BIT-identically to the generator's preordered numbering; coordinates come back in the caller's
    atom order; full parity of the permuted library against the oracle (which rotates the listed
    atoms directly, no renumbering)."""
    c = vsgen.CONFIGS["C2"]
    lib = vsgen.ligands(400, 41, c["atoms"], c["rot"])
    plib, perm = lib.permuted(9)
    assert any(np.any(np.diff(np.sort(m)) != 1) for i in range(20) for _, _, m in plib.ligand(i)[1])
    pk = vsgen.pocket(101)
    e1, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
    e2, *_ = run(plib, [pk], P=c["P"], K=c["K"], debug=True)
    r1, r2 = e1.results(0), e2.results(0)
    assert np.array_equal(r1.best_score, r2.best_score)
    assert np.array_equal(r1.best_pose, r2.best_pose) and np.array_equal(r1.angles, r2.angles)
    x1, x2 = e1.coords(0), e2.coords(0)
    assert np.array_equal(x2[perm], x1)                 # new[perm[g]] = old[g]
    check(e2, plib, range(0, plib.n, 8), pk, rot, tr, cs)


def test_ligand_ids_pass_through():
    lib = vsgen.ligands(50, 3, (20, 60), (0, 6))
    lib.ligand_id = (np.arange(50, dtype=np.uint64) * np.uint64(1000003) + np.uint64(2 ** 40)).astype(np.uint64)
    e, *_ = run(lib, [vsgen.pocket(101)], P=8, K=8, debug=False)
    r = e.results(0)
    assert np.array_equal(r.ligand_id, lib.ligand_id)
    keys, nv = e.local_topk(0, 10)
    idx, sc, ids = e.merge_topk(keys[:nv], 10, with_ids=True)
    assert list(idx) == list(oracle.topk(r.best_score, 10)) and np.array_equal(ids, lib.ligand_id[idx])


def test_topk_merge_of_padded_lists_smaller_than_k():
    """Ranks with fewer than k ligands pad their lists with UINT64_MAX: merging W padded
    lists (W * k above the 8192-entry scratch) keeps every real ligand, deterministically."""
    import torch
    c = vsgen.CONFIGS["C1"]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    pk = vsgen.pocket(101)
    e, *_ = run(lib, [pk], P=8, K=8, debug=False)
    r = e.results(0)
    for W, k in ((8, 1000), (8, 2000), (3, 8192)):
        parts = []
        for rank in range(W):
            eR, *_ = run(lib, [pk], P=8, K=8, debug=False, rank=rank, world_size=W)
            keys, _ = eR.local_topk(0, k)
            parts.append(keys)
        g = torch.cat(parts)
        assert g.numel() == W * k
        for _ in range(2):
            idx, sc = eR.merge_topk(g, k)
            assert list(idx) == list(oracle.topk(r.best_score, k))      # all 16 ligands, ranked
            assert np.array_equal(sc, r.best_score[idx])


def test_mixed_layout_pockets_in_one_submit():
    """A 32^3 pocket (fixed-stride layout), a 36 x 30 x 26 pocket (runtime strides) and a 56^3 pocket
    (window + global) in ONE submit: each launch uses its own layout's class table; full
    parity in all three."""
    pk1 = vsgen.pocket(101)
    pk2 = vsgen.pocket(107, n=(36, 30, 26), spacing=0.9, center_offset=(0.5, -0.5, 0.25))
    pk3 = vsgen.pocket(109, n=56, spacing=0.75)                       # WIN mode
    lib = vsgen.ligands(40, 23, (20, 120), (0, 12))
    e = engine(debug_poses=True)
    rot, tr, cs, ids = setup(e, [pk1, pk2, pk3], 8, 8)
    e.submit_library(lib, ids)
    e.wait()
    for slot, pk in enumerate([pk1, pk2, pk3]):
        check(e, lib, range(lib.n), pk, rot, tr, cs, slot=slot)


# ----------------------------------------------------------------------------- grids beyond shared
# memory (VERDICT r1 "missing" 3): the WIN mode -- a 32^3-node window around the docking centre in
# shared memory, every other cell from the padded global copy through L1 / L2

@pytest.mark.parametrize("n,h,offset", [(64, 1.0, (0.0, 0.0, 0.0)), (48, 0.5, (0.0, 0.0, 0.0)),
                                        (64, 1.0, (19.0, -21.5, 12.0))])
def test_large_grids_window_plus_global_path(n, h, offset):
    """64^3 at 1 A (ligands inside the window: shared-memory path), 48^3 at 0.5 A (the window spans
    only +-7.75 A: many corners come from global memory), and a 64^3 pocket whose centre sits near
    a corner (the window clamps to the grid edge).  Score hook against the oracle everywhere
    (inside / outside the window / outside the grid), then docking parity, every pose replayed."""
    pk = vsgen.pocket(108, n=n, spacing=h, center_offset=offset)
    e = engine()
    pid = e.load_pocket(pk)
    rng = np.random.default_rng(n)
    lo = np.array(pk.origin) - 4.0
    hi = np.array(pk.origin) + h * (n - 1) + 4.0
    pts = rng.uniform(lo, hi, size=(40000, 3)).astype(np.float32)
    near = (np.array(pk.center) + rng.normal(0, 6.0, size=(20000, 3))).astype(np.float32)
    pts = np.concatenate([pts, near])
    g = e.score_points(pid, pts)
    ref = oracle.grid_score(pk, pts.astype(np.float64))
    tol = 2e-6 if h == 1.0 else 2e-5      # 1/h inexact for h != 1 (see the non-cubic test)
    assert np.max(np.abs(g - ref) / np.maximum(1, np.abs(ref))) < tol
    lib = vsgen.ligands(24, 50 + n, (20, 120), (0, 12))
    e2, rot, tr, cs = run(lib, [pk], P=8, K=8)
    check(e2, lib, range(lib.n), pk, rot, tr, cs)


# ----------------------------------------------------------------------------- owned-only input
# (VERDICT r1 "missing" 5): mapped pinned host arrays read in place, per-rank a1 ingest

def test_mapped_host_input_matches_device_input_and_counts_owned_bytes():
    """on_device = 2: the offsets are copied and the kernels read coordinates / axes / moving atoms /
    ids from pinned host memory.  Bit-identical to device input; with W virtual ranks each rank moves
    only the offsets plus its own ligands' arrays (vs_stats.h2d_bytes)."""
    import torch
    c = vsgen.CONFIGS["C2"]
    lib = vsgen.ligands(3000, 61, c["atoms"], c["rot"])
    pk = vsgen.pocket(101)
    e, rot, tr, cs = run(lib, [pk], P=16, K=8, debug=False)
    r = e.results(0)
    pinned = [torch.from_numpy(a).pin_memory() for a in lib.arrays()]
    e2 = engine()
    setup(e2, [pk], 16, 8)
    e2.submit(*pinned, [0], on_device=2)
    e2.wait()
    r2 = e2.results(0)
    assert np.array_equal(r.best_score, r2.best_score) and np.array_equal(r.angles, r2.angles)
    assert np.array_equal(r2.ligand_id, lib.ligand_id) and np.array_equal(e.coords(0), e2.coords(0))
    full = sum(a.nbytes for a in lib.arrays())
    assert e2.stats()["h2d_bytes"] == full
    offs = lib.atom_off.nbytes + lib.frag_off.nbytes + lib.move_off.nbytes
    tot = 0
    for rank in range(4):
        eR = engine(rank=rank, world_size=4)
        setup(eR, [pk], 16, 8)
        eR.submit(*pinned, [0], on_device=2)
        eR.wait()
        rr = eR.results(0)
        own = ~np.isnan(rr.best_score)
        assert np.array_equal(rr.best_score[own], r.best_score[own])
        b = eR.stats()["h2d_bytes"] - offs
        assert 0 < b < 0.4 * (full - offs)
        tot += b
    assert tot == full - offs                       # the shards move every ligand's arrays exactly once


def test_rank_local_ingest_errors():
    """a1's per-atom checks run on each rank's own ligands: with 2 virtual ranks, an invalid ligand
    makes only its owner's submit fail (the other rank docks its share), naming the ligand."""
    from paper_2303_06150_b200 import VsError
    base = vsgen.ligands(400, 5, (20, 60), (1, 6))
    ligs = []
    for i in range(base.n):
        x, f = base.ligand(i)
        ligs.append((np.array(x, copy=True), vsgen.Frags(np.array(f.axis, copy=True), [np.array(m) for m in f.moves])))
    bad = 137
    ligs[bad][1].moves[0] = np.concatenate([ligs[bad][1].moves[0], ligs[bad][1].moves[0][:1]])   # duplicate entry
    lib = mk_lib(ligs)
    pk = vsgen.pocket(101)
    outcomes = {}
    for rank in range(2):
        e = engine(rank=rank, world_size=2)
        setup(e, [pk], 8, 8)
        try:
            e.submit_library(lib, [0])
            e.wait()
            outcomes[rank] = e.results(0)
        except VsError as err:
            outcomes[rank] = err
    errs = [o for o in outcomes.values() if isinstance(o, VsError)]
    assert len(errs) == 1 and errs[0].ligand == bad and "listed twice" in str(errs[0])
    ok = [o for o in outcomes.values() if not isinstance(o, VsError)][0]
    assert np.isnan(ok.best_score[bad]) and np.isfinite(ok.best_score).sum() > 100


def test_pipelined_zero_copy_matches():
    """PipelinedDocker with zero_copy (the multi-GPU default): identical outputs on one GPU."""
    import torch
    from paper_2303_06150_b200.pipeline import PipelinedDocker
    lib = vsgen.ligands(2000, 62, (20, 120), (0, 20))
    pk = vsgen.pocket(101)
    e, rot, tr, cs = run(lib, [pk], P=16, K=8, debug=False)
    r = e.results(0)
    pd = PipelinedDocker()
    pd.setup(rot, tr, cs, [pk])
    h = [torch.from_numpy(a).pin_memory() for a in lib.arrays()]
    out = pd.run(*h, k=50, chunks=0, zero_copy=True)
    assert np.array_equal(out["best_score"][0], r.best_score) and np.array_equal(out["xyz"][0], e.coords(0))
    assert list(out["topk"][0][0]) == list(oracle.topk(r.best_score, 50))
    pd.close()


def test_offsets_relative_to_their_first_entry():
    """A slice of a larger library (offsets starting at b != 0, data arrays starting at the slice) is
    docked exactly like the same ligands as a stand-alone batch, for host, device and mapped input."""
    import torch
    lib = vsgen.ligands(600, 63, (20, 120), (0, 20))
    lo, hi = 217, 431
    sub = lib.subset(np.arange(lo, hi))
    pk = vsgen.pocket(101)
    e, *_ = run(sub, [pk], P=8, K=8, debug=False)
    want, want_xyz = e.results(0), e.coords(0)
    a0, a1 = int(lib.atom_off[lo]), int(lib.atom_off[hi])
    f0, f1 = int(lib.frag_off[lo]), int(lib.frag_off[hi])
    m0, m1 = int(lib.move_off[f0]), int(lib.move_off[f1])
    sl = [lib.ligand_id[lo:hi], lib.atom_off[lo:hi + 1], lib.xyz[a0:a1], lib.frag_off[lo:hi + 1],
          lib.frag_axis[f0:f1], lib.move_off[f0:f1 + 1], lib.move_atoms[m0:m1]]
    variants = {0: [np.ascontiguousarray(a) for a in sl], 1: [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in sl],
                2: [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in sl]}
    for mode, arrs in variants.items():
        e2 = engine()
        setup(e2, [pk], 8, 8)
        e2.submit(*arrs, [0], on_device=mode, max_atoms=120)
        e2.wait()
        r = e2.results(0)
        assert np.array_equal(r.best_score, want.best_score) and np.array_equal(r.angles, want.angles), mode
        assert np.array_equal(r.ligand_id, lib.ligand_id[lo:hi]) and np.array_equal(e2.coords(0), want_xyz), mode


# ----------------------------------------------------------------------------- fused multi-site
# docking: one cluster launch per class docks every pocket

@pytest.mark.parametrize("S", [2, 3, 4, 8])
def test_fused_multisite_bit_identical_to_per_pocket_launches(S):
    """Thread-block clusters of S CTAs (one per pocket, records multicast once per cluster) give the
    same bits as one launch per pocket, for every pocket; one pocket's outputs pass the oracle."""
    lib = vsgen.ligands(1500 if S < 8 else 600, 70 + S, (20, 120), (0, 20))
    pks = [vsgen.pocket(101 + q, center_offset=(0.5 * q, -0.25 * q, 0.0)) for q in range(S)]
    outs = {}
    for fused in (True, False):
        e = engine(fused_sites=fused)
        rot, tr, cs, ids = setup(e, pks, 16, 8)
        e.submit_library(lib, ids)
        e.wait()
        st = e.stats()
        assert (st["fused_launches"] > 0) == fused
        outs[fused] = [(e.results(q), e.coords(q)) for q in range(S)]
    for q in range(S):
        (a, xa), (b, xb) = outs[True][q], outs[False][q]
        assert np.array_equal(a.best_score, b.best_score) and np.array_equal(a.best_pose, b.best_pose), q
        assert np.array_equal(a.angles, b.angles) and np.array_equal(xa, xb), q
    assert not np.array_equal(outs[True][0][0].best_score, outs[True][S - 1][0].best_score)
    r, x = outs[True][S - 1]
    rep = parity.check(lib, range(0, lib.n, 50), pks[S - 1], rot, tr, cs, r.best_score, r.best_pose, r.angles, x,
                       band=BAND, tol_score=TOL_S, tol_xyz=TOL_X)
    assert rep.ok, rep.summary() + str(rep.failures[:5])


# ----------------------------------------------------------------------------- third bucketing key
# (SURVEY 8(f) 4(d)): the moving-atom count sum_r |M_r|

@pytest.mark.parametrize("grid", [(6, 23, 4), (4, 5, 8), (1, 1, 3)])
def test_third_bucketing_key_manifest_bit_exact_and_results_unchanged(c2, grid):
    """Cells (atom class, rotamer class, moving-atom class): the GPU manifest equals the oracle's
    stable sort by the three keys chunked at capacity, and docking results are bit-identical to the
    two-key grid (the kernel's lane map does not depend on the cell)."""
    c, lib, pk = c2
    na, nr, nm = grid
    e, *_ = run(lib, [pk], P=16, K=8, debug=False, atom_clusters=na, rot_clusters=nr, move_clusters=nm,
                bucket_multiple=1)
    buckets, perm = e.manifest()
    cls = e.classes()
    M = lib.moving_per_ligand
    ab = oracle.atom_boundaries(na, 32, int(lib.n_atoms.max()))
    rb = oracle.rotamer_boundaries(nr, int(lib.n_frags.max()))
    mb = oracle.rotamer_boundaries(nm, int(M.max()))
    ref = oracle.bucketize(lib.n_atoms, lib.n_frags, ab, rb, [cl["capacity"] for cl in cls], n_move=M, move_b=mb)
    assert len(ref) == len(buckets) and len({b["move_class"] for b in buckets}) == len(mb)
    assert np.array_equal(perm, np.concatenate([b.ligands for b in ref]).astype(np.uint32))
    for b, rbk in zip(buckets, ref):
        assert (b["atom_class"], b["rot_class"], b["move_class"]) == rbk.cell and b["size"] == len(rbk.ligands)
    e2, *_ = run(lib, [pk], P=16, K=8, debug=False, atom_clusters=na, rot_clusters=nr)
    r, r2 = e.results(0), e2.results(0)
    assert np.array_equal(r.best_score, r2.best_score) and np.array_equal(r.angles, r2.angles)


# ----------------------------------------------------------------------------- rigid refinement (Q23)

def run_refine(lib, pk, P, K, n_ref, table, debug=True, **kw):
    e = engine(debug_poses=debug, **kw)
    rot, tr, cs, ids = setup(e, [pk], P, K)
    e.set_refine(n_ref, *table)
    e.submit_library(lib, ids)
    e.wait()
    return e, rot, tr, cs


def check_refine(e, lib, idx, pk, rot, tr, cs, n_ref, table, debug=True):
    r = e.results(0)
    xyz = e.coords(0)
    ps, pa = e.pose_debug(0) if debug else (None, None)
    prf = e.pose_refine_debug(0) if debug else None
    rep = parity.check(lib, idx, pk, rot, tr, cs, r.best_score, r.best_pose, r.angles, xyz, ps, pa, band=BAND,
                       tol_score=TOL_S, tol_xyz=TOL_X, refine=(n_ref,) + tuple(table), gpu_refine=e.refine(0),
                       gpu_pose_refine=prf)
    assert rep.ok, rep.summary() + "\n" + "\n".join(map(str, rep.failures[:10]))
    return rep, r


def test_refine_c1_full_parity_every_pose():
    """sweeps, then 2 rounds of 13 rigid moves (two lane groups of 8); every pose's
    angle AND refinement choices replayed in fp64, best-pose coordinates include the moves."""
    c = vsgen.CONFIGS["C1"]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    pk = vsgen.pocket(101)
    table = vsgen.refine_table()
    e, rot, tr, cs = run_refine(lib, pk, c["P"], c["K"], 2, table)
    rep, r = check_refine(e, lib, range(lib.n), pk, rot, tr, cs, 2, table)
    assert rep.independent_checked >= lib.n // 2 and rep.independent_equal == rep.independent_checked
    mv = e.refine(0)
    assert mv.shape == (lib.n, 2) and mv.max() < table[0].shape[0] and (mv != 0).any()
    # refinement never raises a pose's score: compare with the unrefined run
    e0, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
    assert np.all(r.best_score <= e0.results(0).best_score + 1e-5 * np.maximum(1, np.abs(r.best_score)))


def test_refine_c2_sample_parity_and_layout_invariance(c2):
    c, lib, pk = c2
    table = vsgen.refine_table(0.3, 8.0)
    e, rot, tr, cs = run_refine(lib, pk, c["P"], c["K"], 1, table)
    rng = np.random.default_rng(5)
    idx = rng.choice(lib.n, 300, replace=False)
    rep, r = check_refine(e, lib, idx, pk, rot, tr, cs, 1, table)
    assert rep.independent_equal == rep.independent_checked > 100
    # bit-identical under another cluster grid / launch structure (same lane map)
    e2, *_ = run_refine(lib, pk, c["P"], c["K"], 1, table, debug=False, atom_clusters=1, rot_clusters=1,
                        bucket_multiple=3)
    r2 = e2.results(0)
    assert np.array_equal(r2.best_score, r.best_score) and np.array_equal(r2.best_pose, r.best_pose)
    assert np.array_equal(e2.refine(0), e.refine(0))


def test_refine_identity_table_keeps_the_sweep_result():
    """A one-move (identity) table changes no pose, angle or coordinate; scores agree to fp32 rounding
    (the refined mode re-scores every atom at the end instead of finalising own regions)."""
    c = vsgen.CONFIGS["C1"]
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    pk = vsgen.pocket(101)
    q, d = vsgen.refine_table()
    e, *_ = run_refine(lib, pk, c["P"], c["K"], 3, (q[:1], d[:1]), debug=False)
    e0, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
    r, r0 = e.results(0), e0.results(0)
    assert np.array_equal(r.best_pose, r0.best_pose) and np.array_equal(r.angles, r0.angles)
    assert np.max(np.abs(r.best_score - r0.best_score) / np.maximum(1, np.abs(r0.best_score))) < 1e-6
    assert np.array_equal(e.coords(0), e0.coords(0))
    assert not e.refine(0).any()


def test_refine_table_validation():
    e = engine()
    q, d = vsgen.refine_table()
    from paper_2303_06150_b200.vsdock import VsError
    with pytest.raises(VsError, match="identity"):
        e.set_refine(1, q[1:], d[1:])
    with pytest.raises(VsError):
        e.set_refine(9, q, d)
    bad = d.copy()
    bad[3, 1] = np.nan
    with pytest.raises(VsError, match="non-finite"):
        e.set_refine(1, q, bad)
    e.set_refine(0)


# ----------------------------------------------------------------------------- per-atom-type grid channels
# (Q24): TYPED layout -- one QUAD window per channel in shared memory,
# the padded channels in global memory behind them

@pytest.mark.parametrize("T", [1, 2, 4, 8])
def test_typed_score_hook_vs_oracle(T):
    """g_{t}(y) on every channel: inside the channel windows, outside them (global path) and outside
    the grid, against the fp64 oracle; node exactness per channel."""
    pk = vsgen.typed_pocket(101, n_types=min(T, 4))
    if T > 4:   # 8 channels: the 4 typed ones and 4 scaled copies
        pk = vsgen.Pocket(np.concatenate([pk.grid, 0.5 * pk.grid]), pk.origin, pk.spacing, pk.center, pk.out_slope)
    e = engine()
    pid = e.load_pocket(pk)
    rng = np.random.default_rng(T)
    pts = np.concatenate([rng.uniform(-5, 36, size=(30000, 3)),
                          np.array(pk.center) + rng.normal(0, 5.0, size=(30000, 3))]).astype(np.float32)
    t = rng.integers(0, T, size=len(pts)).astype(np.uint8)
    g = e.score_points(pid, pts, types=t)
    ref = oracle.grid_score(pk, pts.astype(np.float64), t)
    assert np.max(np.abs(g - ref) / np.maximum(1, np.abs(ref))) < 2e-6
    nodes = rng.integers(0, 32, size=(4000, 3)).astype(np.float32)
    tn = rng.integers(0, T, size=4000).astype(np.uint8)
    g = e.score_points(pid, nodes, types=tn)
    G = pk.grid if pk.grid.ndim == 4 else pk.grid[None]
    assert np.array_equal(g, G[tn, nodes[:, 2].astype(int), nodes[:, 1].astype(int), nodes[:, 0].astype(int)])


def _typed_lib(lib, T, seed=11):
    lib.atom_type = vsgen.atom_types(lib, seed, n_types=min(T, 4))
    return lib


def test_typed_c1_full_parity_every_pose():
    c = vsgen.CONFIGS["C1"]
    lib = _typed_lib(vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"]), 4)
    pk = vsgen.typed_pocket(101, n_types=4)
    e, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"])
    rep, r = check(e, lib, range(lib.n), pk, rot, tr, cs)
    assert rep.independent_checked >= lib.n // 2 and rep.independent_equal == rep.independent_checked


def test_typed_c2_sample_parity_and_layout_invariance(c2):
    """C2 with 4 atom types: 300 ligands replayed (every pose), the independent oracle run
    bit-identical outside near-ties; the same bits from the unsorted grid, a per-bucket launch and
    a 3-stream submit; atom-permuted copies dock bit-identically (types follow their atoms)."""
    c, lib0, _ = c2
    lib = _typed_lib(lib0.subset(np.arange(lib0.n)), 4)
    pk = vsgen.typed_pocket(101, n_types=4)
    e, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"])
    idx = np.random.default_rng(5).choice(lib.n, 300, replace=False)
    rep, r = check(e, lib, idx, pk, rot, tr, cs)
    assert rep.independent_equal == rep.independent_checked > 100
    for kw in (dict(atom_clusters=1, rot_clusters=1), dict(launch_per_bucket=True, bucket_multiple=1),
               dict(n_streams=3)):
        e2, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False, **kw)
        r2 = e2.results(0)
        assert np.array_equal(r.best_score, r2.best_score) and np.array_equal(r.angles, r2.angles)
    sub = lib.subset(np.arange(200))
    lp, perm = sub.permuted(9)
    e3, *_ = run(sub, [pk], P=c["P"], K=c["K"], debug=False)
    e4, *_ = run(lp, [pk], P=c["P"], K=c["K"], debug=False)
    assert np.array_equal(e3.results(0).best_score, e4.results(0).best_score)
    assert np.array_equal(e4.coords(0)[perm], e3.coords(0))


def test_typed_copies_bit_identical_to_untyped(c2):
    """T identical channels and random types: the TYPED layout gives the untyped QUAD bits (the same
    blend on the same values); a typed pocket submitted untyped docks on channel 0."""
    c, lib0, pk = c2
    lib = lib0.subset(np.arange(2000))
    e, *_ = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
    r = e.results(0)
    pk3 = vsgen.Pocket(np.stack([pk.grid] * 3), pk.origin, pk.spacing, pk.center, pk.out_slope)
    lt = _typed_lib(lib.subset(np.arange(lib.n)), 3)
    e2, *_ = run(lt, [pk3], P=c["P"], K=c["K"], debug=False)
    r2 = e2.results(0)
    assert np.array_equal(r.best_score, r2.best_score) and np.array_equal(r.angles, r2.angles)
    assert np.array_equal(e.coords(0), e2.coords(0))
    e3, *_ = run(lib, [pk3], P=c["P"], K=c["K"], debug=False)          # untyped submit: channel 0
    assert np.array_equal(r.best_score, e3.results(0).best_score)


def test_typed_refinement_two_pockets_and_type_errors():
    """Typed docking with rigid refinement (Q23) into two typed pockets of different channel counts
    in one submit, full parity; a type >= a docked pocket's channels is VS_E_PARSE naming the ligand."""
    from paper_2303_06150_b200 import VsError
    lib = _typed_lib(vsgen.ligands(24, 31, (20, 90), (0, 8)), 2)
    pk2 = vsgen.typed_pocket(103, n_types=2)
    pk4 = vsgen.typed_pocket(104, n_types=4, center_offset=(1.5, -1.0, 0.5))
    q, d = vsgen.refine_table()
    e = engine(debug_poses=True)
    rot, tr, cs, ids = setup(e, [pk2, pk4], 8, 8)
    e.set_refine(2, q, d)
    e.submit_library(lib, ids)
    e.wait()
    for slot, pk in enumerate([pk2, pk4]):
        r = e.results(slot)
        ps, pa = e.pose_debug(slot)
        rep = parity.check(lib, range(lib.n), pk, rot, tr, cs, r.best_score, r.best_pose, r.angles, e.coords(slot),
                           ps, pa, band=BAND, tol_score=TOL_S, tol_xyz=TOL_X, refine=(2, q, d),
                           gpu_refine=e.refine(slot), gpu_pose_refine=e.pose_refine_debug(slot))
        assert rep.ok, rep.summary() + "\n" + "\n".join(map(str, rep.failures[:10]))
    bad = lib.subset(np.arange(lib.n))
    bad.atom_type = bad.atom_type.copy()
    bad.atom_type[int(bad.atom_off[5]) + 3] = 2                      # pk2 has channels 0, 1 only
    with pytest.raises(VsError, match="ligand 5"):
        e.submit_library(bad, ids)


def test_typed_pipelined_docker_matches_single_submit(c2):
    """The public host API with atom types (PipelinedDocker.run(atom_type=...), Q24): chunked,
    double-buffered, bit-identical to one typed submit, outputs pass parity on a sample."""
    import torch
    from paper_2303_06150_b200.pipeline import PipelinedDocker
    c, lib0, _ = c2
    lib = _typed_lib(lib0.subset(np.arange(3000)), 4)
    pk = vsgen.typed_pocket(102, n_types=4)
    e, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
    r = e.results(0)
    pd = PipelinedDocker()
    pd.setup(rot, tr, cs, [pk])
    h = [torch.from_numpy(a).pin_memory() for a in lib.arrays()]
    out = pd.run(*h, k=50, chunks=3, atom_type=torch.from_numpy(lib.atom_type).pin_memory())
    assert np.array_equal(out["best_score"][0], r.best_score) and np.array_equal(out["angles"][0], r.angles)
    assert np.array_equal(out["xyz"][0], e.coords(0))
    rep = parity.check(lib, np.arange(0, lib.n, 100), pk, rot, tr, cs, out["best_score"][0], out["best_pose"][0],
                       out["angles"][0], out["xyz"][0], band=BAND, tol_score=TOL_S, tol_xyz=TOL_X)
    assert rep.ok, rep.summary() + str(rep.failures[:5])
    pd.close()


@pytest.mark.parametrize("layout", ["quad", "scalar"])
def test_typed_large_noncubic_grid_window_misses(layout, monkeypatch):
    """TYPED on a 48 x 40 x 44 grid at 0.75 A with the docking centre off-centre, in both channel
    layouts (QUAD windows / scalar windows, VSDOCK_TYPED_LAYOUT): the channel windows cover only
    part of the pocket, so many cells come from the global copy (and beyond the grid, the clamp +
    excess); score hook on every channel against the oracle, then docking parity with every pose
    replayed."""
    monkeypatch.setenv("VSDOCK_TYPED_LAYOUT", layout)
    base = vsgen.typed_pocket(105, n_types=3, n=(48, 40, 44), spacing=0.75, center_offset=(2.0, -1.5, 1.0))
    e = engine(debug_poses=True)
    pid = e.load_pocket(base)
    rng = np.random.default_rng(11)
    lo = np.array(base.origin) - 3.0
    hi = np.array(base.origin) + 0.75 * np.array([47, 39, 43]) + 3.0
    pts = np.concatenate([rng.uniform(lo, hi, size=(30000, 3)),
                          np.array(base.center) + rng.normal(0, 7.0, size=(30000, 3))]).astype(np.float32)
    t = rng.integers(0, 3, size=len(pts)).astype(np.uint8)
    g = e.score_points(pid, pts, types=t)
    ref = oracle.grid_score(base, pts.astype(np.float64), t)
    assert np.max(np.abs(g - ref) / np.maximum(1, np.abs(ref))) < 2e-5     # 1/h inexact for h != 1
    lib = _typed_lib(vsgen.ligands(24, 41, (20, 110), (0, 10)), 3)
    rot, tr, cs = vsgen.pose_table(8)[0], vsgen.pose_table(8)[1], vsgen.angle_table(8)
    e.set_poses(rot, tr)
    e.set_angles(cs)
    e.submit_library(lib, [pid])
    e.wait()
    check(e, lib, range(lib.n), base, rot, tr, cs)


@pytest.mark.parametrize("T", [2, 3, 4])
def test_typed_layouts_quad_and_scalar_bit_identical(c2, T, monkeypatch):
    """The two TYPED channel layouts (QUAD windows: two LDS.128 per point; scalar windows of ~1.6x
    the edge: eight LDS.32) read the same corner values and blend them in the same order, so a
    typed submit docks bit-identically in both; the scalar layout's result passes parity on a
    sample."""
    c, lib0, _ = c2
    lib = _typed_lib(lib0.subset(np.arange(1500)), T)
    pk = vsgen.typed_pocket(106, n_types=T)
    out = {}
    for layout in ("quad", "scalar"):
        monkeypatch.setenv("VSDOCK_TYPED_LAYOUT", layout)
        e, rot, tr, cs = run(lib, [pk], P=c["P"], K=c["K"], debug=False)
        out[layout] = (e.results(0), e.coords(0))
    (rq, xq), (rs, xs) = out["quad"], out["scalar"]
    assert np.array_equal(rq.best_score, rs.best_score) and np.array_equal(rq.angles, rs.angles)
    assert np.array_equal(rq.best_pose, rs.best_pose) and np.array_equal(xq, xs)
    rep = parity.check(lib, np.arange(0, lib.n, 50), pk, rot, tr, cs, rs.best_score, rs.best_pose, rs.angles, xs,
                       band=BAND, tol_score=TOL_S, tol_xyz=TOL_X)
    assert rep.ok, rep.summary() + str(rep.failures[:5])


@pytest.mark.parametrize("layout", ["quad", "scalar"])
def test_typed_grid_smaller_than_the_window(layout, monkeypatch):
    """A 14^3 typed pocket (3 channels) is smaller than either layout's channel window (13 / 20 cells):
    the windows clamp to the grid, nodes past its pads stay zero, and atoms outside the box take the
    clamp + excess; score hook on every channel against the oracle, then docking parity with every
    pose replayed."""
    monkeypatch.setenv("VSDOCK_TYPED_LAYOUT", layout)
    pk = vsgen.typed_pocket(107, n_types=3, n=14, spacing=1.0, shell=(4.0, 6.0), n_receptor=40)
    e = engine(debug_poses=True)
    pid = e.load_pocket(pk)
    rng = np.random.default_rng(5)
    pts = (np.array(pk.center) + rng.normal(0, 6.0, size=(20000, 3))).astype(np.float32)
    t = rng.integers(0, 3, size=len(pts)).astype(np.uint8)
    g = e.score_points(pid, pts, types=t)
    ref = oracle.grid_score(pk, pts.astype(np.float64), t)
    assert np.max(np.abs(g - ref) / np.maximum(1, np.abs(ref))) < 2e-6
    lib = _typed_lib(vsgen.ligands(20, 43, (20, 70), (0, 8)), 3)
    rot, tr = vsgen.pose_table(8, tau=1.0)
    cs = vsgen.angle_table(8)
    e.set_poses(rot, tr)
    e.set_angles(cs)
    e.submit_library(lib, [pid])
    e.wait()
    check(e, lib, range(lib.n), pk, rot, tr, cs)
