"""Pins of the fp64 docking oracle (oracle/oracle.c) to things other than itself.

Each test names the SURVEY 8(c) pin it implements and the DESIGN.md reading it
freezes.  Independent references used here: closed forms (multilinear and
linear grids), scipy.ndimage.map_coordinates (library trilinear interpolation),
scipy.spatial.transform.Rotation (library Rodrigues rotation), invariants of
rigid motions, and an exhaustive numpy brute force over all K^R angle
combinations on tiny ligands.
"""
import itertools
import math

import numpy as np
import pytest
from scipy.ndimage import map_coordinates
from scipy.spatial.transform import Rotation

import oracle
import vsgen


def mkpocket(G, origin=(0.0, 0.0, 0.0), h=1.0, center=None, kappa=1.0):
    G = np.ascontiguousarray(G, np.float32)
    nz, ny, nx = G.shape[-3:]
    if center is None:
        center = tuple(origin[a] + h * (n - 1) / 2 for a, n in enumerate((nx, ny, nz)))
    return vsgen.Pocket(G, tuple(origin), float(h), tuple(center), float(kappa))


def lib_ref_score(pk, pts):
    """Independent g: scipy trilinear (clamped, 'nearest') + kappa*h*L1 excess (reading Q9)."""
    u = (np.asarray(pts, np.float64) - np.array(pk.origin)) / pk.spacing
    nx, ny, nz = pk.dims
    top = np.array([nx - 1, ny - 1, nz - 1], np.float64)
    uc = np.clip(u, 0.0, top)
    e = np.abs(u - uc).sum(axis=1)
    v = map_coordinates(pk.grid.astype(np.float64), [uc[:, 2], uc[:, 1], uc[:, 0]], order=1, mode="nearest")
    return v + pk.out_slope * pk.spacing * e


# ----------------------------------------------------------------------------- a8 interpolation

def test_grid_node_exactness():
    rng = np.random.default_rng(0)
    G = rng.normal(size=(5, 6, 7)).astype(np.float32)
    pk = mkpocket(G, origin=(1.0, -2.0, 0.5), h=0.5)
    pts, want = [], []
    for k in range(5):
        for j in range(6):
            for i in range(7):
                pts.append([1.0 + 0.5 * i, -2.0 + 0.5 * j, 0.5 + 0.5 * k])
                want.append(float(G[k, j, i]))
    got = oracle.grid_score(pk, np.array(pts))
    assert np.array_equal(got, np.array(want))          # bitwise, incl. upper edges (i0 = n-2, f = 1)


def test_grid_multilinear_closed_form():
    # trilinear interpolation reproduces any multilinear polynomial exactly (closed form)
    a, b, c, d, e, f, g, h = 3, -2, 5, 1, 2, -1, 4, -3
    poly = lambda x, y, z: a + b * x + c * y + d * z + e * x * y + f * y * z + g * z * x + h * x * y * z
    Z, Y, X = np.meshgrid(np.arange(6), np.arange(7), np.arange(8), indexing="ij")
    G = poly(X, Y, Z).astype(np.float32)                 # integers: exact in fp32
    pk = mkpocket(G)
    rng = np.random.default_rng(1)
    p = rng.uniform([0, 0, 0], [7, 6, 5], size=(2000, 3))
    got = oracle.grid_score(pk, p)
    want = poly(p[:, 0], p[:, 1], p[:, 2])
    assert np.max(np.abs(got - want)) < 1e-9


def test_grid_matches_scipy_trilinear_inside_and_outside():
    rng = np.random.default_rng(2)
    G = rng.normal(size=(9, 10, 11)).astype(np.float32)
    pk = mkpocket(G, origin=(-3.0, 2.0, 1.0), h=0.75, kappa=2.5)
    lo = np.array(pk.origin) - 4.0
    hi = np.array(pk.origin) + 0.75 * np.array([10, 9, 8]) + 4.0
    p = rng.uniform(lo, hi, size=(5000, 3))
    assert np.max(np.abs(oracle.grid_score(pk, p) - lib_ref_score(pk, p))) < 1e-12


def test_far_atom_penalty_closed_form():
    G = np.full((4, 4, 4), 2.0, np.float32)
    G[3, 3, 3] = 7.0
    pk = mkpocket(G, h=2.0, kappa=1.5)
    # 10 A beyond the upper corner on x, 4 A below 0 on y, inside on z at the top face
    y = np.array([[6.0 + 10.0, -4.0, 6.0]])
    # clamped point = node (3, 0, 3) -> 2.0; excess in grid units = 10/2 + 4/2 = 7
    assert oracle.grid_score(pk, y)[0] == pytest.approx(2.0 + 1.5 * 2.0 * 7.0, abs=1e-12)
    y = np.array([[6.0 + 3.0, 6.0 + 3.0, 6.0 + 3.0]])
    assert oracle.grid_score(pk, y)[0] == pytest.approx(7.0 + 1.5 * 2.0 * 4.5, abs=1e-12)


# ----------------------------------------------------------------------------- a6 placement

@pytest.fixture(scope="module")
def c1():
    c = vsgen.CONFIGS["C1"]
    L = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    return L, vsgen.pocket(101), vsgen.pose_table(c["P"]), vsgen.angle_table(c["K"])


def test_identity_pose(c1):
    L, pk, (rot, tr), _ = c1
    assert np.array_equal(rot[0], np.eye(3, dtype=np.float32)) and not tr.any()
    for i in range(L.n):
        x, _ = L.ligand(i)
        y = oracle.place(pk, x, rot[0], tr[0])
        want = x.astype(np.float64) - x.astype(np.float64).mean(axis=0) + np.array(pk.center)
        assert np.max(np.abs(y - want)) < 1e-12


def test_pose_rotation_invariants(c1):
    L, pk, (rot, tr), _ = c1
    for p in range(rot.shape[0]):
        R = rot[p].astype(np.float64)
        assert np.max(np.abs(R.T @ R - np.eye(3))) < 1e-6
        assert abs(np.linalg.det(R) - 1.0) < 1e-6
    for i in range(4):
        x, _ = L.ligand(i)
        d0 = np.linalg.norm(x[:, None].astype(np.float64) - x[None].astype(np.float64), axis=-1)
        for p in range(rot.shape[0]):
            y = oracle.place(pk, x, rot[p], tr[p])
            d = np.linalg.norm(y[:, None] - y[None], axis=-1)
            assert np.max(np.abs(d - d0)) < 1e-5
            assert np.max(np.abs(y.mean(axis=0) - np.array(pk.center))) < 1e-9
            # closed form R (x - xbar) + c (numpy, independent of the oracle's loops)
            want = (x.astype(np.float64) - x.astype(np.float64).mean(0)) @ rot[p].astype(np.float64).T
            assert np.max(np.abs(y - (want + np.array(pk.center)))) < 1e-9


# ----------------------------------------------------------------------------- a7 fragment rotation

def test_fragment_rotation_matches_scipy_rodrigues(c1):
    L, pk, (rot, tr), _ = c1
    rng = np.random.default_rng(3)
    for i in range(L.n):
        x, fr = L.ligand(i)
        if len(fr) == 0:
            continue
        y = oracle.place(pk, x, rot[1], tr[1])
        for a, b, mv in fr:
            theta = rng.uniform(-math.pi, math.pi)
            got = oracle.rotate(y, (a, b, mv), math.cos(theta), math.sin(theta))
            u = (y[b] - y[a]) / np.linalg.norm(y[b] - y[a])
            want = y.copy()
            want[mv] = Rotation.from_rotvec(theta * u).apply(y[mv] - y[b]) + y[b]
            assert np.max(np.abs(got - want)) < 1e-12          # sign convention: right-hand rule about a->b


def test_fragment_rotation_invariants(c1):
    L, pk, (rot, tr), cs = c1
    for i in range(L.n):
        x, fr = L.ligand(i)
        y = oracle.place(pk, x, rot[2], tr[2])
        for a, b, mv in fr:
            f = (a, b, mv)
            y0 = oracle.rotate(y, f, cs[0, 0], cs[0, 1])
            assert np.array_equal(y0, y)                          # theta_0 = 0 -> identity, bitwise
            y1 = oracle.rotate(y, f, cs[1, 0], cs[1, 1])
            assert np.array_equal(y1[[a, b]], y[[a, b]])          # axis atoms fixed
            mov = np.zeros(len(y), bool); mov[mv] = True
            for grp in (mov, ~mov):                               # both rigid bodies keep their shape
                d0 = np.linalg.norm(y[grp][:, None] - y[grp][None], axis=-1)
                d1 = np.linalg.norm(y1[grp][:, None] - y1[grp][None], axis=-1)
                assert np.max(np.abs(d1 - d0)) < 1e-6
            # distances from the axis atoms to moving atoms are preserved (bond lengths across the axis)
            for ax in (a, b):
                assert np.max(np.abs(np.linalg.norm(y1[mv] - y1[ax], axis=1) - np.linalg.norm(y[mv] - y[ax], axis=1))) < 1e-6
            yk = y
            for _ in range(cs.shape[0]):                          # K steps of 2 pi / K return to start
                yk = oracle.rotate(yk, f, cs[1, 0], cs[1, 1])
            assert np.max(np.abs(yk - y)) < 1e-4


# ----------------------------------------------------------------------------- a7/a9 sweep + best pose

def test_sweep_is_monotone_and_greedy(c1):
    L, pk, (rot, tr), cs = c1
    r = oracle.dock_batch(L, pk, rot, tr, cs)
    P = rot.shape[0]
    for i in range(L.n):
        x, fr = L.ligand(i)
        R = len(fr)
        for p in range(P):
            kseq = r.pose_angles[P * r_off(L, i) + p * R: P * r_off(L, i) + (p + 1) * R]
            s, y, steps = oracle.replay_pose(pk, x, fr, rot[p], tr[p], cs, kseq)
            assert s == r.pose_score[i, p]
            prev = float(oracle.grid_score(pk, oracle.place(pk, x, rot[p], tr[p])).sum())
            for st, k in zip(steps, kseq):
                assert st[k] == st.min() and k == int(np.argmin(st))   # lowest k attaining the min (Q11)
                assert abs(st[0] - prev) < 1e-9                        # k = 0 is the current pose
                assert st[k] <= prev + 1e-12                           # monotone
                prev = st[k]
        assert r.best_pose[i] == int(np.argmin(r.pose_score[i]))
        assert r.best_score[i] == r.pose_score[i].min()


def r_off(L, i):
    return int(L.frag_off[i])


def test_constant_grid_ties_go_to_lowest_index(c1):
    L, _, (rot, tr), cs = c1
    pk = mkpocket(np.full((32, 32, 32), 0.25, np.float32), kappa=0.0)
    r = oracle.dock_batch(L, pk, rot, tr, cs)
    assert (r.best_pose == 0).all() and not r.angles.any()
    assert np.allclose(r.best_score, 0.25 * L.n_atoms, atol=1e-9)


def test_K1_or_R0_is_rigid_only(c1):
    L, pk, (rot, tr), _ = c1
    r = oracle.dock_batch(L, pk, rot, tr, np.array([[1.0, 0.0]], np.float32))
    for i in range(L.n):
        x, _ = L.ligand(i)
        s = [oracle.grid_score(pk, oracle.place(pk, x, rot[p], tr[p])).sum() for p in range(rot.shape[0])]
        assert abs(r.best_score[i] - min(s)) < 1e-9 and r.best_pose[i] == int(np.argmin(s))


@pytest.mark.parametrize("tau,offset", [(0.0, (0.0, 0.0, 0.0)), (1.5, (2.5, -3.0, 1.25))])
def test_linear_grid_closed_form(tau, offset):
    """G = w.u + g0 with every atom inside the box: S = A*g0 + w.sum(u_i).  Without translations every
    initial pose ties (rigid rotation about the centroid keeps sum y), and each greedy step picks
    argmin_k w.M_k v_r with v_r = sum_{i in M_r} (y_i - q) -- computed here with scipy's rotation.
    The second case carries pose translations tau_p != 0 and a docking centre c off the grid centre:
    y = R_p (x - xbar) + c + tau_p (a6)."""
    n, h = 32, 2.0
    w = np.array([0.7, -1.3, 0.4])
    Z, Y, X = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    G = (w[0] * X + w[1] * Y + w[2] * Z + 5.0).astype(np.float64)
    ctr = tuple(h * (n - 1) / 2 + o for o in offset)
    pk = mkpocket(G.astype(np.float32), h=h, center=ctr)
    Gf = pk.grid.astype(np.float64)
    assert np.max(np.abs(Gf - G)) < 1e-5
    L = vsgen.ligands(12, 11, (20, 60), (2, 6))
    rot, tr = vsgen.pose_table(6, tau=tau)
    assert (np.abs(tr[1:]).max() > 0.1) == (tau > 0)
    K = 8
    cs = vsgen.angle_table(K)
    r = oracle.dock_batch(L, pk, rot, tr, cs)
    for i in range(L.n):
        x, fr = L.ligand(i)
        p = int(r.best_pose[i])
        y = ((x.astype(np.float64) - x.astype(np.float64).mean(0)) @ rot[p].astype(np.float64).T + np.array(ctr)
             + tr[p].astype(np.float64))
        init = [oracle.grid_score(pk, oracle.place(pk, x, rot[q], tr[q])).sum() for q in range(6)]
        if tau == 0:
            assert np.ptp(init) < 1e-6 * max(1.0, abs(init[0]))
        else:   # S_p^0 = A g0 + w.(A (c + tau_p - o) / h): the translation enters linearly
            want0 = [x.shape[0] * (5.0 + w @ ((np.array(ctr) + tr[q] - np.array(pk.origin)) / h)) for q in range(6)]
            assert np.max(np.abs(np.array(init) - want0)) < 1e-6 * max(1.0, abs(want0[0]))
        kseq = r.angles[r_off(L, i): r_off(L, i) + len(fr)]
        for (a, b, mv), kg in zip(fr, kseq):
            u = (y[b] - y[a]) / np.linalg.norm(y[b] - y[a])
            v = (y[mv] - y[b]).sum(axis=0)
            vals = [w @ Rotation.from_rotvec(math.atan2(cs[k, 1], cs[k, 0]) * u).apply(v) / h for k in range(K)]
            assert vals[kg] <= min(vals) + 1e-6 * max(1.0, abs(min(vals)))
            y[mv] = Rotation.from_rotvec(math.atan2(cs[kg, 1], cs[kg, 0]) * u).apply(y[mv] - y[b]) + y[b]
        want = x.shape[0] * 5.0 + (w @ ((y - np.array(pk.origin)) / h).sum(axis=0))
        assert abs(r.best_score[i] - want) < 1e-4 * max(1.0, abs(want))


def test_placement_with_translation_and_offcentre_pocket_closed_form():
    """a6 with tau_p != 0 and c != grid centre: numpy R (x - xbar) + c + tau against oracle.place, and
    a replay of the all-zero angle sequence (identity steps) ends at the same coordinates with the
    scipy-trilinear score of them (independent of the oracle's loops)."""
    pk = vsgen.pocket(101, center_offset=(1.75, -2.5, 3.0))
    assert np.max(np.abs(np.array(pk.center) - 15.5 - np.array([1.75, -2.5, 3.0]))) < 1e-12
    rot, tr = vsgen.pose_table(8, tau=2.0)
    assert np.all(np.linalg.norm(tr[1:], axis=1) > 0) and np.all(np.linalg.norm(tr, axis=1) <= 2.0 + 1e-6)
    cs = vsgen.angle_table(8)
    L = vsgen.ligands(6, 1, (20, 40), (1, 4))
    for i in range(L.n):
        x, fr = L.ligand(i)
        xc = x.astype(np.float64) - x.astype(np.float64).mean(0)
        for p in range(rot.shape[0]):
            want = xc @ rot[p].astype(np.float64).T + np.array(pk.center) + tr[p].astype(np.float64)
            y = oracle.place(pk, x, rot[p], tr[p])
            assert np.max(np.abs(y - want)) < 1e-9
            assert np.max(np.abs(y.mean(0) - (np.array(pk.center) + tr[p]))) < 1e-9   # centroid = c + tau_p
            s, yr, _ = oracle.replay_pose(pk, x, fr, rot[p], tr[p], cs, np.zeros(len(fr), np.uint8))
            assert np.array_equal(yr, y)
            assert abs(s - lib_ref_score(pk, want).sum()) < 1e-9 * max(1.0, abs(s))


def test_oracle_invariant_under_atom_renumbering():
    """The moving sets are atom SUBSETS: renumbering the atoms of every ligand (and
    remapping axes and sets) must not change what is docked -- same best pose and angle sequence,
    same score up to fp64 summation order, same coordinates (mapped back)."""
    c = vsgen.CONFIGS["C1"]
    L = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    Lp, perm = L.permuted(5)
    assert any(not np.array_equal(m, np.arange(m.min(), m.max() + 1)) for _, _, m in Lp.ligand(0)[1]) or \
        any(len(Lp.ligand(i)[1]) for i in range(L.n))
    pk = vsgen.pocket(101, center_offset=(0.5, 1.0, -0.75))
    rot, tr = vsgen.pose_table(c["P"], tau=1.0)
    cs = vsgen.angle_table(c["K"])
    a = oracle.dock_batch(L, pk, rot, tr, cs)
    b = oracle.dock_batch(Lp, pk, rot, tr, cs)
    assert np.array_equal(a.best_pose, b.best_pose) and np.array_equal(a.angles, b.angles)
    assert np.max(np.abs(a.best_score - b.best_score) / np.maximum(1, np.abs(a.best_score))) < 1e-12
    assert np.max(np.abs(a.xyz - b.xyz[perm])) < 1e-9      # new[perm[j]] = old[j]


def _brute_force(pk, x, fr, rot, cs):
    """Exhaustive min over all K^R angle combinations and all poses; numpy + scipy only."""
    K = cs.shape[0]
    thetas = [math.atan2(float(cs[k, 1]), float(cs[k, 0])) for k in range(K)]
    best = math.inf
    xc = x.astype(np.float64) - x.astype(np.float64).mean(0)
    for p in range(rot.shape[0]):
        y0 = xc @ rot[p].astype(np.float64).T + np.array(pk.center)
        for combo in itertools.product(range(K), repeat=len(fr)):
            y = y0.copy()
            for (a, b, mv), k in zip(fr, combo):
                u = (y[b] - y[a]) / np.linalg.norm(y[b] - y[a])
                y[mv] = Rotation.from_rotvec(thetas[k] * u).apply(y[mv] - y[b]) + y[b]
            best = min(best, float(lib_ref_score(pk, y).sum()))
    return best


def _star_ligand(rng, arms):
    """Centre atom 0 with `arms` branches (b, then 2 moving atoms), DFS preorder; disjoint M_r and no
    axis atom inside another fragment's moving set -> the score separates over fragments."""
    pts = [np.zeros(3)]
    frags = []
    dirs = [np.array(v, np.float64) / np.linalg.norm(v) for v in ([1, 1, 1], [-1, -1, 1], [-1, 1, -1], [1, -1, -1])]
    for a in range(arms):
        d = dirs[a]
        b = len(pts)
        pts.append(1.5 * d)
        perp = np.cross(d, [0.3, 0.5, 0.8]); perp /= np.linalg.norm(perp)
        pts.append(1.5 * d + 1.5 * (0.33 * d + 0.94 * perp) + rng.normal(scale=0.05, size=3))
        pts.append(pts[-1] + 1.5 * d + rng.normal(scale=0.05, size=3))
        frags.append([0, b, b + 1, b + 3])
    x = (np.array(pts) + np.array([15.5, 15.5, 15.5])).astype(np.float32)
    return x, vsgen.Frags.from_ranges(np.array(frags, np.int32))


def test_brute_force_star_ligands_greedy_is_exact():
    rng = np.random.default_rng(4)
    pk = vsgen.pocket(101)
    rot, tr = vsgen.pose_table(3)
    cs = vsgen.angle_table(8)
    for arms in (1, 2, 3):
        x, fr = _star_ligand(rng, arms)
        lib = vsgen.Library.from_ligands([(x, fr)])
        r = oracle.dock_batch(lib, pk, rot, tr, cs)
        bf = _brute_force(pk, x, fr, rot, cs)
        assert abs(r.best_score[0] - bf) < 1e-9 * max(1.0, abs(bf))
        # the same molecule with shuffled atom numbers: moving sets are arbitrary subsets now
        lp, _ = lib.permuted(arms)
        xp, frp = lp.ligand(0)
        rp = oracle.dock_batch(lp, pk, rot, tr, cs)
        bfp = _brute_force(pk, xp, frp, rot, cs)
        assert abs(bfp - bf) < 1e-9 * max(1.0, abs(bf))
        assert abs(rp.best_score[0] - bfp) < 1e-9 * max(1.0, abs(bfp))


def test_brute_force_general_ligands_greedy_upper_bounds(c1):
    L, pk, (rot, tr), cs = c1
    sel = [i for i in range(L.n) if 1 <= L.n_frags[i] <= 3][:4]
    assert sel
    r = oracle.dock_batch(L.subset(sel), pk, rot[:3], tr[:3], cs)
    for j, i in enumerate(sel):
        x, fr = L.ligand(i)
        bf = _brute_force(pk, x, fr, rot[:3], cs)
        assert r.best_score[j] >= bf - 1e-9 * max(1.0, abs(bf))


# ----------------------------------------------------------------------------- S_w > 1 sweeps (Q13)

def test_second_sweep_extends_the_first_and_never_raises_the_score(c1):
    """The greedy is deterministic, so the first sweep of S_w = 2 replays S_w = 1 exactly
    (identical angle choices) and the second sweep -- angle 0 is always a candidate -- can
    only keep or lower every pose's score; a constant grid keeps every choice at 0."""
    L, pk, (rot, tr), cs = c1
    r1 = oracle.dock_batch(L, pk, rot, tr, cs, S_w=1)
    r2 = oracle.dock_batch(L, pk, rot, tr, cs, S_w=2)
    P = rot.shape[0]
    for i in range(L.n):
        R = int(L.frag_off[i + 1] - L.frag_off[i])
        f0 = int(L.frag_off[i])
        for p in range(P):
            a1 = r1.pose_angles[P * f0 + p * R: P * f0 + (p + 1) * R]
            a2 = r2.pose_angles[P * 2 * f0 + p * 2 * R: P * 2 * f0 + (p + 1) * 2 * R]
            assert np.array_equal(a2[:R], a1)
        assert np.all(r2.pose_score[i] <= r1.pose_score[i] + 1e-12)
    assert np.all(r2.best_score <= r1.best_score + 1e-12)
    flat = mkpocket(np.full((32, 32, 32), 0.25, np.float32), kappa=0.0)
    r3 = oracle.dock_batch(L, flat, rot, tr, cs, S_w=3)
    assert not r3.angles.any() and not r3.best_pose.any()


# ----------------------------------------------------------------------------- rigid refinement (Q23)

def test_rigid_move_matches_scipy_about_the_centroid(c1):
    """Move m about the current centroid: y' = Q (y - ybar) + ybar + d, checked against scipy's
    rotation applied to centred coordinates (Q23)."""
    L, pk, (rot, tr), cs = c1
    q, d = vsgen.refine_table(0.3, 12.0)
    x, _ = L.ligand(3)
    y = oracle.place(pk, x, rot[2], tr[2])
    yb = y.mean(0)
    for m in range(q.shape[0]):
        got = oracle.rigid_move(y, q[m], d[m])
        R = Rotation.from_matrix(q[m].astype(np.float64))
        want = R.apply(y - yb) + yb + d[m].astype(np.float64)
        assert np.max(np.abs(got - want)) < 1e-5   # fp32 table entries vs scipy's orthonormalised matrix
        # rigid: pairwise distances preserved; centroid moves by exactly d
        D0 = np.linalg.norm(y[:, None] - y[None], axis=-1)
        D1 = np.linalg.norm(got[:, None] - got[None], axis=-1)
        assert np.max(np.abs(D0 - D1)) < 1e-5
        assert np.max(np.abs(got.mean(0) - (yb + d[m]))) < 1e-9
    assert np.array_equal(oracle.rigid_move(y, q[0], d[0]), y)   # move 0 is the identity, bit for bit


def test_refinement_identity_table_changes_nothing(c1):
    """A one-move table (the identity) leaves every pose, score and angle exactly as without refinement."""
    L, pk, (rot, tr), cs = c1
    base = oracle.dock_batch(L, pk, rot, tr, cs)
    q, d = vsgen.refine_table()
    r = oracle.dock_batch(L, pk, rot, tr, cs, refine=(3, q[:1], d[:1]))
    assert np.array_equal(r.best_score, base.best_score)
    assert np.array_equal(r.best_pose, base.best_pose)
    assert np.array_equal(r.angles, base.angles)
    assert np.array_equal(r.xyz, base.xyz)
    assert not r.refine.any()


def test_refinement_linear_grid_closed_form():
    """G = w.u + g0 with every atom inside the box: a rotation about the centroid leaves S unchanged
    (sum of w.Q(y_i - ybar) = 0) and a translation d changes it by A w.d / h, so each greedy round
    takes the translation with the most negative w.d (ties -> lowest move index, the identity first)
    and the score falls by exactly A |w.d| / h per round."""
    n, h = 32, 1.0
    w = np.array([0.7, -1.3, 0.4])
    Z, Y, X = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    G = (w[0] * X + w[1] * Y + w[2] * Z + 5.0).astype(np.float32)
    pk = mkpocket(G, h=h, center=(15.5, 15.5, 15.5))
    L = vsgen.ligands(6, 11, (20, 40), (0, 3))
    rot, tr = vsgen.pose_table(3)
    cs = vsgen.angle_table(4)
    q, d = vsgen.refine_table(0.5, 15.0)
    vals = [float(w @ d[m]) for m in range(q.shape[0])]
    m_best = int(np.argmin(vals))                    # -0.5 along y (w_y = -1.3 < 0): move 3
    assert m_best == 3
    base = oracle.dock_batch(L, pk, rot, tr, cs)
    n_ref = 3
    r = oracle.dock_batch(L, pk, rot, tr, cs, refine=(n_ref, q, d))
    A = np.diff(L.atom_off)
    assert np.array_equal(r.refine, np.full((L.n, n_ref), m_best, np.uint8))
    want = base.best_score + n_ref * A * vals[m_best] / h
    # exact up to the fp32 storage of the linear grid's node values (~1e-7 relative)
    assert np.max(np.abs(r.best_score - want) / np.maximum(1, np.abs(want))) < 1e-6
    # translations only: the best pose's coordinates are the unrefined ones shifted n_ref times
    assert np.array_equal(r.best_pose, base.best_pose)
    assert np.max(np.abs(r.xyz - (base.xyz + n_ref * d[m_best]))) < 1e-5


def test_refinement_replay_scores_every_move_and_never_raises_the_score(c1):
    """Replaying the chosen moves reproduces the docked score; every chosen move is the minimum of
    its round's move scores (the identity is a candidate, so no round raises the score)."""
    L, pk, (rot, tr), cs = c1
    q, d = vsgen.refine_table()
    n_ref = 2
    r = oracle.dock_batch(L, pk, rot, tr, cs, refine=(n_ref, q, d))
    base = oracle.dock_batch(L, pk, rot, tr, cs)
    for i in range(L.n):
        x, fr = L.ligand(i)
        p = int(r.best_pose[i])
        kseq = r.angles[r_off(L, i): r_off(L, i) + len(fr)]
        s, y, steps, rs = oracle.replay_pose(pk, x, fr, rot[p], tr[p], cs, kseq, refine=(n_ref, q, d),
                                             mseq=r.refine[i], want_refine=True)
        assert abs(s - r.best_score[i]) < 1e-12 * max(1.0, abs(s))
        prev = rs[0][0]
        for t in range(n_ref):
            assert rs[t][r.refine[i][t]] == rs[t].min()
            assert rs[t][0] == prev if t == 0 else True
            prev = rs[t].min()
        assert rs[-1].min() == s or abs(rs[-1].min() - s) < 1e-12 * max(1.0, abs(s))
        assert r.best_score[i] <= base.pose_score[i, p] + 1e-12 * max(1.0, abs(base.pose_score[i, p]))


# ----------------------------------------------------------------------------- per-atom-type grid channels (Q24)

def _lib_ref_score_typed(pk, pts, types):
    """Independent typed g (Q24): scipy trilinear on channel types[i] + kappa*h*L1 excess."""
    out = np.empty(len(pts))
    for t in range(pk.n_channels):
        sel = np.asarray(types) == t
        if sel.any():
            sub = vsgen.Pocket(pk.grid[t], pk.origin, pk.spacing, pk.center, pk.out_slope)
            out[sel] = lib_ref_score(sub, np.asarray(pts)[sel])
    return out


def test_typed_channels_match_scipy_per_channel():
    """Every point is interpolated on ITS channel: scipy per channel, inside and outside the box."""
    rng = np.random.default_rng(21)
    G = rng.normal(size=(3, 9, 10, 11)).astype(np.float32)
    pk = mkpocket(G, origin=(-3.0, 2.0, 1.0), h=0.75, kappa=2.5)
    lo = np.array(pk.origin) - 3.0
    hi = np.array(pk.origin) + 0.75 * np.array([10, 9, 8]) + 3.0
    p = rng.uniform(lo, hi, size=(4000, 3))
    t = rng.integers(0, 3, size=4000).astype(np.uint8)
    assert np.max(np.abs(oracle.grid_score(pk, p, t) - _lib_ref_score_typed(pk, p, t))) < 1e-12
    with pytest.raises(ValueError):
        oracle.grid_score(pk, p[:2], np.array([0, 3], np.uint8))     # type >= T


def test_typed_linear_channels_closed_form():
    """Channel t = w_t . u + b_t (closed form, exact for trilinear interpolation inside the box): a
    wrong channel index, a transposed channel stride or a dropped type fails it."""
    n = 12
    W = np.array([[0.5, -1.0, 2.0], [-2.0, 0.25, 1.0], [1.5, 1.5, -0.5], [0.0, -3.0, 0.75]])
    b = np.array([1.0, -4.0, 2.5, 0.0])
    Z, Y, X = np.meshgrid(np.arange(n), np.arange(n + 1), np.arange(n + 2), indexing="ij")
    G = np.stack([W[t, 0] * X + W[t, 1] * Y + W[t, 2] * Z + b[t] for t in range(4)]).astype(np.float32)
    pk = mkpocket(G)
    rng = np.random.default_rng(22)
    u = rng.uniform([0, 0, 0], [n + 1, n, n - 1], size=(3000, 3))
    t = rng.integers(0, 4, size=3000)
    want = np.einsum("ij,ij->i", W[t], u) + b[t]
    assert np.max(np.abs(oracle.grid_score(pk, u, t.astype(np.uint8)) - want)) < 1e-9


def test_typed_copies_reduce_to_untyped(c1):
    """T identical channels: any typing docks exactly like the untyped pocket (bitwise)."""
    L, pk, (rot, tr), cs = c1
    pk3 = vsgen.Pocket(np.stack([pk.grid] * 3), pk.origin, pk.spacing, pk.center, pk.out_slope)
    ty = vsgen.atom_types(L, n_types=3)
    a = oracle.dock_batch(L, pk, rot, tr, cs)
    b = oracle.dock_batch(L, pk3, rot, tr, cs, atom_type=ty)
    for f in ("best_score", "best_pose", "angles", "xyz", "pose_score"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_typed_single_type_docks_on_that_channel(c1):
    """Every atom of type t: the result is the untyped docking on G_t."""
    L, _, (rot, tr), cs = c1
    pk = vsgen.typed_pocket(101, n_types=3)
    for t in range(3):
        pt = vsgen.Pocket(pk.grid[t], pk.origin, pk.spacing, pk.center, pk.out_slope)
        a = oracle.dock_batch(L, pt, rot, tr, cs)
        b = oracle.dock_batch(L, pk, rot, tr, cs, atom_type=np.full(int(L.atom_off[-1]), t, np.uint8))
        assert np.array_equal(a.best_score, b.best_score) and np.array_equal(a.angles, b.angles)


def test_typed_channel_relabelling_invariance(c1):
    """Permuting the channels and relabelling the types the same way changes nothing."""
    L, _, (rot, tr), cs = c1
    pk = vsgen.typed_pocket(102, n_types=4)
    ty = vsgen.atom_types(L, n_types=4)
    perm = np.array([2, 0, 3, 1])                       # new channel perm[t] holds old channel t
    Gp = np.empty_like(pk.grid)
    Gp[perm] = pk.grid
    pkp = vsgen.Pocket(Gp, pk.origin, pk.spacing, pk.center, pk.out_slope)
    a = oracle.dock_batch(L, pk, rot, tr, cs, atom_type=ty)
    b = oracle.dock_batch(L, pkp, rot, tr, cs, atom_type=perm[ty].astype(np.uint8))
    assert np.array_equal(a.best_score, b.best_score) and np.array_equal(a.xyz, b.xyz)
    # and the types matter: the untyped docking on channel 0 differs
    c = oracle.dock_batch(L, pk, rot, tr, cs, atom_type=np.zeros_like(ty))
    assert not np.array_equal(a.best_score, c.best_score)


def test_typed_brute_force_star_ligands_greedy_is_exact():
    """Star ligands (separable score) with random atom types: the greedy sweep is the exhaustive
    optimum under the typed score computed by scipy per channel."""
    rng = np.random.default_rng(23)
    pk = vsgen.typed_pocket(101, n_types=4)
    rot, tr = vsgen.pose_table(3)
    cs = vsgen.angle_table(8)
    K = cs.shape[0]
    thetas = [math.atan2(float(cs[k, 1]), float(cs[k, 0])) for k in range(K)]
    for arms in (1, 2, 3):
        x, fr = _star_ligand(rng, arms)
        ty = rng.integers(0, 4, size=len(x)).astype(np.uint8)
        lib = vsgen.Library.from_ligands([(x, fr)])
        r = oracle.dock_batch(lib, pk, rot, tr, cs, atom_type=ty)
        best = math.inf
        xc = x.astype(np.float64) - x.astype(np.float64).mean(0)
        for p in range(rot.shape[0]):
            y0 = xc @ rot[p].astype(np.float64).T + np.array(pk.center)
            for combo in itertools.product(range(K), repeat=len(fr)):
                y = y0.copy()
                for (a, bb, mv), k in zip(fr, combo):
                    u = (y[bb] - y[a]) / np.linalg.norm(y[bb] - y[a])
                    y[mv] = Rotation.from_rotvec(thetas[k] * u).apply(y[mv] - y[bb]) + y[bb]
                best = min(best, float(_lib_ref_score_typed(pk, y, ty).sum()))
        assert abs(r.best_score[0] - best) < 1e-9 * max(1.0, abs(best))


def test_atom_types_are_a_function_of_ligand_id_and_atom_index():
    """The type recipe: slices and renumbered copies keep every atom's type."""
    L = vsgen.ligands(200, 4)
    t = vsgen.atom_types(L)
    sub = vsgen.ligands(50, 4, first=100)
    assert np.array_equal(vsgen.atom_types(sub), t[int(L.atom_off[100]):int(L.atom_off[150])])
    L.atom_type = t
    lp, perm = L.permuted(3)
    assert np.array_equal(lp.atom_type[perm], t)
    freq = np.bincount(vsgen.atom_types(vsgen.ligands(3000, 5)), minlength=4) / 1.0
    assert np.allclose(freq / freq.sum(), vsgen.TYPE_FREQ, atol=0.01)
