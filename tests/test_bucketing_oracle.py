"""Pins of the oracle's bucketing / launch-sizing / sharding / ranking side.

Pinned to SPEC.md's printed worked examples (tests/golden/spec_bucketing.json,
each entry citing its line), Table 1 of PAPER.md, and SPEC's invariants
(S:256-259 conservation, homogeneity, monotonicity, 1x1 = plain batching;
S:157-159 occupancy monotonicity and the t = ws identity).
"""
import json
import os
import random

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_bucketing.json")))


@pytest.mark.parametrize("case", GOLD["atom_boundaries"])
def test_atom_boundaries_spec_examples(case):
    assert oracle.atom_boundaries(*case["args"]) == case["expect"], case["cite"]


@pytest.mark.parametrize("case", GOLD["rotamer_boundaries"])
def test_rotamer_boundaries_spec_examples(case):
    assert oracle.rotamer_boundaries(*case["args"]) == case["expect"], case["cite"]


def test_boundary_errors():
    with pytest.raises(oracle.BucketingError):
        oracle.atom_boundaries(0, 32, 100)
    with pytest.raises(oracle.BucketingError):
        oracle.rotamer_boundaries(0, 20)


def test_atom_boundaries_fallback_reading_q16():
    # S:207 precondition fails for 6 clusters over <=120 atoms (P:337 vs P:412): reading Q16 -> last = 32*n
    assert oracle.atom_boundaries(6, 32, 120) == [32, 64, 96, 128, 160, 192]
    assert oracle.atom_boundaries(4, 32, 120) == [32, 64, 96, 120]


def test_rotamer_boundaries_strictly_increasing_and_dense_low():
    for n in range(1, 24):
        for m in range(0, 33):
            b = oracle.rotamer_boundaries(n, m)
            assert all(x < y for x, y in zip(b, b[1:]))
            assert b[-1] == m
            if n <= m:
                assert len(b) == n
    # "more interested in creating clusters toward lower values":
    # with 3 clusters over 0..20 the classes widen geometrically
    assert list(np.diff([-1] + oracle.rotamer_boundaries(3, 20))) == [4, 6, 11]
    assert list(np.diff([-1] + oracle.rotamer_boundaries(4, 60))) == [5, 8, 16, 32]


def test_assign_spec_examples():
    g = GOLD["assign"]
    for c in g["cases"]:
        if isinstance(c["expect"], str):
            axis = c["expect"].split(":")[1]
            with pytest.raises(oracle.BucketingError) as e:
                oracle.assign(g["grid"]["atoms"], g["grid"]["rot"], *c["ligand"])
            assert e.value.axis == axis, c["cite"]
        else:
            assert list(oracle.assign(g["grid"]["atoms"], g["grid"]["rot"], *c["ligand"])) == c["expect"], c["cite"]


@pytest.mark.parametrize("case", GOLD["bucketizer"])
def test_streaming_bucketizer_spec_examples(case):
    bz = oracle.StreamingBucketizer([32, 64, 96], [3, 9, 20], [case["capacity"]] * 3)
    emitted_at = []
    for t, (a, r) in enumerate(case["ligands"]):
        if bz.push(t, a, r) is not None:
            emitted_at.append(t + 1)
    assert emitted_at == case["emit_after_push"], case["cite"]
    assert sum(len(b) for b in bz.open.values()) == case["open_after"]
    flushed = bz.flush()
    if "flush_sizes" in case:
        assert [len(b.ligands) for b in flushed] == case["flush_sizes"]
    assert sum(len(b.ligands) for b in flushed) == case["open_after"]
    assert bz.flush() == []                      # S:251 freshly flushed state -> empty


@pytest.mark.parametrize("case", GOLD["capacity_native"])
def test_eq1_capacity_examples(case):
    assert oracle.bucket_capacity_native(*case["args"]) == case["expect"], case["cite"]


def test_eq1_table1_exact():
    t = GOLD["table1_active_blocks"]
    for ab in t["cuda"]:
        b = oracle.active_blocks_per_sm(65536, 2048, 32, 167936, 256, 1, 32, 0,
                                        measured_active_blocks=ab, sm_count=t["sm_count"])
        assert oracle.bucket_capacity_native(b, t["sm_count"], 32, 32) == ab


@pytest.mark.parametrize("case", GOLD["occupancy"])
def test_occupancy_examples(case):
    d, k = case["dev"], case["kc"]
    b = oracle.active_blocks_per_sm(d["regs_per_sm"], d["max_threads_per_sm"], d["max_blocks_per_sm"],
                                    d["shared_mem_per_sm"], d["reg_alloc_granularity"], k["regs_per_thread"],
                                    k["block_size"], k["shared_per_block"], k.get("measured_active_blocks"),
                                    k.get("sm_count"))
    assert b == case["expect"], case["cite"]


def test_occupancy_monotone_and_t_eq_ws_identity():
    rng = random.Random(9)
    for _ in range(1000):                        # S:158, S:459 criterion 9
        regs, t, sh = rng.randint(16, 255), 32 * rng.randint(1, 32), rng.randint(0, 100_000)
        base = oracle.active_blocks_per_sm(65536, 2048, 32, 233472, 256, regs, t, sh) if regs * t <= 65536 and sh <= 233472 else None
        if base is None:
            continue
        for r2, t2, s2 in [(regs + rng.randint(0, 30), t, sh), (regs, t, sh + rng.randint(0, 50_000))]:
            try:
                b2 = oracle.active_blocks_per_sm(65536, 2048, 32, 233472, 256, r2, t2, s2)
            except oracle.BucketingError:
                b2 = 0
            assert b2 <= base
        assert oracle.bucket_capacity_native(base, 148, 32, 32) == base * 148


def test_occupancy_errors():
    with pytest.raises(oracle.BucketingError):
        oracle.active_blocks_per_sm(65536, 2048, 32, 1000, 256, 32, 4096, 0)       # S:110 block too big
    with pytest.raises(oracle.BucketingError):
        oracle.active_blocks_per_sm(65536, 2048, 32, 1000, 256, 32, 32, 2000)      # S:110 does not fit
    with pytest.raises(oracle.BucketingError):
        oracle.bucket_capacity_native(1, 1, 48, 32)


def test_footprint_and_multiple():
    assert oracle.ligand_footprint(0, 7, 5) == 7
    assert oracle.ligand_footprint(2, 100, 50) == 200
    assert oracle.max_bucket_multiple(10, 1, 3, 1) == 3
    assert oracle.max_bucket_multiple(12, 2, 3, 2) == 1   # S:153 exact fit
    f1 = oracle.ligand_footprint(4, 100, 50)
    f2 = oracle.ligand_footprint(8, 100, 50)
    assert oracle.max_bucket_multiple(10**6, 10, f2, 2) <= oracle.max_bucket_multiple(10**6, 10, f1, 2)


def _random_features(n, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(20, 121, n), rng.integers(0, 21, n)


def test_bucketize_invariants():
    A, R = _random_features(5000, 3)
    ab, rb = oracle.atom_boundaries(6, 32, 120), oracle.rotamer_boundaries(23, 20)
    caps = [7, 11, 13, 17, 19, 23]
    bk = oracle.bucketize(A, R, ab, rb, caps)
    allidx = [i for b in bk for i in b.ligands]
    assert sorted(allidx) == list(range(5000))             # conservation S:256
    for b in bk:
        assert 0 < len(b.ligands) <= b.capacity
        cells = {oracle.assign(ab, rb, int(A[i]), int(R[i])) for i in b.ligands}
        assert cells == {b.cell}                           # homogeneity S:257
        assert max(A[i] for i in b.ligands) <= ab[b.cell[0]]
        assert b.ligands == sorted(b.ligands)              # input order within a cell (Q18)
    assert [b.cell for b in bk] == sorted(b.cell for b in bk)   # cell-major (Q18)
    # membership equals SPEC's streaming bucketizer (Q18: only the emission order differs)
    bz = oracle.StreamingBucketizer(ab, rb, caps)
    stream = []
    for i in range(5000):
        e = bz.push(i, int(A[i]), int(R[i]))
        if e is not None:
            stream.append(e)
    stream += bz.flush()
    key = lambda b: (b.cell, b.ligands[0])
    assert sorted(((b.cell, tuple(b.ligands)) for b in stream)) == sorted(((b.cell, tuple(b.ligands)) for b in bk))
    assert len([b for b in bk if len(b.ligands) < b.capacity]) <= 6 * 21   # pigeonhole S:253


def test_bucketize_1x1_is_plain_batching():
    A, R = _random_features(1000, 4)
    bk = oracle.bucketize(A, R, [120], [20], [64])
    assert [b.ligands for b in bk] == [list(range(s, min(s + 64, 1000))) for s in range(0, 1000, 64)]


def test_bucketize_overflow_names_axis_and_index():
    with pytest.raises(oracle.BucketingError) as e:
        oracle.bucketize([10, 20, 200], [0, 0, 0], [32, 64], [5], [4, 4])
    assert e.value.axis == "atoms" and e.value.index == 2


def test_boundary_monotonicity():
    # more clusters never widens any cell
    for n in range(1, 6):
        w1 = np.diff([0] + oracle.atom_boundaries(n, 32, 200)).max()
        w2 = np.diff([0] + oracle.atom_boundaries(n + 1, 32, 200)).max()
        assert w2 <= w1
        r1 = np.diff([-1] + oracle.rotamer_boundaries(n, 20)).max()
        r2 = np.diff([-1] + oracle.rotamer_boundaries(n + 1, 20)).max()
        assert r2 <= r1


def test_lpt_balance_and_determinism():
    rng = np.random.default_rng(5)
    w = rng.integers(1, 10**6, 431)
    for W in (1, 2, 4, 8):
        sh = oracle.lpt_shards(w, W)
        assert sorted(b for s in sh for b in s) == list(range(431))
        loads = [sum(int(w[b]) for b in s) for s in sh]
        # Graham's LPT bound: makespan <= (4/3 - 1/(3W)) * OPT, OPT >= mean load
        assert max(loads) <= (4 / 3) * max(np.mean(loads), w.max()) + 1
        assert sh == oracle.lpt_shards(w, W)
    assert oracle.lpt_shards([5, 5, 5], 2) == [[0, 2], [1]]   # ties: id ascending, lowest rank


def test_topk_definition():
    s = np.array([3.0, 1.0, 2.0, 1.0, 0.5])
    assert list(oracle.topk(s, 3)) == [4, 1, 3]                # ties -> lowest index (Q11)
    assert list(oracle.topk(s, 10)) == [4, 1, 3, 2, 0]
    rng = np.random.default_rng(1)
    s = rng.integers(0, 50, 2000).astype(np.float64)
    assert list(oracle.topk(s, 100)) == list(np.lexsort((np.arange(2000), s))[:100])
    parts = [(s[:700], np.arange(700)), (s[700:], np.arange(700, 2000))]
    assert list(oracle.merge_topk(parts, 100)) == list(oracle.topk(s, 100))
