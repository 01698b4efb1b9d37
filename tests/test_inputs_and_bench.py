"""Input generators (SPEC dataset invariants) and the bench.py contract of the reference arm."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import vsgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_generator_ranges_determinism_and_prefix_stability():
    a = vsgen.ligands(300, 9, (20, 120), (0, 20))
    b = vsgen.ligands(300, 9, (20, 120), (0, 20))
    for f in ("atom_off", "xyz", "frag_off", "frags", "frag_axis", "move_off", "move_atoms"):
        assert np.array_equal(getattr(a, f), getattr(b, f))          # S:68 determinism
    assert ((a.n_atoms >= 20) & (a.n_atoms <= 120)).all()             # S:39 in range
    assert ((a.n_frags >= 0) & (a.n_frags <= 20)).all()
    tail = vsgen.ligands(100, 9, (20, 120), (0, 20), first=200)       # ligand i depends only on (seed, i)
    for i in range(100):
        x1, f1 = a.ligand(200 + i)
        x2, f2 = tail.ligand(i)
        assert np.array_equal(x1, x2) and f1 == f2
    assert vsgen.ligands(0, 1).n == 0
    d = vsgen.ligands(3, 5, (5, 5), (0, 0))                            # S:44 degenerate ranges
    assert list(d.n_atoms) == [5, 5, 5] and list(d.n_frags) == [0, 0, 0]
    with pytest.raises(ValueError):
        vsgen.ligands(3, 1, (10, 5), (0, 1))                           # S:40 inverted range


def test_generated_fragments_are_valid_rotatable_bonds():
    lib = vsgen.ligands(200, 3, (20, 120), (0, 20))
    for i in range(lib.n):
        x, fr = lib.ligand_ranges(i)
        A = len(x)
        assert lib.ligand(i)[1] == vsgen.Frags.from_ranges(fr)           # general form == range form
        for a, b, lo, hi in fr:
            assert 0 <= a < A and 0 <= b < A and a != b
            assert 0 <= lo < hi <= A and not (lo <= a < hi) and not (lo <= b < hi)
            assert abs(np.linalg.norm(x[b] - x[a]) - 1.5) < 1e-4     # a -> b is a bond
        assert int(np.sum(fr[:, 3] - fr[:, 2])) == int(lib.n_moving[i])


def test_replicate():
    lib = vsgen.ligands(2, 4, (53, 53), (4, 4))
    r = vsgen.replicate(lib, 1, 4)
    assert r.n == 4 and len(set(r.ligand_id.tolist())) == 4
    for i in range(4):
        assert np.array_equal(r.ligand(i)[0], lib.ligand(1)[0]) and r.ligand(i)[1] == lib.ligand(1)[1]
    assert vsgen.replicate(lib, 0, 1).n == 1


def test_tables():
    rot, tr = vsgen.pose_table(16, 7)
    assert np.array_equal(rot[0], np.eye(3, dtype=np.float32)) and not tr.any()
    cs = vsgen.angle_table(8)
    assert cs[0, 0] == 1.0 and cs[0, 1] == 0.0
    assert np.allclose(np.hypot(cs[:, 0], cs[:, 1]), 1.0, atol=1e-7)


def test_bench_reference_arm_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_pipeline_chunk_schedule():
    """Host-only chunk planning of the double-buffered path (pipeline.chunk_bounds)."""
    from paper_2303_06150_b200.pipeline import chunk_bounds
    for n in (0, 1, 5, 31, 32, 1000, 250_000, 1_000_000):
        b = chunk_bounds(n)
        assert b[0] == 0 and b[-1] == n and all(x < y for x, y in zip(b, b[1:])) or n == 0
        sizes = [y - x for x, y in zip(b, b[1:])]
        if n >= 32 and len(sizes) > 1:
            assert sizes[0] == n // 32 and sizes[-1] == n // 32          # small exposed first H2D / last D2H
            h = (len(sizes) + 1) // 2
            assert all(s2 <= 4 * s1 for s1, s2 in zip(sizes[:h], sizes[1:h]))
            assert all(s1 <= 4 * s2 for s1, s2 in zip(sizes[h - 1:], sizes[h:]))
    assert chunk_bounds(100, 3) == [0, 33, 66, 100]
    assert chunk_bounds(1_000_000) == [0, 31250, 156250, 500000, 843750, 968750, 1_000_000]
