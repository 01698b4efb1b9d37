"""The C-ABI library builds for sm_100a, loads, exports every symbol include/vsdock.h
declares, its struct layouts match the ctypes binding, and its host-only planning
steps (class boundaries, LPT) agree with the oracle.  No GPU needed."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "vsdock.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2303_06150_b200 import build
    build.build()
    from paper_2303_06150_b200 import vsdock
    return vsdock.load_library()


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:vs_status|void|const char\*)\s+(vs_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["vs_create", "vs_load_pocket", "vs_submit", "vs_get_results", "vs_local_topk", "vs_merge_topk"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2303_06150_b200 import vsdock
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(vsdock.SYMBOLS) == declared_symbols()


def test_library_is_sm100a(lib):
    from paper_2303_06150_b200 import vsdock
    out = subprocess.run(["cuobjdump", "--list-elf", vsdock.SO_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_ctypes(tmp_path):
    from paper_2303_06150_b200 import vsdock
    src = tmp_path / "sz.c"
    structs = ["vs_config", "vs_pocket_desc", "vs_ligand_batch", "vs_bucket", "vs_class_info", "vs_stats"]
    src.write_text('#include <stdio.h>\n#include "vsdock.h"\nint main(){' +
                   "".join(f'printf("%zu\\n", sizeof({s}));' for s in structs) + "return 0;}")
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    sizes = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    for s, n in zip(structs, sizes):
        assert ctypes.sizeof(getattr(vsdock, s)) == n, s


def test_no_gpu_means_no_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2303_06150_b200 import Engine
    with pytest.raises(RuntimeError):
        Engine()


def test_plan_boundaries_match_oracle_and_spec(lib):
    import oracle
    from paper_2303_06150_b200.vsdock import plan_boundaries
    # SPEC worked examples through the product's own code
    assert plan_boundaries(3, 96, 3, 20) == ([32, 64, 96], [3, 9, 20])
    assert plan_boundaries(1, 200, 1, 20) == ([200], [20])
    assert plan_boundaries(6, 192, 23, 20)[0] == [32, 64, 96, 128, 160, 192]
    assert plan_boundaries(6, 120, 23, 20)[1] == list(range(21))
    for na in range(1, 9):
        for ub in (20, 33, 64, 97, 120, 150, 200, 256):
            for nr in (1, 2, 3, 5, 8, 21, 23, 33):
                for rub in (0, 1, 4, 20, 25, 32):
                    a, r = plan_boundaries(na, ub, nr, rub)
                    assert a == oracle.atom_boundaries(na, 32, ub)
                    assert r == oracle.rotamer_boundaries(nr, rub)


def test_plan_lpt_matches_oracle(lib):
    import oracle
    from paper_2303_06150_b200.vsdock import plan_lpt
    rng = np.random.default_rng(3)
    for nb in (0, 1, 7, 84, 431):
        w = rng.integers(1, 10 ** 9, nb).astype(np.uint64)
        w[: nb // 3] = w[0] if nb else 0      # force weight ties
        for W in (1, 2, 4, 8):
            owner, order = plan_lpt(w, W)
            ref = oracle.lpt_shards([int(x) for x in w], W)
            for r, bl in enumerate(ref):
                assert [int(b) for b in np.where(owner == r)[0][np.argsort(order[owner == r])]] == bl
