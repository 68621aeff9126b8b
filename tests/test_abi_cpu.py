"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and its pure host planner matches oracle c1 bit-exactly."""
import random
import re
import os

import pytest

from oracle import planner as OP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_header_symbol():
    import ctypes
    from paper_2507_11507_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "mirage.h")).read()
    declared = sorted(set(re.findall(r"\b(mirage_[a-z_0-9]+)\s*\(", hdr)))
    assert len(declared) >= 20
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED) == declared


def test_plan_matches_oracle():
    from paper_2507_11507_b200 import _lib
    rng = random.Random(0)
    cases = [(8, 1, 1, 0, 1, 0), (40, 1, 1, 0, 1000, 0), (32, 1, 2, 0, 1000, 0), (40, 9, 3, 13000, 4000, 0)]
    for _ in range(400):
        n = rng.randint(1, 64)
        cases.append((n, rng.randint(0, n), rng.choice([1, 2, 3]), rng.randint(0, 5000), rng.randint(1, 1000),
                      rng.randint(0, n - 1)))
    for n, a, pol, tt, tc, anc in cases:
        try:
            exp = OP.plan(n, a, pol, tt, tc, anc)
            eerr = None
        except OP.InfeasibleAlpha:
            exp, eerr = None, _lib.ERR_INFEASIBLE
        except OP.RangeError:
            exp, eerr = None, _lib.ERR_RANGE
        try:
            got = _lib.plan(n, a, pol, tt, tc, anc)
            gerr = None
        except _lib.MirageError as e:
            got, gerr = None, e.code
        assert gerr == eerr, (n, a, pol, tt, tc, anc)
        if exp is not None:
            assert (list(got[0]), got[1], got[2]) == (list(exp[0]), exp[1], exp[2]), (n, a, pol, tt, tc, anc)


def test_sizes_match_synth_spec():
    from paper_2507_11507_b200 import _lib
    from synth import models, weights
    for m in models.PRESETS.values():
        S, G, BB = _lib.model_sizes(m)
        assert S == weights.layer_bytes(m) and G == weights.global_bytes(m)
        assert BB == m.n_layers * m.n_kv_heads * 2 * 16 * m.head_dim * 2
        assert S % 256 == 0


def test_header_is_plain_c99():
    """include/mirage.h is a C ABI: it must compile as C99 (no C++ or torch types)."""
    import os
    import shutil
    import subprocess
    import tempfile
    gcc = shutil.which("gcc")
    if gcc is None:
        import pytest
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "h.c")
        with open(src, "w") as f:
            f.write('#include "mirage.h"\nint main(void) { mirage_stats s; (void)s; return 0; }\n')
        r = subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I",
                            os.path.join(root, "include"), src], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
