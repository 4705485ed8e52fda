"""INTEGRATION.md §2 is executable: the ctypes binding a `fastafd` maintainer
would add is extracted from the document and run as written.

CPU: its argtypes agree with the prototypes in include/afd_capi.h.
GPU: `decompose_b200` on BASELINE c0 matches the CPU oracle (bit for bit with
engine "b200", identical poles and 1e-9 with "b200-fast").
"""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

DOC = os.path.join(ROOT, "INTEGRATION.md")
HEADER = os.path.join(ROOT, "include", "afd_capi.h")


def _binding_source():
    text = open(DOC).read()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    src = [b for b in blocks if "# fastafd/b200.py" in b]
    assert len(src) == 1, "INTEGRATION.md must hold exactly one fastafd/b200.py block"
    lib = os.path.join(ROOT, "paper_1711_08604_b200", "lib", "libafd_b200.so")
    return src[0].replace("/path/to/paper_1711_08604_b200/lib/libafd_b200.so", lib)


def _prototype_arity(name):
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    m = re.search(r"\b%s\s*\((.*?)\)\s*;" % name, src, flags=re.S)
    assert m, name
    args = [a for a in m.group(1).split(",") if a.strip() and a.strip() != "void"]
    return len(args)


def test_binding_argtypes_match_the_header():
    from paper_1711_08604_b200 import build as b
    b.build()
    ns = {}
    exec(compile(_binding_source(), "INTEGRATION.md:fastafd/b200.py", "exec"), ns)
    lib = ns["_lib"]
    for fn in ("afd_plan_create", "afd_plan_set_engine", "afd_decompose_host"):
        assert len(getattr(lib, fn).argtypes) == _prototype_arity(fn), fn
    assert ns["STEP"].itemsize == 72


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["b200", "b200-fast"])
def test_binding_decomposes_like_the_oracle(engine):
    import oracle as O
    from paper_1711_08604_b200 import core, workloads as W
    ns = {}
    exec(compile(_binding_source(), "INTEGRATION.md:fastafd/b200.py", "exec"), ns)
    w = W.CONFIGS["c0"]
    g = W.signal_for("c0")
    grid = core.ParameterGrid(W.radii_for(w.m), w.n)
    rec, initial, rem = ns["decompose_b200"](g, grid, w.steps, None, False, engine)
    o = O.decompose(g, np.array(grid.radii), max_terms=w.steps)
    assert len(rec) == len(o.steps) == w.steps
    assert np.array_equal(rec["j"], o.steps["j"]) and np.array_equal(rec["radius"],
                                                                      o.steps["radius"])
    if engine == "b200":
        for k in ("c_re", "c_im", "residual"):
            assert np.array_equal(rec[k], o.steps[k]), k
        assert np.array_equal(rem, o.remainder)
    else:
        for k in ("c_re", "c_im", "residual"):
            assert np.all(np.abs(rec[k] - o.steps[k]) <= 1e-9 * np.abs(o.steps[k])), k
        assert np.max(np.abs(rem - o.remainder)) <= 1e-9 * np.max(np.abs(o.remainder))
