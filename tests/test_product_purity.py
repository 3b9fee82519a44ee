"""The product path never touches the oracle and never falls back to CPU."""

import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2409_16781_b200")


def test_package_never_imports_the_oracle():
    pat = re.compile(r"^\s*(from|import)\s+oracle\b|liboracle|oracle/", re.M)
    for dirpath, _, files in os.walk(PKG):
        for name in files:
            if name.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, name)).read()
                code = "\n".join(l for l in text.splitlines()
                                 if not l.lstrip().startswith(("#", "//", "*", "/*")))
                code = re.sub(r'""".*?"""', "", code, flags=re.S)
                assert not pat.search(code), f"{name} references the oracle"


def test_only_tests_smoke_and_the_bench_cpu_arm_use_the_oracle():
    pat = re.compile(r"^\s*(from|import)\s+oracle\b", re.M)
    tools = os.path.join(ROOT, "tools")
    for name in os.listdir(tools):
        if name.endswith(".py"):
            assert not pat.search(open(os.path.join(tools, name)).read()), f"tools/{name}"
    # bench.py: only as the timed CPU arm (cpu_arm) and as the CHECKER of the GPU result
    # (parity_and_cpu_baseline at N = 1, preflight at N > 1) - never inside the functions
    # that produce the GPU numbers; __graft_entry__.py: inside smoke only
    bench = open(os.path.join(ROOT, "bench.py")).read()
    allowed = {bench.find("\ndef " + fn) for fn in ("cpu_arm", "parity_and_cpu_baseline",
                                                      "preflight")}
    assert -1 not in allowed
    assert [m.start() for m in pat.finditer(bench)] and all(
        bench.rfind("\ndef ", 0, m.start()) in allowed for m in pat.finditer(bench))
    entry = open(os.path.join(ROOT, "__graft_entry__.py")).read()
    assert all(entry.rfind("\ndef ", 0, m.start()) == entry.find("\ndef smoke")
               for m in pat.finditer(entry))


def test_no_reference_sources_read_at_run_time():
    for name in ("bench.py", "__graft_entry__.py"):
        assert "/root/reference" not in open(os.path.join(ROOT, name)).read()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_compute_path_fails_loudly_without_a_gpu():
    import numpy as np
    from paper_2409_16781_b200 import boundaries as B, cases, engine
    from paper_2409_16781_b200.fields import Layout, Precision
    from paper_2409_16781_b200.kernels import KernelPlan
    with pytest.raises(RuntimeError):
        KernelPlan(8, 8, 8, Layout.ROW, Precision.SINGLE,
                   B.flatten_mask(B.cavity_mask(8, 8, 8)), 1.0)
    state = cases.init(cases.CaseSpec("ldc", 8, 8, 8), Precision.SINGLE)
    with pytest.raises(RuntimeError):
        engine.run(state, engine.RunConfig(steps=1))
    with pytest.raises(RuntimeError):
        state.macro()
    assert isinstance(state.f_pre.data, np.ndarray)


def test_backend_selection(monkeypatch):
    # mirrors test_kernels.py:262-287
    from paper_2409_16781_b200 import kernels
    monkeypatch.delenv("MLB_BACKEND", raising=False)
    assert kernels._pick_backend() == "cuda"
    monkeypatch.setenv("MLB_BACKEND", " CUDA ")
    assert kernels._pick_backend() == "cuda"
    monkeypatch.setenv("MLB_BACKEND", "")
    assert kernels._pick_backend() == "cuda"
    monkeypatch.setenv("MLB_BACKEND", "numpy")
    with pytest.raises(ValueError, match="MLB_BACKEND"):
        kernels._pick_backend()
