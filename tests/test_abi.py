"""CPU: the C-ABI library loads and exports exactly what include/laq_b200.h
declares; host-only entry points (cost model) match the reference."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "laq_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(laq_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_python_binding():
    from paper_2306_08367_b200 import _abi
    assert header_functions() == sorted(_abi.EXPORTED)


def test_library_exports_every_header_symbol():
    from paper_2306_08367_b200 import _abi
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("liblaq_b200.so not built")
    lib = C.CDLL(_abi.LIB_PATH)
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert b"sm_100a" in _abi.lib().laq_version()


def test_cost_model_through_abi_matches_reference():
    from paper_2306_08367_b200 import errors, fusion
    from paper_2306_08367_b200 import _abi
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("liblaq_b200.so not built")
    for c in load_golden("fusion.json")["cost"]:
        ci = fusion.CostInputs(c["i"], c["k"], c["l"], c["k"], c["dims"])
        assert fusion.speedup_ratio_linear(ci) == float.fromhex(c["linear"])
        assert fusion.speedup_ratio_tree(ci) == float.fromhex(c["tree"])
        assert fusion.decide_fusion(fusion.speedup_ratio_linear(ci)) == c["fuse"]
    with pytest.raises(errors.DomainError):
        fusion.speedup_ratio_linear(fusion.CostInputs(0, 8, 2, 8, [100]))
    with pytest.raises(errors.DomainError):
        fusion.speedup_ratio_tree(fusion.CostInputs(10, 8, 2, 8, [0]))
    with pytest.raises(errors.DomainError):
        fusion.decide_fusion(float("nan"))
    # planner: k/l = 64/256 -> non-fused; k/l large -> fused
    assert fusion.plan_linear(60_000_000, 64, 256, [300_000, 800_000]) == "nonfused"
    assert fusion.plan_linear(1_000_000, 16, 1, [10_000]) == "fused"


def test_product_never_imports_oracle():
    """The product package must not import oracle/ (the checker)."""
    pkg = os.path.join(ROOT, "paper_2306_08367_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f


def test_gpu_path_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2306_08367_b200 import errors
    from paper_2306_08367_b200.device import Context
    with pytest.raises(errors.CudaError):
        Context(0)
