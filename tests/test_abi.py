"""The C-ABI boundary: library loads, exports every symbol include/csrc_gpu.h
declares, and fails loudly (nonzero status + message) instead of falling back."""
import os
import re

import numpy as np
import pytest

import paper_1003_0952_b200 as P
import paper_1003_0952_b200._lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "csrc_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(csrc_\w+)\s*\(", src)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "csrc_gpu_plan_create" in names and "csrc_gpu_spmv" in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    missing = [n for n in declared_functions() if not hasattr(L.lib, n)]
    assert not missing, f"libcsrc_b200.so lacks {missing}"


def test_python_binding_covers_the_abi():
    assert sorted(L.EXPORTED) == declared_functions()


def test_abi_version():
    assert L.abi_version() == 1


def test_library_is_in_tree():
    assert os.path.dirname(L.LIB_PATH) == os.path.join(ROOT, "paper_1003_0952_b200")


def test_plan_creation_reports_errors_not_fallbacks():
    # reference error paths (parallel.hpp:231-233) are checked before any device work
    a = P.CsrcMatrix(2, [1.0, 1.0], [0, 0, 1], [0], [5.0], [7.0])
    with pytest.raises(P.Error, match="thread count must be >= 1"):
        P.GpuSpmv(a, P.Strategy(P.StrategyKind.local_buffers, p=0))
    with pytest.raises(P.Error, match="sequential strategy requires p = 1"):
        P.GpuSpmv(a, P.Strategy(P.StrategyKind.sequential, p=2))


def test_structure_errors_are_reported():
    bad = P.CsrcMatrix(3, np.ones(3), [0, 0, 1, 2], [1, 0], [1.0, 1.0], [1.0, 1.0])
    with pytest.raises(P.Error, match="strictly increasing and < row"):
        P.GpuSpmv(bad, P.Strategy(P.StrategyKind.windowed))


def test_without_gpu_the_product_fails_loudly():
    if L.device_count() > 0:
        pytest.skip("a CUDA device is present")
    a = P.CsrcMatrix(2, [1.0, 1.0], [0, 0, 1], [0], [5.0], [7.0])
    with pytest.raises(P.Error, match="CUDA"):
        P.spmv_csrc(a, [1.0, 2.0])


def test_model_bytes_and_flops():
    # working_set.hpp:11-23 and cost_model.hpp:80-86
    assert L.model_bytes(262144, 6859000, 0, 0) == 73308596
    assert L.model_bytes(16777216, 449455096, 0, 1) == 2864502740
    assert L.model_flops(9, 33) == 57
