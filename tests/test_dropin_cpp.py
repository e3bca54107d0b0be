"""C++ drop-in: the reference's own types/calls through include/csrc_gpu.hpp
(tests/cpp/dropin_test.cpp, built by oracle/Makefile against the reference
headers) agree with the reference CPU results on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_test not built (needs the reference headers)")
def test_cpp_dropin_against_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failures 0" in r.stdout


def test_cpp_wrapper_header_compiles_standalone(tmp_path):
    """The wrapper needs only csrc_gpu.h when used with its own types."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "csrc_gpu.hpp"\nint main(){ csrc::gpu::Strategy s = csrc::gpu::Strategy::windowed();'
                   ' static_assert(sizeof(csrc::gpu::BandSpmv) > 0 && sizeof(csrc::gpu::ParallelSpmv) > 0, "");'
                   ' return s.kind == CSRC_KIND_WINDOWED ? 0 : 1; }\n')
    r = subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                        str(tmp_path / "t")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(tmp_path / "t")]).returncode == 0
