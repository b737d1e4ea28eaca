"""Stage-level drop-in API (reference proj/include/trijoin/{filter,refine,knn,index}.hpp) on the
GPU: tests/cpp/test_stages.cpp restates the reference's doctest checks of those functions
(proj/tests/test_filter.cpp, test_refine.cpp, test_knn.cpp, test_index.cpp) and checks that
the staged pipeline reproduces run_join's records bit for bit."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_stage_api_cpp():
    exe = os.path.join(HERE, "cpp", "test_stages")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(HERE, "cpp")], check=True)
    p = subprocess.run([exe, os.path.join(HERE, "golden")], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout
