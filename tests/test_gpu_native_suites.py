"""Native test programs on the GPU: the reference's own test_registry
(compiled from /root/reference against this library) and the C++ fusion
soundness suite."""
import pathlib
import subprocess

import pytest

pytestmark = pytest.mark.gpu
REPO = pathlib.Path(__file__).resolve().parent.parent


def _run(exe, timeout=900, env=None):
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=timeout, env=env)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]
    assert "failed: 0" in out.stdout


def test_reference_registry_tests_pass_on_b200():
    exe = REPO / "oracle" / "_ref" / "bin" / "test_registry"
    if not exe.exists():
        pytest.skip("built from /root/reference in the build container (oracle/Makefile)")
    _run(exe)


def test_reference_expr_and_graph_tests():
    for name in ("test_expr", "test_graph_core"):
        exe = REPO / "oracle" / "_ref" / "bin" / name
        if exe.exists():
            _run(exe)


def test_cpp_fusion_soundness_and_boundaries():
    _run(REPO / "tests" / "cpp" / "bin" / "test_graphvx")
