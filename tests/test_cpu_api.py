"""Host-side checks that need no GPU: the C-ABI libraries load and export
every declared symbol, the reference's own unit tests pass against this
library (drop-in proof), and the C++ API tests in CPU mode."""
import os
import pathlib
import re
import subprocess

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent


def declared(header):
    text = (REPO / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gvx[bc]_[a-z0-9_]+)\s*\(", text)))


def exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_gvxb_exports_every_declared_symbol(gvx):
    syms = exported(gvx.LIB_CUDA)
    missing = [s for s in declared("gvxb.h") if s not in syms]
    assert not missing, missing


def test_gvx_c_exports_every_declared_symbol(gvx):
    syms = exported(gvx.LIB_GRAPH)
    missing = [s for s in declared("gvx_c.h") if s not in syms]
    assert not missing, missing


def test_libraries_load_without_gpu(gvx):
    c, g = gvx.libraries()
    assert c.gvxb_abi_version() == 1


@pytest.mark.parametrize("name", ["test_expr", "test_graph_core"])
def test_reference_unit_tests_pass_against_graphvx(name):
    exe = REPO / "oracle" / "_ref" / "bin" / name
    if not exe.exists():
        pytest.skip("reference tests are compiled from /root/reference (oracle/Makefile)")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "failed: 0" in out.stdout


def test_cpp_api_cases_cpu_mode():
    exe = REPO / "tests" / "cpp" / "bin" / "test_graphvx"
    env = dict(os.environ, GVX_TEST_CPU_ONLY="1")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stdout + out.stderr


def test_config_plans_on_host(gvx):
    """Verification + optimisation run on the host: reference-granularity fusion,
    transfer reduction."""
    want = {1: (4, 3, 2), 2: (10, 5, 2), 3: (4, 1, 2), 4: (5, 4, 6)}
    for cfg, (nodes, launches, transfers) in want.items():
        g = gvx.ConfigGraph(cfg, 64, 32)
        st = g.pass_stats()
        assert st["nodes_before"] == nodes and st["launches_after"] == launches
        assert st["transfers_optimized"] == transfers and st["transfers_naive"] == 2 * nodes


def test_no_device_means_no_execution(gvx):
    if gvx.device_count() > 0:
        pytest.skip("a device is present")
    g = gvx.ConfigGraph(1, 16, 16)
    import numpy as np
    with pytest.raises(gvx.GraphvxError) as e:
        g.run_host(np.zeros((16, 16), np.uint8))
    assert e.value.code == "UnsupportedKind"
