"""Every built-in kernel of the registry (28; tests/kernel_graphs.py) as a
one-node graph file at border-heavy sizes, executed on the B200 through
run_plan and run_naive and compared bit-for-bit with the UNMODIFIED
reference engine's run_naive (SHA-256 of the serialised outputs in
tests/golden/kernels.json, from tests/golden/make_kernel_golden.py), event
counters included.  ScaleImage and EqualizeHist cannot run on the
reference through graph files (its MissingCast / CrossGraphVirtual defects,
recorded in the golden file); for those run_plan == run_naive here, and the
reference's own oracle tests (test_registry: "image scaling", "histogram
equalization") check them in tests/test_gpu_native_suites.py."""
import hashlib
import json
import pathlib
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO / "tests"))
import kernel_graphs  # noqa: E402

GOLDEN = json.loads((REPO / "tests" / "golden" / "kernels.json").read_text())
CASES = kernel_graphs.all_cases()


def blob(outs):
    b = bytearray()
    for kind, payload in outs:
        b += kind.to_bytes(4, "little") + len(payload).to_bytes(4, "little") + payload
    return bytes(b)


def test_every_registry_kernel_is_covered():
    covered = {json.loads(t)["nodes"][0]["kernel"] for _, t in CASES}
    assert covered == set(kernel_graphs.KERNELS) and len(kernel_graphs.KERNELS) == 28
    refd = {json.loads(t)["nodes"][0]["kernel"] for c, t in CASES if c in GOLDEN["cases"]}
    assert set(kernel_graphs.KERNELS) - refd == {"ScaleImage", "EqualizeHist"}


@pytest.mark.parametrize("case,text", CASES, ids=[c for c, _ in CASES])
def test_kernel_matches_reference(case, text, gvx):
    g = gvx.GraphFile(text)
    plan, pc = g.run(naive=False, seed=GOLDEN["seed"])
    naive, nc = g.run(naive=True, seed=GOLDEN["seed"])
    assert blob(plan) == blob(naive), case
    gold = GOLDEN["cases"].get(case)
    if gold is None:
        assert case in GOLDEN["reference_errors"]
        return
    assert hashlib.sha256(blob(naive)).hexdigest() == gold["sha256"], case
    assert [nc["pixels_read"], nc["pixels_written"], nc["transfers_executed"]] == gold["counters"][1:], case
