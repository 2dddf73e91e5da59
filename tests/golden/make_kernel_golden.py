"""Generates tests/golden/kernels.json: every built-in kernel as a one-node
graph file (tests/kernel_graphs.py) executed by the UNMODIFIED reference
engine (oracle/_ref, run_naive on random_buffer inputs, seed + object id);
stores the SHA-256 of the serialised outputs and the event counters.
Run in the build container:  python tests/golden/make_kernel_golden.py
"""
import hashlib
import json
import pathlib
import sys

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))
import oracle  # noqa: E402
import kernel_graphs  # noqa: E402

SEED = 29


def main():
    out, failed = {}, []
    for case, text in kernel_graphs.all_cases():
        try:
            blob, counters = oracle.ref_json_run(text, SEED)
        except RuntimeError as e:
            failed.append((case, str(e)))
            continue
        out[case] = {"sha256": hashlib.sha256(blob).hexdigest(), "bytes": len(blob), "counters": counters}
    (HERE / "kernels.json").write_text(json.dumps({"seed": SEED, "cases": out, "reference_errors": dict(failed)},
                                                  indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(out)} cases; reference rejected {len(failed)}: {failed[:5]}")


if __name__ == "__main__":
    main()
