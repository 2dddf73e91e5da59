"""Generates tests/golden/corpus.json from the UNMODIFIED reference
(oracle/_ref/liboracle_ref.so incl. its graph_io.cpp): for every graph file
in examples/, the reference's canonical save_graph_json text and, with
intermediates made non-virtual (the reference's expand() rejects virtual
images), the SHA-256 of its run_naive outputs on random_buffer inputs
(seed + object id, configs/json_runner.hpp) and its event counters.
Run in the build container:  python tests/golden/make_corpus_golden.py
"""
import hashlib
import json
import pathlib
import sys

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
import oracle  # noqa: E402

SEED = 11


def devirtualise(text: str) -> str:
    d = json.loads(text)
    for im in d.get("images", []):
        im.pop("virtual", None)
    return json.dumps(d)


def main():
    out = {}
    for f in sorted((REPO / "examples").glob("*.json")):
        text = f.read_text()
        blob, counters = oracle.ref_json_run(devirtualise(text), SEED)
        out[f.stem] = {"seed": SEED, "sha256": hashlib.sha256(blob).hexdigest(), "bytes": len(blob),
                       "counters": counters, "canonical": oracle.ref_json_roundtrip(text)}
    (HERE / "corpus.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(out)} entries to {HERE / 'corpus.json'}")


if __name__ == "__main__":
    main()
