"""Generates tests/golden/fullsize.json from the UNMODIFIED reference engine
(oracle/_ref/liboracle_ref.so, built from /root/reference by oracle/Makefile).

For every BASELINE config at its configured size (SURVEY.md §8d seeds:
cfg1 = 1, cfg2 = 2, cfg3 = 3, cfg4 = 4 + frame, cfg5 = 5) the reference's own
random_buffer input is run through verify -> expand -> verify -> run_naive
(ref:src/execute.cpp:880-888) and the SHA-256 of the input and of the output
bytes is stored, plus per-block digests of the output (blocks of
`BLOCK_ROWS` rows) so a mismatch on the B200 localises to a row band.
cfg4's histogram / mean / stddev are small and stored in full for `CFG4_FRAMES`
frames of the 64-frame batch.

Run in the build container (where /root/reference exists; cfg5 alone takes
~150 s of reference CPU time):  python tests/golden/make_fullsize_golden.py
"""
import hashlib
import json
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
import oracle  # noqa: E402

SIZES = {1: (1920, 1080), 2: (3840, 2160), 3: (7680, 4320), 4: (3840, 2160), 5: (16384, 16384)}
BLOCK_ROWS = {1: 270, 2: 540, 3: 1080, 5: 2048}
CFG4_FRAMES = 6


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(cfgs):
    path = HERE / "fullsize.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    for cfg in cfgs:
        w, h = SIZES[cfg]
        t0 = time.time()
        if cfg == 4:
            frames = []
            for f in range(CFG4_FRAMES):
                img = oracle.ref_random_u8(w, h, 4 + f)
                (hist, mean, sd), _ = oracle.ref_run(4, img)
                frames.append({"seed": 4 + f, "input_sha256": sha(img), "hist": [int(x) for x in hist],
                               "mean": float(mean).hex(), "stddev": float(sd).hex()})
            out["4"] = {"width": w, "height": h, "frames": frames}
        else:
            img = oracle.ref_random_u8(w, h, cfg)
            res, secs = oracle.ref_run(cfg, img)
            br = BLOCK_ROWS[cfg]
            out[str(cfg)] = {"width": w, "height": h, "seed": cfg, "input_sha256": sha(img),
                             "output_dtype": str(res.dtype), "output_sha256": sha(res), "block_rows": br,
                             "block_sha256": [sha(res[r:r + br]) for r in range(0, h, br)],
                             "reference_run_naive_seconds": round(secs, 2)}
            del res, img
        print(f"cfg{cfg}: {time.time() - t0:.1f} s", flush=True)
        path.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {path}")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5])
