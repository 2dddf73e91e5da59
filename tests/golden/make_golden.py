"""Generates tests/golden/configs.npz from the UNMODIFIED reference engine
(oracle/_ref/liboracle_ref.so, built from /root/reference by oracle/Makefile).

For each BASELINE config and a set of border-heavy sizes, stores the
reference's own random_buffer input (seed) and the reference run_naive
result, plus the reference's event counters.  Run in the build container
(where /root/reference exists):  python tests/golden/make_golden.py
"""
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
import oracle  # noqa: E402

SIZES = [(1, 1), (2, 3), (7, 5), (16, 16), (33, 17), (64, 48), (5, 129), (130, 3)]
CONFIGS = [1, 2, 3, 4]


def main():
    out = {}
    for (w, h) in SIZES:
        for cfg in CONFIGS:
            seed = 1000 * cfg + w * 7 + h
            img = oracle.ref_random_u8(w, h, seed)
            res, _ = oracle.ref_run(cfg, img)
            cnt = oracle.ref_counters(cfg, img)
            key = f"c{cfg}_{w}x{h}"
            out[key + "_in"] = img
            out[key + "_seed"] = np.array(seed)
            if cfg == 4:
                out[key + "_hist"] = res[0]
                out[key + "_stats"] = np.array([res[1], res[2]])
            else:
                out[key + "_out"] = res
            out[key + "_counters"] = np.array([cnt["kernel_launches"], cnt["pixels_read"], cnt["pixels_written"],
                                               cnt["transfers_executed"]], np.int64)
    np.savez_compressed(HERE / "configs.npz", **out)
    print(f"wrote {len(out)} arrays to {HERE / 'configs.npz'}")


if __name__ == "__main__":
    main()
