"""Quick GPU shake-out: every config through run_plan / run_naive / sessions
against the oracles at small and medium sizes.  Prints one line per case;
exits non-zero on the first mismatch.  (The pytest suite is the real gate;
this is a fast developer loop for gpurun.)"""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2008_11476_b200 as gvx  # noqa: E402


def expect(cfg, img):
    if oracle.have_ref():
        return oracle.ref_run(cfg, img)[0]
    return oracle.port_run(cfg, img)


def same(cfg, a, b):
    if cfg == 4:
        return bool((a[0] == b[0]).all() and a[1] == b[1] and a[2] == b[2])
    return bool((a == b).all())


def main():
    print("devices:", gvx.device_count(), "ref oracle:", oracle.have_ref())
    bad = 0
    for (w, h) in [(1, 1), (2, 3), (7, 5), (33, 17), (64, 48), (513, 77), (1000, 300), (1920, 1080)]:
        img = gvx.random_u8(w, h, 11)
        for cfg in (1, 2, 3, 4):
            try:
                want = expect(cfg, img)
                g = gvx.ConfigGraph(cfg, w, h, True)
                t0 = time.time()
                got_p, cnt_p = g.run_host(img, naive=False)
                got_n, cnt_n = g.run_host(img, naive=True)
                ok = same(cfg, got_p, want) and same(cfg, got_n, want)
                if not ok:
                    bad += 1
                    if cfg != 4:
                        dp = np.argwhere(got_p != want)
                        dn = np.argwhere(got_n != want)
                        print("   plan mismatches", len(dp), dp[:5].tolist(), "naive mismatches", len(dn), dn[:5].tolist())
                        if len(dp):
                            y, x = dp[0]
                            print("   plan", got_p[y, x], "want", want[y, x], "naive", got_n[y, x])
                    else:
                        print("   plan", got_p[1:], "naive", got_n[1:], "want", want[1:],
                              (got_p[0] != want[0]).sum(), (got_n[0] != want[0]).sum())
                print(f"{w}x{h} cfg{cfg} ok={ok} plan={cnt_p} naive={cnt_n} t={time.time() - t0:.2f}s", flush=True)
            except Exception:
                bad += 1
                print(f"{w}x{h} cfg{cfg} EXCEPTION")
                traceback.print_exc()
    # describe the lowered programs
    for cfg in (1, 2, 3, 4):
        g = gvx.ConfigGraph(cfg, 256, 128, True)
        print(g.describe(False))
        print(g.pass_stats())
    print("BAD", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
