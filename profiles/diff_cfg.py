# where a config's GPU output differs from the C restatement (rows / columns of the mismatches)
import sys; sys.path.insert(0, '.')
import numpy as np, paper_2008_11476_b200 as gvx, oracle
cfg, w, h = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
img = gvx.random_u8(w, h, 3)
import time
t0 = time.time()
g = gvx.ConfigGraph(cfg, w, h)
got, _ = g.run_host(img)
t1 = time.time()
want = oracle.port_run(cfg, img)
print('gpu s', round(t1 - t0, 2), 'oracle s', round(time.time() - t1, 2), flush=True)
if cfg == 4:
    print("cfg 4", w, h, "equal:", got[1:] == want[1:]); sys.exit()
bad = np.argwhere(got != want)
print("cfg", cfg, w, h, "mismatches", len(bad))
if len(bad):
    ys, xs = np.unique(bad[:, 0]), np.unique(bad[:, 1])
    print(" rows", ys[:40], "... n", len(ys))
    print(" cols", xs[:40], "... n", len(xs))
