import sys; sys.path.insert(0,'.')
import numpy as np, paper_2008_11476_b200 as gvx, oracle
cfg = int(sys.argv[1]); w = int(sys.argv[2]); h = int(sys.argv[3])
img = gvx.random_u8(w,h,3)
g = gvx.ConfigGraph(cfg,w,h)
got,_ = g.run_host(img)
want = oracle.port_run(cfg, img)
print("cfg", cfg, w, h, "equal:", bool(np.array_equal(got, want)) if cfg != 4 else got[1:] == want[1:])
