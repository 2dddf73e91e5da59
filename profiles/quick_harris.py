import sys; sys.path.insert(0,'.')
import numpy as np, paper_2008_11476_b200 as gvx, oracle
for (w,h) in [(77,41),(1,1),(480,64),(481,65),(3840,2160)]:
    img = gvx.random_u8(w,h,3)
    g = gvx.ConfigGraph(2,w,h)
    got,_ = g.run_host(img)
    print(w,h, np.array_equal(got, oracle.port_run(2,img)), flush=True)
