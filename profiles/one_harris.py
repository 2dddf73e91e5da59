import sys; sys.path.insert(0,'.')
import numpy as np, paper_2008_11476_b200 as gvx
img = gvx.random_u8(77,41,3)
g = gvx.ConfigGraph(2,77,41)
got,_ = g.run_host(img)
print("ok")
