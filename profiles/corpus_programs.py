# plan programs of the example corpus: which units (hand-written groups, local
# chains, per-node NVRTC kernels) each graph runs as, and plan == naive outputs
import glob, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2008_11476_b200 as gvx
for f in sorted(glob.glob("examples/*.json")):
    g = gvx.GraphFile(open(f).read())
    print("==", f.split("/")[-1])
    print(g.describe())
    a, ca = g.run(False)
    b, cb = g.run(True)
    same = repr(a) == repr(b)
    print("plan == naive:", same, "counters", ca, cb)
