# one plan execution of a 4K corpus graph (for an ncu kernel list)
import sys
sys.path.insert(0, ".")
import paper_2008_11476_b200 as gvx
g = gvx.GraphFile(open(sys.argv[1]).read())
print(g.describe())
for _ in range(2):
    g.run(naive=False, seed=1)
