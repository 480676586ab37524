import sys, numpy as np
sys.path.insert(0, ".")
import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import bhtree
g = np.load("tests/golden/trees.npz")
for case in ["octant", "dups_cap6", "uniform300", "grid1200", "dups400", "blob2000", "uniform_cap3"]:
    t = bhtree.build(fga.PointCloud(g[f"{case}/pts"]), g[f"{case}/masses"], int(g[f"{case}/max_depth"]))
    m, rm = t.mass, g[f"{case}/mass"]
    rel = np.abs(m - rm) / np.abs(rm)
    bad = np.nonzero(rel > 1e-12)[0]
    print(case, len(m), "bad", len(bad), "maxrel", rel.max())
    for x in bad[:6]:
        print("   node", x, "depth", t.depth[x], "occ", t.occupancy[x], "mass", m[x], "ref", rm[x], "nchild", (t.children[x] >= 0).sum())
