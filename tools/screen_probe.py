import sys, numpy as np
sys.path.insert(0, "/root/repo")
import bench
from paper_1702_05911_b200 import DeviceIndex
from oracle.bindings import Oracle
hix, Q = bench.make_workload("gist1m", 7, 0, 1)
Q = Q[:200]
from paper_1702_05911_b200._abi import lib
lib().pqtg_set_kernel_variant(2)
dev = DeviceIndex(hix, max_batch=256)
dev.search(Q, 100)
inter = dev.intermediates(len(Q))
o = Oracle(hix)
exact = 0; tot = 0; maxrel = 0
for i in range(len(Q)):
    t = o.traverse(Q[i])
    assert np.array_equal(inter["l2_parent"][i], t["l2_parent"]) and np.array_equal(inter["l2_child"][i], t["l2_child"])
    g, w = inter["l2_dist"][i], t["l2_dist"]
    exact += int((g.view(np.uint32) == w.view(np.uint32)).sum()); tot += g.size
    maxrel = max(maxrel, float(np.max(np.abs(g - w) / np.maximum(w, 1e-30))))
print("exact fraction", exact / tot, "entries per part", exact / tot * g.shape[1], "max rel err", maxrel)

# radius analysis (numpy restatement of screen.cu's screen_radius on the exact distances)
c = hix.config
m = c.dim // c.p_tree
L1 = hix.level1.reshape(c.p_tree, c.k1, m).astype(np.float64)
L2 = hix.level2.reshape(c.p_tree, c.k1 * c.k2, m).astype(np.float64)
mu = L2.mean(axis=1)
u = 2.0 ** -24
ratios, gaps, rads, mand = [], [], [], 0
for i in range(50):
    t = o.traverse(Q[i])
    for p in range(c.p_tree):
        y = Q[i, p * m:(p + 1) * m].astype(np.float64)
        yn = ((y - mu[p]) ** 2).sum()
        d = t["l2_dist"][p].astype(np.float64)
        par, ch = t["l2_parent"][p], t["l2_child"][p]
        j = par * c.k2 + ch
        cpp = L2[p, j] - L1[p, par]
        cn = (cpp ** 2).sum(1)
        l1 = ((y[None, :] - L1[p, par]) ** 2).sum(1)
        g = ((y - mu[p])[None, :] * cpp).sum(1)
        e = 6.1035156e-5 * np.sqrt(yn * cn) + (m + 16) * u * l1 + 4 * u * (2 * abs(g) + cn) + 2.38e-7 * np.sqrt(d * cn)
        R = e + (m + 4) * u * 1.05 * (d + e)
        rads.append(R / d)
        gaps.append(np.diff(d) / d[:-1])
        ratios.append(e / d)
print("median R/d", np.median(np.concatenate([r for r in rads])), "median gap/d", np.median(np.concatenate(gaps)),
      "frac gaps < 2R", np.mean(np.concatenate(gaps) < 2 * np.concatenate([r[:-1] for r in rads])))
print("median tc-part/d", np.median(np.concatenate(ratios)))
