import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_1702_05911_b200 import DeviceIndex
hix, Q = bench.make_workload("gist1m", 7, 0, 4)
dev = DeviceIndex(hix, max_batch=4000)
dev.search(Q[:4000], 100)
c = dev.counters(4000)
t = c["ntuples"].astype(np.int64)
print("T_q percentiles 50/90/99/99.9/max:", np.percentile(t, [50, 90, 99, 99.9]).astype(int), t.max(), "mean", t.mean())
print("frac > 8192:", (t > 8192).mean(), "> 16384:", (t > 16384).mean(), "> 32768:", (t > 32768).mean())
