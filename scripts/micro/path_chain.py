import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1810_04221_b200 as pkg
dev = pkg.Device(0)
for n in (2000, 20000, 100000):
    # path graph 0-1-2-...-(n-1), all weights equal -> one dislodgement chain of ~n/2 links
    xadj = np.zeros(n + 1, np.int64); adj = []
    for i in range(n):
        nb = [j for j in (i - 1, i + 1) if 0 <= j < n]
        adj += nb; xadj[i + 1] = xadj[i] + len(nb)
    adj = np.array(adj, np.int64); w = np.ones(len(adj))
    dev.suitor(xadj, adj, w)
    dev.synchronize()
    ts = []
    for r in range(3):
        t0 = time.perf_counter(); m = dev.suitor(xadj, adj, w); dev.synchronize(); ts.append(time.perf_counter() - t0)
    ok = all(m[2 * k] == 2 * k + 1 for k in range(n // 2))
    print(f"path n={n}: {min(ts)*1e3:.2f} ms -> {min(ts)*1e9/(n/2):.0f} ns per link (greedy pairs ok={ok})")
