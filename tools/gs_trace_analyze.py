"""Critical-path analysis of a traced GS sweep (MGRX_GS_TRACE output)."""
import sys
import numpy as np

for path in sys.argv[1:]:
    with open(path, "rb") as f:
        n, levels, nnz = np.frombuffer(f.read(12), np.int32)
        order = np.frombuffer(f.read(4 * n), np.int32)
        dp = np.frombuffer(f.read(4 * (n + 1)), np.int32)
        dc = np.frombuffer(f.read(4 * nnz), np.int32)
        t0 = np.frombuffer(f.read(8 * n), np.uint64).astype(np.int64)
        t1 = np.frombuffer(f.read(8 * n), np.uint64).astype(np.int64)
    base = t0.min()
    t0 = t0 - base
    t1 = t1 - base
    rows = order
    ready = np.zeros(n, np.int64)
    for p in range(n):
        i = rows[p]
        deps = dc[dp[p]:dp[p + 1]]
        ready[i] = t1[deps].max() if deps.size else 0
    hop = t1 - np.maximum(ready, t0)        # publish after (ready and started)
    late = np.maximum(t0 - ready, 0)         # row started after its deps were ready
    total = t1.max()
    print(f"{path}: n={n} levels={levels} total={total/1e3:.1f}us per-level={total/levels/1e3:.2f}us")
    print("  hop (publish - max(ready,start)) us: p50 %.2f p90 %.2f p99 %.2f" % tuple(np.percentile(hop, [50, 90, 99]) / 1e3))
    print("  late start (start - ready) us:        p50 %.2f p90 %.2f frac>0 %.2f" % (np.percentile(late, 50) / 1e3, np.percentile(late, 90) / 1e3, (late > 0).mean()))
    # critical path walk from the last row
    i = int(np.argmax(t1))
    chain = []
    pos = np.empty(n, np.int64)
    pos[rows] = np.arange(n)
    while True:
        p = pos[i]
        deps = dc[dp[p]:dp[p + 1]]
        chain.append((i, t0[i], t1[i], ready[i]))
        if deps.size == 0:
            break
        i = int(deps[np.argmax(t1[deps])])
    chain = chain[::-1]
    hops = np.array([c[2] - max(c[3], c[1]) for c in chain])
    lates = np.array([max(c[1] - c[3], 0) for c in chain])
    print(f"  critical chain: {len(chain)} rows, mean hop {hops.mean()/1e3:.2f}us, mean late-start {lates.mean()/1e3:.2f}us")
