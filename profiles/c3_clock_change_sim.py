"""How sparse are the clock updates of a C3-like lock trace?

Model of the C3 recipe's lock traffic (workloads.c3_text): T acquiring threads
(lane 0 of every warp), K locks, every iteration each thread acquires a
uniformly random lock, joins the lock's clock (the previous releaser's hb --
with one device-scope instance the lock's accumulated hb equals the last
release clock) and releases it (its own entry + 1, the lock := its clock).
Reports, per join in steady state, the fraction of the T coordinates whose
value changes -- the lower bound on the entries any delta / versioned /
tree-clock representation must touch per join.

    python profiles/c3_clock_change_sim.py [T K iters]
"""
import sys

import numpy as np

T, K, IT = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (2048, 1024, 40)
rng = np.random.default_rng(1)
C = np.zeros((T, T), np.int32)
C[np.arange(T), np.arange(T)] = 1
L = np.zeros((K, T), np.int32)
for it in range(IT):
    changed = 0
    for t in range(T):
        k = rng.integers(K)
        nc = np.maximum(C[t], L[k])
        changed += np.count_nonzero(nc != C[t])
        C[t] = nc
        C[t, t] += 1
        L[k] = C[t]
    if it % 5 == 4 or it == IT - 1:
        print(f"iteration {it:3d}: {changed / T:8.1f} of {T} entries change per join ({changed / T / T:.1%})")
