import sys, traceback; sys.path.insert(0,'.'); sys.path.insert(0,'tests'); sys.path.insert(0,'tests/golden')
import numpy as np, paper_2101_11649_b200 as mx
from concurrent.futures import ThreadPoolExecutor
P = mx.mfd_problem(12, 12, 8, "layered"); t = mx.load_strategy("mfd_mgr_pi_c1_l1j")
H = mx.Hierarchy(mx.Matrix(P.ptr, P.col, P.val), P.partition, t)
g = mx.LocalGroup(2); st = mx.slab_row_starts(P, 2)
S = [mx.Shard(H, r, 2, st, group=g) for r in range(2)]
v = np.random.default_rng(7).uniform(-1, 1, P.n)
def f(s):
    try: return s.apply(v[s.row_begin:s.row_end])
    except Exception as e: traceback.print_exc(); return None
with ThreadPoolExecutor(2) as ex: zs = list(ex.map(f, S))
print("apply ok" if all(z is not None for z in zs) else "apply FAILED")
