"""Off-line: how many faces of an EI-ZO polytope (and of its per-iteration prefixes) are
strictly redundant?  LP per face (scipy HiGHS): max a_f x s.t. the other faces."""
import sys
import time

import numpy as np
from scipy.optimize import linprog

z = np.load(sys.argv[1])
A, b = z["A"], z["b"]
d = A.shape[1]
F0 = 2 * d
nf = 10


def redundant(A, b, idx, margin=1e-7):
    red = []
    for f in idx:
        m = np.ones(A.shape[0], bool)
        m[f] = False
        r = linprog(-A[f], A_ub=A[m], b_ub=b[m], bounds=[(None, None)] * d, method="highs")
        if r.status == 0 and -r.fun <= b[f] - margin:
            red.append(f)
    return red


for F in [int(x) for x in sys.argv[2:]] or [A.shape[0]]:
    t0 = time.perf_counter()
    red = redundant(A[:F], b[:F], range(F))
    print(f"F={F}: {len(red)} strictly redundant ({len(red) / F:.2%}) in {time.perf_counter() - t0:.1f}s; "
          f"domain faces redundant {sum(f < F0 for f in red)}")
