import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2603_14926_b200 import roots, Variant, LaneBatch, batch_mul, batch_add
q = roots.MonicPoly.from_coeffs([(-1.0, 0.0), (0.0, 0.0)])
print("planes", q.planes)
k, n = 2, 2
rad = roots.radius_estimate(q, Variant.BRANCH_FREE)
print("rad", rad)
radb = LaneBatch(np.tile(np.array(rad).reshape(k, 1), (1, n)))
print("radb", radb.planes)
cosv = np.array([[0.73, -0.73], [0.0, 0.0]])
print(batch_mul(radb, LaneBatch(cosv), Variant.BRANCH_FREE).planes)
try:
    st = roots.aberth_init(q, Variant.BRANCH_FREE)
    print(st.re, st.im)
except Exception as e:
    print("ERR", e)
