"""The README usage example (runs on a CUDA device)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2603_14926_b200 as mw
from paper_2603_14926_b200 import gen, multiword
rng = np.random.default_rng(0)
A, B = mw.MWMatrix(gen.g_k(rng, 4, (512, 512))), mw.MWMatrix(gen.g_k(rng, 4, (512, 512)))
C = mw.matmul(A, B, mw.MatMulPlan(scheme="naive", variant="bf"))   # QD GEMM, bit-exact with mwfloat
q = mw.chebyshev_coeffs(64, 3)                                      # TD monic polynomial
state, sweeps = mw.dk_solve(q, mw.Variant.BRANCH_FREE)              # Durand-Kerner on the device
print(multiword.mw_add((1.0, 1e-17), (2.0, 0.0), mw.Variant.BRANCH_FREE))  # scalar K-word ops too
print(C.k, sweeps)
