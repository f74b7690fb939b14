"""Diagnostics: the standalone factorization (INT8 path) against LAPACK at a few orders."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2008_01541_b200 import dense as pd
for nt in (6, 10, 24, 48):
    m = 64 * nt
    d = pd.DenseCholesky(m, int8=True)
    d.synthetic()
    A = d.matrix()
    try:
        d.factor()
        L = d.factor_lower()
        ref = np.linalg.cholesky(A)
        print(m, "max |L - L_lapack| / max|L|:", float(np.abs(L - ref).max() / np.abs(ref).max()))
    except Exception as e:
        print(m, "ERR", e)
