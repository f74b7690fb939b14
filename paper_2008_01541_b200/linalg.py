"""Sparse symmetric containers and the three-step direct solve.

Same API as the reference module (/root/reference/pkg/src/schurpd/linalg.py):
ScalarSparseSym (:30-94), CscLower (:230-254), PartialFactor (:298-319),
partial_cholesky (:329-382), forward_sub / backward_sub (:385-414),
DenseSPD / dense_factor / schur_assemble / dense_solve (:420-461), pcg (:467-504).

Where the computation lives:
  * partial_cholesky / fill_ordering -> native host precompute (C++,
    multifrontal supernodal, nested dissection; csrc/precompute.cpp);
  * forward_sub / backward_sub / dense_factor / dense_solve -> sm_100a
    kernels through the C ABI (no host fallback);
  * ScalarSparseSym, CscLower inspection helpers and the PCG baseline are host
    utilities outside the per-frame hot path.
"""

from __future__ import annotations

from typing import Callable, Optional, Tuple

import numpy as np
import scipy.io
import scipy.sparse as sp

from . import _native
from .errors import IndefiniteMatrixError, IndefiniteOperatorError, InvalidArgumentError

PIVOT_TOLERANCE = 1e-13  # linalg.py:227


class ScalarSparseSym:
    """Symmetric n x n scalar block stored as its upper triangle (CSC, sorted);
    the 3n x 3n operator is this block on each coordinate."""

    def __init__(self, upper: sp.spmatrix):
        if upper.shape[0] != upper.shape[1]:
            raise InvalidArgumentError("matrix must be square")
        u = sp.csc_matrix(upper)
        u.sum_duplicates()
        u.sort_indices()
        if sp.tril(u, -1).nnz:
            raise InvalidArgumentError("strictly-lower entries passed to upper-triangle storage")
        self.upper = u
        self._full = None

    @classmethod
    def from_coo(cls, n: int, rows, cols, vals) -> "ScalarSparseSym":
        """Symmetric triplets (both halves present), duplicates summed."""
        full = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsc()
        full.sum_duplicates()
        return cls(sp.triu(full, format="csc"))

    @classmethod
    def from_dense(cls, a: np.ndarray) -> "ScalarSparseSym":
        a = np.asarray(a, dtype=np.float64)
        tol = 1e-12 * max(1.0, np.abs(a).max(initial=0.0))
        if not np.allclose(a, a.T, rtol=0, atol=tol):
            raise InvalidArgumentError("matrix is not symmetric")
        return cls(sp.triu(sp.csc_matrix(a), format="csc"))

    @property
    def n(self) -> int:
        return self.upper.shape[0]

    @property
    def nnz_upper(self) -> int:
        return self.upper.nnz

    def full(self) -> sp.csr_matrix:
        if self._full is None:
            u = self.upper
            f = (u + u.T - sp.diags(u.diagonal())).tocsr()
            f.sort_indices()
            self._full = f
        return self._full

    def diagonal(self) -> np.ndarray:
        return self.upper.diagonal()

    def matvec(self, x: np.ndarray) -> np.ndarray:
        return self.full() @ x

    def toarray(self) -> np.ndarray:
        return self.full().toarray()

    def permuted(self, order: np.ndarray) -> "ScalarSparseSym":
        """Symmetric permutation, order[new] = old."""
        order = np.asarray(order)
        if order.shape != (self.n,) or not np.array_equal(np.sort(order), np.arange(self.n)):
            raise InvalidArgumentError("order is not a permutation of 0..n-1")
        return ScalarSparseSym(sp.triu(self.full()[order][:, order], format="csc"))

    def __repr__(self):
        return f"ScalarSparseSym(n={self.n}, nnz_upper={self.nnz_upper})"


def write_matrix_market(path, mat) -> None:
    if isinstance(mat, ScalarSparseSym):
        mat = mat.full()
    scipy.io.mmwrite(path, sp.coo_matrix(mat))


class CscLower:
    """Lower-triangular factor in CSC arrays (diagonal first in each column)."""

    def __init__(self, n: int, indptr: np.ndarray, indices: np.ndarray, data: np.ndarray):
        self.n = int(n)
        self.indptr = indptr
        self.indices = indices
        self.data = data

    @property
    def nnz(self) -> int:
        return int(self.indptr[self.n])

    def to_scipy(self) -> sp.csc_matrix:
        return sp.csc_matrix((self.data, self.indices, self.indptr), shape=(self.n, self.n))

    def solve_lower(self, b: np.ndarray) -> np.ndarray:
        """Inspection helper (host); the solver's sweeps run on the device."""
        from scipy.sparse.linalg import spsolve_triangular

        return spsolve_triangular(self.to_scipy().tocsr(), np.asarray(b, dtype=np.float64), lower=True)

    def solve_lower_t(self, b: np.ndarray) -> np.ndarray:
        from scipy.sparse.linalg import spsolve_triangular

        return spsolve_triangular(self.to_scipy().T.tocsr(), np.asarray(b, dtype=np.float64), lower=False)


def fill_ordering(pattern, coords: Optional[np.ndarray] = None) -> np.ndarray:
    """Fill-reducing ordering (order[new] = old): nested dissection (graph
    bisection, or geometric bisection when rest coordinates are given)."""
    if isinstance(pattern, ScalarSparseSym):
        pattern = pattern.upper
    pattern = sp.csc_matrix(pattern)
    n = pattern.shape[0]
    up = sp.triu(pattern + pattern.T, format="csc") if (sp.tril(pattern, -1).nnz) else sp.triu(pattern, format="csc")
    up.sort_indices()
    perm = _native.fill_ordering(n, up, coords)
    if len(perm) != n or not np.array_equal(np.bincount(perm, minlength=n), np.ones(n, dtype=np.int64)):
        raise RuntimeError("fill ordering produced a non-bijective permutation")
    # nested dissection targets meshes; on band-like graphs (a chain) its
    # separators add fill the natural order avoids: keep whichever fills less
    # (symbolic counts only, no factorization)
    if n > 1:
        full = (up + sp.triu(up, 1).T).tocsr()
        nd = _native.symbolic_nnz(n, sp.triu(full[perm][:, perm], format="csc"))
        nat = _native.symbolic_nnz(n, up)
        if nat <= nd:
            return np.arange(n, dtype=np.int64)
    return perm


class PartialFactor:
    """Partial Cholesky of an SPD matrix split at n1 (reference linalg.py:298-319):
    l1 l1^T = P1 A11 P1^T, coupling = A21 P1^T L1^-T, sigma0 = A22 - C C^T.
    l1 and coupling are exported lazily from the native supernodal factor."""

    def __init__(self, native: _native.NativeFactor, n1: int, n2: int):
        self.native = native
        self.n1 = n1
        self.n2 = n2
        self.fill_perm = native.fill_perm()
        self._l1 = None
        self._coupling = None
        self._sigma0 = None

    @property
    def n(self) -> int:
        return self.n1 + self.n2

    @property
    def l1(self) -> CscLower:
        if self._l1 is None:
            ip, ix, dx = self.native.l1_csc()
            self._l1 = CscLower(self.n1, ip, ix, dx)
        return self._l1

    @property
    def coupling(self) -> sp.csr_matrix:
        if self._coupling is None:
            ip, ix, dx = self.native.coupling_csr()
            self._coupling = sp.csr_matrix((dx, ix, ip), shape=(self.n2, self.n1))
        return self._coupling

    @property
    def sigma0(self) -> np.ndarray:
        if self._sigma0 is None:
            self._sigma0 = self.native.sigma0()
        return self._sigma0


def _columns(b) -> Tuple[np.ndarray, bool]:
    b = np.asarray(b, dtype=np.float64)
    if b.ndim == 1:
        return b[:, None], True
    return b, False


def partial_cholesky(A: ScalarSparseSym, n1: int, use_fill_ordering: bool = True,
                     coords: Optional[np.ndarray] = None) -> PartialFactor:
    """Eliminate the leading n1 unknowns of A and retain the dense Schur
    complement of the trailing block (fill ordering inside x1 only)."""
    n = A.n
    if not 0 <= n1 <= n:
        raise InvalidArgumentError(f"n1 = {n1} out of range for n = {n}")
    try:
        nat = _native.NativeFactor(n, n1, A.upper, coords=coords,
                                   ordering=1 if (use_fill_ordering and n1 > 1) else 0,
                                   relax=1 if use_fill_ordering else 0)
    except IndefiniteMatrixError as err:
        raise IndefiniteMatrixError(
            f"leading block is not positive definite: non-positive pivot (original index {err.column})",
            column=err.column,
        ) from None
    return PartialFactor(nat, n1, n - n1)


def forward_sub(f: PartialFactor, b1, b2):
    """y1 = L1^-1 b1[fill] (factored basis), y2 = b2 - C y1 (device sweep)."""
    b1c, squeeze = _columns(b1)
    b2c, _ = _columns(b2)
    if b1c.shape[0] != f.n1 or b2c.shape[0] != f.n2:
        raise InvalidArgumentError("right-hand side sizes do not match the factor split")
    y1, y2 = f.native.forward_sub(b1c, b2c)
    if squeeze:
        return y1[:, 0], y2[:, 0]
    return y1, y2


def backward_sub(f: PartialFactor, y1, x2) -> np.ndarray:
    """x1 = L1^-T (y1 - C^T x2), returned in the partition basis (device sweep)."""
    y1c, squeeze = _columns(y1)
    x2c, _ = _columns(x2)
    if y1c.shape[0] != f.n1 or x2c.shape[0] != f.n2:
        raise InvalidArgumentError("vector sizes do not match the factor split")
    x1 = f.native.backward_sub(y1c, x2c)
    return x1[:, 0] if squeeze else x1


class DenseSPD:
    """Dense SPD matrix with its lower Cholesky factor."""

    def __init__(self, h: np.ndarray, chol: np.ndarray):
        self.h = h
        self.chol = chol

    @property
    def m(self) -> int:
        return self.h.shape[0]


def dense_factor(h: np.ndarray) -> DenseSPD:
    """Lower Cholesky of a dense SPD matrix on the device (tile kernel)."""
    h = np.ascontiguousarray(h, dtype=np.float64)
    if h.size == 0:
        return DenseSPD(h.reshape(0, 0), h.reshape(0, 0))
    try:
        chol = _native.op_dense_factor(h)
    except IndefiniteMatrixError as err:
        raise IndefiniteMatrixError(f"dense factorization failed: {err}", column=err.column) from None
    return DenseSPD(h, chol)


def schur_assemble(sigma0: np.ndarray, c22: sp.spmatrix) -> DenseSPD:
    """Additive Schur update sigma0 + C22, then the dense refactorization."""
    m = sigma0.shape[0]
    if c22.shape != (m, m):
        raise InvalidArgumentError(f"c22 shape {c22.shape} does not match sigma0 {sigma0.shape}")
    return dense_factor(sigma0 + c22.toarray())


def dense_solve(f: DenseSPD, g) -> np.ndarray:
    """H^-1 g with the two triangular sweeps on the device."""
    if f.m == 0:
        return np.zeros_like(np.asarray(g, dtype=np.float64))
    gc, squeeze = _columns(g)
    x = _native.op_dense_solve(f.chol, gc)
    return x[:, 0] if squeeze else x


def pcg(apply_A: Callable[[np.ndarray], np.ndarray], b: np.ndarray, jacobi_diag: np.ndarray, tol: float,
        max_iters: int, callback: Optional[Callable[[np.ndarray], None]] = None) -> Tuple[np.ndarray, int]:
    """Jacobi-preconditioned CG baseline (host; the comparison solver of
    PAPER.md §5.4, not the Schur hot path). Stops at |r|/|b| <= tol."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return x, 0
    dinv = 1.0 / np.asarray(jacobi_diag, dtype=np.float64)
    r = b.copy()
    z = dinv * r
    p = z.copy()
    rz = float(r @ z)
    for it in range(1, max_iters + 1):
        q = apply_A(p)
        pq = float(p @ q)
        if pq <= 0.0:
            raise IndefiniteOperatorError(f"p'Ap = {pq:.3e} at iteration {it}")
        alpha = rz / pq
        x += alpha * p
        r -= alpha * q
        if callback is not None:
            callback(x)
        if np.linalg.norm(r) / bnorm <= tol:
            return x, it
        z = dinv * r
        rz_next = float(r @ z)
        p = z + (rz_next / rz) * p
        rz = rz_next
    return x, max_iters
