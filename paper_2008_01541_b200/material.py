"""Corotated PD material with free per-element rotations, the bi-phasic
stretch-limited variant, and the constant scalar stiffness block.

API of the reference module (/root/reference/pkg/src/schurpd/material.py).
The hot-path math (sign-carrying 3x3 SVD, rotations, clamp, element forces,
energy) runs in the sm_100a element kernels (csrc/element.cu) through the C ABI;
the stiffness assembly is host-side scene setup.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native
from .errors import InvalidArgumentError
from .linalg import ScalarSparseSym
from .mesh import RestData, TetMesh


@dataclass(frozen=True)
class MaterialParams:
    """mu (Pa); lam fixed at 0; mu_prime > 0 enables the bi-phasic term with
    principal stretches limited to [sigma_min, sigma_max] (material.py:24-49)."""

    mu: float
    lam: float = 0.0
    mu_prime: float = 0.0
    sigma_min: float = 0.9
    sigma_max: float = 1.1

    def __post_init__(self):
        if self.mu <= 0:
            raise InvalidArgumentError(f"mu must be positive, got {self.mu}")
        if self.lam != 0.0:
            raise InvalidArgumentError("the volumetric lambda term is not supported; lam must be 0")
        if self.mu_prime < 0:
            raise InvalidArgumentError(f"mu_prime must be >= 0, got {self.mu_prime}")
        if not (0.0 < self.sigma_min <= 1.0 <= self.sigma_max):
            raise InvalidArgumentError(
                f"need 0 < sigma_min <= 1 <= sigma_max, got [{self.sigma_min}, {self.sigma_max}]"
            )

    @property
    def biphasic(self) -> bool:
        return self.mu_prime > 0.0


class RotationCache:
    """Per-element projections: rotations r (ne,3,3) and, bi-phasic, q.

    When owned by a device-resident solver state the arrays are pulled from
    the GPU lazily on first access after a frame (the solver sets `_pull`)."""

    def __init__(self, r: np.ndarray, q: Optional[np.ndarray] = None):
        self._r = r
        self._q = q
        self._pull = None  # callable returning (r, q) when the device copy is newer

    def _sync(self):
        if self._pull is not None:
            pull, self._pull = self._pull, None
            r, q = pull()
            self._r[...] = r
            if q is not None and self._q is not None:
                self._q[...] = q

    @property
    def r(self) -> np.ndarray:
        self._sync()
        return self._r

    @r.setter
    def r(self, value):
        self._pull = None
        self._r = value

    @property
    def q(self) -> Optional[np.ndarray]:
        self._sync()
        return self._q

    @q.setter
    def q(self, value):
        self._sync()
        self._q = value

    @classmethod
    def identity(cls, num_elements: int, biphasic: bool = False) -> "RotationCache":
        eye = np.broadcast_to(np.eye(3), (num_elements, 3, 3)).copy()
        return cls(eye, eye.copy() if biphasic else None)

    def copy(self) -> "RotationCache":
        self._sync()
        return RotationCache(self._r.copy(), None if self._q is None else self._q.copy())


def signed_svd(f: np.ndarray):
    """One 3x3: (U, s, V), f = U diag(s) V^T, U, V proper rotations,
    s0 >= s1 >= |s2|, s2 < 0 iff det f < 0 (device kernel)."""
    out = _native.op_svd(np.reshape(f, (1, 3, 3)), want=("U", "S", "V"))
    return out["U"][0], out["S"][0], out["V"][0]


def polar_rotations(F: np.ndarray) -> np.ndarray:
    """Best-fit rotations of a stack of 3x3 (det +1 for singular/inverted F)."""
    return _native.op_svd(F, want=("R",))["R"]


def polar_rotation(f: np.ndarray) -> np.ndarray:
    return polar_rotations(np.reshape(f, (1, 3, 3)))[0]


def biphasic_projections(F: np.ndarray, params: MaterialParams) -> np.ndarray:
    """Nearest matrices with singular values clamped to [sigma_min, sigma_max]."""
    if not params.biphasic:
        raise InvalidArgumentError("biphasic projection requires mu_prime > 0")
    return _native.op_svd(F, want=("Q",), sigma_min=params.sigma_min, sigma_max=params.sigma_max)["Q"]


def biphasic_projection(f: np.ndarray, params: MaterialParams) -> np.ndarray:
    return biphasic_projections(np.reshape(f, (1, 3, 3)), params)[0]


def energy_density(f, r, q, params: MaterialParams) -> float:
    """mu |f - r|^2 (+ mu' |f - q|^2) of one element (scalar helper)."""
    d = np.asarray(f) - r
    e = params.mu * float(np.sum(d * d))
    if q is not None:
        dq = np.asarray(f) - q
        e += params.mu_prime * float(np.sum(dq * dq))
    return e


def piola_stress(f, r, q, params: MaterialParams) -> np.ndarray:
    """2 mu (f - r) (+ 2 mu' (f - q)) of one element (scalar helper)."""
    p = 2.0 * params.mu * (np.asarray(f) - r)
    if q is not None:
        p = p + 2.0 * params.mu_prime * (np.asarray(f) - q)
    return p


def element_forces(mesh: TetMesh, rest: RestData, e: int, p: np.ndarray) -> np.ndarray:
    """(4,3) node forces of one element from its Piola stress (rows sum to 0)."""
    if not 0 <= e < mesh.num_elements:
        raise InvalidArgumentError(f"element index {e} out of range")
    g = -rest.volume[e] * (p @ rest.dm_inverse[e].T)
    out = np.empty((4, 3))
    out[1:] = g.T
    out[0] = -g.sum(axis=1)
    return out


def elastic_forces(mesh: TetMesh, rest: RestData, x: np.ndarray, rotations: RotationCache,
                   params: MaterialParams, elements: Optional[np.ndarray] = None,
                   out: Optional[np.ndarray] = None) -> np.ndarray:
    """Node forces of the fixed-projection energy over a subset (device kernel;
    deterministic slot-major element-order gather)."""
    q = rotations.q if (rotations.q is not None and params.biphasic) else None
    f, _ = _native.op_elastic(mesh.tets, rest.dm_inverse, rest.volume, x, rotations.r, q, params.mu,
                              params.mu_prime if q is not None else 0.0, elements=elements, forces=True)
    if out is None:
        return f
    out += f
    return out


def elastic_energy(mesh: TetMesh, rest: RestData, x: np.ndarray, rotations: RotationCache,
                   params: MaterialParams, elements: Optional[np.ndarray] = None) -> float:
    """Volume-integrated fixed-projection energy over a subset (device kernel)."""
    q = rotations.q if (rotations.q is not None and params.biphasic) else None
    _, e = _native.op_elastic(mesh.tets, rest.dm_inverse, rest.volume, x, rotations.r, q, params.mu,
                              params.mu_prime if q is not None else 0.0, elements=elements, forces=False,
                              energy=True)
    return e


def element_scalar_stiffness(rest: RestData, params: MaterialParams) -> np.ndarray:
    """(ne,4,4) blocks 2 (mu + mu') vol B B^T of the shared coordinate block."""
    dmi = rest.dm_inverse
    B = np.concatenate([-dmi.sum(axis=1, keepdims=True), dmi], axis=1)  # (ne,4,3)
    coef = 2.0 * (params.mu + params.mu_prime) * rest.volume
    return coef[:, None, None] * np.einsum("eaj,ebj->eab", B, B)


def assemble_stiffness(mesh: TetMesh, rest: RestData, params: MaterialParams) -> ScalarSparseSym:
    """Constant n x n scalar stiffness (identical for x, y, z; zero row sums)."""
    ke = element_scalar_stiffness(rest, params)
    rows = np.repeat(mesh.tets, 4, axis=1).ravel()
    cols = np.tile(mesh.tets, (1, 4)).ravel()
    return ScalarSparseSym.from_coo(mesh.num_nodes, rows, cols, ke.ravel())
