"""Standalone dense Cholesky on the GPU (BASELINE config 4) through the C ABI.

Parity: the factor of the tile kernel against LAPACK dpotrf (scipy, the
reference's own dense_factor path, linalg.py:432-440) at 1e-12 relative; the
failing column of an indefinite matrix equals dpotrf's `info`; full-size
orders are checked through ||A v - L L^T v|| / ||A v|| on the device.

Tile-cyclic data path: the emulated mode factors P ranks' replicas in ONE
launch on this one GPU (CTA b serves rank b % P; finished tiles are pushed
into the other replicas and released with system-scope flags). Every replica
must come out bit-identical to the single-GPU factor: a tile's arithmetic does
not depend on which rank computed it.
"""

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _spd(rng, m, kappa=1e3):
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    w = np.geomspace(1.0, kappa, m)
    return (q * w) @ q.T


@pytest.mark.parametrize("m", [1, 5, 63, 64, 65, 130, 500])
def test_factor_matches_lapack(rng, m):
    from paper_2008_01541_b200.dense import DenseCholesky

    a = _spd(rng, m) + 10.0 * np.eye(m)
    d = DenseCholesky(m)
    d.set_matrix(a)
    d.factor()
    L = d.factor_lower()
    ref = sla.cholesky(a, lower=True)
    assert np.max(np.abs(L - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert np.array_equal(np.triu(L, 1), np.zeros_like(L))


def test_indefinite_column_matches_dpotrf(rng):
    from paper_2008_01541_b200.dense import DenseCholesky
    from paper_2008_01541_b200.errors import IndefiniteMatrixError

    m = 300
    a = _spd(rng, m)
    a[170, 170] = -5.0
    _, info = sla.lapack.dpotrf(a, lower=1)
    assert info > 0
    d = DenseCholesky(m)
    d.set_matrix(a)
    with pytest.raises(IndefiniteMatrixError) as ei:
        d.factor()
    assert ei.value.column == info


def test_synthetic_matrix_and_factor():
    from paper_2008_01541_b200.dense import DenseCholesky, SYNTH_A, SYNTH_B, SYNTH_ELL

    m = 1500
    d = DenseCholesky(m)
    d.synthetic()
    a = d.matrix()
    g = int(np.ceil(np.sqrt(m)))
    r = np.arange(m)
    p = np.stack([r % g, r // g], 1).astype(float)
    dist = np.sqrt(((p[:, None, :] - p[None, :, :]) ** 2).sum(-1))
    want = SYNTH_A * np.exp(-dist / SYNTH_ELL) + SYNTH_B * np.eye(m)
    assert np.max(np.abs(a - want)) <= 1e-12 * np.max(np.abs(want))
    d.factor(reps=2)
    L = d.factor_lower()
    ref = sla.cholesky(a, lower=True)
    assert np.max(np.abs(L - ref)) <= 1e-12 * np.max(np.abs(ref))
    rr, aa = d.residual(np.random.default_rng(1).standard_normal(m))
    assert rr <= 1e-14 * aa * 10


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_emulated_tile_cyclic_replicas_bit_identical(P):
    from paper_2008_01541_b200.dense import DenseCholesky

    m = 1000 if P != 8 else 2100
    one = DenseCholesky(m, int8=False)  # the tile-cyclic ranks run the FP64 DMMA kernel
    one.synthetic()
    one.factor()
    ref = one.factor_lower()
    emu = DenseCholesky(m, nranks=P, emulate=True)
    emu.synthetic()
    for _ in range(2):  # the reset between factorizations clears every replica's flags
        emu.factor()
        for r in range(P):
            assert np.array_equal(emu.factor_lower(replica=r), ref), f"replica {r} of {P}"


def test_emulated_indefinite_reports_first_column(rng):
    from paper_2008_01541_b200.dense import DenseCholesky
    from paper_2008_01541_b200.errors import IndefiniteMatrixError

    m = 400
    a = _spd(rng, m)
    a[250, 250] = -1.0
    _, info = sla.lapack.dpotrf(a, lower=1)
    emu = DenseCholesky(m, nranks=4, emulate=True)
    emu.set_matrix(a)
    with pytest.raises(IndefiniteMatrixError) as ei:
        emu.factor()
    assert ei.value.column == info


@pytest.mark.parametrize("m", [6144, 12288])
def test_full_size_residual(m):
    from paper_2008_01541_b200.dense import DenseCholesky

    d = DenseCholesky(m)
    d.synthetic()
    d.factor()
    rr, aa = d.residual(np.random.default_rng(m).standard_normal(m))
    assert rr <= 1e-13 * aa


@pytest.mark.parametrize("m", [700, 3000, 6197])
def test_int8_tensor_core_factor_matches_fp64(m):
    """The emulated-FP64 factor (INT8 tcgen05 trailing updates, 8 digit
    planes) against the FP64 DMMA factor of the same matrix: 1e-13 of max|L|,
    and the residual ||A v - L L^T v|| / ||A v|| at the FP64 level."""
    from paper_2008_01541_b200.dense import DenseCholesky

    a = DenseCholesky(m, int8=True)
    b = DenseCholesky(m, int8=False)
    assert a.int8 and not b.int8
    for d in (a, b):
        d.synthetic()
        d.factor()
    La, Lb = a.factor_lower(), b.factor_lower()
    assert np.abs(La - Lb).max() <= 1e-13 * np.abs(Lb).max()
    v = np.random.default_rng(m).standard_normal(m)
    rr, aa = a.residual(v)
    assert rr <= 1e-14 * aa * 10
