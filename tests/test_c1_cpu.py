"""CPU pins of the BASELINE C1 restatement (2-level spatial T. Chan
preconditioner of A = I (x) T_x + T_y (x) I): the numpy FFT solve equals a
dense solve with the circulants built from the reference's T. Chan first
columns (circulant.cpp:10-26, ref_tchan in oracle/_ref)."""
import numpy as np
import pytest

from oracle.pyoracle import circulant_dense, spatial_precond_solve


@pytest.mark.parametrize("shape", [(1, 5, 7), (2, 8, 8), (3, 13, 6), (1, 31, 17)])
def test_spatial_precond_matches_dense(ref, shape):
    nt, n1, n2 = shape
    cy, ry = ref.build_riesz(1.7, n1, 1.0 / (n1 + 1))
    cx, rx = ref.build_riesz(1.3, n2, 1.0 / (n2 + 1))
    fy, ly = ref.tchan(cy, ry)
    fx, lx = ref.tchan(cx, rx)
    Cy, Cx = circulant_dense(fy), circulant_dense(fx)
    A2 = np.kron(Cy, np.eye(n2)) + np.kron(np.eye(n1), Cx)
    rng = np.random.default_rng(7)
    r = rng.standard_normal(nt * n1 * n2)
    z = spatial_precond_solve(shape, ly, lx, r)
    zd = np.concatenate([np.linalg.solve(A2, r[k * n1 * n2:(k + 1) * n1 * n2]) for k in range(nt)])
    assert np.linalg.norm(z - zd) <= 1e-11 * np.linalg.norm(zd)


def test_c1_eigenvalues_real(ref):
    """Symmetric Riesz factors -> real, even T. Chan spectra (the GPU's Hartley
    formulation relies on it)."""
    for beta, n in ((1.3, 1023), (1.7, 1023), (1.5, 64)):
        c, r = ref.build_riesz(beta, n, 1.0 / (n + 1))
        _, lam = ref.tchan(c, r)
        assert np.max(np.abs(lam.imag)) <= 1e-12 * np.max(np.abs(lam))
        assert np.allclose(lam.real[1:], lam.real[1:][::-1], rtol=1e-12, atol=0)


def test_pfa_1023_index_maps():
    """The Good-Thomas plan of csrc/fdg_pfa.cu, executed step for step in
    numpy on one lane: pass-A gather x[(31 a + 33 b) mod 1023] -> DFT_31 ->
    slot k2 * 33 + a; pass B DFT_33 as DFT_3 x DFT_11 over
    a = (11 i + 3 j) mod 33 -> slot k2 * 33 + (22 c + 12 d) mod 33; X[k] read
    back at (k mod 31) * 33 + k mod 33 equals the 1023-point DFT."""
    N, PA, PB = 1023, 33, 31
    rng = np.random.default_rng(11)
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    E = np.zeros(N, complex)
    for a in range(PA):
        E[np.arange(PB) * PA + a] = np.fft.fft(x[(31 * a + 33 * np.arange(PB)) % N])
    X2 = np.zeros(N, complex)
    i, j = np.meshgrid(np.arange(3), np.arange(11), indexing="ij")
    c, d = i, j
    for t in range(PB):
        r = E[t * PA + (11 * i + 3 * j) % PA]
        r = np.fft.fft(np.fft.fft(r, axis=0), axis=1)
        X2[t * PA + (22 * c + 12 * d) % PA] = r
    k = np.arange(N)
    X = X2[(k % PB) * PA + k % PA]
    ref = np.fft.fft(x)
    assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
