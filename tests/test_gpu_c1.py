"""BASELINE C1 operator microbenchmark path on the GPU: the 2-level Toeplitz
matvec A = I (x) T_x + T_y (x) I and its 2-level T. Chan preconditioner
(Bluestein Hartley passes, any level size) against the CPU oracle.

Tolerance 1e-11 relative (BASELINE north_star, operator / preconditioner)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _factors(port, shape):
    nt, n1, n2 = shape
    ty = port.build_riesz(1.7, n1, 1.0 / (n1 + 1))
    tx = port.build_riesz(1.3, n2, 1.0 / (n2 + 1))
    return (np.zeros(nt), np.zeros(nt)), ty, tx


SHAPES = [(2, 31, 47), (3, 64, 64), (1, 128, 96), (2, 100, 17), (1, 7, 1023), (2, 1023, 1023), (3, 1, 5)]


@pytest.mark.parametrize("shape", SHAPES)
def test_c1_precond_vs_numpy(gpu_ctx, ref, shape):
    from oracle.pyoracle import spatial_precond_solve
    from paper_1907_13428_b200 import SpatialPreconditioner
    nt, n1, n2 = shape
    cy, ry = ref.build_riesz(1.7, n1, 1.0 / (n1 + 1))
    cx, rx = ref.build_riesz(1.3, n2, 1.0 / (n2 + 1))
    _, ly = ref.tchan(cy, ry)
    _, lx = ref.tchan(cx, rx)
    pc = SpatialPreconditioner.from_eigs(nt, ly, lx, ctx=gpu_ctx)
    r = np.random.default_rng(sum(shape)).standard_normal(nt * n1 * n2)
    assert rel(pc.solve(r), spatial_precond_solve(shape, ly, lx, r)) < TOL


@pytest.mark.parametrize("shape", SHAPES)
def test_c1_matvec_vs_port(gpu_ctx, port, shape):
    from paper_1907_13428_b200 import ConstraintOperator
    time, ty, tx = _factors(port, shape)
    op = ConstraintOperator(time, ty, tx, -1.0, ctx=gpu_ctx)
    pop = port.op(shape, time, ty, tx, -1.0)
    x = np.random.default_rng(3 + sum(shape)).standard_normal(op.size)
    assert rel(op.apply(x), pop.apply(x)) < TOL


def test_c1_assemble_matches_eigs(gpu_ctx, ref):
    """assemble_spatial_precond(op) (host T. Chan of the operator's factors)
    equals the preconditioner built from the reference's T. Chan spectra."""
    from paper_1907_13428_b200 import SpatialPreconditioner, make_c1
    shape = (2, 45, 33)
    op, pc = make_c1(shape, ctx=gpu_ctx)
    cy, ry = ref.build_riesz(1.7, 45, 1.0 / 46)
    cx, rx = ref.build_riesz(1.3, 33, 1.0 / 34)
    pc2 = SpatialPreconditioner.from_eigs(2, ref.tchan(cy, ry)[1], ref.tchan(cx, rx)[1], ctx=gpu_ctx)
    r = np.random.default_rng(5).standard_normal(op.size)
    assert rel(pc.solve(r), pc2.solve(r)) < 1e-13


def test_c1_precond_inverts_circulant(gpu_ctx, ref):
    """z = C2^-1 r: applying the 2-level circulant (numpy) to z gives r back."""
    from oracle.pyoracle import circulant_dense
    from paper_1907_13428_b200 import SpatialPreconditioner
    nt, n1, n2 = 2, 24, 19
    cy, ry = ref.build_riesz(1.7, n1, 1.0 / (n1 + 1))
    cx, rx = ref.build_riesz(1.3, n2, 1.0 / (n2 + 1))
    fy, ly = ref.tchan(cy, ry)
    fx, lx = ref.tchan(cx, rx)
    A2 = np.kron(circulant_dense(fy), np.eye(n2)) + np.kron(np.eye(n1), circulant_dense(fx))
    r = np.random.default_rng(9).standard_normal(nt * n1 * n2)
    z = SpatialPreconditioner.from_eigs(nt, ly, lx, ctx=gpu_ctx).solve(r)
    back = np.concatenate([A2 @ z[k * n1 * n2:(k + 1) * n1 * n2] for k in range(nt)])
    assert rel(back, r) < TOL


def test_c1_full_size_slices(gpu_ctx, port):
    """Full C1 (256 x 1023 x 1023, N = 268M): the slices are independent for
    both operations, so slices 0, 127 and 255 of the full-size GPU results are
    checked against the oracle run on those slices alone."""
    import torch
    from oracle.pyoracle import spatial_precond_solve
    from paper_1907_13428_b200 import make_c1, randn
    op, pc = make_c1(ctx=gpu_ctx)
    nt, n1, n2 = op.shape
    S = n1 * n2
    x = torch.from_numpy(randn(1, op.size)).cuda()
    ax = torch.empty_like(x)
    z = torch.empty_like(x)
    torch.cuda.synchronize()
    op.apply_dev(x, ax)
    pc.solve_dev(x, z)
    gpu_ctx.synchronize()
    time, ty, tx = _factors(port, (1, n1, n2))
    pop = port.op((1, n1, n2), time, ty, tx, -1.0)
    _, ly = port.tchan(*ty)
    _, lx = port.tchan(*tx)
    for k in (0, 127, 255):
        xs = x[k * S:(k + 1) * S].cpu().numpy()
        assert rel(ax[k * S:(k + 1) * S].cpu().numpy(), pop.apply(xs)) < TOL
        assert rel(z[k * S:(k + 1) * S].cpu().numpy(), spatial_precond_solve((1, n1, n2), ly, lx, xs)) < TOL
