"""dt_matmul / core.matmul (core.py:63-77) on the any-major tcgen05 GEMM (k_tc_xgemm.cu).

Every operand order the backward uses (plain, aᵀ, bᵀ, both) in tf32 and bf16, ragged shapes,
split-K, against f64 products of the same inputs (bf16: the bf16-rounded inputs, exact products
and fp32 sums -> <= 1e-4; tf32: inputs truncated to 10-bit mantissas -> <= 3e-3 of max|e|, the
reference's rel_error metric). Plus the reference's DimensionError text and determinism."""

import numpy as np
import pytest
import torch

from oracle import deepthin_oracle as O

import paper_1802_06944_b200 as D
from paper_1802_06944_b200.core import matmul

pytestmark = pytest.mark.gpu


def operand(rows, cols, trans, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if trans:  # a transposed view of a row-major (cols x rows) buffer
        return torch.randn(cols, rows, device="cuda", generator=g).to(dtype).t()
    return torch.randn(rows, cols, device="cuda", generator=g).to(dtype)


@pytest.mark.parametrize("mma", ["tf32", "bf16"])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("shape", [(300, 200, 1000), (1024, 512, 4096), (256, 24, 2816),
                                   (128, 1024, 65536), (64, 64, 64)])
def test_matmul_orders_and_shapes(mma, ta, tb, shape):
    M, N, K = shape
    dt = torch.float32 if mma == "tf32" else torch.bfloat16
    a = operand(M, K, ta, dt, 1)
    b = operand(K, N, tb, dt, 2)
    c = matmul(a, b, mma=mma)
    assert c.shape == (M, N) and c.dtype == torch.float32
    want = a.double().cpu().numpy() @ b.double().cpu().numpy()
    err = O.rel_error(c.double().cpu().numpy(), want)
    assert err <= (3e-3 if mma == "tf32" else 1e-4), (mma, ta, tb, shape, err)
    c2 = matmul(a, b, mma=mma)
    assert torch.equal(c, c2)  # fixed-order split-K: bitwise repeatable


def test_matmul_shape_error_and_numpy():
    with pytest.raises(D.DimensionError, match="cannot multiply 3x4 by 5x2"):
        matmul(np.zeros((3, 4)), np.zeros((5, 2)))
    a = np.random.default_rng(0).standard_normal((33, 17))
    b = np.random.default_rng(1).standard_normal((17, 9))
    got = matmul(a, b)
    assert isinstance(got, np.ndarray) and got.shape == (33, 9)
    assert O.rel_error(got, a @ b) <= 3e-3
