"""GPU parity of the raw operators through the C ABI against the oracle and
exact integer references (restating proj/tests/test_quant.cpp and
test_tensor.cpp). int8: bit-exact. fp32 (3xTF32): 2e-5 relative to the
largest output. bf16: 1e-2 relative."""

import numpy as np
import pytest

import oracle_lib as o
import paper_2008_04885_b200 as mt

pytestmark = pytest.mark.gpu


def int32_ref(qa, sa, qb, sb):
    return (qa.astype(np.int64) @ qb.astype(np.int64)).astype(np.float32) * (
        np.float32(1.0) / (np.float32(sa) * np.float32(sb)))


@pytest.mark.parametrize("x", [[2.0, -2.0, 1.0], [0.0, 0.0], [1.0], [127.0, 0.5, -0.5]])
def test_quantize_kats(x):  # test_quant.cpp:38-64
    qg, sg = mt.quantize(np.array(x, np.float32))
    qo, so = o.quantize(np.array(x, np.float32))
    assert sg == so and np.array_equal(qg, qo)


def test_quantize_random_bit_exact():
    rng = np.random.default_rng(4)
    for shape in ((16, 16), (3, 1000), (70001,)):
        x = (rng.standard_normal(shape) * rng.uniform(0.1, 10)).astype(np.float32)
        qg, sg = mt.quantize(x)
        qo, so = o.quantize(x)
        assert sg == so and np.array_equal(qg, qo)


def test_quantize_rejects_nonfinite():
    with pytest.raises(mt.ValueError_):
        mt.quantize(np.array([1.0, np.inf], np.float32))


@pytest.mark.parametrize("m,k,n", [(3, 7, 5), (8, 64, 16), (1, 33, 17), (5, 128, 48),
                                   (320, 512, 1536), (320, 2048, 512), (1664, 512, 2048),
                                   (257, 512, 32000)])
def test_qmatmul_bit_exact(m, k, n):  # test_quant.cpp:85-100 + model shapes
    rng = np.random.default_rng(m * 7 + k + n)
    qa, sa = o.quantize(rng.uniform(-2, 2, (m, k)).astype(np.float32))
    qb, sb = o.quantize(rng.uniform(-2, 2, (k, n)).astype(np.float32))
    got = mt.qmatmul(qa, sa, qb, sb)
    assert np.array_equal(got, int32_ref(qa, sa, qb, sb))
    if m * n <= 4096:
        assert np.array_equal(got, o.qmatmul(qa, sa, qb, sb))


def test_qmatmul_nt_subset_and_errors():  # test_quant.cpp:112-138, 159-173
    rng = np.random.default_rng(35)
    qa, sa = o.quantize(rng.uniform(-2, 2, (3, 20)).astype(np.float32))
    qb, sb = o.quantize(rng.uniform(-2, 2, (12, 20)).astype(np.float32))
    full = mt.qmatmul_nt(qa, sa, qb, sb)
    assert np.array_equal(full, int32_ref(qa, sa, qb.T.copy(), sb))
    sub = [7, 0, 11, 3]
    assert np.array_equal(mt.qmatmul_nt(qa, sa, qb, sb, sub), full[:, sub])
    with pytest.raises(mt.IndexError_):
        mt.qmatmul_nt(qa, sa, qb, sb, [12])
    a = np.zeros((1, 65537), np.int8)
    with pytest.raises(mt.ValueError_):
        mt.qmatmul(a, 1.0, np.zeros((65537, 1), np.int8), 1.0)


def test_qmatmul_error_bound():  # test_quant.cpp:140-157
    rng = np.random.default_rng(36)
    for _ in range(10):
        af = rng.uniform(-3, 3, (6, 32)).astype(np.float32)
        bf = rng.uniform(-3, 3, (32, 8)).astype(np.float32)
        qa, sa = mt.quantize(af)
        qb, sb = mt.quantize(bf)
        exact = af.astype(np.float64) @ bf.astype(np.float64)
        da, db = 0.5 / sa, 0.5 / sb
        bound = 32 * (da * np.abs(bf).max() + db * np.abs(af).max() + da * db)
        assert np.all(np.abs(mt.qmatmul(qa, sa, qb, sb) - exact) <= bound * 1.0001)


def test_gemm_kats():  # test_tensor.cpp:47-64
    a = np.array([[1, 2], [3, 4]], np.float32)
    b = np.array([[5, 6], [7, 8]], np.float32)
    for prec in (mt.F32, mt.BF16):
        assert np.array_equal(mt.gemm(a, b, prec), np.array([[19, 22], [43, 50]], np.float32))
    # test_tensor.cpp:57-64 asks bit-exact identity of the CPU fp32 GEMM; the
    # 3xTF32 tensor-core path reproduces x to within 1 ulp (hi + lo summed in
    # the MMA's fp32 accumulator).
    x = np.random.default_rng(7).uniform(-3, 3, (5, 8)).astype(np.float32)
    y = mt.gemm(x, np.eye(8, dtype=np.float32), mt.F32)
    assert np.all(np.abs(y - x) <= np.spacing(np.abs(x)))


@pytest.mark.parametrize("m,k,n", [(3, 7, 5), (130, 512, 300), (320, 512, 32000), (1664, 2048, 512)])
def test_gemm_f32_and_bf16_accuracy(m, k, n):
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    want = a.astype(np.float64) @ b.astype(np.float64)
    scale = np.abs(want).max()
    assert np.abs(mt.gemm(a, b, mt.F32) - want).max() / scale < 2e-5
    assert np.abs(mt.gemm(a, b, mt.BF16) - want).max() / scale < 1e-2
