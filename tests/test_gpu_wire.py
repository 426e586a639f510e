"""GPU: the COO wire codec (okt_wire_encode / okt_wire_decode, the
reference's sparse.cpp:275-312) against the reference's own wire_encode /
wire_decode: byte-identical images, identical decodes, the same rejections
(test_sparse_core.cpp:200-225), at up to the allreduce's u sizes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def okm(gpus):
    from paper_2201_07598_b200 import oktopk
    return oktopk


def test_documented_layout(okm):
    s = okm.SparseGrad(32, np.array([3, 7], np.uint32), np.array([1.5, -2.0]))
    b = okm.wire_encode(s)
    assert b == bytes([2, 0, 0, 0, 3, 0, 0, 0, 7, 0, 0, 0, 0, 0, 0xc0, 0x3f, 0, 0, 0, 0xc0])
    back = okm.wire_decode(b, 32)
    assert back == s


def test_rejects_malformed(okm):
    good = okm.wire_encode(okm.SparseGrad(8, np.array([1], np.uint32), np.array([4.0])))
    for bad, n in ((good[:-1], 8), (good + b"\0", 8), (bytes([1, 2]), 8), (good, 1)):
        with pytest.raises(okm.DecodeError):
            okm.wire_decode(bad, n)
    twice = okm.wire_encode(okm.SparseGrad(8, np.array([5, 5], np.uint32), np.array([1.0, 2.0])))
    with pytest.raises(okm.DecodeError):
        okm.wire_decode(twice, 8)
    assert okm.wire_decode(bytes(4), 8).nnz() == 0


@pytest.mark.parametrize("nnz", [1, 1000, 147_283, 1_000_000])
def test_matches_reference(okm, reference, nnz):
    rng = np.random.default_rng(nnz)
    n = max(4 * nnz, 64)
    idx = np.sort(rng.choice(n, nnz, replace=False)).astype(np.uint32)
    val = rng.standard_normal(nnz) * 10.0 ** rng.integers(-40, 40, nnz)  # fp64 values: exercises the f32 rounding
    b = okm.wire_encode(okm.SparseGrad(n, idx, val))
    assert b == reference.wire_encode(idx, val)
    back = okm.wire_decode(b, n)
    ri, rv = reference.wire_decode(b, n)
    assert np.array_equal(back.indices, ri) and np.array_equal(back.values, rv)
