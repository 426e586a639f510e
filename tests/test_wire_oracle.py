"""CPU: the oracle's restatement of the COO wire codec (okt_oracle.c,
sparse.cpp:275-312) against the reference's own wire_encode / wire_decode
(oracle/_ref/libokref.so): the documented layout case and the malformed
buffers of test_sparse_core.cpp:200-225, and random images."""
import numpy as np
import pytest


def test_documented_layout(oracle, reference):
    want = bytes([2, 0, 0, 0, 3, 0, 0, 0, 7, 0, 0, 0, 0x00, 0x00, 0xc0, 0x3f, 0x00, 0x00, 0x00, 0xc0])
    for impl in (oracle, reference):
        assert impl.wire_encode(np.array([3, 7]), np.array([1.5, -2.0])) == want
        idx, val = impl.wire_decode(want, 32)
        assert list(idx) == [3, 7] and list(val) == [1.5, -2.0]


def test_malformed_buffers(oracle, reference):
    good = oracle.wire_encode(np.array([1]), np.array([4.0]))
    for impl in (oracle, reference):
        assert impl.wire_decode(good[:-1], 8) is None          # truncated
        assert impl.wire_decode(good + b"\0", 8) is None        # trailing byte
        assert impl.wire_decode(bytes([1, 2]), 8) is None       # no header
        assert impl.wire_decode(good, 1) is None                # index >= n
        bad_order = impl.wire_encode(np.array([5, 5]), np.array([1.0, 2.0]))
        assert impl.wire_decode(bad_order, 8) is None           # not strictly increasing
        empty = impl.wire_decode(bytes(4), 8)                  # nnz = 0 is a valid image
        assert empty is not None and len(empty[0]) == 0


@pytest.mark.parametrize("seed", range(5))
def test_random_images_match_reference(oracle, reference, seed):
    rng = np.random.default_rng(seed)
    n = 100_000
    idx = np.sort(rng.choice(n, 1000, replace=False)).astype(np.uint32)
    val = rng.standard_normal(1000) * 10.0 ** rng.integers(-30, 30, 1000)  # not fp32-exact: rounding path
    a, b = oracle.wire_encode(idx, val), reference.wire_encode(idx, val)
    assert a == b
    ia, va = oracle.wire_decode(a, n)
    ib, vb = reference.wire_decode(b, n)
    assert np.array_equal(ia, ib) and np.array_equal(va, vb)
