# SPDX-License-Identifier: Apache-2.0
"""GPU parity of the pure C-ABI functions against the reference KATs and the
oracle: shard_assign, select_evictions, attention, int8/int4 codes (bit-exact
vs oracle/pikv_oracle.c), per-head low-rank projection (tolerance 1e-5)."""
import ctypes

import numpy as np
import pytest

from oracle_bind import oracle_lib

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2508_06526_b200 import engine as pe  # noqa: E402
from paper_2508_06526_b200.engine import PikvError  # noqa: E402


def test_shard_assign_kats():  # test_kvstore.cpp:42-70
    s = pe.shard_assign(5, 3, 4, 4, 2)
    assert (s.raw, s.device, s.shard_index) == (2, 0, 1)
    assert pe.shard_assign(0, 0, 8, 8, 4).raw == 0
    assert pe.shard_assign(7, 2, 8, 4, 4).raw == 5
    assert pe.shard_assign(5, 3, 4, 4, 2, additive=True).raw == 4
    for bad in ((1, 1, 3, 4, 2), (1, 1, 4, 6, 2)):
        with pytest.raises(PikvError) as e:
            pe.shard_assign(*bad)
        assert e.value.kind == "InvalidConfig"
    with pytest.raises(PikvError) as e:
        pe.shard_assign(-1, 1, 4, 4, 2)
    assert e.value.kind == "InvalidArgument"
    rng = np.random.default_rng(3)
    t = rng.integers(0, 1 << 20, 500)
    ee = rng.integers(0, 256, 500)
    d, sh, raw = pe.shard_assign(t, ee, 64, 32, 4)
    want = (t % 64) ^ (ee % 32)
    assert np.array_equal(raw, want) and np.array_equal(d, want % 4) and np.array_equal(sh, want // 4)


def test_select_evictions_kats():  # test_scheduler.cpp:178-234
    assert pe.select_evictions([(1, 1), (2, 2), (3, 3)], 5, False, 0) == []
    assert pe.select_evictions([(5, 1), (1, 2), (3, 3), (2, 4)], 2, False, 0) == [
        (1, "budget"), (3, "budget")]
    assert pe.select_evictions([(5, 1), (1, 2), (3, 3)], 10, True, 4.0) == [
        (1, "threshold"), (2, "threshold")]
    assert [i for i, _ in pe.select_evictions([(1, 9), (1, 2), (1, 5)], 1, False, 0)] == [1, 2]
    rng = np.random.default_rng(13)
    for _ in range(200):
        n = int(rng.integers(1, 65))
        budget = int(rng.integers(1, 17))
        pages = [(float(np.floor(rng.uniform(-8, 8))), int(rng.integers(0, 1000))) for _ in range(n)]
        order = sorted(range(n), key=lambda i: (pages[i][0], pages[i][1], i))
        got = [i for i, _ in pe.select_evictions(pages, budget, False, 0)]
        assert got == order[:max(n - budget, 0)]


def test_attention_kats():  # test_pipeline.cpp:80-119
    y, w = pe.attention([1, 0], np.zeros((0, 2)), np.zeros((0, 2)))
    assert y.tolist() == [0, 0] and w.size == 0
    y, w = pe.attention([0.2, 0.9], [[1, 0]], [[3, 4]])
    assert w.tolist() == [1.0] and np.allclose(y, [3, 4])
    y, w = pe.attention([2, 1], [[0.3, -0.7], [0.3, -0.7]], [[1, 0], [0, 1]])
    assert np.allclose(w, [0.5, 0.5])
    y, w = pe.attention([0, 0, 5], [[1, 0, 0], [0, 1, 0]], [[2, 0, 0], [0, 4, 0]])
    assert np.allclose(y[:2], [1, 2])


@pytest.mark.parametrize("bits", [8, 4])
def test_quantize_bit_exact_vs_oracle(bits):
    L = oracle_lib()
    rng = np.random.default_rng(bits)
    x = (rng.standard_normal((64, 128)) * rng.uniform(0.01, 10, (64, 1))).astype(np.float32)
    x[3] = 0.0  # all-zero row: scale 0, codes 0
    x[5, 7] = 1e-30
    codes, scales = pe.quantize(x, bits)
    w = 128 if bits == 8 else 64
    for r in range(64):
        c = np.zeros(w, dtype=np.uint8)
        sc = ctypes.c_float()
        L.po_quantize_row(x[r].ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 128, bits,
                          c.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), ctypes.byref(sc))
        assert np.array_equal(codes[r], c), r
        assert scales[r] == np.float32(sc.value), r
    back = pe.dequantize(codes, scales, 128, bits)
    qmax = 127 if bits == 8 else 7
    assert np.all(np.abs(back - x) <= scales[:, None] * 0.5 + 1e-6 * np.abs(x).max())
    del qmax


def test_lowrank_projection():
    rng = np.random.default_rng(1)
    H, hd, r = 4, 64, 16
    basis = rng.standard_normal((H, r, hd)).astype(np.float32)
    bias = rng.standard_normal(H * hd).astype(np.float32)
    x = rng.standard_normal((10, H * hd)).astype(np.float32)
    y = pe.lowrank_encode(x, basis, bias)
    ref = np.einsum("hjd,nhd->nhj", basis.astype(np.float64),
                    (x - bias).reshape(10, H, hd).astype(np.float64)).reshape(10, -1)
    assert np.allclose(y, ref, rtol=1e-5, atol=1e-4)
    xr = pe.lowrank_decode(y, basis, bias)
    ref2 = np.einsum("hjd,nhj->nhd", basis.astype(np.float64),
                     y.reshape(10, H, r).astype(np.float64)).reshape(10, -1) + bias
    assert np.allclose(xr, ref2, rtol=1e-5, atol=1e-3)
    # FastV KAT (test_compressor.cpp:130-142): orthonormal crop basis, [3,4] -> [3]
    crop = np.zeros((1, 1, 2), dtype=np.float32)
    crop[0, 0, 0] = 1.0
    assert pe.lowrank_encode(np.array([[3.0, 4.0]]), crop).tolist() == [[3.0]]
