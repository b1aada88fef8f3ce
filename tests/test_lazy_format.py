"""CPU tests for SURVEY.md §8(f) row 4: the reference's binary Tucker format
(save_tucker / load_tucker, src/tucker.cpp:329-383) in the host mirror, and the
oracle's Lazy rounding (tucker_rounding, src/tucker.cpp:285-296) checked against
the reference's own assertions (proj/tests/test_tucker_core.cpp)."""
import io
import struct

import numpy as np
import pytest

import oracle as O
from helpers import dense_rel_error, random_tucker
from paper_2603_13532_b200 import tucksum as T


def test_serialization_round_trip():
    """test_tucker_core.cpp:260-277."""
    x = random_tucker([5, 4, 3], [2, 2, 2], (34, 0))
    y = random_tucker([5, 4, 3], [1, 2, 1], (34, 1))
    s = T.tucker_axby(1.0, x, 2.0, y)
    buf = io.BytesIO()
    T.save_tucker(buf, s)
    buf.seek(0)
    back = T.load_tucker(buf)
    assert back.dims == s.dims and back.ranks == s.ranks and len(back.blocks) == len(s.blocks)
    for a, b in zip(back.factors, s.factors):
        assert np.array_equal(a, b)
    for a, b in zip(back.blocks, s.blocks):
        assert list(a.offsets) == list(b.offsets) and np.array_equal(a.data, b.data)


def test_serialization_byte_layout_and_truncation(tmp_path):
    """src/tucker.cpp:329-352 field order, little-endian u64 / f64; truncated streams raise."""
    x = T.TuckerTensor(np.arange(4.0).reshape((2, 2), order="F"), [np.eye(3)[:, :2], np.ones((2, 2))])
    path = tmp_path / "x.tucker"
    T.save_tucker(str(path), x)
    raw = path.read_bytes()
    head = struct.unpack("<5Q", raw[:40])
    assert head == (2, 3, 2, 2, 2)  # order, dims, ranks
    f0 = np.frombuffer(raw[40:88], dtype="<f8")
    assert np.array_equal(f0, np.eye(3)[:, :2].ravel(order="F"))
    assert struct.unpack("<Q", raw[120:128])[0] == 1  # one block
    assert struct.unpack("<4Q", raw[128:160]) == (0, 0, 2, 2)
    assert np.array_equal(np.frombuffer(raw[160:], dtype="<f8"), np.arange(4.0))
    assert len(raw) == 160 + 32
    back = T.load_tucker(str(path))
    assert np.array_equal(back.dense_core(), x.dense_core())
    with pytest.raises(RuntimeError):
        T.load_tucker(io.BytesIO(raw[:-8]))
    with pytest.raises(RuntimeError):
        T.load_tucker(io.BytesIO(struct.pack("<Q", 0)))


def test_oracle_rounding_honors_budget():
    """test_tucker_core.cpp:208-220."""
    x = random_tucker([8, 7, 6], [5, 4, 5], (29, 0))
    dense = O.reconstruct(x)
    for tau in (1e-1, 1e-4, 1e-8):
        r = O.lazy_sum([x], [1.0], tau)
        assert np.linalg.norm(O.reconstruct(r) - dense) <= tau * np.linalg.norm(dense) + 1e-13 * np.linalg.norm(dense)
        for u in r.factors:
            assert np.linalg.norm(u.T @ u - np.eye(u.shape[1])) <= 1e-12


def test_oracle_rounding_recovers_copies_and_floor():
    """test_tucker_core.cpp:222-251."""
    x = random_tucker([9, 8, 7], [3, 2, 4], (30, 0))
    r = O.lazy_sum([x] * 4, [0.25] * 4, 1e-10)
    assert r.ranks == x.ranks
    assert O.rel_error_to_sum(r, [x], [1.0]) <= 1e-9
    u0 = O.gaussian_matrix(6, 2, (31, 0))
    f = [np.concatenate([u0, u0[:, :1]], axis=1), O.gaussian_matrix(5, 2, (31, 1)), O.gaussian_matrix(4, 2, (31, 2))]
    core = O.gaussian_matrix(12, 1, (31, 3))[:, 0].reshape((3, 2, 2), order="F")
    y = T.TuckerTensor(core, f)
    r = O.lazy_sum([y], [1.0], 0.0)
    assert r.ranks == [2, 2, 2]
    assert O.rel_error_to_sum(r, [y], [1.0]) <= 1e-12
    zero = T.TuckerTensor(np.zeros((2, 2)), [O.gaussian_matrix(4, 2, (32, 0)), O.gaussian_matrix(3, 2, (32, 1))])
    r = O.lazy_sum([zero], [1.0], 1e-6)
    assert r.ranks == [1, 1]
    assert O.tucker_norm(r) == 0.0


def test_oracle_lazy_random_sums():
    """test_sketch_sum.cpp:266-299 (Lazy branch, ≤ 1e-6)."""
    from helpers import dense_weighted_sum

    rng = np.random.Generator(np.random.MT19937(907))
    for trial in range(10):
        xs, ws = [], []
        for i in range(5):
            ranks = [int(v) for v in rng.integers(1, 4, size=3)]
            xs.append(random_tucker([14, 11, 9], ranks, (1000 + trial, i)))
            ws.append((1.0 if rng.integers(0, 2) == 0 else -1.0) * rng.uniform(0.5, 2.0))
        assert dense_rel_error(O.lazy_sum(xs, ws, 1e-6), dense_weighted_sum(xs, ws)) <= 1e-6
