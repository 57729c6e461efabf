"""The seeded generator: numpy (uint64) and torch (int64 wraparound) implementations agree bit for bit."""
import numpy as np
import torch

import synth


def test_hash_numpy_torch_identical():
    idx = np.concatenate([np.arange(0, 5000), np.array([2**31 - 1, 2**31, 2**32 + 7, 2_097_151_999, 2**40 + 3])])
    for seed in (0, 1, 4, 123456789):
        for stream in (synth.STREAM_X, synth.STREAM_J):
            a = synth.hash_uniform_np(seed, stream, idx.astype(np.uint64))
            b = synth.hash_uniform_torch(seed, stream, torch.from_numpy(idx.astype(np.int64))).numpy()
            assert np.array_equal(a, b)
            assert a.min() >= 0.0 and a.max() < 1.0


def test_x_and_jac_draws():
    w = synth.CONFIGS[2]
    x = synth.x_np(w, 1000, 500)
    xt = synth.x_torch(w, 1000, 500).numpy()
    assert np.array_equal(x, xt)
    assert x.min() >= -1 and x.max() < 1
    cells = np.array([0, 1, w.plane_cells, w.plane_cells * 3 + 17])
    J = synth.jac_cells_np(w, cells)
    Jt = synth.jac_planes_torch(w, 0, 4).numpy()[cells]
    assert np.array_equal(J, Jt)
    h = 1.0 / 64
    E = J.reshape(-1, 3, 3) / h - np.eye(3)
    assert np.abs(E).max() <= 0.1 and np.abs(E).max() > 0.05
    xb = synth.x_cells_np(w, cells)
    n3 = w.n ** 3
    for i, c in enumerate(cells):
        assert np.array_equal(xb[i], synth.x_np(w, int(c) * n3, n3))


def test_wrap_planes_and_sample():
    w = synth.CONFIGS[3]
    Jt = synth.jac_planes_torch(w, -1, 2)          # planes N0-1 and 0
    assert Jt.shape == (2 * w.plane_cells, 9)
    s = synth.sample_cells(w, nrandom=100, plane_cap=64, wrap_plane_cells=32)
    assert s.min() >= 0 and s.max() < w.ncells and len(np.unique(s)) == len(s)
