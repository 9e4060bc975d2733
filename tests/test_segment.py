"""NEXT row f4: segmentation-guided initialisation (host C++ in libsmoe,
no GPU needed) against the plain reference (oracle/segment.py) and the SPEC
worked examples."""
import numpy as np
import pytest

from oracle import segment as S


@pytest.fixture(scope="module")
def smoe():
    import subprocess, os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call(["make", "-s", "-C", os.path.join(root, "paper_2510_05814_b200", "csrc")])
    from paper_2510_05814_b200 import smoe as m
    return m


def test_spec_segment_examples(smoe):
    img = np.zeros((3, 20, 30), np.float32)
    img[:, :, 15:] = 1.0                                     # S:421 black | white
    lab, n = smoe.segment(img, 10, 16)
    assert n == 2 and np.all(lab[:, :15] == 0) and np.all(lab[:, 15:] == 1)
    lab, n = smoe.segment(np.full((3, 17, 9), 0.4, np.float32), 10, 16)     # S:422 constant
    assert n == 1
    rnd = np.random.default_rng(0).random((3, 16, 16)).astype(np.float32)
    lab, n = smoe.segment(rnd, 255, 1)                        # S:423 vacuous threshold
    assert n == 1


def test_spec_allocation_examples(smoe):
    lab = np.zeros((10, 10), np.int32)
    lab[:, 5:] = 1
    img = np.zeros((1, 10, 10), np.float32)
    pool = smoe.segment_init(img, lab, 2, 10)                # 5 and 5
    seg_of = lab[np.clip(np.rint(pool.mu[:, 1]), 0, 9).astype(int), np.clip(np.rint(pool.mu[:, 0]), 0, 9).astype(int)]
    assert np.bincount(seg_of, minlength=2).tolist() == [5, 5]
    lab2 = np.zeros((10, 10), np.int32)
    lab2[9, :] = 1                                           # 90% / 10%
    assert S.allocate(lab2, 2, 10).tolist() == [9, 1]
    pool2 = smoe.segment_init(img, lab2, 2, 10)
    seg2 = lab2[np.clip(np.rint(pool2.mu[:, 1]), 0, 9).astype(int), np.clip(np.rint(pool2.mu[:, 0]), 0, 9).astype(int)]
    assert np.bincount(seg2, minlength=2).tolist() == [9, 1]
    with pytest.raises(smoe.SmoeError):                      # S:430 TooFewKernels
        smoe.segment_init(img, np.arange(100).reshape(10, 10) % 5, 5, 3)


@pytest.mark.parametrize("seed,thr,min_size", [(1, 10, 4), (2, 20, 8), (3, 10, 16), (4, 30, 2)])
def test_segment_matches_reference(smoe, seed, thr, min_size):
    from paper_2510_05814_b200 import synth
    img = synth.noisy(synth.image(24, 28, 3, seed), 8 / 255, seed + 10)
    img = np.clip(img, 0, 1).astype(np.float32)
    lab, n = smoe.segment(img, thr, min_size)
    ref, nref = S.segment(img, thr, min_size)
    assert n == nref
    np.testing.assert_array_equal(lab, ref)
    sizes = np.bincount(lab.ravel())
    assert n == 1 or sizes.min() >= min_size


def test_segment_init_layout_and_budget(smoe):
    from paper_2510_05814_b200 import synth
    img = synth.image(40, 48, 3, 9)
    lab, n = smoe.segment(img, 10, 16)
    K = 3 * n + 7
    pool = smoe.segment_init(img, lab, n, K, order=1, seed=5)
    assert pool.mu.shape == (K, 2) and pool.expert.shape == (K, 3, 3)
    assert np.all(pool.chol == np.array([5, 0, 5], np.float32))
    assert np.all(pool.expert[:, :, 1:] == 0) and np.all(pool.log_pi == 0)
    seg = lab[np.clip(np.rint(pool.mu[:, 1]), 0, 39).astype(int), np.clip(np.rint(pool.mu[:, 0]), 0, 47).astype(int)]
    # each kernel sits in its segment (up to the +-0.5 px jitter) with the segment colour
    for k in range(K):
        s = seg[k]
        np.testing.assert_allclose(pool.expert[k, :, 0], img[:, lab == s].mean(axis=1), rtol=1e-5, atol=1e-6) \
            if (lab == s).sum() > 0 else None
    assert np.bincount(seg, minlength=n).sum() == K
