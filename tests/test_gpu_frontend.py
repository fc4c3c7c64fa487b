"""GPU parity of the f2 front end (snn_filter_bank, snn_local_norm, snn_lateral_inhibition) against the
CPU oracle, bit-exact (R33-R35 fix the arithmetic order; the kernels use explicitly rounded
operations).  Sizes span several 8 x 32 tiles with ragged tails; edge cases: B = 0, S = 1, a window
larger than the image, all-equal intensities (ties), zero images, n = 0."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1903_02440_b200 import build, snn
    build.build()
    snn.lib()
    return snn


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


FB_CASES = [  # (images, bank, pad, mode, threshold)
    ("stroke", 6, "dog", 3, 1, float("-inf")),
    ("stroke", 3, "gabor", 2, 2, float("-inf")),
    ("shape", 2, "gabor", 2, 2, float("-inf")),
    ("rand37x45", 3, "rand5", 0, 0, 0.25),
    ("rand37x45", 2, "rand1", 0, 0, float("-inf")),
    ("rand37x45", 2, "rand5", 4, 1, float("-inf")),
    ("zero", 2, "dog", 3, 1, float("-inf")),
]


def _images(kind, n, seed=5):
    if kind == "stroke":
        return synth.stroke_images(seed, n)
    if kind == "shape":
        return synth.shape_images(seed, n)
    if kind == "zero":
        return np.zeros((n, 28, 28))
    return np.random.default_rng(seed).random((n, 37, 45))


def _bank(kind):
    rng = np.random.default_rng(9)
    return {"dog": synth.dog_bank(), "gabor": synth.gabor_bank(), "rand5": rng.standard_normal((3, 5, 5)),
            "rand1": rng.standard_normal((2, 1, 1))}[kind]


@pytest.mark.parametrize("case", FB_CASES, ids=[f"{c[0]}-{c[2]}-m{c[4]}" for c in FB_CASES])
def test_filter_bank(G, case):
    kind, n, bank, pad, mode, thr = case
    img, ker = _images(kind, n), _bank(bank)
    ref = oracle.filter_bank(img, ker, pad, mode=mode, threshold=thr)
    got = G.filter_bank(cu(img), cu(ker), pad, mode=mode, threshold=thr).cpu().numpy()
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_filter_bank_empty_and_errors(G):
    ker = cu(synth.dog_bank())
    out = G.filter_bank(torch.zeros((0, 28, 28), dtype=torch.float64, device="cuda"), ker, 3, mode=1)
    assert out.shape == (0, 6, 28, 28)
    with pytest.raises(G.SNNError):
        G.filter_bank(cu(np.zeros((1, 8, 8))), ker, 3, mode=3)
    with pytest.raises(G.SNNError):
        G.filter_bank(cu(np.zeros((1, 4, 4))), ker, 0, mode=1)  # 7x7 kernel on an unpadded 4x4 image


LN_CASES = [("rand", (2, 3, 37, 45), 2), ("rand", (1, 2, 160, 250), 8), ("rand", (1, 1, 5, 6), 7),
            ("rand", (2, 2, 17, 33), 0), ("zero", (1, 2, 9, 9), 1), ("dog", (4, 6, 28, 28), 3)]


def _planes(kind, shape, seed=3):
    rng = np.random.default_rng(seed)
    if kind == "zero":
        return np.zeros(shape, np.float32)
    if kind == "dog":
        return synth._dog_input(seed, shape[0])
    if kind == "ties":
        return (rng.integers(0, 5, shape) / 4.0).astype(np.float32)
    return rng.random(shape).astype(np.float32)


@pytest.mark.parametrize("case", LN_CASES, ids=[f"{c[0]}-{'x'.join(map(str, c[1]))}-r{c[2]}" for c in LN_CASES])
def test_local_norm(G, case):
    kind, shape, radius = case
    x = _planes(kind, shape)
    ref = oracle.local_norm(x, radius)
    got = G.local_norm(cu(x), radius).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


LI_CASES = [("ties", (2, 3, 37, 45), [0.5, 0.8]), ("rand", (1, 2, 160, 250), [0.3, 0.5, 0.7, 0.9]),
            ("ties", (1, 1, 3, 3), [0.5, 0.6, 0.7, 0.8, 0.9]), ("rand", (2, 2, 17, 33), []),
            ("dog", (4, 6, 28, 28), [0.4]), ("zero", (1, 1, 9, 40), [0.5])]


@pytest.mark.parametrize("case", LI_CASES, ids=[f"{c[0]}-{'x'.join(map(str, c[1]))}-n{len(c[2])}" for c in LI_CASES])
def test_lateral_inhibition(G, case):
    kind, shape, factors = case
    x = _planes(kind, shape)
    ref = oracle.lateral_inhibition(x, factors)
    got = G.lateral_inhibition(cu(x), cu(np.asarray(factors, np.float32))).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_front_chain_then_encode(G):
    """filter bank -> local norm -> lateral inhibition -> encode, all on the GPU, equals the oracle chain."""
    img = synth.stroke_images(21, 8)
    ker = synth.dog_bank()
    x = oracle.lateral_inhibition(oracle.local_norm(oracle.filter_bank(img, ker, 3, mode=1), 2), [0.5, 0.75])
    ref = oracle.encode(x, 15)
    g = G.lateral_inhibition(G.local_norm(G.filter_bank(cu(img), cu(ker), 3, mode=1), 2),
                             cu(np.asarray([0.5, 0.75], np.float32)))
    assert np.array_equal(G.encode(g, 15).cpu().numpy(), ref)
