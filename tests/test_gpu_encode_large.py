"""GPU parity of the large-image encode path (C*H*W > 16384, readings R1/R2, R36): two radix
levels, pass 3 (latencies of every element outside the cut prefixes + the candidates), the per-image
finish, and the device-gated level 2-4 fallback for images with more than kEncCandCap candidates.
Bit-exact against the oracle's encode, planar and channels-last outputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_1903_02440_b200 import build, snn
    build.build()
    snn.lib()
    return snn


def _check(G, orc, x, T, bins=0, nhwc=False, xt=None):
    got = G.encode(xt if xt is not None else torch.from_numpy(x).cuda(), T, bins=bins, nhwc=nhwc).cpu().numpy()
    ref = orc.encode(x, T, bins=bins) if bins else orc.encode(x, T)
    if nhwc:
        ref = ref.transpose(0, 2, 3, 1)
    assert np.array_equal(got, ref)


def _continuous(rng, shape, zero=0.5):
    x = rng.random(shape, dtype=np.float32)
    x[rng.random(shape) < zero] = 0
    return x


@pytest.mark.parametrize("nhwc", [False, True])
@pytest.mark.parametrize("shape,T", [((2, 32, 64, 64), 32), ((2, 8, 45, 47), 15), ((3, 4, 160, 250), 30),
                                     ((1, 1, 1, 16387), 254), ((2, 300, 8, 8), 12)])
def test_encode_large_continuous(G, orc, shape, T, nhwc):
    rng = np.random.default_rng(sum(shape) + T)
    x = _continuous(rng, shape)
    x.reshape(-1)[5::211] = -0.5
    x.reshape(-1)[7] = np.nan
    _check(G, orc, x, T, nhwc=nhwc)


@pytest.mark.parametrize("nhwc", [False, True])
@pytest.mark.parametrize("T", [1, 15, 254])
def test_encode_large_all_equal_fallback(G, orc, T, nhwc):
    """every positive value equal: one prefix holds the whole image (candidate overflow -> levels 2-4)"""
    x = np.full((2, 4, 100, 100), 0.375, np.float32)
    x[1, :, ::3] = 0
    _check(G, orc, x, T, nhwc=nhwc)


@pytest.mark.parametrize("nhwc", [False, True])
def test_encode_large_mixed_batch(G, orc, nhwc):
    """one image finishes from its candidates, the next overflows: the fallback is gated per image"""
    rng = np.random.default_rng(3)
    x = _continuous(rng, (3, 6, 80, 90), 0.3)
    x[1] = (rng.integers(0, 3, size=x[1].shape) / 2).astype(np.float32)
    _check(G, orc, x, 32, nhwc=nhwc)


@pytest.mark.parametrize("bins", [1, 2])
def test_encode_large_bins(G, orc, bins):
    rng = np.random.default_rng(bins)
    x = _continuous(rng, (2, 16, 50, 60))
    _check(G, orc, x, 30, bins=bins)
    _check(G, orc, x, 30, bins=bins, nhwc=True)


def test_encode_large_misaligned_and_repeated(G, orc):
    """a view at a 4-byte (not 16-byte) offset takes the scalar loads; two calls in a row (state reset)"""
    rng = np.random.default_rng(9)
    x = _continuous(rng, (2, 8, 48, 64))
    flat = torch.zeros(x.size + 1, dtype=torch.float32, device="cuda")
    flat[1:] = torch.from_numpy(x.reshape(-1)).cuda()
    xt = flat[1:].view(x.shape)
    _check(G, orc, x, 32, xt=xt)
    _check(G, orc, x, 32, xt=xt, nhwc=True)
    _check(G, orc, x, 32)


def test_encode_large_forced_all_levels(G, orc, monkeypatch):
    monkeypatch.setenv("SNN_ENCODE_LEVELS", "5")
    rng = np.random.default_rng(4)
    x = _continuous(rng, (2, 32, 40, 40))
    _check(G, orc, x, 32)
    _check(G, orc, x, 32, nhwc=True)
