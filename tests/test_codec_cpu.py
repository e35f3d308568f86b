"""XC4 weight-unit format (K9): the C oracle round-trips every bf16 bit
pattern, the frame geometry splits units evenly over 1/2/4/8 ranks, and the
encoded size matches the format's arithmetic.  No GPU needed."""
import numpy as np
import pytest

from oracle import xc4_ref
from paper_2505_10259_b200 import codec


def _gauss_bf16(n, std=0.02, seed=0):
    x = np.random.default_rng(seed).normal(0, std, n).astype(np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)  # truncation is fine: any bit pattern must round-trip


@pytest.mark.parametrize("bits", [0, 3, 4])
@pytest.mark.parametrize("n,F", [(16, 4096), (4096, 4096), (4112, 4096), (3 * 8192 + 48, 8192),
                                 (1 << 20, 1 << 18)])
def test_oracle_round_trip_gaussian(n, F, bits):
    w = _gauss_bf16(n, seed=n)
    if bits == 3 and n % 32:
        with pytest.raises(ValueError):
            xc4_ref.encode(w, F, bits)
        return
    unit = xc4_ref.encode(w, F, bits)
    assert np.array_equal(xc4_ref.decode(unit), w)
    h = xc4_ref.header(unit)
    assert h["total_bytes"] == unit.size and h["n_frames"] == -(-n // F)
    if bits:
        assert h["version"] == (2 if bits == 3 else 1)


@pytest.mark.parametrize("bits,coded", [(4, 15), (3, 7)])
def test_oracle_round_trip_every_bit_pattern(bits, coded):
    # all 65536 patterns (NaN, ±Inf, ±0, subnormals): 256 exponents → most escape
    w = np.random.default_rng(1).permutation(np.arange(1 << 16, dtype=np.uint32)).astype(np.uint16)
    w = np.concatenate([w, w[::-1]])
    unit = xc4_ref.encode(w, 8192, bits)
    assert np.array_equal(xc4_ref.decode(unit), w)
    h = xc4_ref.header(unit)
    assert h["n_escapes"] == w.size - w.size * coded // 256  # `coded` of 256 exponents, equal counts


def test_width_choice_rule():
    # uniform exponents: 11 + 8·249/256 < 12 + 8·241/256 bits → 3-bit codes
    w = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    assert xc4_ref.header(xc4_ref.encode(w, 8192))["version"] == 2
    # 15 equally likely exponents: no 4-bit escapes, 8/15 of the weights escape at 3 bits → 4-bit codes
    e = np.repeat(np.arange(100, 115, dtype=np.uint16), 2048)
    assert xc4_ref.header(xc4_ref.encode((e << 7) | 5, 4096))["version"] == 1
    # a unit whose size is not a multiple of 32 stays 4-bit
    assert xc4_ref.header(xc4_ref.encode(_gauss_bf16(4112), 4096))["version"] == 1


def test_code_table_rule():
    # exponent counts: 130 ×3, 127 ×3 (tie → lower exponent first), 120 ×1
    def bf(e, m=0):
        return np.uint16((e << 7) | m)
    w = np.array([bf(130)] * 3 + [bf(127, 5)] * 3 + [bf(120)] + [bf(0)] * 9, dtype=np.uint16)
    h = xc4_ref.header(xc4_ref.encode(w, 4096))
    assert list(h["exp_of_code"][:4]) == [0, 127, 130, 120] and h["n_escapes"] == 0


def test_gaussian_ratios():
    w = _gauss_bf16(1 << 22)
    r4 = xc4_ref.encode(w, 1 << 20, 4).size / (2 * w.size)
    assert 0.75 <= r4 < 0.7515, r4   # 12 bits/weight + ~2e-4 escapes + tables
    unit = xc4_ref.encode(w, 1 << 20)
    r = unit.size / (2 * w.size)
    assert xc4_ref.header(unit)["version"] == 2
    assert 0.695 < r < 0.70, r      # 11 bits/weight + 8 bits × ~2.1% escapes


@pytest.mark.parametrize("n", [18 << 27, 21 << 26, 3 * 5 * 2**20, 4096 * 7, 48])
def test_frame_geometry(n):
    f = codec.frame_elems_for(n)
    assert f % 4096 == 0 and f <= codec.MAX_FRAME_ELEMS
    if n % (8 * 4096) == 0:
        assert n % (8 * f) == 0  # whole frames, evenly over 8 ranks
    if n == 18 << 27:  # Mixtral-8x22B FFN unit: 24 frames of 96 Mi weights (3 per rank at N = 8)
        assert f == 3 << 25 and n // f == 24


def test_bad_geometry_rejected():
    with pytest.raises(ValueError):
        xc4_ref.encode(np.zeros(24, np.uint16), 4096)
