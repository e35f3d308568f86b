"""K9 parity on the B200: the GPU XC4 encoder writes the oracle's bytes, the
decoder restores every weight bit for bit (also at the full Mixtral-8x22B
unit size), and a streamed pass over encoded units fills the HBM window with
exactly the raw layer bytes."""
import numpy as np
import pytest
import torch

from oracle import xc4_ref
from paper_2505_10259_b200 import codec, native
from paper_2505_10259_b200.streamer import LayerStreamer

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _gauss(n, seed, std=0.02):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return torch.empty(n, dtype=torch.bfloat16, device=DEV).normal_(0.0, std, generator=g)


def _encode_dev(w, F, bits=0):
    scratch = torch.empty(native.xc4_scratch_bytes(w.numel(), F), dtype=torch.uint8, device=DEV)
    nb, _ = native.xc4_encode(w, F, None, scratch, code_bits=bits)
    dst = torch.empty(nb, dtype=torch.uint8, device=DEV)
    nb2, h = native.xc4_encode(w, F, dst, scratch, code_bits=bits)
    assert nb2 == nb == h.total_bytes
    return dst, h


CASES = [(16, 4096), (4096, 4096), (4112, 4096), (3 * 8192 + 48, 8192), (1 << 22, 1 << 20),
         (5 * (1 << 20) + 4096 * 3 + 16, 1 << 20)]


@pytest.mark.parametrize("bits", [0, 3, 4])
@pytest.mark.parametrize("n,F", CASES)
def test_encoder_bytes_equal_oracle(n, F, bits):
    if bits == 3 and n % 32:
        pytest.skip("3-bit codes need whole 32-weight groups")
    w = _gauss(n, seed=n)
    if n > 64:  # sprinkle rare exponents (escapes) and specials
        idx = torch.arange(0, n, 97, device=DEV)
        w.view(torch.int16)[idx] = torch.tensor([0x7f80, -32768, 0x0001, 0x7fc1, 0x3f80, 0x0080],
                                                dtype=torch.int16, device=DEV).repeat(idx.numel() // 6 + 1)[
            : idx.numel()]
    dev, h = _encode_dev(w, F, bits)
    want = xc4_ref.encode(_bits(w), F, bits)
    got = dev.cpu().numpy()
    assert got.size == want.size
    assert np.array_equal(got, want)


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("n,F", CASES)
def test_decoder_bit_exact(n, F, bits):
    if bits == 3 and n % 32:
        pytest.skip("3-bit codes need whole 32-weight groups")
    w = _gauss(n, seed=n + 1)
    w.view(torch.int16)[::31] = torch.randint(-32768, 32767, (len(range(0, n, 31)),), dtype=torch.int16,
                                              device=DEV)  # arbitrary patterns: heavy escapes
    dev, h = _encode_dev(w, F, bits)
    assert h.version == (2 if bits == 3 else 1)
    host = dev.cpu().pin_memory()
    out = torch.full((n,), -1, dtype=torch.int16, device=DEV)
    native.xc4_decode(host.data_ptr(), dev.data_ptr(), 0, h.n_frames, out.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(out, w.view(torch.int16))


@pytest.mark.parametrize("bits", [3, 4])
def test_every_bit_pattern_round_trips(bits):
    w = torch.arange(-32768, 32768, dtype=torch.int32, device=DEV).to(torch.int16)
    w = w[torch.randperm(w.numel(), device=DEV)].repeat(4).view(torch.bfloat16)
    dev, h = _encode_dev(w, 1 << 16, bits)
    out = torch.empty_like(w)
    native.xc4_decode(dev.cpu().pin_memory().data_ptr(), dev.data_ptr(), 0, h.n_frames, out.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), w.view(torch.int16))


def test_full_size_8x22b_unit_round_trip():
    """Size-independent property at BASELINE's full size: one Mixtral-8x22B FFN
    unit (4.83 GB, 24 frames) decodes to itself; 3-bit codes, ratio ≈ 0.698."""
    n = 4_831_838_208 // 2
    w = _gauss(n, seed=7)
    enc = codec.Encoder(DEV)
    dev, h = enc.encode(w)
    assert h.n_frames == 24
    assert h.version == 2 and 0.695 < dev.numel() / (2 * n) < 0.70
    host = dev.cpu().pin_memory()
    out = torch.empty_like(w)
    native.xc4_decode(host.data_ptr(), dev.data_ptr(), 0, h.n_frames, out.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), w.view(torch.int16))


@pytest.mark.parametrize("world", [1, 2, 4])
def test_streamed_window_equals_raw_layers(world):
    """Three passes over 5 encoded layers through a 2-slot window: every acquire
    sees the raw layer bytes.  world > 1: this rank's frame range decodes to
    exactly its slice_bounds bytes (the all-gather supplies the rest)."""
    from paper_2505_10259_b200.streamer import slice_bounds

    n = 8 * (1 << 20)
    raw = {li: _gauss(n, seed=100 + li) for li in range(5)}
    enc = codec.Encoder(DEV)
    host = {li: codec.encode_to_host(w, enc) for li, w in raw.items()}
    for rank in range(world):
        st = LayerStreamer(2 * n, {}, host, 5, DEV, n_slots=2, rank=rank, world=world) if world == 1 else None
        if world == 1:
            s = torch.cuda.Stream(device=DEV)
            for _ in range(3):
                for li in range(5):
                    p = st.acquire(li, s)
                    with torch.cuda.stream(s):
                        slot = next(t for t in st.slots if t.data_ptr() == p)
                        ok = torch.equal(slot.view(torch.bfloat16).view(torch.int16), raw[li].view(torch.int16))
                    assert ok, li
                    st.release(li, s)
            assert st.bytes_issued < 0.70 * st.raw_bytes_issued
        else:
            u = host[0]
            f0, f1 = u.frame_range(rank, world)
            out = torch.zeros(n, dtype=torch.int16, device=DEV)
            dev = u.data.to(DEV)
            native.xc4_decode(u.data.data_ptr(), dev.data_ptr(), f0, f1, out.data_ptr())
            torch.cuda.synchronize()
            lo, hi = slice_bounds(2 * n, rank, world)
            assert torch.equal(out[lo // 2:hi // 2], raw[0].view(torch.int16)[lo // 2:hi // 2])
            assert int(out[: lo // 2].abs().sum()) == 0 and int(out[hi // 2:].abs().sum()) == 0
