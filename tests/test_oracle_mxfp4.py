"""Oracle pins for the mxfp4 dequantisation (NEXT #1), CPU only."""

from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import mxfp4
from tests.conftest import golden_rows


def test_e2m1_table_matches_ocp_spec():
    for code, val in golden_rows("ocp_e2m1.txt"):
        s, mag = mxfp4.e2m1_value(int(code))
        assert float(s * mag) == float(val)
        assert (s < 0) == val.startswith("-")


def test_e8m0_matches_torch_float8_e8m0fnu():
    """Library routine: torch's float8_e8m0fnu -> float32 conversion."""
    x = torch.arange(256, dtype=torch.int32).to(torch.uint8).view(torch.float8_e8m0fnu)
    ref = x.to(torch.float32).numpy()
    for v in range(256):
        sc = mxfp4.e8m0_scale(v)
        if v == 255:
            assert sc is None and np.isnan(ref[v])
        else:
            assert float(sc) == float(ref[v])


def test_dequant_exact_for_every_code_and_scale():
    """bf16 bits decode back to exactly e2m1 * 2^(x-127) (Fraction arithmetic),
    inf above the bf16 range, NaN for the NaN scale -- all 16 x 256 pairs."""
    tab = mxfp4.dequant_table()
    vals = torch.from_numpy(tab.view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()
    for x in range(256):
        for c in range(16):
            v = vals[x, c]
            if x == 255:
                assert np.isnan(v)
                continue
            s, mag = mxfp4.e2m1_value(c)
            exact = s * mag * Fraction(2) ** (x - 127)
            if abs(exact) > mxfp4.BF16_MAX:
                assert np.isinf(v) and (v > 0) == (s > 0)
            else:
                assert Fraction(float(v)) == exact
                assert np.signbit(v) == (s < 0)


def test_known_values():
    assert mxfp4.dequant_bits(2, 127) == 0x3F80          # 1.0 * 2^0
    assert mxfp4.dequant_bits(15, 128) == 0xC140         # -6 * 2 = -12
    assert mxfp4.dequant_bits(1, 0) == 0x0020            # 0.5 * 2^-127 = 2^-128 (subnormal)
    assert mxfp4.dequant_bits(7, 254) == 0x7F80          # 6 * 2^127 -> inf
    assert mxfp4.dequant_bits(8, 100) == 0x8000          # -0


# --- upcast_np pinned against an independent library routine ----------------------
#
# transformers' MXFP4 dequantisation (transformers.integrations.mxfp4,
# the gpt-oss checkpoint loader) takes blocks [.., G, 16] of packed E2M1 bytes
# and one E8M0 scale per block of 32 values ([.., G]), low nibble first --
# written independently of this repository.  It fixes what the paper leaves to
# the OCP MX format: which nibble holds k = 2kb, and which scale a
# byte uses (row m, group kb >> 4 of K/32 groups).  A wrong nibble order, or
# kb >> 5 instead of kb >> 4, fails these tests.

def _tf_dequant(packed_mk, scales_mg):
    """[M, KB] packed bytes + [M, KB/16] scales -> [M, 2 KB] bf16 bits (uint16),
    via transformers' convert_moe_packed_tensors."""
    tfm = pytest.importorskip("transformers.integrations.mxfp4")
    M, KB = packed_mk.shape
    blocks = torch.from_numpy(packed_mk.reshape(1, M, KB // 16, 16).copy())
    sc = torch.from_numpy(scales_mg.reshape(1, M, KB // 16).copy())
    out = tfm.convert_moe_packed_tensors(blocks, sc, dtype=torch.bfloat16)   # [1, K, M]
    return out[0].transpose(0, 1).contiguous().view(torch.int16).numpy().view(np.uint16)


def _rowmajor_bytes(m_bits, kb_bits):
    from oracle.layout import Layout
    out = [("m", m_bits), ("kb", kb_bits)]
    unit = [(0, 1 << k) for k in range(kb_bits)] + [(1 << k, 0) for k in range(m_bits)]
    return Layout([("offset", m_bits + kb_bits)], out, {"offset": unit})


def _mx_inputs(m_bits, kb_bits, seed):
    rng = np.random.default_rng(seed)
    M, KB = 1 << m_bits, 1 << kb_bits
    packed = rng.integers(0, 256, size=(M, KB), dtype=np.uint8)
    # scales vary along m and along k (4+ groups per row); the range keeps
    # every product a normal bf16 so the library's float arithmetic is exact
    scales = rng.integers(110, 141, size=(M, KB // 16), dtype=np.uint8)
    return packed, scales


def test_upcast_np_matches_transformers_rowmajor():
    packed, scales = _mx_inputs(3, 6, 1)
    L = _rowmajor_bytes(3, 6)
    got = mxfp4.upcast_np(packed.reshape(-1), L, scales.reshape(-1), L)
    exp = _tf_dequant(packed, scales).reshape(-1)
    assert got.tobytes() == exp.tobytes()


def test_upcast_np_hand_example():
    """One row, K = 64 (two scale groups): byte 0x21 at kb = 0 -> (1.0, 0.5)
    * 2^(s0 - 127); byte 0xF7 at kb = 16 -> (6, -6) * 2^(s1 - 127)."""
    packed = np.zeros((1, 32), dtype=np.uint8)
    packed[0, 0] = 0x21
    packed[0, 16] = 0xF7
    scales = np.array([[128, 126]], dtype=np.uint8)     # x2, x0.5
    L = _rowmajor_bytes(0, 5)
    got = mxfp4.upcast_np(packed.reshape(-1), L, scales.reshape(-1), L)
    f = torch.from_numpy(got.view(np.int16).copy()).view(torch.bfloat16).float().numpy()
    assert f[0] == 1.0 and f[1] == 2.0        # low nibble 0x1 = 0.5, high nibble 0x2 = 1.0, x2
    assert f[32] == 3.0 and f[33] == -3.0     # 0x7 = 6, 0xF = -6, x0.5
    assert not np.any(np.delete(f, [0, 1, 32, 33]))


def test_upcast_np_matches_transformers_through_config5_layouts():
    """Config-5 layout family (reading A22): destination byte h holds the
    packed byte B(h) = (m, kb); its bf16 pair must equal the library's
    dequantised W[m, 2kb], W[m, 2kb + 1]."""
    from oracle import convert
    from oracle.layout import Layout
    from workloads import configs
    c = configs.cfg5(m_bits=8, kb_bits=7)
    A, B = Layout(**c["A"]), Layout(**c["B"])
    packed_buf = np.random.default_rng(5).integers(0, 256, size=1 << A.in_bits, dtype=np.uint8)
    scales = np.random.default_rng(6).integers(110, 141, size=(1 << 8) * (1 << 7) // 16, dtype=np.uint8)
    got = mxfp4.upcast_np(packed_buf, A, scales, B)
    # the logical [M, KB] matrix: byte (m, kb) is the source byte at A's preimage
    rows = convert.convert_np(packed_buf, A, _rowmajor_bytes(8, 7)).reshape(1 << 8, 1 << 7)
    W = _tf_dequant(rows, scales.reshape(1 << 8, -1))
    h = np.arange(1 << B.in_bits)
    x = convert.apply_np(B.cols, h)
    m, kb = x >> 7, x & 127
    assert got[0::2].tobytes() == W[m, 2 * kb].tobytes()
    assert got[1::2].tobytes() == W[m, 2 * kb + 1].tobytes()


def test_upcast_np_chunks_concatenate_to_upcast_np():
    from oracle.layout import Layout
    from workloads import configs
    c = configs.cfg5(m_bits=8, kb_bits=7)
    A, B = Layout(**c["A"]), Layout(**c["B"])
    packed = np.random.default_rng(8).integers(0, 256, size=1 << A.in_bits, dtype=np.uint8)
    scales = np.random.default_rng(9).integers(0, 256, size=(1 << 15) // 16, dtype=np.uint8)
    whole = mxfp4.upcast_np(packed, A, scales, B)
    parts = [o for _, o in mxfp4.upcast_np_chunks(packed, A, scales, B, chunk=1 << 10)]
    assert np.concatenate(parts).tobytes() == whole.tobytes()
