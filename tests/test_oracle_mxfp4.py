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
