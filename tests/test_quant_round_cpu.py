"""The E4M3 encode in csrc/prologue.cu (write_codes) rounds v = fl(z fl(7/m)) to the nearest integer, ties to even (R10),
as (v + 1.5*2^23) - 1.5*2^23 in f32: exact because |v| < 7.5 < 2^22 and numbers in [2^23, 2^24) have ulp 1.  It must
equal rint(v) bit for bit, with the canonical +0 for values that round to zero (code byte 0x00, R10/R11).  Checked here
in f32 on a dense grid, every half-integer tie and the signed zeros / tiny values."""
import numpy as np


def test_magic_add_rounding_equals_rint_ties_to_even():
    v = np.concatenate([np.linspace(-7.6, 7.6, 2_000_001, dtype=np.float32),
                        np.arange(-15, 16, dtype=np.float32) / 2,
                        np.nextafter(np.arange(-15, 16, dtype=np.float32) / 2, np.float32(np.inf)),
                        np.nextafter(np.arange(-15, 16, dtype=np.float32) / 2, np.float32(-np.inf)),
                        np.array([-0.0, 0.0, -1e-30, 1e-30, -0.49999997, 0.49999997, -0.5, 0.5], np.float32)])
    M = np.float32(12582912.0)
    got = (v + M).astype(np.float32) - M
    want = (np.rint(v) + np.float32(0.0)).astype(np.float32)  # rint, -0 -> +0
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.all(np.signbit(got[got == 0]) == False)  # noqa: E712
    assert np.array_equal(np.rint(np.arange(-15, 16, dtype=np.float32) / 2)[[0, 1, 2]], np.float32([-8, -7, -6]))
