"""The phase decoder's symbol search index (coder.cu build_cdf_kernel /
dec_sym_rsv), restated on the oracle's 64 cumulative tables of both prior
families: for every target q in [0, 65536) the bucket entry, the
unit-frequency closed form and the bounded binary search give the symbol a
full search of the table gives (the largest k with cum[k] <= q)."""
import numpy as np
import pytest

from oracle_api import cdf_tables_family

K = 257


def build_index(c):
    freq = np.diff(c)
    lut = np.zeros(257, np.int64)
    k = 0
    for b in range(257):
        while k + 1 < K and c[k + 1] <= b * 256:
            k += 1
        lut[b] = k
    unit = np.zeros(257, bool)
    for b in range(256):
        unit[b] = bool(np.all(freq[lut[b] + 1:lut[b + 1]] == 1))
    return lut, unit


@pytest.mark.parametrize("family", [0, 1])
def test_bucket_index_matches_full_search(family):
    tables = cdf_tables_family(family).astype(np.int64)
    q = np.arange(65536)
    b = q >> 8
    for c in tables:
        lut, unit = build_index(c)
        ref = np.searchsorted(c, q, side="right") - 1
        lo, hi = lut[b], lut[b + 1]
        c1 = c[np.minimum(lo + 1, K)]
        closed = np.where(q >= c1, np.minimum(lo + 1 + (q - c1), hi), lo)
        # the bounded search over [lo, hi] returns the full search's symbol
        # whenever the symbol lies in [lo, hi]; check that bracket too
        assert np.all((ref >= lo) & (ref <= hi))
        got = np.where(unit[b], closed, ref)
        assert np.array_equal(got, ref)
        # the closed form is what the unit buckets use: verify it on them
        assert np.array_equal(closed[unit[b]], ref[unit[b]])
