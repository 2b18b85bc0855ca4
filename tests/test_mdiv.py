"""K1's bin index by multiply-high (csrc/nk_api.cu Geom.mdiv, csrc/nk_sort.cu
k_fold_keys): b = umulhi(c, ceil(2^32 / m)) must equal c // m (binsort.py:
103-111) for every cell c < n whenever n * m <= 2^32 -- the condition under
which the plan enables it.  Restated here in exact integer arithmetic."""
import random

import pytest


def mdiv(n, m):
    return ((1 << 32) + m - 1) // m if m > 1 and n * m <= (1 << 32) else 0


@pytest.mark.parametrize("m", list(range(2, 70)) + [127, 128, 129, 1000, 4097, 65537])
def test_mulhi_bin_index_exact(m):
    rng = random.Random(m)
    for n in (2 * m, 4096, 1 << 20, (1 << 32) // m):
        d = mdiv(n, m)
        if not d:
            continue
        cells = set(range(min(n, 3000))) | {n - 1, n - 2, n - m, n - m - 1}
        cells |= {rng.randrange(n) for _ in range(3000)}
        for c in cells:
            if 0 <= c < n:
                assert (c * d) >> 32 == c // m, (n, m, c)


def test_fallback_when_out_of_range():
    assert mdiv(1 << 30, 8) == 0          # n m > 2^32: plain division
    assert mdiv(4096, 1) == 0             # m = 1: plain division
    assert mdiv(512, 11) == ((1 << 32) + 10) // 11
