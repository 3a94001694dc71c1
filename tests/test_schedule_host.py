"""Host logic of the attention kernel's tail schedule (stream-K, DESIGN.md
Sec 6) through tm_schedule_tail_host, without a GPU: the ranges are
contiguous, non-empty and cover every tail tile exactly once; there are at
most min(148, max(units, tiles / 4)) of them (no 1-tile shredding of short
problems); units shorter than 4 tiles stay whole; and the ranges are
balanced to within one unit's worth of per-item cost."""
import itertools

import pytest

from paper_2506_03099_b200 import tm


SHAPES = [(u, n) for u, n in itertools.product([1, 2, 3, 5, 36, 40, 60, 92, 120, 147],
                                               [1, 2, 3, 4, 7, 24, 56, 59, 112])]


@pytest.mark.parametrize("units,n", SHAPES)
def test_tail_ranges_partition_the_tiles(units, n):
    C = 148
    b = tm.tm_schedule_tail_host(units, n, C)
    G = len(b) - 1
    W = units * n
    assert b[0] == 0 and b[-1] == W
    assert all(b[i + 1] > b[i] for i in range(G)), "empty range"
    assert 1 <= G <= C
    assert G <= max(units, W // 4), "ranges shorter than the minimum piece"
    if n < 4:                                  # short units are never split
        assert all(x % n == 0 for x in b)


@pytest.mark.parametrize("units,n", [(36, 56), (60, 56), (92, 56), (120, 56), (72, 112)])
def test_tail_ranges_are_balanced(units, n):
    """tiles + 3 per extra item, the cost the host greedy equalises: max <= mean + one unit."""
    b = tm.tm_schedule_tail_host(units, n, 148)
    costs = []
    for lo, hi in zip(b, b[1:]):
        items = len(set(range(lo // n, (hi - 1) // n + 1)))
        costs.append((hi - lo) + 3 * (items - 1))
    mean = sum(costs) / len(costs)
    assert max(costs) <= mean + n, (max(costs), mean)


@pytest.mark.parametrize("units,n", [(1, 630), (1, 2000), (2, 1000), (3, 300)])
def test_long_units_have_at_most_65_pieces(units, n):
    """A split unit's merger tracks its contributors in a 64-bit mask: however
    long a unit, the schedule never cuts it into more than 65 pieces (the
    minimum piece is raised from 4 until that holds), the ranges still
    partition the tiles, and the cap does not collapse the parallelism (a
    one-unit problem keeps more than 32 ranges)."""
    b = tm.tm_schedule_tail_host(units, n, 148)
    assert b[0] == 0 and b[-1] == units * n
    assert all(b[i + 1] > b[i] for i in range(len(b) - 1))
    for u in range(units):
        first = max(i for i in range(len(b) - 1) if b[i] <= u * n)
        last = max(i for i in range(len(b) - 1) if b[i] <= u * n + n - 1)
        assert last - first + 1 <= 65, (u, last - first + 1)
    if units * n // 4 > 148:                   # enough work for every CTA at the first minimum
        assert len(b) - 1 > 32


def test_invalid_query():
    with pytest.raises(tm.TMError):
        tm.tm_schedule_tail_host(0, 56, 148)
    with pytest.raises(tm.TMError):
        tm.tm_schedule_tail_host(10, 56, 200)
