"""The device reductions fold the 2048-block partials in chunks of
kFoldChunk = 4096 (solve.cu fold_any): fold(partials) = fold(fold(chunk_0),
fold(chunk_1), ...). This holds bit for bit for the reference's pairwise
combine with the odd tail carried (proj/src/vector_ops.cpp:16-25) because
chunk boundaries stay even at every level below log2(chunk). Checked here on
the reference's own combine order (a pure-Python restatement; CPU)."""
import random

import pytest


def combine(p):
    """proj/src/vector_ops.cpp:16-25."""
    p = list(p)
    if not p:
        return 0.0
    m = len(p)
    while m > 1:
        half = m // 2
        for i in range(half):
            p[i] = p[2 * i] + p[2 * i + 1]
        if m % 2:
            p[half] = p[m - 1]
        m = (m + 1) // 2
    return p[0]


def chunked(p, c):
    if len(p) <= c:
        return combine(p)
    return combine([combine(p[i:i + c]) for i in range(0, len(p), c)])


@pytest.mark.parametrize("chunk", [2, 4, 64, 4096])
def test_chunked_fold_is_the_reference_fold(chunk):
    rng = random.Random(chunk)
    sizes = list(range(1, 200)) + [4095, 4096, 4097, 8191, 8195, 12289, 20021]
    for m in sizes:
        p = [rng.uniform(-1, 1) * 10.0 ** rng.randint(-12, 12) for _ in range(m)]
        a, b = combine(p), chunked(p, chunk)
        assert a == b or (a != a and b != b), (m, chunk)
