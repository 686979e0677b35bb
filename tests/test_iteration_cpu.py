"""NEXT-2 host policy: the adaptive (d, w) control of P:L880-884."""
import pytest

from paper_2501_12162_b200.iteration import IterationShape, adaptive_params


def test_adaptive_params_formula_examples():
    # d = clip(D_max, D_min, floor(B1/(n + c1)) - 1); w = clip(W_max, 1, floor(B2/n) + c2)
    assert adaptive_params(7, d_max=8, d_min=1, w_max=4, b1=64, b2=16, c1=1, c2=0)[0] == 7
    assert adaptive_params(64, d_max=8, d_min=1, w_max=4, b1=64, b2=16, c1=1, c2=0)[1] == 1   # lower clip
    assert adaptive_params(1, d_max=8, d_min=1, w_max=4, b1=64, b2=16, c1=1, c2=0)[0] == 8    # upper clip
    assert adaptive_params(200, d_max=8, d_min=2, w_max=4, b1=64, b2=16, c1=1, c2=0)[0] == 2  # d_min binds
    with pytest.raises(ValueError):
        adaptive_params(0, 8, 1, 4, 64, 16)


def test_adaptive_params_monotone_in_load():
    """More active requests -> never deeper or wider trees."""
    prev = None
    for n in range(1, 300):
        d, w = adaptive_params(n, d_max=8, d_min=1, w_max=8, b1=4096, b2=512, c1=4, c2=1)
        assert 1 <= d <= 8 and 1 <= w <= 8
        if prev:
            assert d <= prev[0] and w <= prev[1]
        prev = (d, w)


def test_shape_key_distinguishes_shapes():
    a = IterationShape(64, 64 * 65, 8, 31, 2048, 32, 8, 128, 4096, 64, 40, 9)
    b = IterationShape(64, 64 * 65, 8, 31, 2048, 32, 8, 128, 4096, 64, 40, 10)
    assert a.key() != b.key() and a.key() == IterationShape(*[getattr(a, f) for f in a.__dataclass_fields__]).key()
