"""CPU: pin the oracle (oracle/) to the reference's own outputs.

The golden vectors were produced by importing the reference package
(tests/golden/make_golden.py). If the oracle agrees with them bit for bit, it
can stand in for the reference where the reference itself cannot run
(large N, the GPU box).
"""

import numpy as np
import pytest

from conftest import battery_cases, random_quantized_mant
from oracle import invop_oracle as O


@pytest.mark.parametrize("name", ["battery_2024", "battery_7"])
def test_oracle_battery_bitwise(golden, name):
    for n, m, mant, x, y_ref, counts in battery_cases(golden(name)):
        plan = O.build_plan(mant, m)
        y, c = O.plan_apply(plan, x)
        assert y.tobytes() == y_ref.tobytes()
        assert c == counts
        assert O.ordered_apply(mant, m, x).tobytes() == y_ref.tobytes()
        yn, cn = O.naive_apply(mant, m, x)
        assert yn.tobytes() == y_ref.tobytes()
        assert cn == (counts[1], counts[1])
        nz, distinct = O.sparsity_stats(mant)
        assert (sum(distinct), nz) == counts


def test_oracle_grid_cases(golden):
    g = golden("grid_cases")
    for side in (5, 11):
        inv = g["g%d_inverse" % side]
        ours = O.invert_dense(_full_grid_uniform(side))
        assert np.abs(ours - inv).max() <= 1e-14
        for m in (1, 2, 3, 5):
            mant = O.quantize(inv, m)
            assert (mant == g["g%d_m%d_mant" % (side, m)]).all()
            y = O.ordered_apply(mant, m, g["g%d_rhs" % side])
            assert y.tobytes() == g["g%d_m%d_y" % (side, m)].tobytes()
            if side == 5:
                plan = O.build_plan(mant, m)
                for k in ("col_ptr", "group_abs_mantissa", "group_coeff", "group_ptr",
                          "entry_rows", "entry_signs"):
                    assert np.array_equal(plan[k], g["g5_m%d_%s" % (m, k)]), k
        assert O.dense_matvec(inv, g["g%d_rhs" % side]).tobytes() == g["g%d_dense_y" % side].tobytes()


def _full_grid_uniform(side):
    n = side * side
    a = np.eye(n)
    for p in range(n):
        i, j = divmod(p, side)
        if 0 < i < side - 1 and 0 < j < side - 1:
            for q in (p - side, p + side, p - 1, p + 1):
                a[p, q] = -0.25
    return a


def test_oracle_quant_cases(golden):
    g = golden("quant_cases")
    for m in range(7):
        assert (O.quantize(g["vals"], m) == g["m%d" % m]).all()
    for m in (0, 3, 6, 12):
        assert (O.quantize(g["rand8"], m) == g["rand8_m%d" % m]).all()
    with pytest.raises(OverflowError):
        O.quantize(np.array([[1.0, 1e300]]), 2)


def test_oracle_config1(golden):
    g = golden("config1")
    mant = O.quantize(g["inverse"], 3)
    assert (mant == g["mant"]).all()
    assert O.ordered_apply(mant, 3, g["x"]).tobytes() == g["y"].tobytes()


def test_oracle_reference_known_answers():
    # pkg/tests/test_applyplan.py:57-63 — [[10,-5],[0,20]] at m=1, x=(2,4) -> (0, 8)
    y, c = O.naive_apply(np.array([[10, -5], [0, 20]]), 1, [2.0, 4.0])
    assert list(y) == [0.0, 8.0] and c == (3, 3)
    # pkg/tests/test_applyplan.py:27-38 — shared |25| in one column
    mant = np.zeros((4, 4), dtype=np.int64)
    mant[:, 0] = [25, 25, -25, 0]
    plan = O.build_plan(mant, 2)
    y, c = O.plan_apply(plan, [1.0, 0, 0, 0])
    assert list(y) == [0.25, 0.25, -0.25, 0.0] and c == (1, 3)
    # pkg/tests/test_quant.py:19-24 — half away from zero
    assert O.quantize(np.array([-0.005]), 2)[0] == -1
    assert O.quantize(np.array([0.005]), 2)[0] == 1
    assert O.quantize(np.array([0.025]), 1)[0] == 0
    assert O.quantize(np.array([-0.35]), 1)[0] == -4


def test_oracle_matches_reference_compiled_kernel():
    """oracle/_ref is the reference's own Cython kernel compiled from its source."""
    ref = O.reference_native()
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(2, 40))
        mant = random_quantized_mant(rng, n, 3)
        plan = O.build_plan(mant, 3)
        x = rng.standard_normal(n)
        out = np.zeros(n)
        counts = ref.plan_apply(plan["col_ptr"], plan["group_coeff"], plan["group_ptr"],
                                plan["entry_rows"], plan["entry_signs"], x, out)
        y, c = O.plan_apply(plan, x)
        assert out.tobytes() == y.tobytes() and tuple(counts) == c


def test_config2_fixture_consistency(golden):
    """The oracle rebuilds config 2 (N=2500) from scratch and must reproduce
    the reference's outputs on the reference's mantissas' checksums."""
    g = golden("config2")
    from paper_1602_00001_b200.grid import uniform_interior

    a = uniform_interior(50).to_dense()
    inv = O.invert_dense(a)
    mant = O.quantize(inv, 4)
    assert mant.sum() == g["mant_sum"][0]
    assert (mant[g["rows_sample"]] == g["mant_rows"]).all()
    Y = O.ordered_apply(mant, 4, g["X"])
    assert Y.tobytes() == g["Y"].tobytes()
