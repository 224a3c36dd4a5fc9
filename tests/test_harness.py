"""Table 1 / scaling harness on the device path against the reference's
recorded run (/root/reference/pkg/test_output.txt:11-19)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_table1_matches_reference_run(tmp_path):
    import paper_1602_00001_b200 as invop

    rows = invop.run_table1([5, 11, 21, 41], ["none", 5])
    got = {(r.n, r.digits): r.error for r in rows}
    # reference run: unrounded 0.0658436 / 0.0106893 / 0.00258888 / 0.000647352; n=41 m=5 0.000647285
    for n, ref in ((5, 0.0658436), (11, 0.0106893), (21, 0.00258888), (41, 0.000647352)):
        assert "%.6g" % got[(n, "none")] == "%.6g" % ref
    assert "%.6g" % got[(41, 5)] == "0.000647285"
    invop.emit_csv(rows, tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_text().startswith("n,digits,error\n5,none,0.0658436\n")


def test_cli_goldens():
    """reference test_cli.py:16-30 golden lines"""
    import paper_1602_00001_b200 as invop

    (r1,) = invop.run_table1([5], ["none"])
    (r2,) = invop.run_table1([11], [2])
    assert "grid 5x5 digits=none relative error: %.6g" % r1.error == "grid 5x5 digits=none relative error: 0.0658436"
    assert "%.6g" % r2.error == "0.0111585"


def test_scaling_slopes_match_reference_run():
    import paper_1602_00001_b200 as invop

    rep = invop.run_scaling([11, 21, 41], [2])
    s_mult, s_add = rep.slopes[2]
    assert round(s_mult, 4) == 1.4537 and round(s_add, 4) == 2.0966
    assert all(r.naive_mult == r.big_n ** 2 for r in rep.rows)


def test_large_grid_beyond_dense_limit():
    """n=129 full grid (N=16641 > MAX_DENSE_N): the device path has no dense limit."""
    import paper_1602_00001_b200 as invop

    (row,) = invop.run_table1([129], [6])
    assert 0 < row.error < 5e-4
