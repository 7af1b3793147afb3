"""CPU tests of host-side scheduling logic (no GPU needed)."""
from unittest import mock

import pytest


class _Props:
    multi_processor_count = 148


@pytest.mark.parametrize("n", [1, 1000, 18944, 18944 * 5 + 3, 18944 * 16, 18944 * 16 + 1,
                               1 << 20, 8388608])
def test_pipeline_bounds_cover_and_align(n):
    """The pipelined numpy projection's chunks tile [0, n) contiguously. Every chunk except the
    last is a whole number of voxel-tile-per-SM units (128 x SMs voxels). Long inputs ramp
    1, 2, 4 units up and 4, 2, 1 down."""
    from paper_1810_01967_b200 import projection as P
    unit = 128 * _Props.multi_processor_count
    with mock.patch("torch.cuda.get_device_properties", return_value=_Props()):
        b = P._pipeline_bounds(n, 0)
    assert b[0][0] == 0 and b[-1][1] == n
    assert all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
    assert all(hi > lo for lo, hi in b)
    assert all((hi - lo) % unit == 0 for lo, hi in b[:-1])
    total = -(-n // unit)
    if total > 16:
        sizes = [(hi - lo) // unit for lo, hi in b]
        assert sizes[:3] == [1, 2, 4]
        assert max(sizes) <= 8 and (total < 22 or max(sizes) == 8)
        assert sizes[-3:-1] == [4, 2] and b[-1][1] - b[-1][0] <= unit


def test_bench_cpu_ipg_model_fields():
    """bench.cpu_ipg_model: the modelled CPU denominators of the large IPG legs (projection at
    the measured CPU rate + per-frame FFTs) are finite, positive and consistent."""
    import bench
    res = {"parity": {"first": {"D": 120624}}, "projection_trials": 52, "iterations": 22,
           "ms_per_iter": 2.3}
    m = bench.cpu_ipg_model("cfg2", res, 5.0e9)
    assert m["kind"] == "model"
    assert m["projection_ms"] > 0 and m["operator_ms"] > 0
    assert abs(m["ms_per_iter"] - (m["projection_ms"] + m["operator_ms"])) < 1e-6 * m["ms_per_iter"]
    # r n D 2s / rate
    r = 52 / 22
    assert abs(m["projection_ms"] - 1e3 * r * 65536 * 120624 * 40 / 5.0e9) < 1e-6 * m["projection_ms"]
    assert abs(m["speedup_vs_model"] - m["ms_per_iter"] / 2.3) < 1e-6 * m["speedup_vs_model"]
