"""Measured latency grid in the reference's profiler schema:
abscissae equal the reference's make_points, and the CSV loads with the
reference's own grid_from_csv / profile_lookup (oracle/_ref)."""
import pytest

import oracle
from paper_2510_18121_b200 import profiler


def test_grid_points_match_reference_synth_grid():
    # make_points (P/src/cost.cpp:172-185) with tile 128, max_len 1000
    assert profiler.grid_points(128, 1000) == [32, 64, 128, 256, 384, 512, 640, 896, 1000]
    assert profiler.grid_points(128, 100) == [32, 64, 128]


def test_csv_roundtrip_through_reference_parser():
    q, kv = [128, 256], [128, 256, 512]
    lat = [1e-5 * (i + 1) for i in range(len(q) * len(kv))]
    csv = profiler.grid_to_csv(q, kv, lat)
    assert csv.splitlines()[0] == "q,kv,latency_s"
    got = oracle.ref_lib().ref_grid_lookup(csv.encode(), 1e15, 4.0 * 4096, 128, 128, 256)
    assert got == pytest.approx(lat[1])


@pytest.mark.gpu
def test_measured_grid_loads_in_reference():
    from paper_2510_18121_b200 import configs as CF
    q, kv, lat = profiler.measure_grid(CF.LLAMA8B, 1024, q_points=[128, 512, 1024], kv_points=[128, 512, 1024])
    assert all(x > 0 for x in lat)
    csv = profiler.grid_to_csv(q, kv, lat)
    got = oracle.ref_lib().ref_grid_lookup(csv.encode(), 1e18, 4.0 * 4096, 128, 512, 1024)
    assert got == pytest.approx(lat[1 * 3 + 2], rel=1e-9)
