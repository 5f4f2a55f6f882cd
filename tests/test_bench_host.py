"""Host-side logic of bench.py (no GPU): the conv2 design-ceiling model reported next to the roofline."""
import bench


def test_conv2_design_ceiling_lowrate():
    # 64x64: ten 6-row units of 416 MMA columns (balanced 205 + 204 -> 208 + 208) and a 4-row unit (271 -> 136 + 135 ->
    # 144 + 144) for 4096
    # outputs; 11 of 12 column-tap slots useful
    expected = 11 / 12 * 4096 / (10 * 416 + 288)
    assert abs(bench.conv2_useful_mac_ceiling(64, 64) - expected) < 1e-12


def test_conv2_design_ceiling_pitch74_and_bounds():
    # two column segments: pitch 74 (448 columns per full 6-row unit of 384 outputs)
    c128 = bench.conv2_useful_mac_ceiling(128, 128)
    assert 0.75 < c128 < 11 / 12 * 384 / 416
    for n in (16, 33, 64, 100, 256):
        assert 0.0 < bench.conv2_useful_mac_ceiling(n, n) < 11 / 12


def test_clock_sampler_keeps_only_rows_inside_the_timed_region(tmp_path):
    """The NVML child writes timestamped rows; summary() keeps those between __enter__ and __exit__ and reports
    the median SM clock of the rows under load and the union of throttle reasons (B200_PROFILING.md clocks line)."""
    s = bench.ClockSampler(0)
    s.kind, s.t0, s.t1 = "nvml", 100.0, 200.0
    s.path = str(tmp_path / "clk.csv")
    rows = [(50.0, 1000, 1965, 500.0, "0,0,0,1"),      # before the region: ignored
            (120.0, 1800, 1965, 400.0, "0,0,0,1"),
            (150.0, 1900, 1965, 420.0, "0,0,0,0"),
            (180.0, 1700, 1965, 250.0, "0,0,0,0"),      # inside but idle (power <= 300 W): not under load
            (250.0, 900, 1965, 450.0, "1,0,0,0")]       # after the region: ignored
    with open(s.path, "w") as f:
        for t, sm, mx, pw, rs in rows:
            f.write(f"{t},{sm},{mx},{pw},{rs}\n")
    d = s.summary()
    assert d["samples"] == 3 and d["samples_under_load"] == 2
    assert d["sm_mhz"] == 1850.0 and d["sm_max_mhz"] == 1965.0
    assert d["reasons"] == ["sw_power_cap"] and d["window"] == "timed region only"
