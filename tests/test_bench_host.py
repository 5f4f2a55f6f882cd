"""Host-side logic of bench.py (no GPU): the conv2 design-ceiling model reported next to the roofline."""
import bench


def test_conv2_design_ceiling_lowrate():
    # 64x64 (mixed row-block heights): four 7-row units of 478 positions (237 + 241 outputs -> 240 + 256
    # MMA columns) and six 6-row units (205 + 204 -> 208 + 208) for 4096 outputs; 11 of 12 column-tap slots useful
    expected = 11 / 12 * 4096 / (4 * 496 + 6 * 416)
    assert abs(bench.conv2_useful_mac_ceiling(64, 64) - expected) < 1e-12
    assert bench.conv2_row_blocks(64, 64) == [(0, 7), (7, 7), (14, 7), (21, 7)] + [(28 + 6 * i, 6) for i in range(6)]


def test_conv2_row_blocks_rule():
    # uniform where mixing saves no tile: two column segments (a 7-row unit of pitch 74 needs 3 tiles), n1 = 9 / 33
    assert bench.conv2_row_blocks(128, 128) == [(r, min(6, 128 - r)) for r in range(0, 128, 6)]
    assert bench.conv2_row_blocks(9, 13) == [(0, 6), (6, 3)]
    assert bench.conv2_row_blocks(33, 33) == [(r, min(6, 33 - r)) for r in range(0, 33, 6)]
    # the blocks tile the image exactly, heights R or R + 1, tall ones first
    for n1, n2 in [(64, 64), (61, 64), (50, 40), (20, 20), (64, 16)]:
        blocks = bench.conv2_row_blocks(n1, n2)
        assert blocks[0][0] == 0 and sum(h for _, h in blocks) == n1
        assert all(b[0] + b[1] == c[0] for b, c in zip(blocks, blocks[1:]))
    assert bench._conv2_tiles(478) == [237, 241] and bench._conv2_tiles(409) == [205, 204]


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
            (180.0, 1700, 1965, 250.0, "0,0,0,0"),      # inside: under load whatever the (lagging) power reading
            (250.0, 900, 1965, 450.0, "1,0,0,0")]       # after the region: ignored
    with open(s.path, "w") as f:
        for t, sm, mx, pw, rs in rows:
            f.write(f"{t},{sm},{mx},{pw},{rs}\n")
    d = s.summary()
    assert d["samples"] == 3 and d["samples_under_load"] == 3
    assert d["sm_mhz"] == 1800.0 and d["sm_max_mhz"] == 1965.0
    assert d["reasons"] == ["sw_power_cap"] and d["window"] == "timed region only"


def test_clock_sampler_uses_instant_power_and_names_other_events(tmp_path):
    """Rows of the current NVML child carry the instantaneous draw and the raw clocks-event mask: every row inside the
    timed region counts as under load (both power readings lag a short region), both draws are reported, and event
    bits other than the four throttle reasons are named, so a clock below max is never reported without its reason."""
    s = bench.ClockSampler(0)
    s.kind, s.t0, s.t1 = "nvml", 100.0, 200.0
    s.path = str(tmp_path / "clk.csv")
    rows = [(110.0, 1950, 1965, 250.0, "0,0,0,0", 980.0, 0x0),      # averaged power still low, instant draw high
            (120.0, 1900, 1965, 260.0, "0,0,0,1", 1010.0, 0x4),
            (130.0, 1500, 1965, 270.0, "0,0,0,0", 990.0, 0x80),     # hw power brake: not one of the four columns
            (140.0, 1965, 1965, 280.0, "0,0,0,0", 120.0, 0x0)]      # a lagging low reading: still inside, still counted
    with open(s.path, "w") as f:
        for t, sm, mx, pw, rs, pin, mask in rows:
            f.write(f"{t},{sm},{mx},{pw},{rs},{pin},{mask}\n")
    d = s.summary()
    assert d["samples"] == 4 and d["samples_under_load"] == 4
    assert d["sm_mhz"] == 1925.0
    assert d["reasons"] == ["sw_power_cap"] and d["other_clock_events"] == ["hw_power_brake_slowdown"]
    assert d["power_w_max"] == 1010.0 and d["power_avg_w_max"] == 280.0
