"""Host-side logic of bench.py (no GPU): the conv2 design-ceiling model reported next to the roofline."""
import bench


def test_conv2_design_ceiling_lowrate():
    # 64x64: ten 6-row units of 416 MMA columns (253 + 156 -> 256 + 160) and a 4-row unit (271 -> 256 + 32) for 4096
    # outputs; 11 of 12 column-tap slots useful
    expected = 11 / 12 * 4096 / (10 * 416 + 288)
    assert abs(bench.conv2_useful_mac_ceiling(64, 64) - expected) < 1e-12


def test_conv2_design_ceiling_pitch74_and_bounds():
    # two column segments: pitch 74 (448 columns per full 6-row unit of 384 outputs)
    c128 = bench.conv2_useful_mac_ceiling(128, 128)
    assert 0.75 < c128 < 11 / 12 * 384 / 416
    for n in (16, 33, 64, 100, 256):
        assert 0.0 < bench.conv2_useful_mac_ceiling(n, n) < 11 / 12
