"""Seeded synthetic inputs shared by tests, smoke() and bench.py (no method arithmetic)."""
from .configs import CONFIGS, ORDER, Config  # noqa: F401
from .dtypes import bf16_bits_to_f32, f32_to_bf16_bits, round_bf16  # noqa: F401
from .generators import KSIZE, WIDTHS, Params, make_images, make_params, make_phi, measure  # noqa: F401
