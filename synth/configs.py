"""The five workloads of BASELINE.json ``configs`` (index order preserved)."""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    n: int                 # image side, N = n*n
    m: int                 # measurements
    batch: int             # images per GPU
    n_blobs: int
    n_rects: int
    texture_var: float
    precisions: tuple      # storage/compute modes the config is run in
    note: str = ""

    @property
    def N(self) -> int:
        return self.n * self.n


CONFIGS = {
    "tiny": Config("tiny", 16, 64, 4, 4, 0, 0.0, ("f32", "bf16"),
                   "BASELINE.json configs[0]: 16x16, M=64, batch 4, 4 blobs, fp32"),
    "paper": Config("paper", 64, 1024, 256, 8, 4, 0.0, ("f32", "tf32"),
                    "configs[1]: 64x64, M/N=0.25, batch 256, fp32 and TF32, 1 GPU"),
    "lowrate": Config("lowrate", 64, 410, 4096, 8, 4, 0.0, ("bf16",),
                      "configs[2]: 64x64, M/N=0.1 (M=410), batch 4096/GPU, bf16 in, fp32 acc"),
    "larger": Config("larger", 128, 4096, 1024, 16, 8, 0.0, ("bf16",),
                     "configs[3]: 128x128, M=4096, batch 1024/GPU, bf16"),
    "stress": Config("stress", 256, 16384, 256, 32, 16, 0.01, ("bf16",),
                     "configs[4]: 256x256, M=16384, Phi 2.1 GB bf16, batch 256/GPU, texture N(0,0.01)"),
}

ORDER = ["tiny", "paper", "lowrate", "larger", "stress"]
