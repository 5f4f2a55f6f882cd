"""Multi-GPU runs on real ranks: one process per GPU over NCCL, launched the way
the driver launches bench.py.  They need >= 2 visible GPUs and skip otherwise (the 1-GPU pool); the host logic of
the same paths is covered over 2 gloo ranks in tests/test_multiproc.py."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch
    return torch.cuda.device_count()


need2 = pytest.mark.skipif("_gpus() < 2", reason="needs >= 2 GPUs")


def _torchrun(script, args, n):
    import bench
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", f"--master-port={bench.free_port()}", os.path.join(ROOT, script), *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)


@need2
def test_bench_launches_n_ranks_and_checks_the_gathered_outputs():
    n = min(2, _gpus())
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "3", "--warmup",
                        "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == n and line["config"]["global_batch"] == n * line["config"]["batch_per_gpu"]
    g = line["gather_check"]
    assert g["pass"] and g["ranks"] == n and g["bitwise_vs_rank0_recovery"]


@need2
def test_data_parallel_training_allreduce():
    r = _torchrun("tools/train_dp.py", ["3", "64", "paper", "bf16"], 2)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["world"] == 2 and d["loss_first_last"][1] < d["loss_first_last"][0]


@need2
def test_row_sharded_recovery_on_peers():
    r = _torchrun("tools/rowshard_check.py", ["64", "1024", "16"], 2)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["pass"] and d["world"] == 2


def test_same_launchers_with_one_rank():
    """The scripts above through the same torchrun launcher with a single rank (runs on the 1-GPU pool)."""
    r = _torchrun("tools/rowshard_check.py", ["64", "1024", "8"], 1)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["pass"]
    r = _torchrun("bench.py", ["--gpus", "1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--batch", "512"], 1)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["gather_check"]["pass"]
