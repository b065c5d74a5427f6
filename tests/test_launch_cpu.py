"""bench.py's one-process-per-GPU launcher (paper_2409_14309_b200/launch.py)
on CPU: --gpus N without a launcher re-executes under torch.distributed.run
and forms an N-rank world (gloo here); a world that does not match --gpus,
or too few devices, fails loudly instead of running on one GPU."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env_extra=None, timeout=240):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                          text=True, env=env, cwd=str(ROOT), timeout=timeout)


@pytest.mark.timeout(300)
def test_launch_forms_world_of_four():
    out = _run(["--gpus", "4", "--launch-check"])
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["world"] == 4 and line["n_gpus"] == 4
    assert line["rank_sum"] == 1 + 2 + 3 + 4
    assert line["launcher"] == "torchrun"
    assert line["backend"] == ("nccl" if torch.cuda.device_count() >= 4 else "gloo")


def test_world_mismatch_fails_loudly():
    out = _run(["--gpus", "2", "--launch-check"], {"WORLD_SIZE": "3", "RANK": "0"})
    assert out.returncode == 2
    assert "WORLD_SIZE=3 but --gpus 2" in out.stderr


@pytest.mark.skipif(torch.cuda.device_count() >= 64, reason="needs a node with < 64 GPUs")
def test_too_few_devices_fails_loudly():
    out = _run(["--gpus", "64", "--steps", "1"])
    assert out.returncode == 2
    assert "needs 64 CUDA devices" in out.stderr


def test_single_rank_needs_no_launcher():
    from paper_2409_14309_b200.launch import ensure_world, torchrun_argv

    saved = {k: os.environ.pop(k) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK")
             if k in os.environ}
    try:
        assert ensure_world(1, "bench.py", []) == (0, 1, 0)
    finally:
        os.environ.update(saved)
    argv = torchrun_argv(8, "bench.py", ["--gpus", "8"], port=1234)
    assert argv[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in argv and "127.0.0.1" in argv and argv[-2:] == ["--gpus", "8"]
