"""One process per GPU: the launcher behind ``bench.py --gpus N``.

A multi-GPU run is N processes, one per device, that meet in a
``torch.distributed`` process group (NCCL over NVLink for the data plane
where one is needed, the plumbing otherwise).  When a script is started
without a launcher (``WORLD_SIZE`` unset) and asked for N > 1 ranks, it
re-executes itself under ``torch.distributed.run`` with N local workers on
127.0.0.1; under a launcher the world size must equal the N asked for, so
a run can never silently report fewer GPUs than requested.
"""

from __future__ import annotations

import os
import socket
import sys


class LaunchError(RuntimeError):
    """The requested world cannot be formed (too few devices, wrong launcher)."""


def env_world() -> tuple[int, int, int] | None:
    """(rank, world, local_rank) from the launcher's environment, or None
    when no launcher started this process."""
    if "WORLD_SIZE" not in os.environ:
        return None
    return (int(os.environ.get("RANK", "0")), int(os.environ["WORLD_SIZE"]),
            int(os.environ.get("LOCAL_RANK", "0")))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun_argv(nproc: int, script: str, args: list[str], port: int | None = None) -> list[str]:
    """Command line that runs ``script args`` as ``nproc`` local ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
            "--master-port", str(port or free_port()), script, *args]


def require_devices(nproc: int) -> None:
    """Fail loudly unless this node has ``nproc`` CUDA devices."""
    import torch

    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < nproc:
        raise LaunchError(f"--gpus {nproc} needs {nproc} CUDA devices, this node has {have}")


def ensure_world(nproc: int, script: str, args: list[str], need_gpus: bool = True) -> tuple[int, int, int]:
    """Make this process one of ``nproc`` ranks.

    * Under a launcher: check that its world size is ``nproc`` and return
      (rank, world, local_rank).
    * Without one and ``nproc`` == 1: (0, 1, 0).
    * Without one and ``nproc`` > 1: re-exec under torch.distributed.run
      (does not return); with ``need_gpus`` the node must have ``nproc``
      devices first."""
    w = env_world()
    if w is not None:
        if w[1] != nproc:
            raise LaunchError(f"launched with WORLD_SIZE={w[1]} but --gpus {nproc}")
        return w
    if nproc <= 1:
        return 0, 1, 0
    if need_gpus:
        require_devices(nproc)
    argv = torchrun_argv(nproc, script, args)
    sys.stdout.flush()
    sys.stderr.flush()
    os.execv(argv[0], argv)
    raise AssertionError("unreachable")  # pragma: no cover
