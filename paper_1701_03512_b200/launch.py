"""One process per GPU: (re)launch a script under torchrun.

``python bench.py --gpus N`` must measure N GPUs, not silently one
(VERDICT r1).  When the process is not already a torchrun rank
(``WORLD_SIZE`` unset) and N > 1, ``ensure_world`` checks that N devices are
visible and re-executes the same command line under
``python -m torch.distributed.run --nnodes=1 --nproc-per-node N`` with the
rendezvous on 127.0.0.1; inside a torchrun rank it checks that
``WORLD_SIZE`` equals N.  Either mismatch is an error, never a downgrade.

The reference's scaling harness (pkg/src/binpaths/bench.py:55-93) times M
worker threads in one process; here M is the number of GPU ranks.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from typing import Optional, Sequence


class LaunchError(RuntimeError):
    """A multi-GPU run that cannot run on the requested number of GPUs."""


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_cmd(script: str, argv: Sequence[str], nproc: int, port: Optional[int] = None) -> list:
    """The torchrun command line for `script argv` on `nproc` local ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr=127.0.0.1", f"--master-port={port or free_port()}", script, *argv]


def visible_devices() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:  # noqa: BLE001
        return 0


def ensure_world(n: int, script: str, argv: Sequence[str], need_devices: bool = True,
                 env: Optional[dict] = None) -> Optional[int]:
    """None when this process may run as one of `n` ranks (n == 1 outside
    torchrun, or a torchrun rank of a world of n); otherwise runs the command
    under torchrun with n ranks and returns its exit code.  Raises
    LaunchError when fewer than n devices are visible (need_devices) or when
    an existing torchrun world has a different size."""
    if n < 1:
        raise LaunchError(f"--gpus must be >= 1, got {n}")
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != n:
            raise LaunchError(f"running as a rank of a world of {world} processes but --gpus {n} was asked")
        return None
    if n == 1:
        return None
    if need_devices:
        have = visible_devices()
        if have < n:
            raise LaunchError(f"--gpus {n} needs {n} visible CUDA devices, found {have}")
    return subprocess.call(torchrun_cmd(os.path.abspath(script), list(argv), n), env=env)
