"""Build liblmx.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")


def build(jobs: int = 4, extra: str = "") -> str:
    cmd = ["make", "-s", f"-j{jobs}", "-C", CSRC]
    if extra:
        cmd.append(f"EXTRA={extra}")
    subprocess.run(cmd, check=True)
    return os.path.join(HERE, "liblmx.so")


if __name__ == "__main__":
    print(build())
