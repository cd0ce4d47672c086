"""Build libhalftime_b200.so in-tree with nvcc for sm_100a (csrc/Makefile)."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def build(verbose: bool = False) -> str:
    csrc = os.path.join(HERE, "csrc")
    cmd = ["make", "-C", csrc] + ([] if verbose else ["-s"])
    subprocess.check_call(cmd)
    return os.path.join(HERE, "libhalftime_b200.so")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
