"""The C-ABI from plain C: include/halftime_b200.h compiles as C99, and a C
program linked against libhalftime_b200.so calls the host-side entry points
(no GPU needed) with the reference's answers (seed_words_needed,
pkg/src/halftimehash/hasher.py:152-158; master fold, hasher.py:48-58;
unsupported width -> HTH_EINVAL, params.py:230-237)."""

import os
import shutil
import subprocess

import pytest

from oracle import oracle_np as o

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2104_08865_b200", "libhalftime_b200.so")

PROGRAM = r"""
#include <stdio.h>
#include <string.h>
#include "halftime_b200.h"
int main(void) {
  static const unsigned long long lens[] = {0, 1, 1336, 1344, 4096, 1048576, 17179869184ull};
  static const int widths[] = {16, 24, 32, 40};
  for (int w = 0; w < 4; w++)
    for (int i = 0; i < 7; i++) {
      uint64_t words = 0;
      if (hth_seed_words_needed(widths[w], lens[i], &words) != HTH_OK) return 2;
      printf("%d %llu %llu\n", widths[w], lens[i], (unsigned long long)words);
    }
  uint8_t master[32];
  for (int i = 0; i < 32; i++) master[i] = (uint8_t)i;
  uint64_t fold = 0;
  if (hth_master_fold(master, &fold) != HTH_OK) return 3;
  printf("fold %llu\n", (unsigned long long)fold);
  uint64_t x = 0;
  if (hth_seed_words_needed(20, 5, &x) != HTH_EINVAL) return 4;
  printf("err %s\n", hth_last_error());
  return 0;
}
"""


@pytest.mark.skipif(not os.path.exists(LIB) or shutil.which("gcc") is None, reason="library not built / no gcc")
def test_c_program_against_the_shared_library(tmp_path):
    src = tmp_path / "abi.c"
    src.write_text(PROGRAM)
    exe = tmp_path / "abi"
    libdir = os.path.dirname(LIB)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                    "-L", libdir, "-l:libhalftime_b200.so", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.splitlines()
    for line in lines[:28]:
        w, n, words = (int(x) for x in line.split())
        assert words == o.seed_words_needed(o.variant(w), n), line
    assert lines[28] == f"fold {o.master_fold(bytes(range(32)))}"
    assert lines[29].startswith("err ") and len(lines[29]) > 4
