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


GPU_PROGRAM = r"""
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime.h>
#include "halftime_b200.h"
/* config 1's shape: 1024 strings x 4096 B, 24-byte digests, through the C-ABI
 * only (device buffers, one stream), data read from stdin */
int main(void) {
  const uint64_t B = 1024, n = 4096, k = 3;
  uint8_t* h = (uint8_t*)malloc(B * n);
  if (fread(h, 1, B * n, stdin) != B * n) return 2;
  uint8_t master[32];
  for (int i = 0; i < 32; i++) master[i] = (uint8_t)(7 * i + 1);
  uint64_t fold, cap, ws_bytes;
  if (hth_master_fold(master, &fold) || hth_seed_words_needed(24, n, &cap) ||
      hth_workspace_size_fixed(24, B, n, &ws_bytes)) return 3;
  void *d_data, *ws; uint64_t *d_seed, *d_out;
  cudaMalloc(&d_data, B * n); cudaMalloc(&ws, ws_bytes); cudaMemset(ws, 0, ws_bytes);
  cudaMalloc((void**)&d_seed, cap * 8); cudaMalloc((void**)&d_out, B * k * 8);
  cudaMemcpy(d_data, h, B * n, cudaMemcpyHostToDevice);
  cudaStream_t st; cudaStreamCreate(&st);
  if (hth_expand_seed(fold, 0, cap, d_seed, st)) return 4;
  int rc = hth_hash_fixed(24, d_data, B, n, n, fold, d_seed, cap, d_out, ws, ws_bytes, st);
  if (rc) { fprintf(stderr, "%s\n", hth_last_error()); return 5; }
  uint64_t* out = (uint64_t*)malloc(B * k * 8);
  cudaMemcpyAsync(out, d_out, B * k * 8, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  fwrite(out, 8, B * k, stdout);
  return 0;
}
"""


@pytest.mark.gpu
def test_c_program_hashes_on_the_gpu(tmp_path):
    import numpy as np

    from oracle import c as coracle

    cuda = "/usr/local/cuda"
    src = tmp_path / "abi_gpu.c"
    src.write_text(GPU_PROGRAM)
    exe = tmp_path / "abi_gpu"
    libdir = os.path.dirname(LIB)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
                    str(src), "-L", libdir, "-l:libhalftime_b200.so", f"-Wl,-rpath,{libdir}",
                    "-L", f"{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{cuda}/lib64", "-o", str(exe)], check=True)
    rng = np.random.default_rng(17)
    data = rng.integers(0, 256, 1024 * 4096, dtype=np.uint8)
    r = subprocess.run([str(exe)], input=data.tobytes(), capture_output=True)
    assert r.returncode == 0, r.stderr
    got = np.frombuffer(r.stdout, dtype=np.uint64).reshape(1024, 3)
    master = bytes((7 * i + 1) & 0xFF for i in range(32))
    S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(24), 4096))
    want = coracle.hash_fixed(24, data, 1024, 4096, 4096, S)
    assert np.array_equal(got, want)
