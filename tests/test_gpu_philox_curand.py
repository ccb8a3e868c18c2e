"""Independent pin of the device Philox4x32-10: the
library's generator (ens_philox4x32_10, and the SDE noise stream's raw words
from ens_sde_noise) must equal cuRAND's own curand_Philox4x32_10 device
function (curand_philox4x32_x.h, shipped with the CUDA toolkit) word for word.
The cuRAND side is a separate tiny program compiled here with nvcc; it shares
nothing with the library (-m gpu)."""
import os
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2304_06835_b200 as ens

pytestmark = pytest.mark.gpu

CURAND_REF = r'''
#include <cstdio>
#include <cstdint>
#include <vector>
#include <curand_philox4x32_x.h>
__global__ void k(const uint4* c, const uint2* key, uint4* o, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = curand_Philox4x32_10(c[i], key[i]);
}
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int n; if (fread(&n, 4, 1, f) != 1) return 2;
  std::vector<uint4> c(n); std::vector<uint2> key(n), dummy;
  if (fread(c.data(), 16, n, f) != (size_t)n || fread(key.data(), 8, n, f) != (size_t)n) return 3;
  fclose(f);
  uint4 *dc, *dout; uint2* dk;
  cudaMalloc(&dc, 16 * n); cudaMalloc(&dk, 8 * n); cudaMalloc(&dout, 16 * n);
  cudaMemcpy(dc, c.data(), 16 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, key.data(), 8 * n, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(dc, dk, dout, n);
  std::vector<uint4> o(n);
  if (cudaMemcpy(o.data(), dout, 16 * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 4;
  f = fopen(argv[2], "wb"); fwrite(o.data(), 16, n, f); fclose(f);
  return 0;
}
'''


def _nvcc():
    for c in [os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")]:
        if c and os.path.exists(c):
            return c
    pytest.skip("nvcc not available")


def _curand_philox(tmp_path: Path, ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
    src = tmp_path / "curand_ref.cu"
    src.write_text(CURAND_REF)
    exe = tmp_path / "curand_ref"
    subprocess.run([_nvcc(), "-O2", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe), str(src)],
                   check=True, capture_output=True)
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    n = ctr.shape[0]
    with open(inp, "wb") as f:
        f.write(np.int32(n).tobytes())
        f.write(np.ascontiguousarray(ctr, dtype=np.uint32).tobytes())
        f.write(np.ascontiguousarray(key, dtype=np.uint32).tobytes())
    subprocess.run([str(exe), str(inp), str(out)], check=True)
    return np.fromfile(out, dtype=np.uint32).reshape(n, 4)


def test_philox_equals_curand(tmp_path):
    rng = np.random.default_rng(0x9E3779B9)
    n = 1 << 16
    ctr = rng.integers(0, 1 << 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 1 << 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    ctr[:4] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4, [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [1, 2, 3, 4]]
    key[:4] = [[0, 0], [0xFFFFFFFF] * 2, [0xA4093822, 0x299F31D0], [5, 6]]
    ref = _curand_philox(tmp_path, ctr, key)
    dev = torch.device("cuda:0")
    got = ens.philox4x32_10(torch.from_numpy(ctr.view(np.int32)).to(dev), torch.from_numpy(key.view(np.int32)).to(dev))
    np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), ref)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_noise_stream_words_equal_curand(tmp_path, dtype):
    """Trajectory g's call c has counter (c lo, g lo, g hi, c hi) and key = seed (DESIGN R8)."""
    seed, N, nsteps, step0, off = 0xC4C4C4C4DEADBEEF, 300, 9, 5, (1 << 33) + 7
    words, _ = ens.sde_noise(N, nsteps, seed=seed, dtype=dtype, step0=step0, index_offset=off)
    per = 4 if dtype == torch.float32 else 2
    c0 = 3 * step0 // per
    ncalls = words.shape[0]
    g = off + np.arange(N, dtype=np.uint64)
    c = c0 + np.arange(ncalls, dtype=np.uint64)
    G, C = np.meshgrid(g, c)                       # [ncalls, N]
    ctr = np.stack([C & 0xFFFFFFFF, G & 0xFFFFFFFF, G >> 32, C >> 32], -1).reshape(-1, 4).astype(np.uint32)
    key = np.tile(np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint64), (ctr.shape[0], 1)).astype(np.uint32)
    ref = _curand_philox(tmp_path, ctr, key).reshape(ncalls, N, 4).transpose(0, 2, 1)
    np.testing.assert_array_equal(words.cpu().numpy().view(np.uint32), ref)
