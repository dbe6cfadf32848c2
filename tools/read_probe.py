"""Pure-read HBM ceiling with plain 16-byte loads (LDG.128), for comparison with the
TMA-fed kernels' read rates.  Builds a tiny extension with nvcc."""
import os, sys
import torch
from torch.utils.cpp_extension import load_inline
src = r"""
#include <torch/extension.h>
__global__ void rd(const uint4* __restrict__ p, long n, unsigned* out, int unroll) {
  unsigned acc = 0;
  long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  #pragma unroll 8
  for (; i < n; i += stride) { uint4 v = __ldg(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void cp(const uint4* __restrict__ p, uint4* __restrict__ q, long n) {
  long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  #pragma unroll 8
  for (; i < n; i += stride) q[i] = __ldg(p + i);
}
void run_rd(torch::Tensor x, torch::Tensor out, int blocks, int threads) {
  rd<<<blocks, threads>>>((const uint4*)x.data_ptr(), x.numel() * x.element_size() / 16, (unsigned*)out.data_ptr(), 8);
}
void run_cp(torch::Tensor x, torch::Tensor y, int blocks, int threads) {
  cp<<<blocks, threads>>>((const uint4*)x.data_ptr(), (uint4*)y.data_ptr(), x.numel() * x.element_size() / 16);
}
"""
m = load_inline("rdprobe", cpp_sources="void run_rd(torch::Tensor x, torch::Tensor out, int blocks, int threads); void run_cp(torch::Tensor x, torch::Tensor y, int blocks, int threads);",
                cuda_sources=src, functions=["run_rd", "run_cp"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                build_directory=os.environ.get("TMPBUILD", "/tmp/rdprobe"), verbose=False)
x = torch.empty(512 << 20, dtype=torch.uint8, device="cuda"); x.fill_(1)
y = torch.empty_like(x)
out = torch.zeros(1, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for blocks, threads in [(148 * 4, 512), (148 * 8, 256), (148 * 16, 256)]:
    for name, f, by in (("read", lambda: m.run_rd(x, out, blocks, threads), x.numel()),
                        ("copy", lambda: m.run_cp(x, y, blocks, threads), 2 * x.numel())):
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[5]
        print(f"{name} grid {blocks}x{threads}: {by / t / 1e6:.0f} GB/s", flush=True)
