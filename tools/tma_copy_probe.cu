// Ceiling of the TC kernels' HBM access pattern: copy a [B, L, H, 128] bf16 tensor
// with the same TMA boxes (64 channels x T tokens of one head, 128B swizzle), the same
// persistent contiguous-range walk over (line, block-group) items and an NI-stage
// mbarrier ring -- but no compute -- timed back to back (no L2 flush; 2 x 128 MiB
// footprint > L2) against a grid-stride 16-byte LDG/STG copy and cudaMemcpyAsync.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_copy_probe \
//        tools/tma_copy_probe.cu -lcuda
//   tools/tma_copy_probe [B L H]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));            \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity), "r"(1000000)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
               "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

struct Maps {
  CUtensorMap in, in2, out;
};

// item order 0: (b, h, m) -- a CTA's range walks one head's tokens (the TC kernels);
// order 1: (b, m, h) -- heads fastest (all heads of a token range together)
// NIN input tensors per item (2: the backward's read:write = 2:1), one output
template <int T, int NI, int ORDER, int NIN = 1>
__global__ void __launch_bounds__(64, 1) tcopy(const __grid_constant__ Maps maps, int B, int L, int H) {
  constexpr int kHalf = T * 128, kStage = 2 * kHalf * NIN;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NI * kStage);
  uint64_t* empty = full + NI;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NI; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nbi = L / T;
  const long total = (long)B * H * nbi;
  const int g0 = (int)((long)blockIdx.x * total / gridDim.x), g1 = (int)(((long)blockIdx.x + 1) * total / gridDim.x);
  auto coords = [&](int gi, int& b, int& h, int& t) {
    if (ORDER == 0) {
      const int line = gi / nbi;
      t = (gi - line * nbi) * T;
      b = line / H;
      h = line - b * H;
    } else {
      const int bm = gi / H;
      h = gi - bm * H;
      b = bm / nbi;
      t = (bm - b * nbi) * T;
    }
  };
  if (lane != 0) return;
  if (warp == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int gi = g0; gi < g1; ++gi) {
      int b, h, t;
      coords(gi, b, h, t);
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* st = smem + s * kStage;
      mbar_expect_tx(&full[s], kStage);
      tma_load_4d(st, &maps.in, &full[s], 0, h, t, b);
      tma_load_4d(st + kHalf, &maps.in, &full[s], 64, h, t, b);
      if (NIN == 2) {
        tma_load_4d(st + 2 * kHalf, &maps.in2, &full[s], 0, h, t, b);
        tma_load_4d(st + 3 * kHalf, &maps.in2, &full[s], 64, h, t, b);
      }
      if (++s == NI) s = 0, ph ^= 1;
    }
  } else {
    int s = 0, sp = 0;
    uint32_t ph = 0;
    for (int gi = g0; gi < g1; ++gi) {
      int b, h, t;
      coords(gi, b, h, t);
      mbar_wait(&full[s], ph);
      uint8_t* st = smem + s * kStage;
      tma_store_4d(&maps.out, st, 0, h, t, b);
      tma_store_4d(&maps.out, st + kHalf, 64, h, t, b);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (gi - g0 >= 2) {  // keep two store groups reading
        bulk_wait_read<2>();
        mbar_arrive(&empty[sp]);
        if (++sp == NI) sp = 0;
      }
      if (++s == NI) s = 0, ph ^= 1;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void ldst_copy(const uint4* __restrict__ a, uint4* __restrict__ b, long n) {
  const long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 x0 = a[i], x1 = a[i + stride], x2 = a[i + 2 * stride], x3 = a[i + 3 * stride];
    b[i] = x0;
    b[i + stride] = x1;
    b[i + 2 * stride] = x2;
    b[i + 3 * stride] = x3;
  }
  for (; i < n; i += stride) b[i] = a[i];
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}
static void map4(CUtensorMap* m, void* ptr, int B, int L, int H, int T) {
  cuuint64_t dims[4] = {128, (cuuint64_t)H, (cuuint64_t)L, (cuuint64_t)B};
  cuuint64_t str[3] = {256, (cuuint64_t)H * 256, (cuuint64_t)L * H * 256};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)T, 1}, es[4] = {1, 1, 1, 1};
  if (enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, ptr, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("map failed\n");
    exit(1);
  }
}

template <typename F>
static float b2b(F f, int n = 30, int warm = 5) {
  for (int i = 0; i < warm; ++i) f();
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  for (int i = 0; i < n; ++i) f();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms * 1e3f / n;
}

template <int T, int NI, int ORDER, int NIN = 1>
static float run_tma(const char* name, void* a, void* a2, void* b, int B, int L, int H, int sms, bool print = true) {
  Maps m;
  map4(&m.in, a, B, L, H, T);
  map4(&m.in2, a2, B, L, H, T);
  map4(&m.out, b, B, L, H, T);
  const int smem = NI * 2 * T * 128 * NIN + 1024 + 1024;
  CK(cudaFuncSetAttribute(tcopy<T, NI, ORDER, NIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const float us = b2b([&] { tcopy<T, NI, ORDER, NIN><<<sms, 64, smem>>>(m, B, L, H); });
  CK(cudaGetLastError());
  const double bytes = (double)B * L * H * 256 * (NIN + 1);
  if (print)
    printf("%-22s in=%d T=%3d NI=%2d stage=%3d KB inflight=%4d KB: %7.1f us %6.0f GB/s\n", name, NIN, T, NI,
           2 * T * 128 * NIN / 1024, NI * 2 * T * 128 * NIN / 1024, us, bytes / us / 1e3);
  return us;
}
// a step-like pair back to back: 1-in copy (fwd traffic) then 2-in copy (bwd traffic)
template <int TF, int NF, int TB, int NB>
static void run_step(void* a, void* a2, void* b, void* b2, int B, int L, int H, int sms) {
  Maps mf, mb;
  map4(&mf.in, a, B, L, H, TF);
  map4(&mf.in2, a, B, L, H, TF);
  map4(&mf.out, b, B, L, H, TF);
  map4(&mb.in, a, B, L, H, TB);
  map4(&mb.in2, a2, B, L, H, TB);
  map4(&mb.out, b2, B, L, H, TB);
  const int sf = NF * 2 * TF * 128 + 2048, sb = NB * 4 * TB * 128 + 2048;
  CK(cudaFuncSetAttribute(tcopy<TF, NF, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sf));
  CK(cudaFuncSetAttribute(tcopy<TB, NB, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb));
  const float us = b2b([&] {
    tcopy<TF, NF, 0, 1><<<sms, 64, sf>>>(mf, B, L, H);
    tcopy<TB, NB, 0, 2><<<sms, 64, sb>>>(mb, B, L, H);
  });
  const double bytes = (double)B * L * H * 256 * 5;
  printf("step-like pair fwd T=%d NI=%d + bwd T=%d NI=%d: %7.1f us %6.0f GB/s\n", TF, NF, TB, NB, us, bytes / us / 1e3);
}

// initcheck probe (tma_copy_probe init): a TMA store into fresh memory, then a plain
// kernel reads it -- does compute-sanitizer initcheck count the TMA write?
static int init_probe() {
  const int B = 1, L = 64, H = 16;
  const size_t nbytes = (size_t)B * L * H * 128 * 2;
  void *a, *b, *c;
  CK(cudaMalloc(&a, nbytes));
  CK(cudaMalloc(&b, nbytes));  // never written by the host: only the TMA stores write it
  CK(cudaMalloc(&c, nbytes));
  CK(cudaMemset(a, 1, nbytes));
  Maps m;
  map4(&m.in, a, B, L, H, 32);
  map4(&m.in2, a, B, L, H, 32);
  map4(&m.out, b, B, L, H, 32);
  const int smem = 4 * 2 * 32 * 128 + 2048;
  CK(cudaFuncSetAttribute(tcopy<32, 4, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  tcopy<32, 4, 0, 1><<<4, 64, smem>>>(m, B, L, H);
  ldst_copy<<<4, 128>>>((const uint4*)b, (uint4*)c, (long)(nbytes / 16));  // reads the TMA-written bytes
  CK(cudaDeviceSynchronize());
  unsigned char h[4];
  CK(cudaMemcpy(h, c, 4, cudaMemcpyDeviceToHost));
  printf("init probe: first bytes %d %d (expect 1 1)\n", h[0], h[1]);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "init") return init_probe();
  const int B = argc > 1 ? atoi(argv[1]) : 8, L = argc > 2 ? atoi(argv[2]) : 4096, H = argc > 3 ? atoi(argv[3]) : 16;
  const size_t n = (size_t)B * L * H * 128, nbytes = n * 2;
  const double bytes = 2.0 * nbytes;  // read + write (plain copies)
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void *a, *b;
  CK(cudaMalloc(&a, nbytes));
  CK(cudaMalloc(&b, nbytes));
  CK(cudaMemset(a, 1, nbytes));
  CK(cudaMemset(b, 0, nbytes));
  printf("B=%d L=%d H=%d D=128 bf16: %.1f MiB per tensor, %d SMs\n", B, L, H, nbytes / 1048576.0, sms);
  float us = b2b([&] { CK(cudaMemcpyAsync(b, a, nbytes, cudaMemcpyDeviceToDevice)); });
  printf("%-34s %7.1f us %6.0f GB/s\n", "cudaMemcpyAsync D2D", us, bytes / us / 1e3);
  for (int per : {4, 8, 16}) {
    us = b2b([&] { ldst_copy<<<sms * per, 256>>>((const uint4*)a, (uint4*)b, (long)(nbytes / 16)); });
    printf("ldst_copy grid=%3d x SMs x 256 thr      %7.1f us %6.0f GB/s\n", per, us, bytes / us / 1e3);
  }
  void *a2, *b2;
  CK(cudaMalloc(&a2, nbytes));
  CK(cudaMalloc(&b2, nbytes));
  CK(cudaMemset(a2, 1, nbytes));
  run_tma<64, 8, 0>("line-major (fwd now)", a, a2, b, B, L, H, sms);
  run_tma<64, 4, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<64, 6, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<32, 4, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<32, 6, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<32, 8, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<32, 12, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<16, 8, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<16, 12, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<16, 16, 0>("line-major", a, a2, b, B, L, H, sms);
  run_tma<32, 8, 0, 2>("line-major (bwd now)", a, a2, b, B, L, H, sms);
  run_tma<32, 3, 0, 2>("line-major", a, a2, b, B, L, H, sms);
  run_tma<32, 4, 0, 2>("line-major", a, a2, b, B, L, H, sms);
  run_tma<32, 6, 0, 2>("line-major", a, a2, b, B, L, H, sms);
  run_tma<16, 6, 0, 2>("line-major", a, a2, b, B, L, H, sms);
  run_tma<16, 8, 0, 2>("line-major", a, a2, b, B, L, H, sms);
  run_tma<16, 12, 0, 2>("line-major", a, a2, b, B, L, H, sms);
  run_tma<32, 4, 1, 2>("heads-fastest", a, a2, b, B, L, H, sms);
  run_tma<32, 8, 1>("heads-fastest", a, a2, b, B, L, H, sms);
  run_step<64, 8, 32, 8>(a, a2, b, b2, B, L, H, sms);
  run_step<32, 8, 32, 4>(a, a2, b, b2, B, L, H, sms);
  run_step<32, 6, 32, 4>(a, a2, b, b2, B, L, H, sms);
  run_step<16, 16, 16, 8>(a, a2, b, b2, B, L, H, sms);
  return 0;
}
