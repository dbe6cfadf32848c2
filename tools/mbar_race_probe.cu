// Does compute-sanitizer racecheck understand an mbarrier hand-off?  Warp 0 writes a
// shared buffer and arrives (release) on an mbarrier; warp 1 waits on the phase
// (acquire) and reads it; then the roles swap through a second mbarrier, twice -- the
// pattern of the TC kernels' slot rings.  Correct by the PTX memory model; a racecheck
// report here is the tool not modelling mbarrier phases.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/mbar_race_probe tools/mbar_race_probe.cu
//   compute-sanitizer --tool racecheck tools/mbar_race_probe
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}

__global__ void probe(float* out) {
  __shared__ float buf[32];
  __shared__ uint64_t full, empty;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  for (int it = 0; it < 4; ++it) {
    const uint32_t ph = it & 1;
    if (warp == 0) {
      if (it > 0) wait(&empty, ph ^ 1);  // the reader released the buffer
      buf[lane] = (float)(it * 32 + lane);
      __syncwarp();
      if (lane == 0) arrive(&full);
    } else {
      wait(&full, ph);
      acc += buf[lane ^ 1];
      __syncwarp();
      if (lane == 0) arrive(&empty);
    }
  }
  if (warp == 1) out[lane] = acc;
}

int main() {
  float* d;
  cudaMalloc(&d, 32 * sizeof(float));
  probe<<<1, 64>>>(d);
  float h[32];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("probe %s: out[0] = %.0f (expect %d)\n", cudaGetErrorString(cudaGetLastError()), h[0], 1 + 33 + 65 + 97);
  return 0;
}
