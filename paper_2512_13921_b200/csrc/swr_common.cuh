// swr_common.cuh -- internal types shared by the libswr.so kernels (NOT part of
// the C ABI; see include/swr.h for that).  Nothing here is shared with oracle/.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace swr {

constexpr int kEll = 16;  // block length ell = 16

// Everything a kernel needs, passed by value (__grid_constant__-style).
struct Params {
  // SWR operands
  const void* u;
  const void* a;
  void* x;
  const void* dx;
  void* du;
  void* da;
  // Phalanx mixer operands
  const void* q;
  const void* k;
  const void* v;
  void* y;
  const void* dy;
  void* dq;
  void* dk;
  void* dv;
  // carries, fp32 [B,H,D] contiguous
  const float* carry_in;
  float* carry_out;
  const float* mu_in;
  float* mu_out;
  // geometry (elements)
  int64_t B, L, H, D;
  int64_t sx_b, sx_l, sx_h;
  int64_t sa_b, sa_l, sa_h;
  int64_t nb;  // number of 16-token blocks, ceil(L/16)
  int64_t K;   // blocks per walk (FFMA path)
  // Phalanx layer around the mixer (phalanx_layer_mix*):
  // logit_a / logit_k: a / k hold logits, the kernels apply sigma
  // and the backward writes the logits' gradients; q and k are group-shared
  // [B, L, G, D] tensors, head h reading group h / hq (resp. h / hk).
  // The plain mixer ops run with hq = hk = 1 and q/k strides equal to sx.
  int logit_a, logit_k;
  int64_t hq, hk;               // heads per q group, per k group
  int64_t sq_b, sq_l, sq_h;     // element strides of q and dq
  int64_t sk_b, sk_l, sk_h;     // element strides of k and dk
  // tensor-core layer backward with shared groups: per-head dq / dk scratch ([B, L, H, D]
  // contiguous, in the caller's workspace) summed over each group by a second kernel;
  // NULL = not used
  void* gq;
  void* gk;
  // exact-mode forward on the tensor cores (swr_exact_fwd): the exact carrier s_t at
  // the end of every block, [B*H][nb][D] fp32 (from the look-back scan); NULL = B2P
  const float* ex_S;
  float* ex_C;  // exact first pass (Cfg<7>): c_t per block [B*H][nb]; v_t goes to ex_S
  unsigned long long* trace;  // diagnostics (swr_set_trace), NULL = off
  int64_t trace_n;
  uint32_t epoch;  // TC path: launch ticket of the range claims (set by launch_tc)
};

// Recurrence-mode decode step (one token per (b, h); swr_decode_step in swr.h)
struct DecParams {
  const void* u;  // SWR input, or k of the mixer (u^ = k (.) v)
  const void* v;  // mixer: v (pre-gate factor and residual)
  const void* q;  // mixer: q (post-gate)
  const void* a;
  void* x;        // x~ (SWR) or y (mixer)
  float* w;       // state [B,H,D]: local state of the current block
  float* vc;      // state [B,H,D]: carrier v_{t-1}
  float* g;       // state [B,H]: g_t[i]
  int64_t B, H, D;
  int64_t sx_b, sx_h, sa_b, sa_h;
  int64_t pos;    // sequence position of the token
};

// sigma(z) = 1 / (1 + e^-z) in fp32 (the featurization's bounding activation,
// P:1562): e^-z from ex2 and the reciprocal from rcp.approx (__fdividef), a few
// ulp in all (~1e-6 relative at |z| <= 10, inside the fp32 tolerance 1e-5); saturates
// to exactly 0 / 1 for |z| large (__fdividef(1, inf) = 0).
__device__ __forceinline__ float sigmoid_f(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }
// The key gate's sigma for storage type T: bf16 storage takes the single-MUFU
// 1/2 + tanh(z/2)/2 (tanh.approx.f32, ~2^-11 relative, below the bf16 rounding of the
// outputs -- the tensor-core family's form), fp32 storage the accurate sigmoid_f.
template <typename T>
__device__ __forceinline__ float sigmoid_gate(float z) {
  if constexpr (sizeof(T) == 2) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * z));
    return fmaf(0.5f, t, 0.5f);
  } else {
    return sigmoid_f(z);
  }
}

// ---------------------------------------------------------------------------
// storage-dtype traits: 2-channel vector loads/stores, scalar decay access
// ---------------------------------------------------------------------------
template <typename T>
struct IO;

template <>
struct IO<float> {
  using raw = float2;
  static __device__ __forceinline__ raw ld(const float* p) {
    return __ldg(reinterpret_cast<const float2*>(p));
  }
  static __device__ __forceinline__ raw zero() { return make_float2(0.f, 0.f); }
  static __device__ __forceinline__ float2 f2(raw r) { return r; }
  static __device__ __forceinline__ void st(float* p, float x, float y) {
    *reinterpret_cast<float2*>(p) = make_float2(x, y);
  }
  static __device__ __forceinline__ float ld1(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ void st1(float* p, float x) { *p = x; }
};

template <>
struct IO<__nv_bfloat16> {
  using raw = uint32_t;  // two bf16, channel c in the low half (little endian)
  static __device__ __forceinline__ raw ld(const __nv_bfloat16* p) {
    return __ldg(reinterpret_cast<const unsigned int*>(p));
  }
  static __device__ __forceinline__ raw zero() { return 0u; }
  static __device__ __forceinline__ float2 f2(raw r) {
    return make_float2(__uint_as_float(r << 16), __uint_as_float(r & 0xffff0000u));
  }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float x, float y) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(x, y);
  }
  static __device__ __forceinline__ float ld1(const __nv_bfloat16* p) {
    return __bfloat162float(__ldg(p));
  }
  static __device__ __forceinline__ void st1(__nv_bfloat16* p, float x) {
    *p = __float2bfloat16_rn(x);
  }
};

// ---------------------------------------------------------------------------
// deterministic transpose-reduce of 16 per-token partial sums over a group of
// GS lanes (GS power of two, <= 32, lanes of one group contiguous and aligned).
// After the call lane l holds NV = max(1, 16/GS) sums in p[0..NV-1]; p[j] is the
// group total for token tok + j.  Fixed shuffle order => bitwise reproducible.
// ---------------------------------------------------------------------------
template <int KD, int NV>
struct GroupReduce {
  static __device__ __forceinline__ void run(float* p, int lane, int& tok) {
    if constexpr (NV > 1) {
      constexpr int HALF = NV / 2;
      const bool up = (lane & KD) != 0;
#pragma unroll
      for (int j = 0; j < HALF; ++j) {
        const float send = up ? p[j] : p[j + HALF];
        const float keep = up ? p[j + HALF] : p[j];
        p[j] = keep + __shfl_xor_sync(0xffffffffu, send, KD);
      }
      if (up) tok += HALF;
      if constexpr (KD > 1) GroupReduce<KD / 2, HALF>::run(p, lane, tok);
    } else {
      p[0] += __shfl_xor_sync(0xffffffffu, p[0], KD);
      if constexpr (KD > 1) GroupReduce<KD / 2, 1>::run(p, lane, tok);
    }
  }
};

}  // namespace swr
