// swr_ffma.cu -- the portable kernel family (SWR_PATH_FFMA): Block Two-Pass on
// CUDA cores, any storage dtype, D in {16, 32, 64, 128}.
//
// Mapping.  A thread owns one vector of adjacent channels of one (b, h) -- 16
// bytes in the forward (fwd_stream), four channels in the backward
// (bwd_ffma_vec) -- and walks a run of K consecutive 16-token blocks ("chunk").
// For every block it
//   * loads the 16 decays and 16 token vectors of its channels (coalesced across
//     the lanes of the head: consecutive lanes own consecutive channel vectors),
//   * Pass I  (Alg. 4, Alg. 5): w_t = L_t u_t as the block-local
//     recurrence w[i] = a[i] w[i-1] + u[i], w[0] = u[0] (L_t excludes a_t[0],
//     P:594) -- the same product as the dense 16x16 transfer, 16x fewer FLOPs,
//   * carrier v_t = w_t[15] kept in registers for the next block,
//   * Pass II (Alg. 4): x~_t[i] = w_t[i] + g_t[i] v_{t-1} with
//     g_t[i] = a_t[0]...a_t[i] built by running products (products
//     only, never ratios).
// The first block of a chunk gets v_{t-1} by recomputing the previous block's
// Pass I with the SAME device function (halo), so results do not depend on the
// chunk size.  Backward walks the chunk in reverse time order carrying
// mu_t = a_{t+1}[0] lambda_{t+1}[0] (DESIGN.md Appendix "backward").
#include <algorithm>
#include <type_traits>

#include "swr_common.cuh"

namespace swr {

// ---------------------------------------------------------------------------
// forward, streamed: a thread owns one 16-byte vector of channels (VC = 8 bf16 or
// 4 fp32) and walks its chunk token by token -- Pass I as the local recurrence
// (restarted at each block start, w[0] = u[0]), g_t[i] = a_t[0]...a_t[i] as
// a running product (products only), Pass II x~ = w + g v_{t-1},
// v_t = w_t[15] -- with one 16-byte load and store per token and tensor and no
// per-block arrays.
// ---------------------------------------------------------------------------
template <typename T>
struct Vec16;
template <>
struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void to_f(const uint4& r, float (&f)[8]) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      f[2 * q] = __uint_as_float(w[q] << 16);
      f[2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
    }
  }
  static __device__ __forceinline__ uint4 from_f(const float (&f)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 b2 = __floats2bfloat162_rn(f[2 * q], f[2 * q + 1]);
      w[q] = *reinterpret_cast<uint32_t*>(&b2);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct Vec16<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void to_f(const uint4& r, float (&f)[4]) {
    f[0] = __uint_as_float(r.x);
    f[1] = __uint_as_float(r.y);
    f[2] = __uint_as_float(r.z);
    f[3] = __uint_as_float(r.w);
  }
  static __device__ __forceinline__ uint4 from_f(const float (&f)[4]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
};

// Pass-I input of one token: u (SWR) or u^ = k (.) v (pre-gate); LAYER: k
// may be a logit, k = sigma(zk), read from its group's tensor at ko.
template <typename T, bool MIX, bool LAYER>
__device__ __forceinline__ void load_u16(const Params& p, int64_t off, int64_t ko, bool valid,
                                         float (&u)[Vec16<T>::N]) {
  constexpr int VC = Vec16<T>::N;
  if (!valid) {
#pragma unroll
    for (int e = 0; e < VC; ++e) u[e] = 0.f;
    return;
  }
  if constexpr (!MIX) {
    Vec16<T>::to_f(__ldg(reinterpret_cast<const uint4*>((const T*)p.u + off)), u);
  } else {
    float kk[VC], vv[VC];
    Vec16<T>::to_f(__ldg(reinterpret_cast<const uint4*>((const T*)p.k + (LAYER ? ko : off))), kk);
    Vec16<T>::to_f(__ldg(reinterpret_cast<const uint4*>((const T*)p.v + off)), vv);
    if (LAYER && p.logit_k) {
#pragma unroll
      for (int e = 0; e < VC; ++e) kk[e] = sigmoid_gate<T>(kk[e]);
    }
#pragma unroll
    for (int e = 0; e < VC; ++e) u[e] = __fmul_rn(kk[e], vv[e]);
  }
}

// decay of token n: a, or (LAYER, logit_a) a = sigma(za); pad a = 1 past L
template <typename T, bool LAYER>
__device__ __forceinline__ float ld_decay(const Params& p, const T* A, int64_t n, bool valid) {
  if (!valid) return 1.f;
  const float z = IO<T>::ld1(A + n * p.sa_l);
  return (LAYER && p.logit_a) ? sigmoid_f(z) : z;
}

#ifndef SWR_FFMA_FWD_SG
#define SWR_FFMA_FWD_SG 16  // SWR forward: tokens whose loads are issued together
#endif
#ifndef SWR_FFMA_FWD_MINB
#define SWR_FFMA_FWD_MINB 1
#endif
#ifndef SWR_FFMA_MIXF_MINB
#define SWR_FFMA_MIXF_MINB 4  // mixer forward: 128 registers, 4 CTAs per SM (fp32 d=128 252 -> 180 us, d=16 208 -> 189 us)
#endif
#ifndef SWR_FFMA_MIXF_GROUP
#define SWR_FFMA_MIXF_GROUP 4  // mixer forward: tokens whose loads are issued together
#endif
// LAYER: the Phalanx layer around the mixer (phalanx_layer_mix): logits and
// group-shared q / k (Params); otherwise the plain SWR / mixer ops.
template <typename T, bool MIX, bool LAYER>
__global__ void __launch_bounds__(128, MIX ? SWR_FFMA_MIXF_MINB : SWR_FFMA_FWD_MINB) fwd_stream(const Params p) {
  constexpr int VC = Vec16<T>::N;
  const int TPH = (int)p.D / VC;  // threads per head
  const int HPC = 128 / TPH;      // heads per CTA
  const int tid = threadIdx.x;
  const int hh = tid / TPH;
  const int c = VC * (tid % TPH);
  const int64_t b = blockIdx.z;
  const int64_t h = (int64_t)blockIdx.y * HPC + hh;
  if (h >= p.H) return;
  const int64_t t_lo = (int64_t)blockIdx.x * p.K;
  const int64_t t_hi = min(t_lo + p.K, p.nb);
  const T* A = (const T*)p.a + b * p.sa_b + h * p.sa_h;
  const int64_t xo = b * p.sx_b + h * p.sx_h + c;
  // group-shared gates (LAYER): q of group h / hq, k of group h / hk
  const int64_t qo = LAYER ? b * p.sq_b + (h / p.hq) * p.sq_h + c : xo;
  const int64_t ko = LAYER ? b * p.sk_b + (h / p.hk) * p.sk_h + c : xo;
  const int64_t sql = LAYER ? p.sq_l : p.sx_l, skl = LAYER ? p.sk_l : p.sx_l;
  const int64_t co = (b * p.H + h) * p.D + c;

  float v[VC];  // carrier v_{t-1}; v_{-1} = carry_in or 0
#pragma unroll
  for (int e = 0; e < VC; ++e) v[e] = 0.f;
  if (t_lo == 0) {
    if (p.carry_in) {
#pragma unroll
      for (int e = 0; e < VC; ++e) v[e] = p.carry_in[co + e];
    }
  } else {  // halo: Pass I of block t_lo - 1
    float w[VC];
#pragma unroll
    for (int i = 0; i < kEll; ++i) {
      const int64_t n = (t_lo - 1) * kEll + i;
      const bool valid = n < p.L;
      const float a = ld_decay<T, LAYER>(p, A, n, valid);
      float u[VC];
      load_u16<T, MIX, LAYER>(p, xo + n * p.sx_l, ko + n * skl, valid, u);
#pragma unroll
      for (int e = 0; e < VC; ++e) w[e] = (i == 0) ? u[e] : fmaf(a, w[e], u[e]);
    }
#pragma unroll
    for (int e = 0; e < VC; ++e) v[e] = w[e];
  }

  for (int64_t t = t_lo; t < t_hi; ++t) {
    float w[VC];
    float g = 1.f;
    // SWR: the block's loads first (stores to x may alias them, so the compiler
    // cannot hoist them past the stores): 16 decays and 16 raw 16-byte vectors.
    // Mixer: the loads of MG tokens at a time (a, k, v, q; v serves the pre-gate and
    // the residual), then their arithmetic and stores.
    if constexpr (!MIX) {
      constexpr int SG = SWR_FFMA_FWD_SG;
#pragma unroll
      for (int i0 = 0; i0 < kEll; i0 += SG) {
        float ab[SG];
        uint4 ub[SG];
#pragma unroll
        for (int m = 0; m < SG; ++m) {
          const int64_t n = t * kEll + i0 + m;
          const bool valid = n < p.L;
          ab[m] = valid ? IO<T>::ld1(A + n * p.sa_l) : 1.f;  // pad: a = 1 (carry_out = state at L-1)
          ub[m] = valid ? __ldg(reinterpret_cast<const uint4*>((const T*)p.u + xo + n * p.sx_l)) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int m = 0; m < SG; ++m) {
          const int i = i0 + m;
          const int64_t n = t * kEll + i;
          float u[VC];
          Vec16<T>::to_f(ub[m], u);
          g *= ab[m];  // g_t[i] = a_t[0] ... a_t[i]
          float x[VC];
#pragma unroll
          for (int e = 0; e < VC; ++e) {
            w[e] = (i == 0) ? u[e] : fmaf(ab[m], w[e], u[e]);  // Pass I
            x[e] = fmaf(g, v[e], w[e]);                         // Pass II: x~ = w + g v_{t-1}
          }
          if (n < p.L) *reinterpret_cast<uint4*>((T*)p.x + xo + n * p.sx_l) = Vec16<T>::from_f(x);
        }
      }
    } else {
      constexpr int MG = SWR_FFMA_MIXF_GROUP;
#pragma unroll
      for (int i0 = 0; i0 < kEll; i0 += MG) {
        float ar[MG];
        uint4 kr[MG], vr[MG], qr[MG];
#pragma unroll
        for (int m = 0; m < MG; ++m) {
          const int64_t n = t * kEll + i0 + m;
          const bool valid = n < p.L;
          ar[m] = valid ? IO<T>::ld1(A + n * p.sa_l) : 1.f;
          kr[m] = valid ? __ldg(reinterpret_cast<const uint4*>((const T*)p.k + ko + n * skl)) : make_uint4(0, 0, 0, 0);
          vr[m] = valid ? __ldg(reinterpret_cast<const uint4*>((const T*)p.v + xo + n * p.sx_l)) : make_uint4(0, 0, 0, 0);
          qr[m] = valid ? __ldg(reinterpret_cast<const uint4*>((const T*)p.q + qo + n * sql)) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int m = 0; m < MG; ++m) {
          const int i = i0 + m;
          const int64_t n = t * kEll + i;
          float a = ar[m];
          if (LAYER && p.logit_a && n < p.L) a = sigmoid_f(a);  // a = sigma(za)
          float kk[VC], vv[VC], qq[VC], u[VC];
          Vec16<T>::to_f(kr[m], kk);
          Vec16<T>::to_f(vr[m], vv);
          Vec16<T>::to_f(qr[m], qq);
          if (LAYER && p.logit_k) {
#pragma unroll
            for (int e = 0; e < VC; ++e) kk[e] = sigmoid_gate<T>(kk[e]);  // k = sigma(zk)
          }
#pragma unroll
          for (int e = 0; e < VC; ++e) u[e] = __fmul_rn(kk[e], vv[e]);  // u^ = k (.) v
          g *= a;
          float x[VC];
#pragma unroll
          for (int e = 0; e < VC; ++e) {
            w[e] = (i == 0) ? u[e] : fmaf(a, w[e], u[e]);  // Pass I
            x[e] = fmaf(g, v[e], w[e]);                      // Pass II
            x[e] = fmaf(qq[e], x[e], vv[e]);                 // post-gate with residual
          }
          if (n < p.L) *reinterpret_cast<uint4*>((T*)p.y + xo + n * p.sx_l) = Vec16<T>::from_f(x);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < VC; ++e) v[e] = w[e];  // v_t = w_t[15]
  }
  if (t_hi == p.nb && p.carry_out) {
#pragma unroll
    for (int e = 0; e < VC; ++e) p.carry_out[co + e] = v[e];
  }
}

// ---------------------------------------------------------------------------
// backward, vectorised: a three-pass walk per block with a thread owning
// VC channels (one 8- or 16-byte vector per tensor and token), per-block base
// pointers advanced by the token stride (no per-token 64-bit index products), and
// the adjoint lambda_t staged in dynamic shared memory as [token][VC/4][thread]
// float4s.  The da sum over the head's channels is VC-channel chains, then the lane
// transpose-reduce.
// ---------------------------------------------------------------------------
#ifndef SWR_FFMA_BWD_VC
#define SWR_FFMA_BWD_VC 4  // bf16 channels per thread (4: 8-byte vectors; 8: 16-byte, 20% slower at d=16)
#endif
#ifndef SWR_FFMA_BWDV_UNROLL
#define SWR_FFMA_BWDV_UNROLL 4  // pass C unroll (16 spills 1.3 KB: 3x slower; 2 or 8: 5-15% slower)
#endif
#ifndef SWR_FFMA_MIXBV_UNROLL
#define SWR_FFMA_MIXBV_UNROLL 1  // the mixer pass C: groups of SWR_FFMA_BWD_CG tokens, not unrolled further (spills)
#endif
#ifndef SWR_FFMA_BWD_MINB
#define SWR_FFMA_BWD_MINB 4  // 128 registers
#endif
#ifndef SWR_FFMA_BWD_CG
#define SWR_FFMA_BWD_CG 4  // Pass C: tokens whose loads are issued together
#endif
template <bool MIX>
struct CUnrollV {
  static constexpr int v = MIX ? SWR_FFMA_MIXBV_UNROLL : SWR_FFMA_BWDV_UNROLL;
};

template <typename T, int VC>
struct VecN {
  static_assert(sizeof(T) * VC == 8 || sizeof(T) * VC == 16, "8- or 16-byte vectors");
  using raw = typename std::conditional<sizeof(T) * VC == 8, uint2, uint4>::type;
  static __device__ __forceinline__ raw ld(const T* p) { return __ldg(reinterpret_cast<const raw*>(p)); }
  static __device__ __forceinline__ raw zero() { raw r; memset(&r, 0, sizeof r); return r; }
  static __device__ __forceinline__ void to_f(const raw& r, float (&f)[VC]) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&r);
    if constexpr (sizeof(T) == 2) {
#pragma unroll
      for (int q = 0; q < VC / 2; ++q) {
        f[2 * q] = __uint_as_float(w[q] << 16);
        f[2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
      }
    } else {
#pragma unroll
      for (int q = 0; q < VC; ++q) f[q] = __uint_as_float(w[q]);
    }
  }
  static __device__ __forceinline__ void st(T* p, const float (&f)[VC]) {
    raw r;
    uint32_t* w = reinterpret_cast<uint32_t*>(&r);
    if constexpr (sizeof(T) == 2) {
#pragma unroll
      for (int q = 0; q < VC / 2; ++q) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(f[2 * q], f[2 * q + 1]);
        w[q] = *reinterpret_cast<uint32_t*>(&b2);
      }
    } else {
#pragma unroll
      for (int q = 0; q < VC; ++q) w[q] = __float_as_uint(f[q]);
    }
    *reinterpret_cast<raw*>(p) = r;
  }
};

// LAYER (phalanx_layer_mix_bwd, mixer only): a and k may be logits (sigma applied
// on load; dza = da a (1 - a), dzk = dk k (1 - k)), and q / k are group-shared
// tensors [B, L, G, D] read by hq / hk consecutive heads; their gradients are the
// sums over the group's heads, formed in the CTA in a fixed head
// order (deterministic): the CTA holds NTH / TPH heads, a multiple of hq and hk.
// dq is staged over the lambda slots it replaces, dk in a second buffer.
template <typename T, int VC, int TPH, bool MIX, bool LAYER = false, int NTH = 128>
__global__ void __launch_bounds__(NTH, NTH == 128 ? ((LAYER || (!MIX && sizeof(T) == 2)) ? 3 : SWR_FFMA_BWD_MINB) : 1)
    bwd_ffma_vec(const Params p) {
  using V = VecN<T, VC>;
  using io = IO<T>;
  static_assert(!LAYER || MIX, "the layer options apply to the mixer");
  constexpr int HPC = NTH / TPH;
  constexpr int GS = TPH;  // lanes per head (<= 32)
  constexpr int NQ = VC / 4;
  extern __shared__ float4 slam[];  // [kEll][NQ][NTH]; LAYER: then dk staging [kEll][NQ][NTH]
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int hh = tid / TPH;
  const int c = VC * (tid % TPH);
  const int64_t b = blockIdx.z;
  const int64_t h = (int64_t)blockIdx.y * HPC + hh;
  const bool act = h < p.H;
  const int64_t hc = act ? h : p.H - 1;  // inactive threads read a valid head, store nothing
  const int64_t t_lo = (int64_t)blockIdx.x * p.K;
  const int64_t t_hi = min(t_lo + p.K, p.nb);
  const int64_t sl = p.sx_l, sal = p.sa_l;
  const int64_t xo = b * p.sx_b + hc * p.sx_h + c;
  // group-shared gates (LAYER): q of group h / hq, k of group h / hk
  const int64_t qo = LAYER ? b * p.sq_b + (hc / p.hq) * p.sq_h + c : xo;
  const int64_t ko = LAYER ? b * p.sk_b + (hc / p.hk) * p.sk_h + c : xo;
  const int64_t sql = LAYER ? p.sq_l : sl, skl = LAYER ? p.sk_l : sl;
  const bool sig_a = LAYER && p.logit_a, sig_k = LAYER && p.logit_k;
  const int64_t co = (b * p.H + hc) * p.D + c;
  const T* A0 = (const T*)p.a + b * p.sa_b + hc * p.sa_h;
  T* dA = (T*)p.da + b * p.sa_b + hc * p.sa_h;
  auto lam_at = [&](int i, int q) -> float4& { return slam[(i * NQ + q) * NTH + tid]; };
  auto dk_at = [&](int i, int q, int th) -> float4& { return slam[((kEll + i) * NQ + q) * NTH + th]; };
  auto dq_at = [&](int i, int q, int th) -> float4& { return slam[(i * NQ + q) * NTH + th]; };
  auto decay = [&](const T* ap) {  // a, or a = sigma(za)
    const float z = io::ld1(ap);
    return sig_a ? sigmoid_f(z) : z;
  };

  // decays of a block (pad a = 1 past L)
  auto load_a = [&](int64_t n0, int lim, float (&a)[kEll]) {
    const T* ap = A0 + n0 * sal;
#pragma unroll
    for (int i = 0; i < kEll; ++i) {
      a[i] = (i < lim) ? decay(ap) : 1.f;
      ap += sal;
    }
  };
  // A stream of Pass-I inputs (u, or u^ = k (.) v: pre-gate) or of adjoint
  // inputs (dx, or G = dy (.) q), walked by pointers stepped by the token strides.
  struct Src {
    const T* p0;
    const T* p1;   // mixer: the second factor
    int64_t s0, s1;
    bool sig0;     // LAYER: p0 holds logits (k = sigma(zk))
    __device__ __forceinline__ void load(bool valid, float (&x)[VC]) const {
      if constexpr (!MIX) {
        V::to_f(valid ? V::ld(p0) : V::zero(), x);
      } else {
        float f0[VC], f1[VC];
        V::to_f(valid ? V::ld(p0) : V::zero(), f0);
        V::to_f(valid ? V::ld(p1) : V::zero(), f1);
        if (LAYER && sig0) {
#pragma unroll
          for (int e = 0; e < VC; ++e) f0[e] = valid ? sigmoid_gate<T>(f0[e]) : 0.f;
        }
#pragma unroll
        for (int e = 0; e < VC; ++e) x[e] = __fmul_rn(f0[e], f1[e]);
      }
    }
    __device__ __forceinline__ void fwd() {
      p0 += s0;
      if constexpr (MIX) p1 += s1;
    }
    __device__ __forceinline__ void back() {
      p0 -= s0;
      if constexpr (MIX) p1 -= s1;
    }
  };
  auto src_u = [&](int64_t n) {
    return MIX ? Src{(const T*)p.k + ko + n * skl, (const T*)p.v + xo + n * sl, skl, sl, sig_k}
               : Src{(const T*)p.u + xo + n * sl, nullptr, sl, 0, false};
  };
  auto src_g = [&](int64_t n) {
    return MIX ? Src{(const T*)p.dy + xo + n * sl, (const T*)p.q + qo + n * sql, sl, sql, false}
               : Src{(const T*)p.dx + xo + n * sl, nullptr, sl, 0, false};
  };

  // mu for block t_hi - 1: a_{t_hi}[0] lambda_{t_hi}[0] from the right halo block, or mu_in
  float mu[VC];
#pragma unroll
  for (int e = 0; e < VC; ++e) mu[e] = 0.f;
  if (t_hi == p.nb) {
    if (p.mu_in) {
#pragma unroll
      for (int e = 0; e < VC; ++e) mu[e] = p.mu_in[co + e];
    }
  } else {
    const int64_t n0 = t_hi * kEll;
    const int lim = (p.L - n0 < kEll) ? (int)(p.L - n0) : kEll;
    float a[kEll];
    load_a(n0, lim, a);
    float l[VC];
    Src gsrc = src_g(n0 + kEll - 1);
    gsrc.load(kEll - 1 < lim, l);  // l[15] = G[15]
#pragma unroll
    for (int i = kEll - 2; i >= 0; --i) {
      float g[VC];
      gsrc.back();
      gsrc.load(i < lim, g);
#pragma unroll
      for (int e = 0; e < VC; ++e) l[e] = fmaf(a[i + 1], l[e], g[e]);
    }
#pragma unroll
    for (int e = 0; e < VC; ++e) mu[e] = a[0] * l[e];
  }

  if constexpr (!MIX && sizeof(T) == 2) {
    // SWR (bf16): every u block is read once and nothing lives in local memory.  Per block t
    // (reverse walk): A) w_{t-1} by the local solve of block t-1 into one of two w stash
    // slots, v_{t-1} = w_{t-1}[15]; BC) one reverse sweep: lambda[i] = G[i] + a[i+1]
    // lambda[i+1], r[i] = a[i+1] r[i+1], du = lambda + r mu, and the da terms
    // du . w_t[i-1] (w_t from the other stash slot, written by A one step earlier) and
    // g[i-1] lambda . v_{t-1}.  Fully unrolled: every per-token array is registers.
    // The chunk's last block first fills its stash slot from u_t.
    auto w_at = [&](int slot, int i, int q) -> float4& {
      return slam[((slot * kEll + i) * NQ + q) * NTH + tid];
    };
    auto solve_into = [&](int64_t nb0, int slot, int lim, float (&wl)[VC]) {  // Pass I of a block into a slot
      const T* ap = A0 + nb0 * sal;
      Src usrc = src_u(nb0);
#pragma unroll 4
      for (int i = 0; i < kEll; ++i) {
        const float a = (i < lim) ? decay(ap) : 1.f;
        float u[VC];
        usrc.load(i < lim, u);
        ap += sal;
        usrc.fwd();
#pragma unroll
        for (int e = 0; e < VC; ++e) wl[e] = (i == 0) ? u[e] : fmaf(a, wl[e], u[e]);
#pragma unroll
        for (int q = 0; q < NQ; ++q) w_at(slot, i, q) = make_float4(wl[4 * q], wl[4 * q + 1], wl[4 * q + 2], wl[4 * q + 3]);
      }
    };
    int cur = 0;  // stash slot holding w_t of the block being processed
    {
      const int64_t n0 = (t_hi - 1) * kEll;
      float wl[VC];
      solve_into(n0, cur, (p.L - n0 < kEll) ? (int)(p.L - n0) : kEll, wl);
    }
    for (int64_t t = t_hi - 1; t >= t_lo; --t) {
      const int64_t n0 = t * kEll;
      const int lim = (p.L - n0 < kEll) ? (int)(p.L - n0) : kEll;
      float acur[kEll];
      load_a(n0, lim, acur);
      // the block's G vectors first: their loads are in flight during A
      typename V::raw graw[kEll];
      {
        const T* gp = (const T*)p.dx + xo + n0 * sl;
#pragma unroll
        for (int i = 0; i < kEll; ++i) {
          graw[i] = (i < lim) ? V::ld(gp) : V::zero();
          gp += sl;
        }
      }
      // A) w_{t-1} into the other slot (block t-1 is whole), v_{t-1} = w_{t-1}[15]
      float vprev[VC];
      if (t > 0) {
        solve_into(n0 - kEll, cur ^ 1, kEll, vprev);
      } else {
#pragma unroll
        for (int e = 0; e < VC; ++e) vprev[e] = p.carry_in ? p.carry_in[co + e] : 0.f;
      }
      float gsv[kEll];  // g[i] = a[0] ... a[i]
      gsv[0] = acur[0];
#pragma unroll
      for (int i = 1; i < kEll; ++i) gsv[i] = gsv[i - 1] * acur[i];
      // BC) reverse sweep over the block
      float part[kEll];
      float lam[VC], mu_next[VC];
      float rr = 1.f;
      T* dup = (T*)p.du + xo + (n0 + kEll - 1) * sl;
#pragma unroll
      for (int i = kEll - 1; i >= 0; --i) {
        float g[VC];
        V::to_f(graw[i], g);
        if (i == kEll - 1) {
#pragma unroll
          for (int e = 0; e < VC; ++e) lam[e] = g[e];  // lambda[15] = G[15]
        } else {
#pragma unroll
          for (int e = 0; e < VC; ++e) lam[e] = fmaf(acur[i + 1], lam[e], g[e]);
          rr *= acur[i + 1];  // r_t[i] = a_t[i+1] ... a_t[15]
        }
        float du[VC];
#pragma unroll
        for (int e = 0; e < VC; ++e) du[e] = fmaf(rr, mu[e], lam[e]);
        float sdot = 0.f, lv = 0.f;  // sum_c du[i] w[i-1] (w[-1] = 0), sum_c lambda[i] v_{t-1}
        if (i > 0) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const float4 w4 = w_at(cur, i - 1, q);
            const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) {
              const int e = 4 * q + e4;
              sdot = (e == 0) ? du[e] * wv[e4] : fmaf(du[e], wv[e4], sdot);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < VC; ++e) lv = (e == 0) ? lam[e] * vprev[e] : fmaf(lam[e], vprev[e], lv);
        part[i] = fmaf(i > 0 ? gsv[i - 1] : 1.f, lv, sdot);
        if (act && i < lim) V::st(dup, du);
        dup -= sl;
        if (i == 0) {
#pragma unroll
          for (int e = 0; e < VC; ++e) mu_next[e] = acur[0] * lam[e];  // mu_{t-1} = a_t[0] lambda_t[0]
        }
      }
#pragma unroll
      for (int e = 0; e < VC; ++e) mu[e] = mu_next[e];
      if (t == 0 && act && p.mu_out) {
#pragma unroll
        for (int e = 0; e < VC; ++e) p.mu_out[co + e] = mu[e];
      }
      cur ^= 1;
      // da: deterministic reduction over the head's channels
      int tok = 0;
      if constexpr (GS > 1) GroupReduce<GS / 2, kEll>::run(part, lane, tok);
      constexpr int NV = GS >= kEll ? 1 : kEll / GS;
      const bool owner = (GS < 32) || ((lane & 1) == 0);
      if (act && owner) {
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (tok + j < lim) io::st1(dA + (n0 + tok + j) * sal, part[j]);
      }
    }
    return;
  }

  // LAYER group sums: does this CTA stage dq / dk (more than one head per group)?
  const bool grp_q = LAYER && p.hq > 1, grp_k = LAYER && p.hk > 1;
  for (int64_t t = t_hi - 1; t >= t_lo; --t) {
    const int64_t n0 = t * kEll;
    const int lim = (p.L - n0 < kEll) ? (int)(p.L - n0) : kEll;
    // A) carrier v_{t-1} = w_{t-1}[15] (block t-1 is whole: only the last block is ragged)
    float vprev[VC];
    if (t > 0) {
      const T* ap = A0 + (n0 - kEll) * sal;
      Src usrc = src_u(n0 - kEll);
#pragma unroll
      for (int i = 0; i < kEll; ++i) {
        const float a = decay(ap);
        float u[VC];
        usrc.load(true, u);
        ap += sal;
        usrc.fwd();
#pragma unroll
        for (int e = 0; e < VC; ++e) vprev[e] = (i == 0) ? u[e] : fmaf(a, vprev[e], u[e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < VC; ++e) vprev[e] = p.carry_in ? p.carry_in[co + e] : 0.f;
    }
    // B) lambda_t in reverse (lambda[15] = G[15], lambda[i] = G[i] + a[i+1] lambda[i+1]), r_t
    float acur[kEll], r[kEll];
    load_a(n0, lim, acur);
    {
      float lam[VC];
      float rr = 1.f;
      Src gsrc = src_g(n0 + kEll - 1);
      gsrc.load(kEll - 1 < lim, lam);  // lambda[15] = G[15]
      r[kEll - 1] = 1.f;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        lam_at(kEll - 1, q) = make_float4(lam[4 * q], lam[4 * q + 1], lam[4 * q + 2], lam[4 * q + 3]);
#pragma unroll
      for (int i = kEll - 2; i >= 0; --i) {
        float g[VC];
        gsrc.back();
        gsrc.load(i < lim, g);
#pragma unroll
        for (int e = 0; e < VC; ++e) lam[e] = fmaf(acur[i + 1], lam[e], g[e]);
        rr *= acur[i + 1];
        r[i] = rr;  // r_t[i] = a_t[i+1] ... a_t[15]
#pragma unroll
        for (int q = 0; q < NQ; ++q) lam_at(i, q) = make_float4(lam[4 * q], lam[4 * q + 1], lam[4 * q + 2], lam[4 * q + 3]);
      }
    }
    // C) Pass I of block t forward, du (mixer: dq, dk, dv) and da partials
    float part[kEll];
    float wprev[VC];
    float mu_next[VC];  // mu for block t-1: a_t[0] lambda_t[0]
    float gs = 1.f;  // g[i-1]
    int64_t o = xo + n0 * sl;
    int64_t ok = ko + n0 * skl, oq = qo + n0 * sql;
    // the loads of CG tokens are issued together (the stores in between would keep the
    // compiler from hoisting them): u, or k, v and dy
    constexpr int CG = MIX ? SWR_FFMA_BWD_CG : 1;  // fp32 SWR: unrolled by CUnrollV instead
#pragma unroll CUnrollV<MIX>::v
    for (int i0 = 0; i0 < kEll; i0 += CG) {
      typename V::raw r0[CG], r1[CG], r2[CG];
#pragma unroll
      for (int m = 0; m < CG; ++m) {
        const bool valid = i0 + m < lim;
        const int64_t d = (int64_t)m * sl;
        if constexpr (!MIX) {
          r0[m] = valid ? V::ld((const T*)p.u + o + d) : V::zero();
        } else {
          r0[m] = valid ? V::ld((const T*)p.k + (LAYER ? ok + (int64_t)m * skl : o + d)) : V::zero();
          r1[m] = valid ? V::ld((const T*)p.v + o + d) : V::zero();
          r2[m] = valid ? V::ld((const T*)p.dy + o + d) : V::zero();
        }
      }
#pragma unroll
    for (int m = 0; m < CG; ++m) {
      const int i = i0 + m;
      float lam[VC];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 l4 = lam_at(i, q);
        lam[4 * q] = l4.x; lam[4 * q + 1] = l4.y; lam[4 * q + 2] = l4.z; lam[4 * q + 3] = l4.w;
      }
      if (i == 0) {
#pragma unroll
        for (int e = 0; e < VC; ++e) mu_next[e] = acur[0] * lam[e];
      }
      float du[VC];
      float sdot = 0.f, lv = 0.f;  // sum_c du[i] w[i-1] (w[-1] = 0), sum_c lambda[i] v_{t-1}
#pragma unroll
      for (int e = 0; e < VC; ++e) {
        du[e] = fmaf(r[i], mu[e], lam[e]);
        if (i > 0) sdot = (e == 0) ? du[e] * wprev[e] : fmaf(du[e], wprev[e], sdot);
        lv = (e == 0) ? lam[e] * vprev[e] : fmaf(lam[e], vprev[e], lv);
      }
      part[i] = fmaf(gs, lv, sdot);
      if (sig_a) part[i] *= acur[i] * (1.f - acur[i]);  // dza = da sigma'(za), sigma' = a (1 - a)
      const bool valid = i < lim;
      float kk[VC], vv[VC], u[VC];
      if constexpr (!MIX) {
        V::to_f(r0[m], u);
      } else {
        V::to_f(r0[m], kk);
        V::to_f(r1[m], vv);
        if (sig_k) {
#pragma unroll
          for (int e = 0; e < VC; ++e) kk[e] = valid ? sigmoid_gate<T>(kk[e]) : 0.f;
        }
#pragma unroll
        for (int e = 0; e < VC; ++e) u[e] = __fmul_rn(kk[e], vv[e]);
      }
#pragma unroll
      for (int e = 0; e < VC; ++e) wprev[e] = (i == 0) ? u[e] : fmaf(acur[i], wprev[e], u[e]);
      gs *= acur[i];  // g[i]
      if constexpr (!MIX) {
        if (act && valid) V::st((T*)p.du + o, du);
      } else {
        float dd[VC], dq[VC], dk[VC], dv[VC];
        V::to_f(r2[m], dd);
#pragma unroll
        for (int e = 0; e < VC; ++e) {
          dq[e] = dd[e] * fmaf(gs, vprev[e], wprev[e]);  // dq = dy x~
          dk[e] = du[e] * vv[e];                         // dk = du^ v
          dv[e] = fmaf(du[e], kk[e], dd[e]);             // dv = du^ k + dy
        }
        if (sig_k) {
#pragma unroll
          for (int e = 0; e < VC; ++e) dk[e] *= kk[e] * (1.f - kk[e]);  // dzk = dk sigma'(zk)
        }
        if (act && valid) {
          V::st((T*)p.dv + o, dv);
          if (!grp_q) V::st((T*)p.dq + (LAYER ? oq : o), dq);
          if (!grp_k) V::st((T*)p.dk + (LAYER ? ok : o), dk);
        }
        if constexpr (LAYER) {  // stage the per-head terms of the group sums
          if (grp_q) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) dq_at(i, q, tid) = make_float4(dq[4 * q], dq[4 * q + 1], dq[4 * q + 2], dq[4 * q + 3]);
          }
          if (grp_k) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) dk_at(i, q, tid) = make_float4(dk[4 * q], dk[4 * q + 1], dk[4 * q + 2], dk[4 * q + 3]);
          }
        }
      }
      o += sl;
      ok += skl;
      oq += sql;
    }
    }
#pragma unroll
    for (int e = 0; e < VC; ++e) mu[e] = mu_next[e];
    if (t == 0 && act && p.mu_out) {
#pragma unroll
      for (int e = 0; e < VC; ++e) p.mu_out[co + e] = mu[e];
    }
    // da: deterministic reduction over the head's channels
    int tok = 0;
    if constexpr (GS > 1) GroupReduce<GS / 2, kEll>::run(part, lane, tok);
    constexpr int NV = GS >= kEll ? 1 : kEll / GS;
    const bool owner = (GS < 32) || ((lane & 1) == 0);
    if (act && owner) {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (tok + j < lim) io::st1(dA + (n0 + tok + j) * sal, part[j]);
    }
    if constexpr (LAYER) {
      // group sums of dq (hq heads) and dk (hk heads): the j-th head of a group sums
      // tokens i = j (mod heads per group) over the group's heads in head order
      if (grp_q || grp_k) {
        __syncthreads();
        auto gsum = [&](int64_t hpg, bool is_q) {
          const int j = hh % (int)hpg, th0 = (hh - j) * TPH + (tid % TPH);  // head 0 of the group
          T* base = (T*)(is_q ? p.dq : p.dk) + (is_q ? qo + n0 * sql : ko + n0 * skl);
          const int64_t stl = is_q ? sql : skl;
          for (int i = j; i < lim; i += (int)hpg) {
            float acc[VC];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const float4 x = is_q ? dq_at(i, q, th0) : dk_at(i, q, th0);
              acc[4 * q] = x.x; acc[4 * q + 1] = x.y; acc[4 * q + 2] = x.z; acc[4 * q + 3] = x.w;
            }
            for (int m = 1; m < (int)hpg; ++m) {
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
                const float4 x = is_q ? dq_at(i, q, th0 + m * TPH) : dk_at(i, q, th0 + m * TPH);
                acc[4 * q] += x.x; acc[4 * q + 1] += x.y; acc[4 * q + 2] += x.z; acc[4 * q + 3] += x.w;
              }
            }
            if (act) V::st(base + i * stl, acc);
          }
        };
        if (grp_q) gsum(p.hq, true);
        if (grp_k) gsum(p.hk, false);
        __syncthreads();  // the staging slots are rewritten by the next block
      }
    }
  }
}

// ---------------------------------------------------------------------------
// recurrence-mode decode step ("decoded in recurrence mode",
// P:1888): one token per (b, h), state (w, v_{t-1}, g) carried between calls.
// The ops and their order are those of fwd_stream for the same token, so a
// sequence decoded step by step is bitwise the FFMA forward:
//   i == 0: v <- w, g <- a, w <- u;  else g <- g a, w <- a w + u;  x~ = w + g v
// A thread owns 4 channels; a head's D/4 threads sit in one warp, so the shared g
// is read by all of them before one lane writes it (__syncwarp in between).
// ---------------------------------------------------------------------------
template <typename T, bool MIX>
__global__ void __launch_bounds__(128) decode_step(const DecParams p) {
  using V = VecN<T, 4>;
  const int tph = (int)p.D / 4;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t bh = gt / tph;  // (b, h) flattened
  const int c = 4 * (int)(gt % tph);
  const bool act = bh < p.B * p.H;
  const int64_t b = act ? bh / p.H : 0, h = act ? bh % p.H : 0;
  const int64_t xo = b * p.sx_b + h * p.sx_h + c;
  const int64_t so = bh * p.D + c;
  const int i = (int)(p.pos % kEll);
  float gold = 1.f, a = 1.f;
  if (act) {
    a = IO<T>::ld1((const T*)p.a + b * p.sa_b + h * p.sa_h);
    if (i != 0) gold = p.g[bh];  // a block start does not read the state's g (nor v)
  }
  __syncwarp();  // every lane of the head has read g before lane c == 0 rewrites it
  if (!act) return;
  float u[4];
  if constexpr (!MIX) {
    V::to_f(V::ld((const T*)p.u + xo), u);
  } else {  // u^ = k (.) v
    float kk[4], vv[4];
    V::to_f(V::ld((const T*)p.u + xo), kk);
    V::to_f(V::ld((const T*)p.v + xo), vv);
#pragma unroll
    for (int e = 0; e < 4; ++e) u[e] = __fmul_rn(kk[e], vv[e]);
  }
  const float4 w4 = *reinterpret_cast<const float4*>(p.w + so);
  float w[4] = {w4.x, w4.y, w4.z, w4.w};
  float vc[4];
  float g;
  if (i == 0) {  // block start: the finished block's local end state becomes the carrier
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      vc[e] = w[e];
      w[e] = u[e];
    }
    g = 1.f * a;
    *reinterpret_cast<float4*>(p.vc + so) = make_float4(vc[0], vc[1], vc[2], vc[3]);
  } else {
    const float4 v4 = *reinterpret_cast<const float4*>(p.vc + so);
    vc[0] = v4.x; vc[1] = v4.y; vc[2] = v4.z; vc[3] = v4.w;
    g = gold * a;
#pragma unroll
    for (int e = 0; e < 4; ++e) w[e] = fmaf(a, w[e], u[e]);
  }
  *reinterpret_cast<float4*>(p.w + so) = make_float4(w[0], w[1], w[2], w[3]);
  if (c == 0) p.g[bh] = g;
  float x[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) x[e] = fmaf(g, vc[e], w[e]);  // Pass II
  if constexpr (MIX) {  // y = q x~ + v
    float qq[4], vv[4];
    V::to_f(V::ld((const T*)p.q + xo), qq);
    V::to_f(V::ld((const T*)p.v + xo), vv);
#pragma unroll
    for (int e = 0; e < 4; ++e) x[e] = fmaf(qq[e], x[e], vv[e]);
  }
  V::st((T*)p.x + xo, x);
}

cudaError_t launch_decode(bool mix, bool bf16, const DecParams& p, cudaStream_t st) {
  const int64_t threads = p.B * p.H * (p.D / 4);
  const unsigned grid = (unsigned)((threads + 127) / 128);
  if (bf16) {
    if (mix) decode_step<__nv_bfloat16, true><<<grid, 128, 0, st>>>(p);
    else decode_step<__nv_bfloat16, false><<<grid, 128, 0, st>>>(p);
  } else {
    if (mix) decode_step<float, true><<<grid, 128, 0, st>>>(p);
    else decode_step<float, false><<<grid, 128, 0, st>>>(p);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// exact full-range recurrence (Alg. 2, Thm. 3
// P:657-669): x_n = a_n x_{n-1} + u_n over the whole sequence (Eq. 2.1), in the
// three stages of Alg. 2 --
//   I   exact_local: per block, the local solve's end state v_t = w_t[15] and the
//       block decay product c_t = a_t[0] ... a_t[15] (the carrier system);
//   II  exact_carry: the carrier recurrence s_t = c_t s_{t-1} + v_t (s_{-1} =
//       carry_in), sequential over blocks per (b, h, channel);
//   III exact_out: x~_t[i] = w_t[i] + g_t[i] s_{t-1} -- B2P's Pass II with the full
//       carrier instead of the truncated v_{t-1}.
// Workspace: S [B, H, nb, D] fp32 (v_t, overwritten by s_t), C [B, H, nb] fp32.
// A thread owns 4 channels; padding past L is u = 0, a = 1 as elsewhere.
// ---------------------------------------------------------------------------
#ifndef SWR_EXACT_CHUNKS
#define SWR_EXACT_CHUNKS 32  // exact mode: chunks per SM and (b, head-group) column (8: 15-20% slower)
#endif
struct ExactWs {
  float* S;
  float* C;
};

template <typename T>
__global__ void __launch_bounds__(128) exact_local(const Params p, const ExactWs ws) {
  using V = VecN<T, 4>;
  const int tph = (int)p.D / 4, hpc = 128 / tph;
  const int hh = threadIdx.x / tph, c = 4 * (threadIdx.x % tph);
  const int64_t b = blockIdx.z, h = (int64_t)blockIdx.y * hpc + hh;
  if (h >= p.H) return;
  const int64_t t_lo = (int64_t)blockIdx.x * p.K, t_hi = min(t_lo + p.K, p.nb);
  const T* A = (const T*)p.a + b * p.sa_b + h * p.sa_h;
  const int64_t xo = b * p.sx_b + h * p.sx_h + c;
  const int64_t line = b * p.H + h;
  for (int64_t t = t_lo; t < t_hi; ++t) {
    float w[4], g = 1.f;
#pragma unroll
    for (int i = 0; i < kEll; ++i) {
      const int64_t n = t * kEll + i;
      const bool valid = n < p.L;
      const float a = valid ? IO<T>::ld1(A + n * p.sa_l) : 1.f;
      float u[4];
      V::to_f(valid ? V::ld((const T*)p.u + xo + n * p.sx_l) : V::zero(), u);
      g *= a;
#pragma unroll
      for (int e = 0; e < 4; ++e) w[e] = (i == 0) ? u[e] : fmaf(a, w[e], u[e]);
    }
    *reinterpret_cast<float4*>(ws.S + (line * p.nb + t) * p.D + c) = make_float4(w[0], w[1], w[2], w[3]);
    if (c == 0) ws.C[line * p.nb + t] = g;
  }
}

__global__ void __launch_bounds__(128) exact_carry(const Params p, const ExactWs ws) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int tph = (int)p.D / 4;
  const int64_t line = gt / tph;
  const int c = 4 * (int)(gt % tph);
  if (line >= p.B * p.H) return;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (p.carry_in) s = *reinterpret_cast<const float4*>(p.carry_in + line * p.D + c);
  float4* S = reinterpret_cast<float4*>(ws.S + line * p.nb * p.D + c);
  const float* C = ws.C + line * p.nb;
  const int64_t st = p.D / 4;  // float4 stride between blocks
  // The chain is serial; its loads are not.  Issue a group's loads before its stores
  // (the compiler cannot move them across stores to the same array).
  constexpr int kG = 16;
  for (int64_t t0 = 0; t0 < p.nb; t0 += kG) {
    float cg[kG];
    float4 vg[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const bool ok = t0 + j < p.nb;
      cg[j] = ok ? C[t0 + j] : 0.f;
      vg[j] = ok ? S[(t0 + j) * st] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      if (t0 + j < p.nb) {
        const float ct = cg[j];
        const float4 v = vg[j];
        s = make_float4(fmaf(ct, s.x, v.x), fmaf(ct, s.y, v.y), fmaf(ct, s.z, v.z), fmaf(ct, s.w, v.w));
        S[(t0 + j) * st] = s;
      }
    }
  }
  if (p.carry_out) *reinterpret_cast<float4*>(p.carry_out + line * p.D + c) = s;
}

template <typename T>
__global__ void __launch_bounds__(128) exact_out(const Params p, const ExactWs ws) {
  using V = VecN<T, 4>;
  const int tph = (int)p.D / 4, hpc = 128 / tph;
  const int hh = threadIdx.x / tph, c = 4 * (threadIdx.x % tph);
  const int64_t b = blockIdx.z, h = (int64_t)blockIdx.y * hpc + hh;
  if (h >= p.H) return;
  const int64_t t_lo = (int64_t)blockIdx.x * p.K, t_hi = min(t_lo + p.K, p.nb);
  const T* A = (const T*)p.a + b * p.sa_b + h * p.sa_h;
  const int64_t xo = b * p.sx_b + h * p.sx_h + c;
  const int64_t line = b * p.H + h;
  for (int64_t t = t_lo; t < t_hi; ++t) {
    float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);  // s_{t-1}
    if (t > 0) s4 = *reinterpret_cast<const float4*>(ws.S + (line * p.nb + t - 1) * p.D + c);
    else if (p.carry_in) s4 = *reinterpret_cast<const float4*>(p.carry_in + line * p.D + c);
    const float sp[4] = {s4.x, s4.y, s4.z, s4.w};
    float w[4], g = 1.f;
#pragma unroll
    for (int i = 0; i < kEll; ++i) {
      const int64_t n = t * kEll + i;
      const bool valid = n < p.L;
      const float a = valid ? IO<T>::ld1(A + n * p.sa_l) : 1.f;
      float u[4];
      V::to_f(valid ? V::ld((const T*)p.u + xo + n * p.sx_l) : V::zero(), u);
      g *= a;
      float x[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        w[e] = (i == 0) ? u[e] : fmaf(a, w[e], u[e]);
        x[e] = fmaf(g, sp[e], w[e]);
      }
      if (valid) V::st((T*)p.x + xo + n * p.sx_l, x);
    }
  }
}

// Backward of the exact mode (reverse mode of Eq. 2.1): lambda_n = G_n + a_{n+1}
// lambda_{n+1}, du = lambda, da_n = sum_c lambda_n x_{n-1} (x_{-1} = carry_in),
// mu_out = a_0 lambda_0; mu_in enters as mu for the last block (as in swr_bwd).
// Blockwise: lambda_t[i] = l_t[i] + r_t[i] mu_t with l_t the block-local reverse
// solve, r_t[i] = a_t[i+1]...a_t[15] and mu_t = a_{t+1}[0] lambda_{t+1}[0]; the
// reverse carrier chain is mu_{t-1} = a_t[0] (l_t[0] + r_t[0] mu_t).  Stages:
// exact_local + exact_carry (forward carriers s_t, needed for x_{n-1}),
// exact_bwd_local (E_t = l_t[0] into S2, R_t = r_t[0] into C2),
// exact_bwd_carry (mu_t into S2), exact_bwd_out (du, da).
template <typename T>
__global__ void __launch_bounds__(128) exact_bwd_local(const Params p, const ExactWs ws2) {
  using V = VecN<T, 4>;
  const int tph = (int)p.D / 4, hpc = 128 / tph;
  const int hh = threadIdx.x / tph, c = 4 * (threadIdx.x % tph);
  const int64_t b = blockIdx.z, h = (int64_t)blockIdx.y * hpc + hh;
  if (h >= p.H) return;
  const int64_t t_lo = (int64_t)blockIdx.x * p.K, t_hi = min(t_lo + p.K, p.nb);
  const T* A = (const T*)p.a + b * p.sa_b + h * p.sa_h;
  const int64_t xo = b * p.sx_b + h * p.sx_h + c;
  const int64_t line = b * p.H + h;
  for (int64_t t = t_lo; t < t_hi; ++t) {
    float l[4], r = 1.f;
#pragma unroll
    for (int i = kEll - 1; i >= 0; --i) {
      const int64_t n = t * kEll + i;
      const bool valid = n < p.L;
      float g[4];
      V::to_f(valid ? V::ld((const T*)p.dx + xo + n * p.sx_l) : V::zero(), g);
      if (i == kEll - 1) {
#pragma unroll
        for (int e = 0; e < 4; ++e) l[e] = g[e];
      } else {
        const int64_t n1 = n + 1;
        const float an = n1 < p.L ? IO<T>::ld1(A + n1 * p.sa_l) : 1.f;  // a_t[i+1]
        r *= an;
#pragma unroll
        for (int e = 0; e < 4; ++e) l[e] = fmaf(an, l[e], g[e]);
      }
    }
    *reinterpret_cast<float4*>(ws2.S + (line * p.nb + t) * p.D + c) = make_float4(l[0], l[1], l[2], l[3]);
    if (c == 0) ws2.C[line * p.nb + t] = r;  // r_t[0] = a_t[1] ... a_t[15]
  }
}

template <typename T>
__global__ void __launch_bounds__(128) exact_bwd_carry(const Params p, const ExactWs ws2) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int tph = (int)p.D / 4;
  const int64_t line = gt / tph;
  const int c = 4 * (int)(gt % tph);
  if (line >= p.B * p.H) return;
  const int64_t b = line / p.H, h = line % p.H;
  const T* A = (const T*)p.a + b * p.sa_b + h * p.sa_h;
  float4 mu = make_float4(0.f, 0.f, 0.f, 0.f);  // mu_{nb-1}
  if (p.mu_in) mu = *reinterpret_cast<const float4*>(p.mu_in + line * p.D + c);
  float4* S = reinterpret_cast<float4*>(ws2.S + line * p.nb * p.D + c);
  const float* R = ws2.C + line * p.nb;
  const int64_t st = p.D / 4;
  constexpr int kG = 16;
  for (int64_t t1 = p.nb - 1; t1 >= 0; t1 -= kG) {  // blocks t1, t1-1, ... (groups of 16)
    float rg[kG], ag[kG];
    float4 eg[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const int64_t t = t1 - j;
      const bool ok = t >= 0;
      rg[j] = ok ? R[t] : 0.f;
      eg[j] = ok ? S[t * st] : make_float4(0.f, 0.f, 0.f, 0.f);
      ag[j] = ok ? IO<T>::ld1(A + t * kEll * p.sa_l) : 0.f;  // a_t[0] (t * 16 < L)
    }
#pragma unroll
    for (int j = 0; j < kG; ++j) {
      const int64_t t = t1 - j;
      if (t >= 0) {
        S[t * st] = mu;  // mu_t for block t
        const float r = rg[j], a0 = ag[j];
        const float4 e = eg[j];  // lambda_t[0] = l_t[0] + r_t[0] mu_t; mu_{t-1} = a_t[0] lambda_t[0]
        mu = make_float4(a0 * fmaf(r, mu.x, e.x), a0 * fmaf(r, mu.y, e.y), a0 * fmaf(r, mu.z, e.z),
                         a0 * fmaf(r, mu.w, e.w));
      }
    }
  }
  if (p.mu_out) *reinterpret_cast<float4*>(p.mu_out + line * p.D + c) = mu;
}

template <typename T>
__global__ void __launch_bounds__(128) exact_bwd_out(const Params p, const ExactWs ws, const ExactWs ws2) {
  using V = VecN<T, 4>;
  using io = IO<T>;
  const int tph = (int)p.D / 4, hpc = 128 / tph;
  const int hh = threadIdx.x / tph, c = 4 * (threadIdx.x % tph);
  const int lane = threadIdx.x & 31;
  const int64_t b = blockIdx.z, h0 = (int64_t)blockIdx.y * hpc + hh;
  const bool act = h0 < p.H;
  const int64_t h = act ? h0 : p.H - 1;
  __shared__ float4 slam[kEll][128];
  const int64_t t_lo = (int64_t)blockIdx.x * p.K, t_hi = min(t_lo + p.K, p.nb);
  const T* A = (const T*)p.a + b * p.sa_b + h * p.sa_h;
  T* dA = (T*)p.da + b * p.sa_b + h * p.sa_h;
  const int64_t xo = b * p.sx_b + h * p.sx_h + c;
  const int64_t line = b * p.H + h;
  for (int64_t t = t_lo; t < t_hi; ++t) {
    const int64_t n0 = t * kEll;
    const int lim = (p.L - n0 < kEll) ? (int)(p.L - n0) : kEll;
    float acur[kEll];
#pragma unroll
    for (int i = 0; i < kEll; ++i) acur[i] = i < lim ? io::ld1(A + (n0 + i) * p.sa_l) : 1.f;
    const float4 m4 = *reinterpret_cast<const float4*>(ws2.S + (line * p.nb + t) * p.D + c);
    const float mu[4] = {m4.x, m4.y, m4.z, m4.w};
    // lambda_t[i] = l_t[i] + r_t[i] mu_t, in reverse, staged in shared memory
    {
      float l[4], r = 1.f;
#pragma unroll
      for (int i = kEll - 1; i >= 0; --i) {
        float g[4];
        V::to_f(i < lim ? V::ld((const T*)p.dx + xo + (n0 + i) * p.sx_l) : V::zero(), g);
        if (i < kEll - 1) r *= acur[i + 1];
#pragma unroll
        for (int e = 0; e < 4; ++e) l[e] = (i == kEll - 1) ? g[e] : fmaf(acur[i + 1 < kEll ? i + 1 : i], l[e], g[e]);  // a_t[i+1]
        slam[i][threadIdx.x] = make_float4(fmaf(r, mu[0], l[0]), fmaf(r, mu[1], l[1]), fmaf(r, mu[2], l[2]),
                                           fmaf(r, mu[3], l[3]));
      }
    }
    // forward: x_{n-1} = w[i-1] + g[i-1] s_{t-1}; du = lambda; da = sum_c lambda x_{n-1}
    float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t > 0) s4 = *reinterpret_cast<const float4*>(ws.S + (line * p.nb + t - 1) * p.D + c);
    else if (p.carry_in) s4 = *reinterpret_cast<const float4*>(p.carry_in + line * p.D + c);
    const float sp[4] = {s4.x, s4.y, s4.z, s4.w};
    float part[kEll];
    float xprev[4] = {sp[0], sp[1], sp[2], sp[3]};  // x_{n0-1} = s_{t-1}
    float w[4], g = 1.f;
#pragma unroll
    for (int i = 0; i < kEll; ++i) {
      const float4 l4 = slam[i][threadIdx.x];
      const float lam[4] = {l4.x, l4.y, l4.z, l4.w};
      float d = lam[0] * xprev[0];
#pragma unroll
      for (int e = 1; e < 4; ++e) d = fmaf(lam[e], xprev[e], d);
      part[i] = d;
      if (act && i < lim) V::st((T*)p.du + xo + (n0 + i) * p.sx_l, lam);
      float u[4];
      V::to_f(i < lim ? V::ld((const T*)p.u + xo + (n0 + i) * p.sx_l) : V::zero(), u);
      g *= acur[i];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        w[e] = (i == 0) ? u[e] : fmaf(acur[i], w[e], u[e]);
        xprev[e] = fmaf(g, sp[e], w[e]);
      }
    }
    int tok = 0;
    switch (tph) {  // deterministic reduction over the head's lanes
      case 4: GroupReduce<2, kEll>::run(part, lane, tok); break;
      case 8: GroupReduce<4, kEll>::run(part, lane, tok); break;
      case 16: GroupReduce<8, kEll>::run(part, lane, tok); break;
      default: GroupReduce<16, kEll>::run(part, lane, tok); break;
    }
    const int nv = tph >= kEll ? 1 : kEll / tph;
    const bool owner = (tph < 32) || ((lane & 1) == 0);
    if (act && owner) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < nv && tok + j < lim) io::st1(dA + (n0 + tok + j) * p.sa_l, part[j]);
    }
  }
}

// ---------------------------------------------------------------------------
// exact forward in ONE pass over the sequence: Alg. 2's carrier stage fused by a
// decoupled look-back across CTAs.  The carrier
// recurrence s_t = c_t s_{t-1} + v_t composes associatively,
// (c2, v2) o (c1, v1) = (c2 c1, c2 v1 + v2), so each CTA
//   1) runs the local solve over its chunk of K blocks (from a zero state) to the chunk
//      aggregate (C, V): C = the chunk's decay product, V = its local end state;
//   2) publishes (C, V) (flag 1), or, for chunk 0, the inclusive prefix directly;
//   3) looks back over its predecessors' flags: an aggregate is folded in and the
//      look-back continues, an inclusive prefix S ends it: s_in = C_acc S + V_acc;
//   4) publishes its own inclusive prefix S = C s_in + V (flag 2);
//   5) re-runs the chunk from s_in (Eq. 2.1 token by token) and stores x.
// CTAs take chunks by an atomic ticket in (chunk, column) order, so every predecessor
// a CTA waits for is already resident: no deadlock.  Per (column of HPC heads, chunk):
// a flag; per (b, h, chunk): C, V, S.  The caller's workspace holds them; the flags and
// the ticket are zeroed on the stream first.
// ---------------------------------------------------------------------------
struct ExactLb {
  unsigned* ticket;
  unsigned* flag;  // [ncol][nchunk]
  float* C;        // [B*H][nchunk - 1]  (the last chunk publishes nothing)
  float* V;        // [B*H][nchunk - 1][D]
  float* S;        // [B*H][nchunk - 1][D]
  float* blk;      // the backward's scans: per-block vectors [B*H][nb][D] (in, then out)
  float* blkC;     //   and per-block scalars [B*H][nb]
  int64_t nchunk, ncol;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// CTAs per SM: bf16 8 (64 registers: more CTAs in flight beat hoisting the block's loads),
// fp32 4 (tools/exact_time.py)
template <typename T>
__global__ void __launch_bounds__(128, sizeof(T) == 2 ? 8 : 4) exact_fwd_lb(const Params p, const ExactLb lb) {
  using V = VecN<T, 4>;
  __shared__ unsigned s_ticket, s_flag;
  const int tph = (int)p.D / 4, hpc = 128 / tph;
  if (threadIdx.x == 0) s_ticket = atomicAdd(lb.ticket, 1u);
  __syncthreads();
  const int64_t tk = s_ticket, chunk = tk / lb.ncol, col = tk % lb.ncol;
  const int64_t hgs = (p.H + hpc - 1) / hpc;
  const int64_t b = col / hgs;
  const int hh = threadIdx.x / tph, c = 4 * (threadIdx.x % tph);
  const int64_t h = (col % hgs) * hpc + hh;
  const bool act = h < p.H;
  const int64_t hc = act ? h : p.H - 1;
  const int64_t line = b * p.H + hc;
  const int64_t t_lo = chunk * p.K, t_hi = min(t_lo + p.K, p.nb);
  const int64_t n_lo = t_lo * kEll, n_hi = min(t_hi * kEll, p.L);
  const T* A = (const T*)p.a + b * p.sa_b + hc * p.sa_h;
  const int64_t xo = b * p.sx_b + hc * p.sx_h + c;
  const bool publish = chunk + 1 < lb.nchunk;  // the last chunk has no successor
  const int64_t slot = line * (lb.nchunk - 1) + chunk;

  // 1) chunk aggregate: local end state from 0, decay product
  float v[4] = {0.f, 0.f, 0.f, 0.f}, cprod = 1.f;
  if (publish || chunk == 0) {
    for (int64_t n0 = n_lo; n0 < n_hi; n0 += kEll) {
      float ab[kEll];
      typename V::raw ub[kEll];
#pragma unroll
      for (int i = 0; i < kEll; ++i) {  // the block's loads first, then the chain
        const bool ok = n0 + i < n_hi;
        ab[i] = ok ? IO<T>::ld1(A + (n0 + i) * p.sa_l) : 1.f;
        ub[i] = ok ? V::ld((const T*)p.u + xo + (n0 + i) * p.sx_l) : V::zero();
      }
#pragma unroll
      for (int i = 0; i < kEll; ++i) {
        float u[4];
        V::to_f(ub[i], u);
        cprod *= ab[i];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = fmaf(ab[i], v[e], u[e]);
      }
    }
  }
  // 2) publish the aggregate, or (chunk 0) the inclusive prefix
  float sin[4] = {0.f, 0.f, 0.f, 0.f};
  if (chunk == 0 && p.carry_in)
#pragma unroll
    for (int e = 0; e < 4; ++e) sin[e] = p.carry_in[line * p.D + c + e];
  if (publish) {
    if (act) {
      if (chunk == 0) {
        *reinterpret_cast<float4*>(lb.S + slot * p.D + c) =
            make_float4(fmaf(cprod, sin[0], v[0]), fmaf(cprod, sin[1], v[1]), fmaf(cprod, sin[2], v[2]),
                        fmaf(cprod, sin[3], v[3]));
      } else {
        *reinterpret_cast<float4*>(lb.V + slot * p.D + c) = make_float4(v[0], v[1], v[2], v[3]);
        if (c == 0) lb.C[slot] = cprod;
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(lb.flag + col * lb.nchunk + chunk, chunk == 0 ? 2u : 1u);
  }
  // 3) look back
  if (chunk > 0) {
    float cacc = 1.f, vacc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t j = chunk - 1;; --j) {
      if (threadIdx.x == 0) {
        unsigned f;
        while ((f = ld_acquire(lb.flag + col * lb.nchunk + j)) == 0u) __nanosleep(32);
        s_flag = f;
      }
      __syncthreads();
      const unsigned f = s_flag;
      const int64_t sj = line * (lb.nchunk - 1) + j;
      if (f == 2u) {  // inclusive prefix S_j: s_in = C_acc S_j + V_acc
        const float4 S = __ldcg(reinterpret_cast<const float4*>(lb.S + sj * p.D + c));
        sin[0] = fmaf(cacc, S.x, vacc[0]);
        sin[1] = fmaf(cacc, S.y, vacc[1]);
        sin[2] = fmaf(cacc, S.z, vacc[2]);
        sin[3] = fmaf(cacc, S.w, vacc[3]);
        __syncthreads();  // s_flag is rewritten only after every thread has read it
        break;
      }
      // aggregate (C_j, V_j): fold chunk j in front of the accumulated chunks
      const float4 Vj = __ldcg(reinterpret_cast<const float4*>(lb.V + sj * p.D + c));
      const float Cj = __ldcg(lb.C + sj);
      vacc[0] = fmaf(cacc, Vj.x, vacc[0]);
      vacc[1] = fmaf(cacc, Vj.y, vacc[1]);
      vacc[2] = fmaf(cacc, Vj.z, vacc[2]);
      vacc[3] = fmaf(cacc, Vj.w, vacc[3]);
      cacc *= Cj;
      __syncthreads();
    }
    // 4) publish the inclusive prefix
    if (publish) {
      if (act)
        *reinterpret_cast<float4*>(lb.S + slot * p.D + c) =
            make_float4(fmaf(cprod, sin[0], v[0]), fmaf(cprod, sin[1], v[1]), fmaf(cprod, sin[2], v[2]),
                        fmaf(cprod, sin[3], v[3]));
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release(lb.flag + col * lb.nchunk + chunk, 2u);
    }
  }
  // 5) the chunk from s_in, token by token (Eq. 2.1)
  float x[4] = {sin[0], sin[1], sin[2], sin[3]};
  for (int64_t n0 = n_lo; n0 < n_hi; n0 += kEll) {
    float ab[kEll];
    typename V::raw ub[kEll];
#pragma unroll
    for (int i = 0; i < kEll; ++i) {
      const bool ok = n0 + i < n_hi;
      ab[i] = ok ? IO<T>::ld1(A + (n0 + i) * p.sa_l) : 1.f;
      ub[i] = ok ? V::ld((const T*)p.u + xo + (n0 + i) * p.sx_l) : V::zero();
    }
#pragma unroll
    for (int i = 0; i < kEll; ++i) {
      float u[4];
      V::to_f(ub[i], u);
#pragma unroll
      for (int e = 0; e < 4; ++e) x[e] = fmaf(ab[i], x[e], u[e]);
      if (act && n0 + i < n_hi) V::st((T*)p.x + xo + (n0 + i) * p.sx_l, x);
    }
  }
  if (act && t_hi == p.nb && p.carry_out)
    *reinterpret_cast<float4*>(p.carry_out + line * p.D + c) = make_float4(x[0], x[1], x[2], x[3]);
}

// The backward's two carrier scans by the same decoupled look-back, over per-block
// values stashed by a first pass (no token is read twice within a scan):
//   forward (REV = false): s_t = c_t s_{t-1} + v_t, v_t = block t's local end state,
//     c_t = a_t[0] ... a_t[15], s_{-1} = carry_in; out: s_t per block;
//   reverse (REV = true): mu_{t-1} = R_t mu_t + E_t, E_t = a_t[0] l_t[0] (l_t the block's
//     local reverse solve of G), R_t = a_t[0] r_t[0] = a_t[0] (a_t[1] ... a_t[15]),
//     mu_{nb-1} = mu_in; out: mu_t per block (the adjoint entering block t from the
//     right) and mu_out = mu_{-1}.
// A CTA takes a chunk (tickets in scan order), computes and stashes its blocks' (c, v)
// or (R, E) in blk / blkC while folding them to the chunk aggregate, publishes it, looks
// back (forward scan) or ahead (reverse scan) for its entering carrier, publishes its
// prefix and replaces the stash by the per-block carriers.
// STASHED: the per-block (c, v) are already in blk / blkC (the tensor-core first pass,
// swr_tc.cu Cfg<7>); pass 1 only folds them
template <typename T, bool REV, bool STASHED = false>
__global__ void __launch_bounds__(128, sizeof(T) == 2 ? 8 : 4) exact_scan_lb(const Params p, const ExactLb lb) {
  using V = VecN<T, 4>;
  __shared__ unsigned s_ticket, s_flag;
  const int tph = (int)p.D / 4, hpc = 128 / tph;
  if (threadIdx.x == 0) s_ticket = atomicAdd(lb.ticket, 1u);
  __syncthreads();
  const int64_t tk = s_ticket, k = tk / lb.ncol, col = tk % lb.ncol;
  const int64_t chunk = REV ? lb.nchunk - 1 - k : k;
  const int64_t hgs = (p.H + hpc - 1) / hpc;
  const int64_t b = col / hgs;
  const int hh = threadIdx.x / tph, c = 4 * (threadIdx.x % tph);
  const int64_t h = (col % hgs) * hpc + hh;
  const bool act = h < p.H;
  const int64_t hc = act ? h : p.H - 1;
  const int64_t line = b * p.H + hc;
  const int64_t t_lo = chunk * p.K, t_hi = min(t_lo + p.K, p.nb);
  const T* A = (const T*)p.a + b * p.sa_b + hc * p.sa_h;
  const int64_t xo = b * p.sx_b + hc * p.sx_h + c;
  const bool first = REV ? chunk == lb.nchunk - 1 : chunk == 0;   // has the initial carrier
  const bool publish = REV ? chunk > 0 : chunk + 1 < lb.nchunk;   // has a successor
  const int64_t slot = line * (lb.nchunk - 1) + (REV ? chunk - 1 : chunk);
  float4* BV = reinterpret_cast<float4*>(lb.blk + line * p.nb * p.D + c);
  float* BC = lb.blkC + line * p.nb;
  const int64_t st4 = p.D / 4;

  // 1) per-block values into the stash, folded to the chunk aggregate (C, V)
  float v[4] = {0.f, 0.f, 0.f, 0.f}, cagg = 1.f;
  constexpr int kSG = 8;  // stashed blocks whose loads are issued together
  if constexpr (STASHED) {
    for (int64_t q0 = 0; q0 < t_hi - t_lo; q0 += kSG) {
      float4 y4[kSG];
      float cb[kSG];
#pragma unroll
      for (int m = 0; m < kSG; ++m) {
        const int64_t q = q0 + m;
        const int64_t t = REV ? t_hi - 1 - q : t_lo + q;
        const bool ok = act && q < t_hi - t_lo;
        y4[m] = ok ? BV[t * st4] : make_float4(0.f, 0.f, 0.f, 0.f);
        cb[m] = ok ? BC[t] : 1.f;
      }
#pragma unroll
      for (int m = 0; m < kSG; ++m) {
        v[0] = fmaf(cb[m], v[0], y4[m].x);
        v[1] = fmaf(cb[m], v[1], y4[m].y);
        v[2] = fmaf(cb[m], v[2], y4[m].z);
        v[3] = fmaf(cb[m], v[3], y4[m].w);
        cagg *= cb[m];
      }
    }
  }
  for (int64_t q = 0; q < (STASHED ? 0 : t_hi - t_lo); ++q) {
    const int64_t t = REV ? t_hi - 1 - q : t_lo + q;
    const int64_t n0 = t * kEll;
    float ab[kEll];
    typename V::raw rb[kEll];
#pragma unroll
    for (int i = 0; i < kEll; ++i) {
      const bool ok = n0 + i < p.L;
      ab[i] = ok ? IO<T>::ld1(A + (n0 + i) * p.sa_l) : 1.f;
      rb[i] = ok ? V::ld((const T*)(REV ? p.dx : p.u) + xo + (n0 + i) * p.sx_l) : V::zero();
    }
    float y[4], cb = 1.f;
    if constexpr (!REV) {  // local solve: w[i] = a[i] w[i-1] + u[i], w[0] = u[0]; c_t includes a_t[0]
#pragma unroll
      for (int i = 0; i < kEll; ++i) {
        float u[4];
        V::to_f(rb[i], u);
#pragma unroll
        for (int e = 0; e < 4; ++e) y[e] = (i == 0) ? u[e] : fmaf(ab[i], y[e], u[e]);
        cb *= ab[i];
      }
    } else {  // l[i] = G[i] + a[i+1] l[i+1]; E = a[0] l[0], R = a[0] (a[1] ... a[15])
#pragma unroll
      for (int i = kEll - 1; i >= 0; --i) {
        float g[4];
        V::to_f(rb[i], g);
#pragma unroll
        for (int e = 0; e < 4; ++e) y[e] = (i == kEll - 1) ? g[e] : fmaf(ab[i + 1 < kEll ? i + 1 : i], y[e], g[e]);
        if (i > 0) cb *= ab[i];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) y[e] *= ab[0];
      cb *= ab[0];
    }
    if (act) {
      BV[t * st4] = make_float4(y[0], y[1], y[2], y[3]);
      if (c == 0) BC[t] = cb;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = fmaf(cb, v[e], y[e]);
    cagg *= cb;
  }
  // 2) publish the aggregate, or (first chunk of the scan) the prefix
  float cin[4] = {0.f, 0.f, 0.f, 0.f};
  const float* init = REV ? p.mu_in : p.carry_in;
  if (first && init)
#pragma unroll
    for (int e = 0; e < 4; ++e) cin[e] = init[line * p.D + c + e];
  if (publish) {
    if (act) {
      if (first) {
        *reinterpret_cast<float4*>(lb.S + slot * p.D + c) =
            make_float4(fmaf(cagg, cin[0], v[0]), fmaf(cagg, cin[1], v[1]), fmaf(cagg, cin[2], v[2]),
                        fmaf(cagg, cin[3], v[3]));
      } else {
        *reinterpret_cast<float4*>(lb.V + slot * p.D + c) = make_float4(v[0], v[1], v[2], v[3]);
        if (c == 0) lb.C[slot] = cagg;
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(lb.flag + col * lb.nchunk + chunk, first ? 2u : 1u);
  }
  // 3) look back (forward scan) / ahead (reverse scan)
  if (!first) {
    float cacc = 1.f, vacc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t j = REV ? chunk + 1 : chunk - 1;; j += REV ? 1 : -1) {
      if (threadIdx.x == 0) {
        unsigned f;
        while ((f = ld_acquire(lb.flag + col * lb.nchunk + j)) == 0u) __nanosleep(32);
        s_flag = f;
      }
      __syncthreads();
      const unsigned f = s_flag;
      const int64_t sj = line * (lb.nchunk - 1) + (REV ? j - 1 : j);
      if (f == 2u) {
        const float4 S = __ldcg(reinterpret_cast<const float4*>(lb.S + sj * p.D + c));
        cin[0] = fmaf(cacc, S.x, vacc[0]);
        cin[1] = fmaf(cacc, S.y, vacc[1]);
        cin[2] = fmaf(cacc, S.z, vacc[2]);
        cin[3] = fmaf(cacc, S.w, vacc[3]);
        __syncthreads();
        break;
      }
      const float4 Vj = __ldcg(reinterpret_cast<const float4*>(lb.V + sj * p.D + c));
      const float Cj = __ldcg(lb.C + sj);
      vacc[0] = fmaf(cacc, Vj.x, vacc[0]);
      vacc[1] = fmaf(cacc, Vj.y, vacc[1]);
      vacc[2] = fmaf(cacc, Vj.z, vacc[2]);
      vacc[3] = fmaf(cacc, Vj.w, vacc[3]);
      cacc *= Cj;
      __syncthreads();
    }
    // 4) publish the prefix
    if (publish) {
      if (act)
        *reinterpret_cast<float4*>(lb.S + slot * p.D + c) =
            make_float4(fmaf(cagg, cin[0], v[0]), fmaf(cagg, cin[1], v[1]), fmaf(cagg, cin[2], v[2]),
                        fmaf(cagg, cin[3], v[3]));
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release(lb.flag + col * lb.nchunk + chunk, 2u);
    }
  }
  // 5) the carriers of the chunk's blocks from the stash: forward s_t; reverse mu_t (the
  //    carrier entering block t from the right, stored before applying block t)
  float s4[4] = {cin[0], cin[1], cin[2], cin[3]};
  for (int64_t q0 = 0; q0 < t_hi - t_lo; q0 += kSG) {  // a group's loads before its stores
    float4 yg[kSG];
    float cg[kSG];
#pragma unroll
    for (int m = 0; m < kSG; ++m) {
      const int64_t q = q0 + m;
      const int64_t t = REV ? t_hi - 1 - q : t_lo + q;
      const bool ok = act && q < t_hi - t_lo;
      yg[m] = ok ? BV[t * st4] : make_float4(0.f, 0.f, 0.f, 0.f);
      cg[m] = ok ? BC[t] : 1.f;
    }
#pragma unroll
    for (int m = 0; m < kSG; ++m) {
      const int64_t q = q0 + m;
      const int64_t t = REV ? t_hi - 1 - q : t_lo + q;
      const bool ok = act && q < t_hi - t_lo;
      if constexpr (REV) {
        if (ok) BV[t * st4] = make_float4(s4[0], s4[1], s4[2], s4[3]);
      }
      s4[0] = fmaf(cg[m], s4[0], yg[m].x);
      s4[1] = fmaf(cg[m], s4[1], yg[m].y);
      s4[2] = fmaf(cg[m], s4[2], yg[m].z);
      s4[3] = fmaf(cg[m], s4[3], yg[m].w);
      if constexpr (!REV) {
        if (ok) BV[t * st4] = make_float4(s4[0], s4[1], s4[2], s4[3]);
      }
    }
  }
  if (REV && act && chunk == 0 && p.mu_out)
    *reinterpret_cast<float4*>(p.mu_out + line * p.D + c) = make_float4(s4[0], s4[1], s4[2], s4[3]);
  if (!REV && act && t_hi == p.nb && p.carry_out)  // the exact state at token L-1
    *reinterpret_cast<float4*>(p.carry_out + line * p.D + c) = make_float4(s4[0], s4[1], s4[2], s4[3]);
}

#ifndef SWR_EXACT_SCAN_K
#define SWR_EXACT_SCAN_K 32  // blocks per look-back chunk when the per-block values are stashed
#endif
#ifndef SWR_EXACT_LB_K
#define SWR_EXACT_LB_K 4  // blocks per look-back chunk
#endif
// the single-pass forward (exact_fwd_lb); workspace layout within swr_exact_workspace_bytes
cudaError_t launch_exact_lb(bool bf16, Params p, void* workspace, cudaStream_t st) {
  auto cdiv = [](int64_t x, int64_t y) { return (x + y - 1) / y; };
  const int64_t hpc = 128 / (p.D / 4);
  p.K = p.nb == 1 ? 1 : std::max<int64_t>(2, std::min<int64_t>(SWR_EXACT_LB_K, p.nb));
  ExactLb lb;
  lb.nchunk = cdiv(p.nb, p.K);
  lb.ncol = p.B * cdiv(p.H, hpc);
  const int64_t lines = p.B * p.H;
  // [V | S] floats, then C floats, then ticket + flags (u32), all 16-byte aligned
  uint8_t* base = reinterpret_cast<uint8_t*>(workspace);
  const int64_t nv = lines * (lb.nchunk - 1) * p.D;
  lb.V = reinterpret_cast<float*>(base);
  lb.S = lb.V + nv;
  lb.C = lb.S + nv;
  lb.ticket = reinterpret_cast<unsigned*>(lb.C + (lines * (lb.nchunk - 1) + 3) / 4 * 4);
  lb.flag = lb.ticket + 4;
  const size_t used = (size_t)(reinterpret_cast<uint8_t*>(lb.flag + lb.ncol * lb.nchunk) - base);
  const size_t avail = (size_t)sizeof(float) * (p.B * p.H * p.nb * p.D + (p.B * p.H * p.nb + 3) / 4 * 4);
  if (used > avail) return cudaErrorInvalidValue;  // cannot happen for K >= 2: 2 (nchunk - 1) <= nb - 1
  cudaError_t e = cudaMemsetAsync(lb.ticket, 0, sizeof(unsigned) * (4 + lb.ncol * lb.nchunk), st);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)(lb.ncol * lb.nchunk);
  if (bf16) exact_fwd_lb<__nv_bfloat16><<<grid, 128, 0, st>>>(p, lb);
  else exact_fwd_lb<float><<<grid, 128, 0, st>>>(p, lb);
  return cudaGetLastError();
}

cudaError_t launch_exact(bool bf16, Params p, void* workspace, cudaStream_t st, int sms) {
  auto cdiv = [](int64_t x, int64_t y) { return (x + y - 1) / y; };
  ExactWs ws;
  ws.S = reinterpret_cast<float*>(workspace);
  ws.C = ws.S + p.B * p.H * p.nb * p.D;
  const int64_t hpc = 128 / (p.D / 4);
  const int64_t cols = p.B * cdiv(p.H, hpc);
  const int64_t want = std::max<int64_t>(1, ((int64_t)sms * SWR_EXACT_CHUNKS) / std::max<int64_t>(cols, 1));
  p.K = std::min<int64_t>(std::max<int64_t>(cdiv(p.nb, want), 1), p.nb);
  const dim3 grid((unsigned)cdiv(p.nb, p.K), (unsigned)cdiv(p.H, hpc), (unsigned)p.B);
  const unsigned gc = (unsigned)cdiv(p.B * p.H * (p.D / 4), 128);
  if (bf16) exact_local<__nv_bfloat16><<<grid, 128, 0, st>>>(p, ws);
  else exact_local<float><<<grid, 128, 0, st>>>(p, ws);
  exact_carry<<<gc, 128, 0, st>>>(p, ws);
  if (bf16) exact_out<__nv_bfloat16><<<grid, 128, 0, st>>>(p, ws);
  else exact_out<float><<<grid, 128, 0, st>>>(p, ws);
  return cudaGetLastError();
}

cudaError_t launch_exact_bwd5(bool bf16, Params p, void* workspace, cudaStream_t st, int sms);
static cudaError_t lb_scratch(const Params& p, void* base, size_t avail, ExactLb& lb, cudaStream_t st);

// The exact forward's carrier pass for the tensor-core output pass: the per-block exact
// carriers s_t into the workspace's first [B*H][nb][D] floats (and carry_out), by the
// forward look-back scan over per-block local solves -- computed here from u, or
// (stashed) already written there with c_t by the tensor-core first pass.  Workspace:
// 2 x swr_exact_workspace_bytes (stash, then the scan's scratch).  Returns the carriers.
void exact_stash(const Params& p, void* workspace, float** V, float** C) {
  *V = reinterpret_cast<float*>(workspace);
  *C = *V + p.B * p.H * p.nb * p.D;
}

cudaError_t launch_exact_carriers(bool bf16, Params p, void* workspace, cudaStream_t st, const float** carriers,
                                  bool stashed) {
  const int64_t nS = p.B * p.H * p.nb * p.D, nC = (p.B * p.H * p.nb + 3) / 4 * 4;
  float* S = reinterpret_cast<float*>(workspace);
  float* C = S + nS;
  void* scratch = C + nC;
  const size_t avail = (size_t)sizeof(float) * (nS + nC);
  // a chunk folds stashed per-block values (4 floats per thread and block): longer chunks
  // keep the look-back chains short
  const int64_t K = stashed ? SWR_EXACT_SCAN_K : SWR_EXACT_LB_K;
  p.K = p.nb == 1 ? 1 : std::max<int64_t>(2, std::min<int64_t>(K, p.nb));
  ExactLb lb;
  cudaError_t e = lb_scratch(p, scratch, avail, lb, st);
  if (e != cudaSuccess) return e;
  lb.blk = S;
  lb.blkC = C;
  const unsigned grid = (unsigned)(lb.ncol * lb.nchunk);
  if (stashed) exact_scan_lb<__nv_bfloat16, false, true><<<grid, 128, 0, st>>>(p, lb);
  else if (bf16) exact_scan_lb<__nv_bfloat16, false><<<grid, 128, 0, st>>>(p, lb);
  else exact_scan_lb<float, false><<<grid, 128, 0, st>>>(p, lb);
  *carriers = S;
  return cudaGetLastError();
}

// the look-back kernels' scratch inside `base` (<= swr_exact_workspace_bytes), zeroed flags
static cudaError_t lb_scratch(const Params& p, void* base, size_t avail, ExactLb& lb, cudaStream_t st) {
  auto cdiv = [](int64_t x, int64_t y) { return (x + y - 1) / y; };
  const int64_t hpc = 128 / (p.D / 4), lines = p.B * p.H;
  lb.nchunk = cdiv(p.nb, p.K);
  lb.ncol = p.B * cdiv(p.H, hpc);
  const int64_t nv = lines * (lb.nchunk - 1) * p.D;
  lb.V = reinterpret_cast<float*>(base);
  lb.S = lb.V + nv;
  lb.C = lb.S + nv;
  lb.ticket = reinterpret_cast<unsigned*>(lb.C + (lines * (lb.nchunk - 1) + 3) / 4 * 4);
  lb.flag = lb.ticket + 4;
  lb.blk = nullptr;
  const size_t used = (size_t)(reinterpret_cast<uint8_t*>(lb.flag + lb.ncol * lb.nchunk) - reinterpret_cast<uint8_t*>(base));
  if (used > avail) return cudaErrorInvalidValue;
  return cudaMemsetAsync(lb.ticket, 0, sizeof(unsigned) * (4 + lb.ncol * lb.nchunk), st);
}

// workspace (3 x swr_exact_workspace_bytes): forward per-block (v_t / s_t, c_t), reverse
// per-block (E_t / mu_t, R_t), then the look-back scratch (reused by both scans)
#ifndef SWR_EXACT_BWD_LB_MIN_NB
#define SWR_EXACT_BWD_LB_MIN_NB 1024  // look-back scans from this many blocks per line on
#endif
cudaError_t launch_exact_bwd(bool bf16, Params p, void* workspace, cudaStream_t st, int sms) {
#ifndef SWR_EXACT_3STAGE
  // The look-back scans cost one more pass over the per-block stash than the serial
  // chains they replace; they pay once the chains are long (tools/exact_time.py: L = 32K
  // 1003 -> 772 us; L = 4K 369 -> 382 us, d = 16 at L = 8K 742 -> 878 us).
  if (p.nb < SWR_EXACT_BWD_LB_MIN_NB) return launch_exact_bwd5(bf16, p, workspace, st, sms);
  auto cdiv = [](int64_t x, int64_t y) { return (x + y - 1) / y; };
  const int64_t nS = p.B * p.H * p.nb * p.D, nC = (p.B * p.H * p.nb + 3) / 4 * 4;
  ExactWs ws, ws2;
  ws.S = reinterpret_cast<float*>(workspace);
  ws.C = ws.S + nS;
  ws2.S = ws.C + nC;
  ws2.C = ws2.S + nS;
  void* scratch = ws2.C + nC;
  const size_t avail = (size_t)sizeof(float) * (nS + (p.B * p.H * p.nb + 3) / 4 * 4);
  p.K = p.nb == 1 ? 1 : std::max<int64_t>(2, std::min<int64_t>(SWR_EXACT_LB_K, p.nb));
  ExactLb lb;
  cudaError_t e = lb_scratch(p, scratch, avail, lb, st);
  if (e != cudaSuccess) return e;
  const unsigned grid_lb = (unsigned)(lb.ncol * lb.nchunk);
  lb.blk = ws.S;  // forward: (v_t, c_t), then the carriers s_t
  lb.blkC = ws.C;
  if (bf16) exact_scan_lb<__nv_bfloat16, false><<<grid_lb, 128, 0, st>>>(p, lb);
  else exact_scan_lb<float, false><<<grid_lb, 128, 0, st>>>(p, lb);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = lb_scratch(p, scratch, avail, lb, st)) != cudaSuccess) return e;
  lb.blk = ws2.S;  // reverse: (E_t, R_t), then the carriers mu_t
  lb.blkC = ws2.C;
  if (bf16) exact_scan_lb<__nv_bfloat16, true><<<grid_lb, 128, 0, st>>>(p, lb);
  else exact_scan_lb<float, true><<<grid_lb, 128, 0, st>>>(p, lb);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int64_t hpc = 128 / (p.D / 4);
  const int64_t cols = p.B * cdiv(p.H, hpc);
  const int64_t want = std::max<int64_t>(1, ((int64_t)sms * SWR_EXACT_CHUNKS) / std::max<int64_t>(cols, 1));
  p.K = std::min<int64_t>(std::max<int64_t>(cdiv(p.nb, want), 1), p.nb);
  const dim3 grid((unsigned)cdiv(p.nb, p.K), (unsigned)cdiv(p.H, hpc), (unsigned)p.B);
  if (bf16) exact_bwd_out<__nv_bfloat16><<<grid, 128, 0, st>>>(p, ws, ws2);
  else exact_bwd_out<float><<<grid, 128, 0, st>>>(p, ws, ws2);
  return cudaGetLastError();
#else
  return launch_exact_bwd5(bf16, p, workspace, st, sms);
#endif
}

// the round-1 five-launch backward: forward S, C then backward S2, C2
cudaError_t launch_exact_bwd5(bool bf16, Params p, void* workspace, cudaStream_t st, int sms) {
  auto cdiv = [](int64_t x, int64_t y) { return (x + y - 1) / y; };
  const int64_t nS = p.B * p.H * p.nb * p.D, nC = (p.B * p.H * p.nb + 3) / 4 * 4;  // keep S2 16-byte aligned
  ExactWs ws, ws2;
  ws.S = reinterpret_cast<float*>(workspace);
  ws.C = ws.S + nS;
  ws2.S = ws.C + nC;
  ws2.C = ws2.S + nS;
  const int64_t hpc = 128 / (p.D / 4);
  const int64_t cols = p.B * cdiv(p.H, hpc);
  const int64_t want = std::max<int64_t>(1, ((int64_t)sms * SWR_EXACT_CHUNKS) / std::max<int64_t>(cols, 1));
  p.K = std::min<int64_t>(std::max<int64_t>(cdiv(p.nb, want), 1), p.nb);
  const dim3 grid((unsigned)cdiv(p.nb, p.K), (unsigned)cdiv(p.H, hpc), (unsigned)p.B);
  const unsigned gc = (unsigned)cdiv(p.B * p.H * (p.D / 4), 128);
  Params pf = p;
  pf.carry_out = nullptr;
  if (bf16) {
    exact_local<__nv_bfloat16><<<grid, 128, 0, st>>>(pf, ws);
    exact_carry<<<gc, 128, 0, st>>>(pf, ws);
    exact_bwd_local<__nv_bfloat16><<<grid, 128, 0, st>>>(p, ws2);
    exact_bwd_carry<__nv_bfloat16><<<gc, 128, 0, st>>>(p, ws2);
    exact_bwd_out<__nv_bfloat16><<<grid, 128, 0, st>>>(p, ws, ws2);
  } else {
    exact_local<float><<<grid, 128, 0, st>>>(pf, ws);
    exact_carry<<<gc, 128, 0, st>>>(pf, ws);
    exact_bwd_local<float><<<grid, 128, 0, st>>>(p, ws2);
    exact_bwd_carry<float><<<gc, 128, 0, st>>>(p, ws2);
    exact_bwd_out<float><<<grid, 128, 0, st>>>(p, ws, ws2);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// uniform-window recurrence (Sec. uniform_window P:1104-1113,
// Eq. banded_L): x~ = (I + AZ + ... + (AZ)^{k-1}) u, every token sees the k most
// recent inputs, x~_n = sum_{j<k} (a_{n-j+1} ... a_n) u_{n-j} (u_{<0} = 0).  The
// paper reaches it by stopping Kogge-Stone after log2 k stages; a thread that
// streams tokens evaluates the same band by Horner over a register ring of the
// last k (u, a) pairs: k FMAs per channel and token, inputs read once (plus a
// (k-1)-token halo per chunk).
// ---------------------------------------------------------------------------
template <typename T, int KW>
__global__ void __launch_bounds__(128) uniform_fwd(const Params p) {
  using V = VecN<T, 4>;
  const int tph = (int)p.D / 4, hpc = 128 / tph;
  const int hh = threadIdx.x / tph, c = 4 * (threadIdx.x % tph);
  const int64_t b = blockIdx.z, h = (int64_t)blockIdx.y * hpc + hh;
  if (h >= p.H) return;
  const int64_t n_lo = (int64_t)blockIdx.x * p.K, n_hi = min(n_lo + p.K, p.L);  // K: tokens per chunk
  const T* A = (const T*)p.a + b * p.sa_b + h * p.sa_h;
  const int64_t xo = b * p.sx_b + h * p.sx_h + c;
  float ur[KW][4], ar[KW];
#pragma unroll
  for (int j = 0; j < KW; ++j) {  // slot j <- token n_lo - KW + j (slot = token mod KW)
    const int64_t n = n_lo - KW + j;
    const bool valid = n >= 0;
    ar[j] = valid ? IO<T>::ld1(A + n * p.sa_l) : 1.f;
    V::to_f(valid ? V::ld((const T*)p.u + xo + n * p.sx_l) : V::zero(), ur[j]);
  }
  for (int64_t n0 = n_lo; n0 < n_hi; n0 += KW) {
#pragma unroll
    for (int i = 0; i < KW; ++i) {
      const int64_t n = n0 + i;
      const bool valid = n < n_hi;
      ar[i] = valid ? IO<T>::ld1(A + n * p.sa_l) : 1.f;
      V::to_f(valid ? V::ld((const T*)p.u + xo + n * p.sx_l) : V::zero(), ur[i]);
      // Horner from the oldest token of the window, on packed fp32x2 FMAs (two
      // IEEE fmas each: the same bits as scalar fmaf)
      const int s0 = (i + 1) % KW;
      float2 x01 = make_float2(ur[s0][0], ur[s0][1]), x23 = make_float2(ur[s0][2], ur[s0][3]);
#pragma unroll
      for (int m = 2; m <= KW; ++m) {
        const int sl = (i + m) % KW;
        const float2 aa = make_float2(ar[sl], ar[sl]);
        x01 = __ffma2_rn(aa, x01, make_float2(ur[sl][0], ur[sl][1]));
        x23 = __ffma2_rn(aa, x23, make_float2(ur[sl][2], ur[sl][3]));
      }
      const float x[4] = {x01.x, x01.y, x23.x, x23.y};
      if (valid) V::st((T*)p.x + xo + n * p.sx_l, x);
    }
  }
}

#ifndef SWR_UNIFORM_CHUNKS
#define SWR_UNIFORM_CHUNKS 16  // uniform window, k <= 16: chunks per SM and column (4: k=4 1.7x slower)
#endif
cudaError_t launch_uniform(bool bf16, Params p, int k, cudaStream_t st, int sms) {
  auto cdiv = [](int64_t x, int64_t y) { return (x + y - 1) / y; };
  const int64_t hpc = 128 / (p.D / 4);
  const int64_t cols = p.B * cdiv(p.H, hpc);
  const int64_t per_sm = k >= 32 ? 4 : SWR_UNIFORM_CHUNKS;  // k = 32: the 32-token ring wants fewer CTAs (16: 10% slower)
  const int64_t want = std::max<int64_t>(1, ((int64_t)sms * per_sm) / std::max<int64_t>(cols, 1));
  p.K = std::max<int64_t>(cdiv(cdiv(p.L, want), 64) * 64, 64);  // tokens per chunk, a multiple of 64 >= k
  const dim3 grid((unsigned)cdiv(p.L, p.K), (unsigned)cdiv(p.H, hpc), (unsigned)p.B);
#define SWR_UNIFORM_CASE(KW)                                                     \
  case KW:                                                                       \
    if (bf16) uniform_fwd<__nv_bfloat16, KW><<<grid, 128, 0, st>>>(p);           \
    else uniform_fwd<float, KW><<<grid, 128, 0, st>>>(p);                        \
    break;
  switch (k) {
    SWR_UNIFORM_CASE(1)
    SWR_UNIFORM_CASE(2)
    SWR_UNIFORM_CASE(4)
    SWR_UNIFORM_CASE(8)
    SWR_UNIFORM_CASE(16)
    SWR_UNIFORM_CASE(32)
    default: return cudaErrorInvalidValue;
  }
#undef SWR_UNIFORM_CASE
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#ifndef SWR_FFMA_FWD_CHUNKS
#define SWR_FFMA_FWD_CHUNKS 2  // SWR: target chunks per SM and (b, head-group) column (8: d=16 13% slower)
#endif
#ifndef SWR_FFMA_MIXF_CHUNKS
#define SWR_FFMA_MIXF_CHUNKS 8  // mixer (one CTA per SM: 4 is 65% slower)
#endif
// forward (SWR and mixer): the streamed kernel, 16 bytes of channels per thread
template <typename T, bool MIX, bool LAYER = false>
static cudaError_t launch_fwd_stream(Params p, cudaStream_t st, int sms) {
  const int64_t hpc = 128 / (p.D / Vec16<T>::N);
  const int64_t cols = p.B * ceil_div(p.H, hpc);
  const int64_t per_sm = MIX ? SWR_FFMA_MIXF_CHUNKS : SWR_FFMA_FWD_CHUNKS;
  const int64_t want_chunks = std::max<int64_t>(1, ((int64_t)sms * per_sm) / std::max<int64_t>(cols, 1));
  int64_t K = std::min<int64_t>(std::max<int64_t>(ceil_div(p.nb, want_chunks), 4), p.nb);
  p.K = K;
  dim3 grid((unsigned)ceil_div(p.nb, K), (unsigned)ceil_div(p.H, hpc), (unsigned)p.B);
  fwd_stream<T, MIX, LAYER><<<grid, 128, 0, st>>>(p);
  return cudaGetLastError();
}

#ifndef SWR_FFMA_BWD_CHUNKS
#define SWR_FFMA_BWD_CHUNKS 8  // backward: target chunks per SM and (b, head-group) column
#endif
template <typename T, int VC, int TPH, bool MIX, bool LAYER = false, int NTH = 128>
static cudaError_t launch_bwd_vec(Params p, cudaStream_t st, int sms) {
  constexpr int HPC = NTH / TPH;
  // lambda staging [kEll][VC/4][NTH] float4; LAYER: + the dk staging; bf16 SWR: the two
  // w stash slots instead (fp32 SWR keeps the three-pass walk: 168 registers spill there)
  constexpr int kSmem = kEll * VC * NTH * 4 * ((LAYER || (!MIX && sizeof(T) == 2)) ? 2 : 1);
  if constexpr (kSmem > 48 * 1024) {  // set per call (per device)
    cudaError_t e = cudaFuncSetAttribute(bwd_ffma_vec<T, VC, TPH, MIX, LAYER, NTH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
  }
  const int64_t cols = p.B * ceil_div(p.H, HPC);
  const int64_t want_chunks = std::max<int64_t>(1, ((int64_t)sms * SWR_FFMA_BWD_CHUNKS * 128 / NTH) / std::max<int64_t>(cols, 1));
  int64_t K = std::max<int64_t>(ceil_div(p.nb, want_chunks), 8);
  K = std::min<int64_t>(K, p.nb);
  p.K = K;
  dim3 grid((unsigned)ceil_div(p.nb, K), (unsigned)ceil_div(p.H, HPC), (unsigned)p.B);
  // the layer kernel needs the dk staging only when heads share k
  const int smem = (LAYER && p.hk == 1) ? kSmem / 2 : kSmem;
  bwd_ffma_vec<T, VC, TPH, MIX, LAYER, NTH><<<grid, NTH, smem, st>>>(p);
  return cudaGetLastError();
}

template <typename T, bool MIX>
static cudaError_t launch_bwd_vec_d(const Params& p, cudaStream_t st, int sms) {
  constexpr int VC = sizeof(T) == 2 ? SWR_FFMA_BWD_VC : 4;
  switch (p.D) {
    case 16: return launch_bwd_vec<T, VC, 16 / VC, MIX>(p, st, sms);
    case 32: return launch_bwd_vec<T, VC, 32 / VC, MIX>(p, st, sms);
    case 64: return launch_bwd_vec<T, VC, 64 / VC, MIX>(p, st, sms);
    default: return launch_bwd_vec<T, VC, 128 / VC, MIX>(p, st, sms);
  }
}

// The layer backward: a CTA of NTH threads holds NTH / TPH heads, which must be a
// multiple of the heads per q group and per k group (ffma_layer_supported).
constexpr int kVC4 = 4;
template <typename T>
static cudaError_t launch_layer_bwd(const Params& p, cudaStream_t st, int sms) {
  const int tph = (int)p.D / kVC4;
  const int64_t hpg = std::max(p.hq, p.hk);
  const bool wide = 128 / tph < hpg;  // 256 threads
  switch (p.D) {
    case 16: return wide ? launch_bwd_vec<T, 4, 4, true, true, 256>(p, st, sms) : launch_bwd_vec<T, 4, 4, true, true, 128>(p, st, sms);
    case 32: return wide ? launch_bwd_vec<T, 4, 8, true, true, 256>(p, st, sms) : launch_bwd_vec<T, 4, 8, true, true, 128>(p, st, sms);
    case 64: return wide ? launch_bwd_vec<T, 4, 16, true, true, 256>(p, st, sms) : launch_bwd_vec<T, 4, 16, true, true, 128>(p, st, sms);
    default: return wide ? launch_bwd_vec<T, 4, 32, true, true, 256>(p, st, sms) : launch_bwd_vec<T, 4, 32, true, true, 128>(p, st, sms);
  }
}

template <typename T, bool MIX, bool BWD>
static cudaError_t launch_d(const Params& p, cudaStream_t st, int sms) {
  if constexpr (!BWD)
    return launch_fwd_stream<T, MIX>(p, st, sms);
  else
    return launch_bwd_vec_d<T, MIX>(p, st, sms);
}

// op: 0 = swr_fwd, 1 = swr_bwd, 2 = mix_fwd, 3 = mix_bwd, 4 / 5 = the layer mixer
// (phalanx_layer_mix fwd / bwd); bf16 selects the dtype
bool narrow_supported(int op, bool bf16, const Params& p);
cudaError_t launch_narrow(int op, const Params& p, cudaStream_t st);

cudaError_t launch_ffma(int op, bool bf16, const Params& p, cudaStream_t st, int sms) {
  // narrow heads (the paper's d = 16): the TMA-staged backward (swr_narrow.cu)
  if (narrow_supported(op, bf16, p)) {
    cudaError_t e = launch_narrow(op, p, st);
    if (e != cudaErrorNotSupported) return e;
  }
  if (op == 4)
    return bf16 ? launch_fwd_stream<__nv_bfloat16, true, true>(p, st, sms) : launch_fwd_stream<float, true, true>(p, st, sms);
  if (op == 5) return bf16 ? launch_layer_bwd<__nv_bfloat16>(p, st, sms) : launch_layer_bwd<float>(p, st, sms);
  if (bf16) {
    switch (op) {
      case 0: return launch_d<__nv_bfloat16, false, false>(p, st, sms);
      case 1: return launch_d<__nv_bfloat16, false, true>(p, st, sms);
      case 2: return launch_d<__nv_bfloat16, true, false>(p, st, sms);
      default: return launch_d<__nv_bfloat16, true, true>(p, st, sms);
    }
  }
  switch (op) {
    case 0: return launch_d<float, false, false>(p, st, sms);
    case 1: return launch_d<float, false, true>(p, st, sms);
    case 2: return launch_d<float, true, false>(p, st, sms);
    default: return launch_d<float, true, true>(p, st, sms);
  }
}

// the layer backward's group sums need every group inside one CTA of at most 256 threads
bool ffma_layer_supported(const Params& p) {
  const int64_t tph = p.D / kVC4, hpc = 256 / tph;
  auto ok = [&](int64_t g) { return g >= 1 && (g & (g - 1)) == 0 && g <= hpc && p.H % g == 0; };
  return ok(p.hq) && ok(p.hk);
}

}  // namespace swr
