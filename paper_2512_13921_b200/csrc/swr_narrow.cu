// swr_narrow.cu -- staged CUDA-core backward for narrow heads (bf16, D = 16 / 32: the
// paper's own head shape d = 16, h = 128), SWR (swr_bwd) and the
// Phalanx mixer (phalanx_mix_bwd).
//
// The block math is Alg. 4's backward as in swr_ffma.cu's bwd_ffma_vec (a thread owns
// VC channels of one head; w_t = L_t u_t as the block-local recurrence; lambda_t the
// local reverse solve; du = lambda + r mu with mu_t = a_{t+1}[0] lambda_{t+1}[0]; the
// da terms du . w[i-1] + g[i-1] lambda . v_{t-1}), but the operands reach the SMs as
// TMA boxes [16 tokens][HC heads][D] through an mbarrier ring instead of per-thread
// 8-byte loads: a producer warp keeps NS-2 blocks in flight ahead of the compute warps,
// and every operand is read from HBM once -- block t-1's inputs, needed for the
// carrier v_{t-1} = w_{t-1}[15], stay in their stage for the next step of
// the reverse walk (the register-staged kernel re-reads them).  A CTA walks a chunk of
// K blocks of one (b, group of HC heads) in reverse time order, with one halo block on
// each side (the right one for mu, the left one for v).
//
// Two channels per thread (VC = 2): twice the warps of four-channel threads, which the
// latency chains of the sweeps need (VC = 4: 242 / 702 us).
//
// Roofline: HBM-bound; algorithmic bytes per (token, head) (2 D + 2) 2 read + (D + 1) 2
// written (SWR), (4 D + 1) 2 read + (3 D + 1) 2 written (mixer) -- DESIGN.md 5.3.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <type_traits>

#include "swr_common.cuh"

namespace swr {

bool tma_encode_bf16(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box, uint32_t kind);

namespace nar {

#ifndef SWR_NAR_K
#define SWR_NAR_K 32  // blocks per CTA chunk
#endif
#ifndef SWR_NAR_GR
#define SWR_NAR_GR 2  // layer backward: q / zk group rows per CTA (16 heads: groups of >= 8; smaller groups measured slower than bwd_ffma_vec)
#endif
#ifndef SWR_NAR_MINB_L
#define SWR_NAR_MINB_L 2  // layer backward at D = 16: CTAs per SM the registers are capped for (D = 32: one CTA fits)
#endif
#ifndef SWR_NAR_K_L
#define SWR_NAR_K_L 16  // layer backward (2 CTAs per SM): shorter chunks balance better, 413 -> 382 us
#endif
#ifndef SWR_NAR_CG
#define SWR_NAR_CG 4  // reverse sweep: tokens whose stage reads are issued together
#endif

struct Maps {
  CUtensorMap t[4];  // d-tensors: SWR u, dx; mixer k, v, dy, q
  CUtensorMap a;     // decays
  CUtensorMap o[3];  // TMA-stored outputs: SWR du; mixer dq, dk, dv
};
#ifndef SWR_NAR_TMA_ST
#define SWR_NAR_TMA_ST 1  // outputs through a shared-memory tile and a TMA store (not the layer)
#endif

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity), "r"(1000000)
      : "memory");
  return ok != 0;
}
// a C-level poll loop: the warp reconverges after it (the consumers' shuffles follow)
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  while (!mbar_try(b, parity)) {
  }
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
      "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// VC bf16 channels (VC = 2: one 32-bit word, VC = 4: two) <-> fp32
template <int VC>
__device__ __forceinline__ void ld_bf(const uint8_t* q, float (&f)[VC]) {
  if constexpr (VC == 4) {
    const uint2 r = *reinterpret_cast<const uint2*>(q);
    f[0] = __uint_as_float(r.x << 16);
    f[1] = __uint_as_float(r.x & 0xffff0000u);
    f[2] = __uint_as_float(r.y << 16);
    f[3] = __uint_as_float(r.y & 0xffff0000u);
  } else {
    const uint32_t r = *reinterpret_cast<const uint32_t*>(q);
    f[0] = __uint_as_float(r << 16);
    f[1] = __uint_as_float(r & 0xffff0000u);
  }
}
template <int VC>
__device__ __forceinline__ void st_bf(__nv_bfloat16* p, const float (&f)[VC]) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(f[0], f[1]);
  if constexpr (VC == 4) {
    __nv_bfloat162 hi = __floats2bfloat162_rn(f[2], f[3]);
    uint2 r;
    r.x = *reinterpret_cast<uint32_t*>(&lo);
    r.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(p) = r;
  } else {
    *reinterpret_cast<__nv_bfloat162*>(p) = lo;
  }
}

// channel-pair arithmetic on the packed fp32x2 pipe (FFMA2 / FMUL2: the same per-lane
// IEEE results as fmaf / __fmul_rn, half the instructions): o = s x + y, o = x y, o = x y + z
// (PK = false: scalar fmaf -- measured faster for the SWR backward, whose sweeps are
// shorter: 168 vs 183 us at d = 16; the mixer gains 359 -> 353 us, the layer 520 -> 497 us)
template <int VC, bool PK = true>
__device__ __forceinline__ void vfma_s(float s, const float (&x)[VC], const float (&y)[VC], float (&o)[VC]) {
  if constexpr (!PK) {
#pragma unroll
    for (int e = 0; e < VC; ++e) o[e] = fmaf(s, x[e], y[e]);
  } else {
#pragma unroll
    for (int e = 0; e < VC; e += 2) {
      const float2 r = __ffma2_rn(make_float2(s, s), make_float2(x[e], x[e + 1]), make_float2(y[e], y[e + 1]));
      o[e] = r.x;
      o[e + 1] = r.y;
    }
  }
}
template <int VC>
__device__ __forceinline__ void vmul(const float (&x)[VC], const float (&y)[VC], float (&o)[VC]) {
#pragma unroll
  for (int e = 0; e < VC; e += 2) {
    const float2 r = __fmul2_rn(make_float2(x[e], x[e + 1]), make_float2(y[e], y[e + 1]));
    o[e] = r.x;
    o[e + 1] = r.y;
  }
}
template <int VC>
__device__ __forceinline__ void vfma(const float (&x)[VC], const float (&y)[VC], const float (&z)[VC], float (&o)[VC]) {
#pragma unroll
  for (int e = 0; e < VC; e += 2) {
    const float2 r = __ffma2_rn(make_float2(x[e], x[e + 1]), make_float2(y[e], y[e + 1]), make_float2(z[e], z[e + 1]));
    o[e] = r.x;
    o[e + 1] = r.y;
  }
}

template <bool MIX, int D, int HC, int NS, int VC, bool LAYER = false>
struct Cfg {
  static constexpr int TPH = D / VC;            // threads per head (VC channels each)
  static constexpr int NC = HC * TPH;           // compute threads
  static constexpr int NCW = NC / 32;           // compute warps
  static constexpr int NT = MIX ? 4 : 2;        // d-tensors per block
  static constexpr int kTile = 16 * HC * D * 2; // bytes of one tensor's box
  // LAYER: zk (x = 0) and q (x = 3) boxes hold at most GR group rows per token
  static constexpr int GR = LAYER ? SWR_NAR_GR : HC;
  static constexpr int kTileG = 16 * GR * D * 2;
  static __host__ __device__ constexpr int off(int x) {
    return x == 0 ? 0 : x == 1 ? kTileG : x == 2 ? kTileG + kTile : kTileG + 2 * kTile;
  }
  static constexpr int kAOff = MIX ? 2 * kTileG + 2 * kTile : 2 * kTile;
  static constexpr int kA = 16 * HC * 2;        // the decay box
  // LAYER: the decays a = sigma(za) in fp32, [16][HC], written by the stage's prep
  static constexpr int kAFOff = ((kAOff + kA + 15) / 16) * 16;
  static constexpr int kStage = ((kAFOff + (LAYER ? 16 * HC * 4 : 0) + 127) / 128) * 128;
  // LAYER: the per-head dq / dk terms of a block, [16][HC][D] fp32 each, for the group sums
  static constexpr int kScrG = NS * kStage;
  // TST: the block's output tiles [16][HC][D] bf16 (SWR du; mixer dq, dk, dv), double-
  // buffered, leave through TMA stores (rows past L and heads past H are clipped by TMA).
  // Measured (tools/nar_time.py against -DSWR_NAR_TMA_ST=0): SWR d = 16 168.5 -> 165 us,
  // d = 32 155 -> 148 us, mixer d = 32 338 -> 313 us; the d = 16 mixer (16 heads, one CTA
  // per SM) 354 -> 371 us keeps the per-thread stores
  static constexpr bool TST = SWR_NAR_TMA_ST && !LAYER && !(MIX && D == 16);
  static constexpr int NOUT = MIX ? 3 : 1;
  static constexpr int kOutOff = kScrG + (LAYER ? 2 * 16 * HC * D * 4 : 0);
  static constexpr int kBar = kOutOff + (TST ? 2 * NOUT * kTile : 0);
  static constexpr int kBytes = kBar + 2 * NS * 8;
  static_assert(NC % 32 == 0 && NS >= 3, "whole compute warps; current + previous + prefetch");
};

// da: the head's TPH threads hold partial sums of all 16 tokens; a transpose-reduce
// leaves thread qd with tokens (16 / TPH) qd .. in a fixed order (deterministic)
template <int TPH>
__device__ __forceinline__ void head_reduce(float (&pv)[16], int qd) {
  int n = 16;
#pragma unroll
  for (int m = TPH / 2; m >= 1; m /= 2) {
    n /= 2;
    const bool up = (qd & m) != 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < n) {
        const float mine = up ? pv[k + n] : pv[k];
        const float other = up ? pv[k] : pv[k + n];
        pv[k] = mine + __shfl_xor_sync(0xffffffffu, other, m);
      }
    }
  }
}

// LAYER (phalanx_layer_mix_bwd): a = sigma(za) and k = sigma(zk)
// when the flags say logits (dza = da a (1 - a), dzk = dk k (1 - k)),
// q and zk shared by groups of hq / hk heads -- the boxes of q / zk carry
// the CTA's HC / hq (HC / hk) group rows, and the group sums of dq / dzk are formed in
// shared memory in head order (deterministic); HC is a multiple of hq and hk.
template <bool MIX, int D, int HC, int NS, int VC, bool LAYER = false>
__global__ void __launch_bounds__(Cfg<MIX, D, HC, NS, VC, LAYER>::NC + 32, (LAYER && D == 16) ? SWR_NAR_MINB_L : 1)
    bwd_staged(const __grid_constant__ Maps maps, const Params p) {
  static_assert(!LAYER || MIX, "the layer options apply to the mixer");
  using C = Cfg<MIX, D, HC, NS, VC, LAYER>;
  constexpr int TPH = C::TPH, NT = C::NT;
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + C::kBar);
  uint64_t* empty = full + NS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t b = blockIdx.z;
  const int h0 = blockIdx.y * HC;
  const int64_t t0 = (int64_t)blockIdx.x * p.K;
  const int64_t t1 = min(t0 + p.K, p.nb);
  const bool rhalo = t1 < p.nb, lhalo = t0 > 0;
  const int n_seq = (int)(t1 - t0) + (rhalo ? 1 : 0) + (lhalo ? 1 : 0);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // LAYER: heads per q / k group and the group rows of the CTA's boxes
  const int hq = LAYER ? (int)p.hq : 1, hk = LAYER ? (int)p.hk : 1;
  const int GQ = HC / hq, GK = HC / hk;
  if (warp == C::NCW) {
    // ===== producer: blocks t1 (right halo), t1-1, ..., t0, t0-1 (left halo) =====
    if (lane == 0) {
      for (int j = 0; j < n_seq; ++j) {
        const int s = j % NS;
        mbar_wait(&empty[s], ((j / NS) & 1) ^ 1);
        const int tb = (int)(t1 - 1 - j + (rhalo ? 1 : 0));
        uint8_t* st = sm + s * C::kStage;
        // halo blocks load only what they are read for: the right one the adjoint input
        // (dx / dy, q) for mu, the left one the Pass-I input (u / k, v) for v_{t0-1}
        const bool rh = rhalo && j == 0, lh = lhalo && j == n_seq - 1;
        auto need = [&](int x) {
          const bool u_in = MIX ? x < 2 : x == 0;
          return !(rh && u_in) && !(lh && !u_in);
        };
        auto box_bytes = [&](int x) {
          return (LAYER && x == 0) ? GK * 16 * D * 2 : (LAYER && x == 3) ? GQ * 16 * D * 2 : C::kTile;
        };
        uint32_t bytes = C::kA;
#pragma unroll
        for (int x = 0; x < NT; ++x)
          if (need(x)) bytes += box_bytes(x);
        mbar_expect_tx(&full[s], bytes);
#pragma unroll
        for (int x = 0; x < NT; ++x)
          if (need(x))
            tma_load_4d(st + C::off(x), &maps.t[x], &full[s], 0, (LAYER && x == 0) ? h0 / hk : (LAYER && x == 3) ? h0 / hq : h0,
                        tb * kEll, (int)b);
        tma_load_3d(st + C::kAOff, &maps.a, &full[s], h0, tb * kEll, (int)b);
      }
    }
    return;
  }

  // ===== compute: thread (head hl, channels c .. c+3) =====
  const int hl = tid / TPH, qd = tid % TPH, c = VC * qd;
  const int64_t h = h0 + hl;
  const bool act = h < p.H;
  const int64_t hc = act ? h : p.H - 1;
  const int64_t xo = b * p.sx_b + hc * p.sx_h + c;
  const int64_t co = (b * p.H + hc) * p.D + c;
  __nv_bfloat16* dA = (__nv_bfloat16*)p.da + b * p.sa_b + hc * p.sa_h;
  // operand access inside a stage: tensor x, token i -> this thread's 4 channels
  // rows per token and this thread's row in each tensor's box (LAYER: k and q hold group rows)
  // LAYER: the thread's byte offset in each box and the box's bytes per token, once (the
  // group rows make them runtime values; divisions and products kept out of the sweeps)
  int offx[4], strx[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int rws = (LAYER && x == 0) ? GK : (LAYER && x == 3) ? GQ : HC;
    const int rw = (LAYER && x == 0) ? hl / hk : (LAYER && x == 3) ? hl / hq : hl;
    offx[x] = C::off(x) + (rw * D + c) * 2;
    strx[x] = rws * D * 2;
  }
  auto boff = [&](int x, int i) {
    if constexpr (LAYER) return offx[x] + i * strx[x];
    return C::off(x) + ((i * HC + hl) * D + c) * 2;
  };
  auto ld = [&](const uint8_t* st, int x, int i, float (&f)[VC]) { ld_bf<VC>(st + boff(x, i), f); };
  auto ldA = [&](const uint8_t* st, int i) {  // LAYER: a (= sigma(za)) in fp32 from the prep
    if constexpr (LAYER) return reinterpret_cast<const float*>(st + C::kAFOff)[i * HC + hl];
    return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(st + C::kAOff + (i * HC + hl) * 2));
  };
  auto cbar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(C::NC) : "memory"); };
  // LAYER prep of a stage, once, by all compute threads (then a CTA barrier): a = sigma(za)
  // in fp32 beside the box, k = sigma(zk) over the zk box in bf16 (the
  // tensor-core family's rounding, R20) -- the group's heads share both
  auto prep = [&](uint8_t* st) {
    if constexpr (LAYER) {
      float* af = reinterpret_cast<float*>(st + C::kAFOff);
      const __nv_bfloat16* za = reinterpret_cast<const __nv_bfloat16*>(st + C::kAOff);
      for (int x = tid; x < 16 * HC; x += C::NC) {
        const float z = __bfloat162float(za[x]);
        af[x] = p.logit_a ? sigmoid_f(z) : z;
      }
      if (p.logit_k) {
        __nv_bfloat162* kz = reinterpret_cast<__nv_bfloat162*>(st + C::off(0));
        for (int x = tid; x < 16 * GK * D / 2; x += C::NC) {
          const float2 z = __bfloat1622float2(kz[x]);
          kz[x] = __floats2bfloat162_rn(sigmoid_gate<__nv_bfloat16>(z.x), sigmoid_gate<__nv_bfloat16>(z.y));
        }
      }
      cbar();
    }
  };
  // Pass-I input u (SWR) / u^ = k (.) v, and the adjoint input G = dx / dy (.) q
  auto ld_u = [&](const uint8_t* st, int i, float (&u)[VC]) {
    if constexpr (!MIX) {
      ld(st, 0, i, u);
    } else {
      float kk[VC], vv[VC];
      ld(st, 0, i, kk);
      ld(st, 1, i, vv);
#pragma unroll
      for (int e = 0; e < VC; ++e) u[e] = __fmul_rn(kk[e], vv[e]);
    }
  };
  auto ld_g = [&](const uint8_t* st, int i, float (&g)[VC]) {
    if constexpr (!MIX) {
      ld(st, 1, i, g);
    } else {
      float dd[VC], qq[VC];
      ld(st, 2, i, dd);
      ld(st, 3, i, qq);
#pragma unroll
      for (int e = 0; e < VC; ++e) g[e] = __fmul_rn(dd[e], qq[e]);
    }
  };
  auto release = [&](int s) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  };

  float mu[VC];
#pragma unroll
  for (int e = 0; e < VC; ++e) mu[e] = 0.f;
  int j = 0;
  if (rhalo) {  // mu_{t1-1} = a_{t1}[0] lambda_{t1}[0]: the local reverse solve of block t1
    mbar_wait(&full[0], 0);
    prep(sm);
    const uint8_t* st = sm;
    float lam[VC];
    ld_g(st, 15, lam);  // padding past L: the TMA zero fill gives G = 0, so lambda = 0 there
#pragma unroll
    for (int i = 14; i >= 0; --i) {
      float g[VC];
      ld_g(st, i, g);
      const float a1 = ldA(st, i + 1);
#pragma unroll
      for (int e = 0; e < VC; ++e) lam[e] = fmaf(a1, lam[e], g[e]);
    }
    const float a0 = ldA(st, 0);
#pragma unroll
    for (int e = 0; e < VC; ++e) mu[e] = a0 * lam[e];
    release(0);
    j = 1;
  } else if (p.mu_in) {
#pragma unroll
    for (int e = 0; e < VC; ++e) mu[e] = p.mu_in[co + e];
  }

  // raw operand words (VC bf16) of tensor x, token i, read from the stage in one LDS
  using R = typename std::conditional<VC == 4, uint2, uint32_t>::type;
  auto ldr = [&](const uint8_t* st, int x, int i) {
    return *reinterpret_cast<const R*>(st + boff(x, i));
  };
  auto cvt = [&](const R& r, float (&f)[VC]) { ld_bf<VC>(reinterpret_cast<const uint8_t*>(&r), f); };
  auto cvtk = [&](const R& r, float (&f)[VC]) { cvt(r, f); };  // the key operand (LAYER: sigma applied by the prep)
  float* sq = reinterpret_cast<float*>(sm + C::kScrG);  // LAYER: per-head dq [16][HC][D]
  float* sk = sq + 16 * HC * D;                        // LAYER: per-head dk (before sigma')
  constexpr int CG = SWR_NAR_CG;  // reverse sweep: tokens whose operands are read together

  const int j_first = j;
  for (int64_t t = t1 - 1; t >= t0; --t, ++j) {
    const int s = j % NS;
    mbar_wait(&full[s], (j / NS) & 1);
    if (j == j_first) prep(sm + s * C::kStage);  // later stages were prepped as block t-1
    const uint8_t* st = sm + s * C::kStage;
    const int64_t n0 = t * kEll;
    const int lim_rt = (p.L - n0 < kEll) ? (int)(p.L - n0) : kEll;
    // LAYER: the block body twice, whole blocks (every block but a ragged last one) without
    // the per-token validity tests and the ragged tail with them
    auto block = [&](auto full_t) {
      constexpr bool FULL = decltype(full_t)::value;
      const int lim = FULL ? kEll : lim_rt;
      // A) carrier v_{t-1} = w_{t-1}[15] from the next stage (block t-1 is whole); the
      //    block's operands are read first, then the chain runs on registers
      float vprev[VC];
      if (t > 0) {
        const int s1 = (j + 1) % NS;
        mbar_wait(&full[s1], ((j + 1) / NS) & 1);
        prep(sm + s1 * C::kStage);
        const uint8_t* sp = sm + s1 * C::kStage;
        R r0[kEll], r1[kEll];
        (void)r1;
        float ap[kEll];
  #pragma unroll
        for (int i = 0; i < kEll; ++i) {
          r0[i] = ldr(sp, 0, i);
          if constexpr (MIX) r1[i] = ldr(sp, 1, i);
          ap[i] = ldA(sp, i);
        }
  #pragma unroll
        for (int i = 0; i < kEll; ++i) {
          float u[VC];
          if constexpr (MIX)
            cvtk(r0[i], u);
          else
            cvt(r0[i], u);
          if constexpr (MIX) {
            float vv[VC];
            cvt(r1[i], vv);
            vmul<VC>(u, vv, u);
          }
          if (i == 0) {
  #pragma unroll
            for (int e = 0; e < VC; ++e) vprev[e] = u[e];
          } else {
            vfma_s<VC, MIX>(ap[i], vprev, u, vprev);
          }
        }
      } else {
  #pragma unroll
        for (int e = 0; e < VC; ++e) vprev[e] = p.carry_in ? p.carry_in[co + e] : 0.f;
      }
      // decays of block t (pad a = 1 past L), g[i] = a[0] ... a[i], and Pass I of block t
      // forward with w kept in registers
      float av[kEll], gsv[kEll], w[kEll][VC];
      {
        R r0[kEll], r1[kEll];
        (void)r1;
  #pragma unroll
        for (int i = 0; i < kEll; ++i) {
          r0[i] = ldr(st, 0, i);
          if constexpr (MIX) r1[i] = ldr(st, 1, i);
          av[i] = ldA(st, i);
        }
  #pragma unroll
        for (int i = 0; i < kEll; ++i) {
          if (i >= lim) av[i] = 1.f;
          gsv[i] = i == 0 ? av[0] : gsv[i - 1] * av[i];
          float u[VC];
          if constexpr (MIX)
            cvtk(r0[i], u);
          else
            cvt(r0[i], u);
          if constexpr (MIX) {
            float vv[VC];
            cvt(r1[i], vv);
            vmul<VC>(u, vv, u);
          }
          if (i == 0) {
  #pragma unroll
            for (int e = 0; e < VC; ++e) w[0][e] = u[e];
          } else {
            vfma_s<VC, MIX>(av[i], w[i - 1], u, w[i]);
          }
        }
      }
      // C) one reverse sweep: lambda, r, du (mixer: dq, dk, dv), the da terms
      uint8_t* ob = sm + C::kOutOff + (j & 1) * C::NOUT * C::kTile;  // TST: this block's output tiles
      if constexpr (C::TST) {  // the TMA store of two blocks ago has read this buffer
        if (tid == 0) bulk_wait_read1();
        cbar();
      }
      auto out_at = [&](int x, int i) {
        return reinterpret_cast<__nv_bfloat16*>(ob + x * C::kTile + ((i * HC + hl) * D + c) * 2);
      };
      // per-thread global stores: the block's base offset once, token offsets in 32 bits
      const int64_t ob0 = xo + n0 * p.sx_l;
      const int sxl = (int)p.sx_l;  // < 2^26 (narrow_supported)
      (void)ob0;
      (void)sxl;
      float part[kEll];
      float lam[VC], mu_next[VC];
      float rr = 1.f;
  #pragma unroll
      for (int i0 = kEll - CG; i0 >= 0; i0 -= CG) {
        R rg[CG], rq[CG], rk[CG], rv[CG];
        (void)rq;
        (void)rk;
        (void)rv;
  #pragma unroll
        for (int m = 0; m < CG; ++m) {
          rg[m] = ldr(st, MIX ? 2 : 1, i0 + m);  // dx (SWR) / dy (mixer)
          if constexpr (MIX) {
            rq[m] = ldr(st, 3, i0 + m);
            rk[m] = ldr(st, 0, i0 + m);
            rv[m] = ldr(st, 1, i0 + m);
          }
        }
  #pragma unroll
        for (int m = CG - 1; m >= 0; --m) {
          const int i = i0 + m;
          float g[VC], dd[VC];
          cvt(rg[m], dd);
          if constexpr (MIX) {
            float qq[VC];
            cvt(rq[m], qq);
            vmul<VC>(dd, qq, g);  // G = dy (.) q
          } else {
  #pragma unroll
            for (int e = 0; e < VC; ++e) g[e] = dd[e];
          }
          if (i == kEll - 1) {
  #pragma unroll
            for (int e = 0; e < VC; ++e) lam[e] = g[e];  // lambda[15] = G[15]
          } else {
            vfma_s<VC, MIX>(av[i + 1], lam, g, lam);
            rr *= av[i + 1];  // r_t[i] = a_t[i+1] ... a_t[15]
          }
          float du[VC];
          vfma_s<VC, MIX>(rr, mu, lam, du);
          float sdot = 0.f, lv = 0.f;  // sum_c du[i] w[i-1] (w[-1] = 0), sum_c lambda[i] v_{t-1}
          if (i > 0) {
  #pragma unroll
            for (int e = 0; e < VC; ++e) sdot = (e == 0) ? du[e] * w[i - 1][e] : fmaf(du[e], w[i - 1][e], sdot);
          }
  #pragma unroll
          for (int e = 0; e < VC; ++e) lv = (e == 0) ? lam[e] * vprev[e] : fmaf(lam[e], vprev[e], lv);
          part[i] = fmaf(i > 0 ? gsv[i - 1] : 1.f, lv, sdot);
          // (32-bit token offsets: layer 423 -> 413 us; the mixer measured 1% slower with them)
          const int64_t o = LAYER ? ob0 + i * sxl : xo + (n0 + i) * p.sx_l;
          const bool valid = act && i < lim;
          (void)o;
          (void)valid;
          if constexpr (!MIX) {
            if constexpr (C::TST)
            st_bf<VC>(out_at(0, i), du);
          else if (valid)
            st_bf<VC>((__nv_bfloat16*)p.du + o, du);
          } else {
            float kk[VC], vv[VC];
            cvtk(rk[m], kk);
            cvt(rv[m], vv);
            float dq[VC], dk[VC], dv[VC], xt[VC];
            vfma_s<VC, MIX>(gsv[i], vprev, w[i], xt);  // x~ = w + g v
            vmul<VC>(dd, xt, dq);                 // dq = dy x~
            vmul<VC>(du, vv, dk);                 // dk = du^ v
            vfma<VC>(du, kk, dd, dv);             // dv = du^ k + dy
            if constexpr (LAYER) {  // the group sums below
              float* q2 = sq + (i * HC + hl) * D + c;
              float* k2 = sk + (i * HC + hl) * D + c;
  #pragma unroll
              for (int e = 0; e < VC; ++e) {
                q2[e] = dq[e];
                k2[e] = dk[e];
              }
              if (valid) st_bf<VC>((__nv_bfloat16*)p.dv + o, dv);
            } else if constexpr (C::TST) {
              st_bf<VC>(out_at(0, i), dq);
              st_bf<VC>(out_at(1, i), dk);
              st_bf<VC>(out_at(2, i), dv);
            } else if (valid) {
              st_bf<VC>((__nv_bfloat16*)p.dq + o, dq);
              st_bf<VC>((__nv_bfloat16*)p.dk + o, dk);
              st_bf<VC>((__nv_bfloat16*)p.dv + o, dv);
            }
          }
          if (i == 0) {
  #pragma unroll
            for (int e = 0; e < VC; ++e) mu_next[e] = av[0] * lam[e];  // mu_{t-1} = a_t[0] lambda_t[0]
          }
        }
      }
  #pragma unroll
      for (int e = 0; e < VC; ++e) mu[e] = mu_next[e];
      if (t == 0 && act && p.mu_out) {
  #pragma unroll
        for (int e = 0; e < VC; ++e) p.mu_out[co + e] = mu[e];
      }
      if constexpr (LAYER) {
        // group sums: item (token i, group row g, channel pair) sums the group's heads in
        // head order; dzk = (sum dk) k (1 - k) with the group's k = sigma(zk)
        cbar();
        const int64_t G_q = p.H / hq, G_k = p.H / hk;
        // group counts per CTA are powers of two (HC = 16 is a multiple of hq, hk): shifts
        const int lgq = __ffs(GQ) - 1, lgk = __ffs(GK) - 1;
        for (int it = tid; it < 16 * GQ * TPH; it += C::NC) {
          const int rem = it / TPH, i = rem >> lgq, g = rem & (GQ - 1), cq = VC * (it % TPH);
          float acc[VC];
  #pragma unroll
          for (int e = 0; e < VC; ++e) acc[e] = 0.f;
          for (int m = 0; m < hq; ++m) {
  #pragma unroll
            for (int e = 0; e < VC; ++e) acc[e] += sq[(i * HC + g * hq + m) * D + cq + e];
          }
          const int64_t gg = h0 / hq + g;
          if (gg < G_q && i < lim) st_bf<VC>((__nv_bfloat16*)p.dq + b * p.sq_b + (n0 + i) * p.sq_l + gg * p.sq_h + cq, acc);
        }
        for (int it = tid; it < 16 * GK * TPH; it += C::NC) {
          const int rem = it / TPH, i = rem >> lgk, g = rem & (GK - 1), cq = VC * (it % TPH);
          float acc[VC];
  #pragma unroll
          for (int e = 0; e < VC; ++e) acc[e] = 0.f;
          for (int m = 0; m < hk; ++m) {
  #pragma unroll
            for (int e = 0; e < VC; ++e) acc[e] += sk[(i * HC + g * hk + m) * D + cq + e];
          }
          if (p.logit_k) {
            float kv[VC];
            ld_bf<VC>(st + ((i * GK + g) * D + cq) * 2, kv);  // k = sigma(zk) of the group row (prep)
  #pragma unroll
            for (int e = 0; e < VC; ++e) acc[e] *= kv[e] * (1.f - kv[e]);
          }
          const int64_t gg = h0 / hk + g;
          if (gg < G_k && i < lim) st_bf<VC>((__nv_bfloat16*)p.dk + b * p.sk_b + (n0 + i) * p.sk_l + gg * p.sk_h + cq, acc);
        }
        cbar();  // the scratch is rewritten by the next block
        if (p.logit_a) {  // dza = da sigma'(za), sigma' = a (1 - a)
  #pragma unroll
          for (int i = 0; i < kEll; ++i) part[i] *= av[i] * (1.f - av[i]);
        }
      }
      if constexpr (C::TST) {  // the output tiles are complete: one thread stores them
        fence_proxy_async();
        cbar();
        if (tid == 0) {
#pragma unroll
          for (int x = 0; x < C::NOUT; ++x) tma_store_4d(&maps.o[x], ob + x * C::kTile, 0, h0, (int)n0, (int)b);
          bulk_commit();
        }
      }
      release(s);  // block t's inputs are consumed (block t-1's stay for the next step)
      // da: deterministic reduction over the head's channels
      head_reduce<TPH>(part, qd);
      constexpr int NV = kEll / TPH;
      if (act) {
  #pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int tok = NV * qd + k;
          if (tok < lim) dA[(n0 + tok) * p.sa_l] = __float2bfloat16_rn(part[k]);
        }
      }
    };
    if constexpr (LAYER) {  // (measured: the layer backward gains 465 -> 423 us at d = 16;
      if (lim_rt == kEll)  // the SWR / mixer kernels lose 3-6% to the larger code)
        block(std::true_type{});
      else
        block(std::false_type{});
    } else {
      block(std::false_type{});
    }
  }
  if (C::TST && tid == 0) bulk_wait_all();  // the last stores have read their tiles
}

// heads per CTA and ring stages, measured back to back at d = 16, h = 128, L = 8K, B = 8
// (tools/nar_time.py): SWR 8 heads x 3 stages (25 KB, 8 CTAs per SM) 169 us against
// 172-207 us for 16 / 32 heads, 4-5 stages or 16 / 64-block chunks; mixer 16 heads x 4
// stages (133 KB, one CTA) 361 us against 383-488 us for 8 heads or 6 stages
#ifndef SWR_NAR_HC_S
#define SWR_NAR_HC_S 8
#endif
#ifndef SWR_NAR_NS_S
#define SWR_NAR_NS_S 3
#endif
#ifndef SWR_NAR_HC_M
#define SWR_NAR_HC_M 16
#endif
#ifndef SWR_NAR_NS_M
#define SWR_NAR_NS_M 4
#endif
#ifndef SWR_NAR_HC_L
#define SWR_NAR_HC_L 16  // layer backward: heads per CTA (a multiple of the group sizes)
#endif
#ifndef SWR_NAR_NS_L
#define SWR_NAR_NS_L 3
#endif
#ifndef SWR_NAR_VC
#define SWR_NAR_VC 2  // channels per thread
#endif

template <bool MIX, int D, int HC, int NS, int VC, bool LAYER = false>
static cudaError_t launch(const Params& p0, cudaStream_t st) {
  using C = Cfg<MIX, D, HC, NS, VC, LAYER>;
  Params p = p0;
  p.K = LAYER ? SWR_NAR_K_L : SWR_NAR_K;
  Maps m;
  const void* ts[4] = {MIX ? p.k : p.u, MIX ? p.v : p.dx, p.dy, p.q};
  const uint64_t dims[4] = {(uint64_t)p.D, (uint64_t)p.H, (uint64_t)p.L, (uint64_t)p.B};
  const uint64_t str[3] = {(uint64_t)p.sx_h * 2, (uint64_t)p.sx_l * 2, (uint64_t)p.sx_b * 2};
  const uint32_t box[4] = {(uint32_t)D, (uint32_t)HC, 16, 1};
  for (int x = 0; x < C::NT; ++x) {
    if (LAYER && (x == 0 || x == 3)) {  // group-shared zk / q [B, L, G, D]: HC / hk (HC / hq) group rows
      const int64_t hg = x == 0 ? p.hk : p.hq;
      const uint64_t gd[4] = {(uint64_t)p.D, (uint64_t)(p.H / hg), (uint64_t)p.L, (uint64_t)p.B};
      const uint64_t gs[3] = {(uint64_t)(x == 0 ? p.sk_h : p.sq_h) * 2, (uint64_t)(x == 0 ? p.sk_l : p.sq_l) * 2,
                              (uint64_t)(x == 0 ? p.sk_b : p.sq_b) * 2};
      const uint32_t gb[4] = {(uint32_t)D, (uint32_t)(HC / hg), 16, 1};
      if (!tma_encode_bf16(&m.t[x], ts[x], 4, gd, gs, gb, 256 + (uint32_t)(HC / hg))) return cudaErrorNotSupported;
    } else if (!tma_encode_bf16(&m.t[x], ts[x], 4, dims, str, box, 64 + HC)) {
      return cudaErrorNotSupported;
    }
  }
  if constexpr (C::TST) {
    void* os[3] = {MIX ? p.dq : p.du, p.dk, p.dv};
    for (int x = 0; x < C::NOUT; ++x)
      if (!tma_encode_bf16(&m.o[x], os[x], 4, dims, str, box, 128 + HC)) return cudaErrorNotSupported;
  }
  const uint64_t adims[3] = {(uint64_t)p.H, (uint64_t)p.L, (uint64_t)p.B};
  const uint64_t astr[2] = {(uint64_t)p.sa_l * 2, (uint64_t)p.sa_b * 2};
  const uint32_t abox[3] = {(uint32_t)HC, 16, 1};
  if (!tma_encode_bf16(&m.a, p.a, 3, adims, astr, abox, 96 + HC)) return cudaErrorNotSupported;
  constexpr int smem = C::kBytes;
  static_assert(smem <= 227 * 1024, "shared memory budget");
  // the attributes are per device (per context): set once for each device this process uses
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = -1;
  static std::atomic<bool> attr[64];
  if (dev < 0 || !attr[dev].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(bwd_staged<MIX, D, HC, NS, VC, LAYER>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(bwd_staged<MIX, D, HC, NS, VC, LAYER>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    if (dev >= 0) attr[dev].store(true, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((p.nb + p.K - 1) / p.K), (unsigned)((p.H + HC - 1) / HC), (unsigned)p.B);
  cfg.blockDim = dim3(C::NC + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, bwd_staged<MIX, D, HC, NS, VC, LAYER>, m, p);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace nar

// the staged backward's envelope: bf16, D in {16, 32}, TMA-addressable operands (head
// stride D, 16-byte token / batch strides, 16-byte aligned bases, decays with heads
// contiguous), the plain SWR / mixer ops (the layer options run on bwd_ffma_vec)
bool narrow_supported(int op, bool bf16, const Params& p) {
#ifdef SWR_NAR_OFF
  return false;  // A/B builds: the register-staged kernels everywhere
#endif
  if (!bf16 || (op != 1 && op != 3 && op != 5) || (p.D != 16 && p.D != 32)) return false;
  if (op == 5) {  // layer: q / zk group tensors with heads contiguous, groups inside a CTA's 16 heads
    if (p.sq_h != p.D || p.sk_h != p.D || (p.sq_l * 2) % 16 || (p.sq_b * 2) % 16 || (p.sk_l * 2) % 16 ||
        (p.sk_b * 2) % 16)
      return false;
    if (p.hq < 1 || p.hk < 1 || SWR_NAR_HC_L % p.hq || SWR_NAR_HC_L % p.hk) return false;
    if (SWR_NAR_HC_L / p.hq > SWR_NAR_GR || SWR_NAR_HC_L / p.hk > SWR_NAR_GR) return false;
  }
  if (p.sx_h != p.D || (p.sx_l * 2) % 16 || (p.sx_b * 2) % 16) return false;
  if (p.sa_h != 1 || (p.sa_l * 2) % 16 || (p.sa_b * 2) % 16) return false;
  if (p.B > 65535 || p.H > (int64_t)65535 * 8 || p.L > (int64_t(1) << 30) || p.sx_l > (int64_t(1) << 26))
    return false;
  auto a16 = [](const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  const void* ptrs[] = {p.u, p.dx, p.du, p.q, p.k, p.v, p.dy, p.dq, p.dk, p.dv, p.a};
  for (const void* q : ptrs)
    if (!a16(q)) return false;
  return true;
}

cudaError_t launch_narrow(int op, const Params& p, cudaStream_t st) {
  if (op == 5)
    return p.D == 16 ? nar::launch<true, 16, SWR_NAR_HC_L, SWR_NAR_NS_L, SWR_NAR_VC, true>(p, st)
                     : nar::launch<true, 32, SWR_NAR_HC_L, 3, SWR_NAR_VC, true>(p, st);
  if (op == 1)
    return p.D == 16 ? nar::launch<false, 16, SWR_NAR_HC_S, SWR_NAR_NS_S, SWR_NAR_VC>(p, st)
                     : nar::launch<false, 32, SWR_NAR_HC_S, SWR_NAR_NS_S, SWR_NAR_VC>(p, st);
  // D = 32: half the heads per CTA (the same bytes per stage)
  constexpr int kHc32 = SWR_NAR_HC_M / 2 < 8 ? 8 : SWR_NAR_HC_M / 2;
  return p.D == 16 ? nar::launch<true, 16, SWR_NAR_HC_M, SWR_NAR_NS_M, SWR_NAR_VC>(p, st)
                   : nar::launch<true, 32, kHc32, SWR_NAR_NS_M, SWR_NAR_VC>(p, st);
}

}  // namespace swr
