// swr_tc.cu -- tensor-core kernel family (SWR_PATH_TC) for bf16, D = 128.
//
// Block Two-Pass (Alg. 4) mapped onto sm_100a:
//
//   * Pass I  w_t = L_t u_t is ONE tcgen05.mma per 16-token block with the
//     roles transposed so the accumulator lands channel-major in TMEM:
//         D[c][i] = sum_j  u_t[j][c] * L_t[i][j]      (D = w_t^T, M=128, N=16, K=16)
//     A = u_t^T comes straight from the TMA-staged tile (MN-major, 128B
//     swizzle), B = L_t^T is the 16x16 transfer built by Alg. 3 (linear-space
//     column cumulative products) in bf16, and the fp32
//     accumulator sits in TMEM lanes = channels, columns = tokens.
//   * Backward also computes lambda_t = L_t^T G_t the same way (B = L_t).
//   * The epilogue warps read TMEM with tcgen05.ld (thread = channel, all 16
//     tokens), so Pass II x~ = w + g v_{t-1}, the carrier
//     v_t = w_t[15] and the backward pairings are thread-local; the
//     carrier between consecutive blocks stays in a register (no SMEM/DSMEM
//     exchange, no cross-CTA sync).
//   * One persistent CTA per SM walks a contiguous range of (b, h, block)
//     items; tiles move HBM -> SMEM -> HBM with TMA (cp.async.bulk.tensor),
//     through an NS-stage mbarrier ring; a CTA recomputes one halo block at a
//     range boundary (and, backward, one on the right).
//
// Warp roles: 4*NG epilogue warps in NG groups of 4 (group g handles items
// j = g mod NG; warp w reads TMEM lanes 32*(w%4)..+31), then prep warps (L tiles,
// g/r, mixer pre-gates), then the producer (TMA), then the MMA issuer.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "swr_common.cuh"

namespace swr {
namespace tc {

constexpr int kD = 128;          // head dim served by this family
constexpr int kTile = 4096;      // one 16 x 128 bf16 tile (two 64-channel halves)
constexpr int kHalf = 2048;      // one 64-channel half: 16 rows x 128 B, 128B-swizzled

// ---------------------------------------------------------------------------
// per-op configuration
//   NT   TMA-loaded input tiles per item     NP  prep-computed A tiles
//   NS   pipeline stages                     COLS TMEM columns per stage
// ---------------------------------------------------------------------------
template <int OP>
struct Cfg;
template <>
struct Cfg<0> {  // swr_fwd: in u;            out x  (over u)
  static constexpr int NT = 1, NP = 0, NS = 16, COLS = 16, NPREP = 1, NOUT = 1, NG = 2;
  static constexpr bool BWD = false, MIX = false;
};
template <>
struct Cfg<1> {  // swr_bwd: in u, G;         out du (over G)
  static constexpr int NT = 2, NP = 0, NS = 12, COLS = 32, NPREP = 1, NOUT = 1, NG = 2;
  static constexpr bool BWD = true, MIX = false;
};
template <>
struct Cfg<2> {  // mix fwd: in q, k, v;      out y  (over q);  prep u^ = k v
  static constexpr int NT = 3, NP = 1, NS = 10, COLS = 16, NPREP = 4, NOUT = 1, NG = 2;
  static constexpr bool BWD = false, MIX = true;
};
template <>
struct Cfg<3> {  // mix bwd: in q, k, v, dy;  out dq (over dy), dk (over k), dv (over v)
  static constexpr int NT = 4, NP = 2, NS = 7, COLS = 32, NPREP = 4, NOUT = 3, NG = 2;
  static constexpr bool BWD = true, MIX = true;
};

// stage layout (bytes, every tile 1024-aligned for the 128B swizzle atoms)
template <int OP>
struct Stage {
  using C = Cfg<OP>;
  static constexpr int kTiles = 0;                                // NT input tiles, then NP prep tiles
  static constexpr int kA = (C::NT + C::NP) * kTile;              // decay box [16 tokens][8 heads] bf16
  static constexpr int kLT = kA + 256;                            // B operand of W:      L_t^T  (512 B)
  static constexpr int kL = kLT + 512;                            // B operand of lambda: L_t    (512 B)
  static constexpr int kG = kL + 512;                             // g_t[16] fp32
  static constexpr int kR = kG + 64;                              // r_t[16] fp32
  static constexpr int kRaw = kR + 64;
  static constexpr int kBytes = (kRaw + 1023) / 1024 * 1024;
};

template <int OP>
constexpr int smem_bytes() {
  // stages + barriers/scratch (4 KiB) + 1 KiB alignment slack
  return Cfg<OP>::NS * Stage<OP>::kBytes + 4096 + 1024;
}

struct Maps {
  CUtensorMap in[4];   // TMA load maps of the input d-tensors (op order above)
  CUtensorMap out[3];  // TMA store maps of the outputs
  CUtensorMap a;       // decays, box [16 tokens][8 heads]
};

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "SWR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SWR_WAIT_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(m),
      "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] = A[smem] * B[smem]  (kind::f16, bf16 in, fp32 accumulate, overwrite)
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(0)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return __uint_as_float(r);
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor (sm_100: version 1 at bit 46, layout type at 61..63)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint64_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}
// A = u_t^T from a TMA tile: MN-major, SWIZZLE_128B; 64-channel halves 2048 B apart
// (LBO), 8-token row groups 1024 B apart (SBO).
__device__ __forceinline__ uint64_t desc_A(uint32_t saddr) { return sdesc(saddr, kHalf, 1024, 2); }
// B = 16x16 transfer tile: K-major, no swizzle; core matrices 8 (N) x 16 B (8 K),
// K-halves 128 B apart (LBO), N-halves 256 B apart (SBO).
__device__ __forceinline__ uint64_t desc_B(uint32_t saddr) { return sdesc(saddr, 128, 256, 0); }
// instruction descriptor: D fp32, A/B bf16, A MN-major, B K-major, N = 16, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (0u << 16) |
                            ((16u >> 3) << 17) | ((128u >> 4) << 24);

// byte offset of element (token i, channel c) inside a 4 KiB swizzled tile
__device__ __forceinline__ uint32_t tile_off(int i, int c) {
  const int half = c >> 6, cc = c & 63;
  return half * kHalf + i * 128 + ((((cc >> 3) ^ (i & 7))) << 4) + ((cc & 7) << 1);
}
// byte offset of B-operand element (n, k) in the K-major no-swizzle 16x16 tile
__device__ __forceinline__ uint32_t btile_off(int n, int k) {
  return (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ float bf(const uint8_t* base, uint32_t off) {
  return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(base + off));
}
__device__ __forceinline__ void st_bf(uint8_t* base, uint32_t off, float x) {
  *reinterpret_cast<__nv_bfloat16*>(base + off) = __float2bfloat16_rn(x);
}

// ---------------------------------------------------------------------------
// work list: CTA c owns blocks [g0, g1) of the flattened (line = b*H + h, t)
// space, plus one left halo block (and, backward, one right halo block) when a
// boundary falls inside a line.  Items are walked with an incremental cursor.
// ---------------------------------------------------------------------------
struct Work {
  int64_t first, g0, g1, last;  // items are global block ids gi in [first, last)
};
template <bool BWD>
__device__ __forceinline__ Work work_of(int64_t total, int64_t nb) {
  Work w;
  w.g0 = (int64_t)blockIdx.x * total / gridDim.x;
  w.g1 = ((int64_t)blockIdx.x + 1) * total / gridDim.x;
  w.first = w.g0 - ((w.g0 < w.g1 && w.g0 % nb != 0) ? 1 : 0);
  w.last = w.g1 + ((BWD && w.g0 < w.g1 && w.g1 % nb != 0) ? 1 : 0);
  if (w.g0 >= w.g1) w.first = w.last = w.g0;
  return w;
}

struct Cursor {
  int64_t gi, t, line;
  int b, h;
  __device__ __forceinline__ void init(int64_t g, int64_t nb, int64_t H) {
    gi = g;
    line = g / nb;
    t = g - line * nb;
    b = (int)(line / H);
    h = (int)(line - (int64_t)b * H);
  }
  __device__ __forceinline__ void next(int64_t nb, int64_t H) {
    ++gi;
    if (++t == nb) {
      t = 0;
      ++line;
      if (++h == H) {
        h = 0;
        ++b;
      }
    }
  }
};

// ring position of item j: stage s = j % NS, parity = (j / NS) & 1, advanced incrementally
template <int NS>
struct Ring {
  int s;
  uint32_t ph;
  __device__ __forceinline__ void init(int64_t j) {
    s = (int)(j % NS);
    ph = (uint32_t)((j / NS) & 1);
  }
  __device__ __forceinline__ void next() {
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
};

// pack two fp32 into bf16x2 (lo = first)
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Store 16 per-token values of this thread's channel c into a swizzled tile as
// bf16 pairs: lanes (c, c^1) swap halves so every store is a 4-byte word and
// the two rows of a warp instruction (i, i^4) fall in disjoint banks.
__device__ __forceinline__ void store_col16(uint8_t* tile, int c, int lane, const float (&x)[16]) {
  const bool odd = lane & 1;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i & 4) continue;
    const int i2 = i ^ 4;
    const float send = odd ? x[i] : x[i2];
    const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
    if (!odd)
      *reinterpret_cast<uint32_t*>(tile + tile_off(i, c)) = pack_bf2(x[i], recv);
    else
      *reinterpret_cast<uint32_t*>(tile + tile_off(i2, c - 1)) = pack_bf2(recv, x[i2]);
  }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int OP>
__global__ void __launch_bounds__((4 * Cfg<OP>::NG + Cfg<OP>::NPREP + 2) * 32, 1)
    swr_tc_kernel(const __grid_constant__ Maps maps, const Params p) {
  using C = Cfg<OP>;
  using S = Stage<OP>;
  constexpr int NS = C::NS, NG = C::NG;
  constexpr int kEpi = 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kPrepW0 = 4 * NG, kProdW = kPrepW0 + C::NPREP, kMmaW = kProdW + 1;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* scratch = smem + NS * S::kBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch);
  uint64_t* prepped = full + NS;
  uint64_t* mmad = prepped + NS;
  uint64_t* ready = mmad + NS;
  uint64_t* empty = ready + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty + NS);
  float* red = reinterpret_cast<float*>(scratch + 2048);  // [NG][2][4][16] da partials

  constexpr int kTmemCols = (NS * C::COLS <= 32) ? 32 : (NS * C::COLS <= 64) ? 64
                          : (NS * C::COLS <= 128) ? 128 : (NS * C::COLS <= 256) ? 256 : 512;
  static_assert(NS * C::COLS <= 512, "TMEM budget");
  // stage release: the item itself (after its store read SMEM) and the neighbour
  // items that read its TMEM / g (next; backward also previous)
  constexpr int kUsers = C::BWD ? 3 : 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&prepped[s], C::NPREP * 32);
      mbar_init(&mmad[s], 1);
      mbar_init(&ready[s], 1);
      mbar_init(&empty[s], kUsers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t nb = p.nb, H = p.H;
  const int64_t total = p.B * H * nb;
  const Work W = work_of<C::BWD>(total, nb);
  const int64_t n_items = W.last - W.first;

  if (warp == kProdW) {
    // ===================== TMA producer =====================
    if (lane == 0 && n_items > 0) {
      Cursor cur;
      cur.init(W.first, nb, H);
      Ring<NS> rg;
      rg.init(0);
      for (int64_t j = 0; j < n_items; ++j) {
        mbar_wait(&empty[rg.s], rg.ph ^ 1);
        uint8_t* st = smem + rg.s * S::kBytes;
        const int tt = (int)(cur.t * kEll);
        mbar_expect_tx(&full[rg.s], C::NT * kTile + 256);
#pragma unroll
        for (int x = 0; x < C::NT; ++x) {
          tma_load_4d(st + x * kTile, &maps.in[x], &full[rg.s], 0, cur.h, tt, cur.b);
          tma_load_4d(st + x * kTile + kHalf, &maps.in[x], &full[rg.s], 64, cur.h, tt, cur.b);
        }
        tma_load_3d(st + S::kA, &maps.a, &full[rg.s], cur.h & ~7, tt, cur.b);
        cur.next(nb, H);
        rg.next();
      }
    }
  } else if (warp == kMmaW) {
    // ===================== MMA issuer + readiness =====================
    // ready[j] is arrived once the MMAs of every item whose TMEM item j's
    // epilogue reads are complete: j-1, j (and, backward, j+1).
    Ring<NS> rg, r1, r2;  // item j, j-1, j-2
    rg.init(0);
    r1 = rg;
    r2 = rg;
    for (int64_t j = 0; j < n_items; ++j) {
      mbar_wait(&full[rg.s], rg.ph);
      mbar_wait(&prepped[rg.s], rg.ph);
      tc_fence_after();
      if (lane == 0) {
        uint8_t* st = smem + rg.s * S::kBytes;
        const uint32_t d = tmem_base + (uint32_t)(rg.s * C::COLS);
        const uint32_t aW = su32(st + (C::MIX ? C::NT * kTile : 0));  // u or u^ = k v
        umma_bf16(d, desc_A(aW), desc_B(su32(st + S::kLT)), kIdesc);
        if constexpr (C::BWD) {
          const uint32_t aG = su32(st + (C::MIX ? (C::NT + 1) * kTile : kTile));  // G or dy q
          umma_bf16(d + 16, desc_A(aG), desc_B(su32(st + S::kL)), kIdesc);
        }
        umma_commit(&mmad[rg.s]);
      }
      __syncwarp();
      if (j >= 1) {
        mbar_wait(&mmad[r1.s], r1.ph);  // item j-1 complete
        tc_fence_before();
        if (lane == 0) {
          if constexpr (!C::BWD) mbar_arrive(&ready[r1.s]);
          else if (j >= 2) mbar_arrive(&ready[r2.s]);
        }
        __syncwarp();
      }
      r2 = r1;
      r1 = rg;
      rg.next();
    }
    if (n_items > 0) {  // flush: r1 = last item, r2 = the one before
      mbar_wait(&mmad[r1.s], r1.ph);
      tc_fence_before();
      if (lane == 0) {
        if (C::BWD && n_items >= 2) mbar_arrive(&ready[r2.s]);
        mbar_arrive(&ready[r1.s]);
      }
      __syncwarp();
    }
  } else if (warp >= kPrepW0) {
    // ===================== prep: L tiles (Alg. 3), g, r, pre-gates =====================
    const int pt = threadIdx.x - kPrepW0 * 32;  // 0 .. NPREP*32-1
    Cursor cur;
    if (n_items > 0) cur.init(W.first, nb, H);
    Ring<NS> rg;
    rg.init(0);
    for (int64_t j = 0; j < n_items; ++j) {
      mbar_wait(&full[rg.s], rg.ph);
      uint8_t* st = smem + rg.s * S::kBytes;
      if (pt < 16) {
        // lane j owns column j of L_t.  Alg. 3: tile a down the columns, pre-mask
        // the inclusive upper triangle with 1, column-wise cumulative product,
        // zero the strict upper triangle.  Products only, never ratios.
        const int col = pt;
        const uint8_t* at = st + S::kA + (cur.h & 7) * 2;
        float a[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          a[i] = (cur.t * kEll + i < p.L) ? __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(at + i * 16)) : 1.f;
        float Lc[16];
        float prod = 1.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i > col) prod *= a[i];
          Lc[i] = (i >= col) ? prod : 0.f;  // L[i][col]
        }
        // B of W (L_t^T, K-major): element (n = i, k = col)
#pragma unroll
        for (int i = 0; i < 16; ++i)
          *reinterpret_cast<__nv_bfloat16*>(st + S::kLT + btile_off(i, col)) = __float2bfloat16_rn(Lc[i]);
        if constexpr (C::BWD) {
          // B of lambda (L_t, K-major): element (n = col, k = i), contiguous along k
          uint4 lo, hi;
          lo.x = pack_bf2(Lc[0], Lc[1]);   lo.y = pack_bf2(Lc[2], Lc[3]);
          lo.z = pack_bf2(Lc[4], Lc[5]);   lo.w = pack_bf2(Lc[6], Lc[7]);
          hi.x = pack_bf2(Lc[8], Lc[9]);   hi.y = pack_bf2(Lc[10], Lc[11]);
          hi.z = pack_bf2(Lc[12], Lc[13]); hi.w = pack_bf2(Lc[14], Lc[15]);
          *reinterpret_cast<uint4*>(st + S::kL + btile_off(col, 0)) = lo;
          *reinterpret_cast<uint4*>(st + S::kL + btile_off(col, 8)) = hi;
          reinterpret_cast<float*>(st + S::kR)[col] = prod;  // r_t[j] = L[15][j]
        }
        // g_t[i] = a_t[0] ... a_t[i]: 16-lane multiplicative scan (pattern of Alg. 1 line 8)
        float g = (cur.t * kEll + col < p.L)
                      ? __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(at + col * 16)) : 1.f;
#pragma unroll
        for (int d = 1; d < 16; d <<= 1) {
          const float o = __shfl_up_sync(0x0000ffffu, g, d, 16);
          if (col >= d) g *= o;
        }
        reinterpret_cast<float*>(st + S::kG)[col] = g;
      }
      if constexpr (C::MIX) {
        // pre-gates in the swizzled tile layout (elementwise, layout-agnostic):
        //   u^ = k (.) v and, backward, G = dy (.) q; rounded once to bf16
        const uint4* K4 = reinterpret_cast<const uint4*>(st + 1 * kTile);
        const uint4* V4 = reinterpret_cast<const uint4*>(st + 2 * kTile);
        uint4* U4 = reinterpret_cast<uint4*>(st + C::NT * kTile);
        for (int v = pt; v < kTile / 16; v += C::NPREP * 32) {
          const uint4 kk = K4[v], vv = V4[v];
          uint4 o;
          const uint32_t* ka = &kk.x;
          const uint32_t* va = &vv.x;
          uint32_t* oa = &o.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ka[e]));
            const float2 vf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&va[e]));
            oa[e] = pack_bf2(kf.x * vf.x, kf.y * vf.y);
          }
          U4[v] = o;
          if constexpr (C::BWD) {
            const uint4* Q4 = reinterpret_cast<const uint4*>(st + 0 * kTile);
            const uint4* D4 = reinterpret_cast<const uint4*>(st + 3 * kTile);
            uint4* G4 = reinterpret_cast<uint4*>(st + (C::NT + 1) * kTile);
            const uint4 qq = Q4[v], dd = D4[v];
            const uint32_t* qa = &qq.x;
            const uint32_t* da = &dd.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 qf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qa[e]));
              const float2 df = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&da[e]));
              oa[e] = pack_bf2(df.x * qf.x, df.y * qf.y);
            }
            G4[v] = o;
          }
        }
      }
      fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
      mbar_arrive(&prepped[rg.s]);
      cur.next(nb, H);
      rg.next();
    }
  } else {
    // ===================== epilogue groups: thread = channel c =====================
    const int grp = warp >> 2;                       // epilogue group, items j = grp mod NG
    const int c = threadIdx.x & 127;                 // channel == TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const bool leader = (threadIdx.x & 127) == 0;
    float* red_g = red + grp * 128;                  // [2][4][16]
    int rbuf = 0;
    int pend = -1;                                   // stage of the last stored item (release lags its store)
    Cursor cur;
    if (grp < n_items) cur.init(W.first + grp, nb, H);
    Ring<NS> rg, rp, rn;
    rg.init(grp);
    for (int64_t j = grp; j < n_items; j += NG) {
      rp = rg;  // ring slots of items j-1 and j+1
      if (rp.s == 0) { rp.s = NS - 1; rp.ph ^= 1; } else { --rp.s; }
      rn = rg;
      rn.next();
      const int64_t t = cur.t;
      const int b = cur.b, h = cur.h;
      const bool halo = cur.gi < W.g0 || cur.gi >= W.g1;
      uint8_t* st = smem + rg.s * S::kBytes;
      const float* g = reinterpret_cast<const float*>(st + S::kG);
      const int64_t co = cur.line * kD + c;
      mbar_wait(&ready[rg.s], rg.ph);
      tc_fence_after();
      bool stored = false;
      if (!halo) {
        const uint32_t tslot = tmem_base + lane_base + (uint32_t)(rg.s * C::COLS);
        float w[16];
        tmem_ld16(tslot, w);
        // carrier v_{t-1} = w_{t-1}[15]: column 15 of the previous item's TMEM
        float vprev;
        if (t == 0) {
          vprev = p.carry_in ? p.carry_in[co] : 0.f;  // v_{-1}
        } else {
          vprev = tmem_ld1(tmem_base + lane_base + (uint32_t)(rp.s * C::COLS + 15));
        }
        if constexpr (!C::BWD) {
          tmem_wait_ld();
          float out[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) out[i] = fmaf(g[i], vprev, w[i]);  // Pass II: x~ = w + g v
          if constexpr (C::MIX) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {  // post-gate with residual: y = q x~ + v
              const uint32_t o = tile_off(i, c);
              out[i] = fmaf(bf(st, o), out[i], bf(st + 2 * kTile, o));
            }
          }
          __syncwarp();
          store_col16(st, c, lane, out);
          if (t == nb - 1 && p.carry_out) p.carry_out[co] = w[15];
        } else {
          float lam[16];
          tmem_ld16(tslot + 16, lam);
          float mu;
          if (t == nb - 1) {
            mu = p.mu_in ? p.mu_in[co] : 0.f;
            tmem_wait_ld();
          } else {  // mu_t = a_{t+1}[0] lambda_{t+1}[0] from the next item
            const float l0 = tmem_ld1(tmem_base + lane_base + (uint32_t)(rn.s * C::COLS + 16));
            tmem_wait_ld();
            mu = reinterpret_cast<const float*>(smem + rn.s * S::kBytes + S::kG)[0] * l0;
          }
          const float* r = reinterpret_cast<const float*>(st + S::kR);
          float part[16], du[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float rmu = r[i] * mu;
            du[i] = lam[i] + rmu;                                            // du = lambda + r mu
            const float wp = (i > 0) ? w[i - 1] : 0.f;
            const float xp = (i > 0) ? fmaf(g[i - 1], vprev, w[i - 1]) : vprev;  // x~[i-1]
            part[i] = fmaf(lam[i], xp, rmu * wp);                              // da partial
          }
          __syncwarp();
          if constexpr (!C::MIX) {
            store_col16(st + kTile, c, lane, du);  // du over G
          } else {
            float dq[16], dk[16], dv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t o = tile_off(i, c);
              const float dy = bf(st + 3 * kTile, o), kk = bf(st + kTile, o), vv = bf(st + 2 * kTile, o);
              const float x = fmaf(g[i], vprev, w[i]);
              dq[i] = dy * x;              // dq = dy x~
              dk[i] = du[i] * vv;          // dk = du^ v
              dv[i] = fmaf(du[i], kk, dy);  // dv = du^ k + dy
            }
            __syncwarp();
            store_col16(st + 3 * kTile, c, lane, dq);
            store_col16(st + 1 * kTile, c, lane, dk);
            store_col16(st + 2 * kTile, c, lane, dv);
          }
          if (t == 0 && p.mu_out) p.mu_out[co] = g[0] * lam[0];  // a_0[0] lambda_0[0]
          // da: deterministic reduction over the 128 channels (4 warps of this group)
          int tok = 0;
          GroupReduce<16, 16>::run(part, lane, tok);
          float* rb = red_g + rbuf * 64;
          if ((lane & 1) == 0) rb[(warp & 3) * 16 + tok] = part[0];
          named_bar(1 + NG + grp, kEpi);
          if ((warp & 3) == 0 && lane < 16) {
            const int64_t n = t * kEll + lane;
            if (n < p.L) {
              const float sum = ((rb[lane] + rb[16 + lane]) + rb[32 + lane]) + rb[48 + lane];
              __nv_bfloat16* dA = (__nv_bfloat16*)p.da + (int64_t)b * p.sa_b + (int64_t)h * p.sa_h;
              dA[n * p.sa_l] = __float2bfloat16_rn(sum);
            }
          }
          rbuf ^= 1;
        }
        stored = true;
      }
      // hand back: outputs -> TMA store; release own stage once the store has read
      // SMEM, and the neighbours' stages whose TMEM / g this item read
      tc_fence_before();
      if (stored) fence_proxy_async();
      named_bar(1 + grp, kEpi);
      if (leader) {
        if (stored) {
          const int tt = (int)(t * kEll);
#pragma unroll
          for (int x = 0; x < C::NOUT; ++x) {
            const int tile = (OP == 0) ? 0 : (OP == 1) ? 1 : (OP == 2) ? 0 : (x == 0 ? 3 : x);
            tma_store_4d(&maps.out[x], st + tile * kTile, 0, h, tt, b);
            tma_store_4d(&maps.out[x], st + tile * kTile + kHalf, 64, h, tt, b);
          }
          bulk_commit();
          bulk_wait_read<1>();
          if (pend >= 0) mbar_arrive(&empty[pend]);
          pend = rg.s;
        } else {
          mbar_arrive(&empty[rg.s]);
        }
        if (j >= 1) mbar_arrive(&empty[rp.s]);                       // as "next" of item j-1
        if (C::BWD && j + 1 < n_items) mbar_arrive(&empty[rn.s]);  // as "previous" of item j+1
        if (j == n_items - 1) mbar_arrive(&empty[rg.s]);           // no next item
        if (C::BWD && j == 0) mbar_arrive(&empty[rg.s]);           // no previous item
      }
      for (int k = 0; k < NG; ++k) {
        cur.next(nb, H);
        rg.next();
      }
    }
    if (leader) {
      bulk_wait_all();
      if (pend >= 0) mbar_arrive(&empty[pend]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaW) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static bool map_dtensor(CUtensorMap* m, const void* ptr, const Params& p) {
  cuuint64_t dims[4] = {(cuuint64_t)p.D, (cuuint64_t)p.H, (cuuint64_t)p.L, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)p.sx_h * 2, (cuuint64_t)p.sx_l * 2, (cuuint64_t)p.sx_b * 2};
  cuuint32_t box[4] = {64, 1, 16, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return encoder()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool map_decay(CUtensorMap* m, const void* ptr, const Params& p) {
  cuuint64_t dims[3] = {(cuuint64_t)p.H, (cuuint64_t)p.L, (cuuint64_t)p.B};
  cuuint64_t strides[2] = {(cuuint64_t)p.sa_l * 2, (cuuint64_t)p.sa_b * 2};
  cuuint32_t box[3] = {8, 16, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return encoder()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int OP>
static cudaError_t launch_op(const Params& p, cudaStream_t st, int sms) {
  Maps maps;
  std::memset(&maps, 0, sizeof(maps));
  const void* ins[4] = {nullptr, nullptr, nullptr, nullptr};
  const void* outs[3] = {nullptr, nullptr, nullptr};
  int nin = 0, nout = 0;
  switch (OP) {
    case 0: ins[0] = p.u; outs[0] = p.x; nin = 1; nout = 1; break;
    case 1: ins[0] = p.u; ins[1] = p.dx; outs[0] = p.du; nin = 2; nout = 1; break;
    case 2: ins[0] = p.q; ins[1] = p.k; ins[2] = p.v; outs[0] = p.y; nin = 3; nout = 1; break;
    default:
      ins[0] = p.q; ins[1] = p.k; ins[2] = p.v; ins[3] = p.dy;
      outs[0] = p.dq; outs[1] = p.dk; outs[2] = p.dv; nin = 4; nout = 3;
  }
  for (int i = 0; i < nin; ++i)
    if (!map_dtensor(&maps.in[i], ins[i], p)) return cudaErrorNotSupported;
  for (int i = 0; i < nout; ++i)
    if (!map_dtensor(&maps.out[i], outs[i], p)) return cudaErrorNotSupported;
  if (!map_decay(&maps.a, p.a, p)) return cudaErrorNotSupported;

  constexpr int smem = smem_bytes<OP>();
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(swr_tc_kernel<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int64_t total = p.B * p.H * p.nb;
  const int grid = (int)std::min<int64_t>(sms, std::max<int64_t>(total, 1));
  constexpr int threads = (4 * Cfg<OP>::NG + Cfg<OP>::NPREP + 2) * 32;
  swr_tc_kernel<OP><<<grid, threads, smem, st>>>(maps, p);
  return cudaGetLastError();
}

}  // namespace tc

bool tc_supported(int op, bool bf16, const Params& p) {
  (void)op;
  if (!bf16 || p.D != 128) return false;
  if (tc::encoder() == nullptr) return false;
  auto a16 = [](const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  // decays must be TMA-addressable: heads contiguous, 16-byte token/batch strides
  if (p.sa_h != 1 || (p.sa_l * 2) % 16 != 0 || (p.sa_b * 2) % 16 != 0 || !a16(p.a)) return false;
  if (p.H > (1 << 30) || p.L > (1 << 30) || p.B > (1 << 30)) return false;
  return true;
}

cudaError_t launch_tc(int op, const Params& p, cudaStream_t st, int sms, int* launches) {
  *launches = 0;
  cudaError_t e;
  switch (op) {
    case 0: e = tc::launch_op<0>(p, st, sms); break;
    case 1: e = tc::launch_op<1>(p, st, sms); break;
    case 2: e = tc::launch_op<2>(p, st, sms); break;
    default: e = tc::launch_op<3>(p, st, sms); break;
  }
  if (e == cudaSuccess) *launches = 1;
  return e;
}

}  // namespace swr
