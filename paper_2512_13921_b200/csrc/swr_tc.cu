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
//   * The epilogue warps read TMEM with tcgen05.ld.16x256b in the m16n8 fragment
//     layout (a lane owns 4 channels x 4 tokens), so Pass II x~ = w + g v_{t-1}
//     (P:1478), du = lambda + r mu and the da terms are thread-local, token pairs
//     are packed fp32x2 / bf16x2, and results reach the swizzled output tile with
//     stmatrix.trans; the carrier v_t = w_t[15] passes to the next block
//     in registers (no SMEM/DSMEM exchange, no cross-CTA sync).  The SWR backward
//     computes w through a row-rotated transfer tile so w[i-1] and w[15] are read
//     in place.
//   * One persistent CTA per SM walks a contiguous range of (b, h, block) items,
//     sized for that SM's measured rate (Split), recomputing one halo item at a
//     range boundary (and, backward, one on the right); tiles move HBM -> SMEM ->
//     HBM with TMA (cp.async.bulk.tensor) through mbarrier rings: input stages,
//     decay stages (loaded ahead by their own producer for the SWR ops), work
//     slots (transfer tiles, g/r, TMEM columns) and output slots.
//
// Warp roles: 4*NG epilogue warps in NG groups of 4 (group g handles items
// j = g mod NG; warp w reads TMEM lanes 32*(w%4)..+31), NPW prep warps (transfer
// tiles, g/r/gs, mixer pre-gates), the TMA producer, the MMA issuer (one thread),
// the store warp (TMA stores, da sums, slot release), the retire warp (MMA
// completion in order, input-stage release, readiness) and, for the SWR ops, the
// decay producer.  DESIGN.md section 5.1 has the rings' phase-parity invariants.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "swr_common.cuh"

namespace swr {
namespace tc {

constexpr int kD = 128;          // head dim served by this family
constexpr int kTile = 4096;      // one 16 x 128 bf16 tile (two 64-channel halves)
constexpr int kHalf = 2048;      // one 64-channel half: 16 rows x 128 B, 128B-swizzled

// ---------------------------------------------------------------------------
// per-op configuration.  A pipeline "item" is BPI consecutive 16-token blocks
// of one (b, h) line (the last item of a line may be partial).  Three rings:
//   input  (NI stages, SMEM): TMA load -> prep -> MMA.  For the SWR ops the
//          input tiles are consumed by the MMA alone, so a stage is released
//          when its MMAs complete; the mixer epilogue also reads q/k/v/dy, so
//          there the epilogue releases it.
//   work   (NW slots): the item's TMEM accumulators + g_t/r_t, held from prep
//          until the epilogues of the item and of its neighbours have read them.
//   output (NO slots, SMEM): epilogue -> TMA store.
//   NT   TMA-loaded input regions (d-tensors)  NP   extra prep-computed A regions
//   COLS TMEM columns per block                NPW  prep warps (each owns whole items)
//   NG   epilogue groups of 4 warps
// ---------------------------------------------------------------------------
// ring depths / prep warps: compile-time tuning knobs (tools/build_var.sh -D...)
// ring depths measured back to back (tools/ab_b2b.sh): 2-block forward
// items with 7 stages and 5 backward stages keep 56 / 80 KB of loads in flight per
// SM -- more bytes in flight made the step slower (the TMA-copy probe agrees)
#ifndef SWR_F_NI
#define SWR_F_NI 7
#endif
#ifndef SWR_F_BPI
#define SWR_F_BPI 2
#endif
#ifndef SWR_F_NO
#define SWR_F_NO 3
#endif
#ifndef SWR_F_NA
#define SWR_F_NA 8
#endif
#ifndef SWR_F_NG
#define SWR_F_NG 3
#endif
#ifndef SWR_F_NPW
#define SWR_F_NPW 4
#endif
#ifndef SWR_B_NI
#define SWR_B_NI 5
#endif
#ifndef SWR_B_NA
#define SWR_B_NA 8
#endif
#ifndef SWR_B_NO
#define SWR_B_NO 4
#endif
#ifndef SWR_B_BPI
#define SWR_B_BPI 2
#endif
#ifndef SWR_B_NPW
#define SWR_B_NPW 2
#endif
#ifndef SWR_B_NG
#define SWR_B_NG 3
#endif
#ifndef SWR_MF_NPW
#define SWR_MF_NPW 3
#endif
#ifndef SWR_MF_NI
#define SWR_MF_NI 6
#endif
#ifndef SWR_MB_NPW
#define SWR_MB_NPW 4
#endif
#ifndef SWR_MF_NW
#define SWR_MF_NW 6
#endif
#ifndef SWR_MB_NI
#define SWR_MB_NI 8
#endif
template <int OP>
struct Cfg;
template <>
struct Cfg<0> {  // swr_fwd: in u;  out x
  static constexpr int NT = 1, NP = 0, BPI = SWR_F_BPI, NI = SWR_F_NI, NA = SWR_F_NA, NW = 8, NO = SWR_F_NO, COLS = 16, NPW = SWR_F_NPW, NOUT = 1, NG = SWR_F_NG;
  static constexpr int TU = 0, TG = 0;  // A-operand regions of W and lambda
  static constexpr bool CYC = false;    // w MMA through the row-rotated tile (see Stage::kLc)
  static constexpr bool WC = false;     // a second w MMA through the rotated tile, at column kWc
  static constexpr bool BWD = false, MIX = false, LAYER = false, EXACT = false, EXACT1 = false;
  static constexpr int HS = 1;  // heads walked together (GRP)
  static constexpr bool GRP = false;
};
template <>
struct Cfg<1> {  // swr_bwd: in u, G;  out du
  static constexpr int NT = 2, NP = 0, BPI = SWR_B_BPI, NI = SWR_B_NI, NA = SWR_B_NA, NW = 8, NO = SWR_B_NO, COLS = 32, NPW = SWR_B_NPW, NOUT = 1, NG = SWR_B_NG;
  static constexpr int TU = 0, TG = 1;
  static constexpr bool CYC = true;
  static constexpr bool WC = false;
  static constexpr bool BWD = true, MIX = false, LAYER = false, EXACT = false, EXACT1 = false;
  static constexpr int HS = 1;  // heads walked together (GRP)
  static constexpr bool GRP = false;
};
template <>
struct Cfg<2> {  // mix fwd: in q, k, v;  out y;  prep u^ = k v (over k)
  static constexpr int NT = 3, NP = 0, BPI = 2, NI = SWR_MF_NI, NA = 6, NW = SWR_MF_NW, NO = 4, COLS = 16, NPW = SWR_MF_NPW, NOUT = 1, NG = 3;
  static constexpr int TU = 1, TG = 0;
  static constexpr bool CYC = false;
  static constexpr bool WC = false;
  static constexpr bool BWD = false, MIX = true, LAYER = false, EXACT = false, EXACT1 = false;
  static constexpr int HS = 1;  // heads walked together (GRP)
  static constexpr bool GRP = false;
};
template <>
struct Cfg<3> {  // mix bwd: in q, k, v, dy;  out dq, dk, dv;  prep u^ = k v (region 4), G = dy q (over q)
  static constexpr int NT = 4, NP = 1, BPI = 1, NI = SWR_MB_NI, NA = 8, NW = 8, NO = 3, COLS = 48, NPW = SWR_MB_NPW, NOUT = 3, NG = 3;
  static constexpr int TU = 4, TG = 0;
  static constexpr bool CYC = false;
  static constexpr bool WC = true;  // x~ needs w[i] (dq), da needs w[i-1]: both from TMEM
  static constexpr bool BWD = true, MIX = true, LAYER = false, EXACT = false, EXACT1 = false;
  static constexpr int HS = 1;  // heads walked together (GRP)
  static constexpr bool GRP = false;
};
// the Phalanx layer mixer (phalanx_layer_mix*, NEXT-1): the mixer's pipelines with
// sigma on the decay / key logits and group-shared q / k (forward; the backward's
// group sums run on the CUDA-core family, so here every group is one head)
template <>
struct Cfg<4> : Cfg<2> {
  static constexpr bool LAYER = true;
};
#ifndef SWR_LB_NPW
#define SWR_LB_NPW 4
#endif
#ifndef SWR_LB_NG
#define SWR_LB_NG 3
#endif
template <>
struct Cfg<5> : Cfg<3> {
  static constexpr bool LAYER = true;
  static constexpr int NPW = SWR_LB_NPW, NG = SWR_LB_NG;
};
// the layer mixer backward with q and k shared by pairs of heads (the paper's models:
// H = 16 heads in 8 groups) and the group sums fused: the item walk interleaves
// the two heads of a group block by block, one epilogue group takes both items of a
// block and sums their dq / dz_k terms in fp32 registers (head order), storing the
// group tile once -- no per-head scratch, no second kernel
#ifndef SWR_LG_NG
#define SWR_LG_NG 2
#endif
#ifndef SWR_LG_NO
#define SWR_LG_NO 3
#endif
#ifndef SWR_LG_NI
#define SWR_LG_NI 8
#endif
#ifndef SWR_LG_GRP
#define SWR_LG_GRP 1
#endif
template <>
struct Cfg<8> : Cfg<5> {
  static constexpr int HS = 2;
  static constexpr bool GRP = SWR_LG_GRP;
  static constexpr int NG = SWR_LG_NG, NO = SWR_LG_NO, NI = SWR_LG_NI;
};
// the exact full-range recurrence's output pass (swr_exact_fwd):
// the forward's Pass I on the tensor cores, with the exact carrier s_{t-1} of Alg. 2
// instead of v_{t-1} -- read from the look-back scan's per-block carriers at
// an item's first block, then carried block to block as the exact state at token 15
template <>
struct Cfg<6> : Cfg<0> {
  static constexpr bool EXACT = true;
};
// ... and its first pass: the same Pass I, but instead of x the epilogue writes each
// block's local end state v_t = w_t[15] and decay product c_t = g_t[15] (the carrier
// system of P:610-613) for the scan
#ifndef SWR_X1_NI
#define SWR_X1_NI 12
#endif
template <>
struct Cfg<7> : Cfg<0> {
  static constexpr bool EXACT1 = true;
  static constexpr int NI = SWR_X1_NI;  // read-only traffic: more loads in flight
};

// SMEM layout (bytes; every 4 KiB tile 1024-aligned for the 128B swizzle atoms).
// A d-tensor of an item occupies one region [2 halves][16*BPI tokens][128 B] (one
// TMA box per 64-channel half); block k of it starts k*2 KiB into each half.
// Four rings: input stages (the item's d-tensor tiles), decay stages (its decay
// box, loaded ahead by its own producer so the transfer tiles are built while the
// d-tensor tiles are still in flight), work slots (transfer tiles + g/r/gs + TMEM
// columns) and output slots.
template <int OP>
struct Stage {
  using C = Cfg<OP>;
  static constexpr int kRegion = C::BPI * kTile;
  static constexpr int kHS = C::BPI * kHalf;                   // half stride inside a region
  // input stage: NT loaded d-tensors + NP prep-computed A operands
  static constexpr int kIn = (C::NT + C::NP) * kRegion;
  // decay stage: box [16*BPI tokens][8 heads] bf16
  static constexpr int kAD = 256 * C::BPI;
  // work slot: transfer tile L_t per block (512 B); CYC: a second tile per block with
  // the rows of L_t rotated by one, Lc[i][j] = L[(i - 1) mod 16][j], so the w MMA
  // yields [w_15, w_0, ..., w_14]: w[i-1] for i >= 1 and the carrier w[15] in column 0
  // (SWR backward); then aux per block: g_t[16], r_t[16], gs[16] = g_t shifted by one
  // (gs[0] = 1), fp32, in fragment token order
  static constexpr int kLc = 512 * C::BPI;                     // offset of the CYC tiles
  static constexpr int kAuxOff = kLc + ((C::CYC || C::WC) ? 512 * C::BPI : 0);
  static constexpr int kAuxBlk = C::LAYER ? 64 : 48;  // floats (layer: + a (1 - a), token order)
  static constexpr int kWork = kAuxOff + C::BPI * kAuxBlk * 4;
  // output slot
  static constexpr int kOut = C::NOUT * kRegion;
  static constexpr int kInBase = 0;
  static constexpr int kOutBase = C::NI * kIn;
  static constexpr int kWorkBase = kOutBase + C::NO * kOut;
  static constexpr int kADBase = kWorkBase + C::NW * kWork;
  static constexpr int kScratch = kADBase + C::NA * kAD;       // barriers + da partials (4 KiB)
  static constexpr int kBytes = kScratch + 4096;
  static __device__ __forceinline__ uint8_t* region(uint8_t* st, int x) { return st + x * kRegion; }
  static __device__ __forceinline__ uint8_t* tile(uint8_t* st, int k, int x) {
    return region(st, x) + k * kHalf;
  }
  static __device__ __forceinline__ uint32_t tile(uint32_t st, int k, int x) {  // shared-window address
    return st + x * kRegion + k * kHalf;
  }
};

template <int OP>
constexpr int smem_bytes() {
  return Stage<OP>::kBytes + 1024;  // + alignment slack
}

struct Maps {
  CUtensorMap in[4];   // TMA load maps of the input d-tensors (op order above)
  CUtensorMap out[3];  // TMA store maps of the outputs
  CUtensorMap a;       // decays, box [16*BPI tokens][8 heads]
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
// Blocking wait.  The suspend-time hint (ns) lets the waiting warp sleep until
// the phase completes instead of re-polling on the default short timeout, so
// idle roles do not consume issue slots.
#if SWR_HANG_DEBUG
// diagnostics build (tools/build_var.sh -DSWR_HANG_DEBUG=1): a wait that has not
// completed after ~2^26 polls prints the CTA's per-warp debug words, then traps
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity);
__shared__ int g_dbg[32][4];
#define SWR_DBG(a, b, c, d)                                                            \
  do {                                                                                 \
    if ((threadIdx.x & 31) == 0) {                                                     \
      g_dbg[threadIdx.x >> 5][0] = (a); g_dbg[threadIdx.x >> 5][1] = (b);              \
      g_dbg[threadIdx.x >> 5][2] = (c); g_dbg[threadIdx.x >> 5][3] = (d);              \
    }                                                                                  \
  } while (0)
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
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t n = 0;
  while (!mbar_try(b, parity))
    if (++n == (1u << 13)) {
      if ((threadIdx.x & 31) == 0) {
        printf("HANG cta %d warp %d bar %u parity %u\n", (int)blockIdx.x, (int)(threadIdx.x >> 5),
               (unsigned)su32(b), parity);
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
          printf("  cta %d warp %d dbg %d %d %d %d\n", (int)blockIdx.x, w, g_dbg[w][0], g_dbg[w][1], g_dbg[w][2],
                 g_dbg[w][3]);
      }
      __trap();
    }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "SWR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra SWR_WAIT_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity), "r"(1000000)
      : "memory");
}
#if SWR_DBG_GLOBAL
// diagnostics build: the debug words go to the host-mapped buffer of swr_set_trace
// ([cta][warp][4] ints), readable by the host while the kernel runs
#define SWR_DBG(a, b, c, d)                                                                  \
  do {                                                                                       \
    if ((threadIdx.x & 31) == 0 && p.trace != nullptr) {                                     \
      volatile int* q_ = reinterpret_cast<volatile int*>(p.trace) + (blockIdx.x * 32 + (threadIdx.x >> 5)) * 4; \
      q_[0] = (a); q_[1] = (b); q_[2] = (c); q_[3] = (d);                                    \
      __threadfence_system();                                                                \
    }                                                                                        \
  } while (0)
#else
#define SWR_DBG(a, b, c, d) \
  do {                      \
  } while (0)
#endif
#endif
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
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
__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return __uint_as_float(r);
}
// diagnostics: clock64 stamp (SM cycles) of event ev for item j of CTA 0 (swr_set_trace)
// events: 0 producer got stage, 1 producer issued TMA, 2 prep saw full, 3 prep done,
// 4 mma saw full+prepped, 5 mma issued, 6 mma marked ready, 7 epilogue saw ready,
// 8 epilogue done (before store), 9 store committed, 10 own stage released
// Compiled in only with -DSWR_TRACE=1 (tools/build_var.sh); the product build has none.
#ifndef SWR_TRACE
#define SWR_TRACE 0
#endif
__device__ __forceinline__ void trace(const Params& p, int j, int ev) {
#if SWR_TRACE
  if (p.trace != nullptr && blockIdx.x == 0 && j < p.trace_n) {
    p.trace[j * 16 + ev] = clock64();  // SM cycles (all roles share the SM clock)
  }
#endif
}
// diagnostics: per-CTA %globaltimer span (ns) and SM id after the per-item area:
// slot 16*n + 4*cta + {0: start, 1: end, 2: smid}
__device__ __forceinline__ void trace_cta(const Params& p, int e) {
#if SWR_TRACE
  if (p.trace != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[16 * p.trace_n + 4 * blockIdx.x + e] = t;
    if (e == 0) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      p.trace[16 * p.trace_n + 4 * blockIdx.x + 2] = sm;
    }
  }
#endif
}
__device__ __forceinline__ void tmem_wait_f(float& x) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+f"(x) : : "memory");
}

// UMMA shared-memory descriptor (sm_100: version 1 at bit 46, layout type at 61..63)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint64_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}
// A = u_t^T from a TMA tile: MN-major, SWIZZLE_128B; 64-channel halves HS bytes
// apart (LBO), 8-token row groups 1024 B apart (SBO).
template <int HS>
__device__ __forceinline__ uint64_t desc_A(uint32_t saddr) { return sdesc(saddr, HS, 1024, 2); }
// The 16x16 transfer tile L_t is stored ONCE, column-major in 8x8 core matrices:
// element L[i][j] at byte (j/8)*256 + (i/8)*128 + (j%8)*16 + (i%8)*2, i.e. each
// column j is 32 contiguous-per-core-row bytes written by one lane.
//  * lambda = L_t^T G needs B[k=i][n=j] = L[i][j]: K-major, no swizzle, core rows
//    = n (16 B apart), K-halves 128 B apart (LBO), N-halves 256 B apart (SBO).
//  * w = L_t u needs B[k=j][n=i] = L[i][j]: MN-major, no swizzle, core rows = k
//    (16 B apart), N-halves 128 B apart (SBO), K-halves 256 B apart (LBO).
// The same bytes serve both MMAs; only the descriptor (and the B-major bit) differ.
__device__ __forceinline__ uint64_t desc_Bk(uint32_t saddr) { return sdesc(saddr, 128, 256, 0); }
__device__ __forceinline__ uint64_t desc_Bmn(uint32_t saddr) { return sdesc(saddr, 256, 128, 0); }
// instruction descriptors: D fp32, A/B bf16, A MN-major, N = 16, M = 128; B K- or MN-major
constexpr uint32_t kIdescBk = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (0u << 16) |
                              ((16u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescBmn = kIdescBk | (1u << 16);

// byte offset of L[i][j] in the transfer tile (see desc_Bk / desc_Bmn)
__device__ __forceinline__ uint32_t ltile_off(int i, int j) {
  return (j >> 3) * 256 + (i >> 3) * 128 + (j & 7) * 16 + (i & 7) * 2;
}


// ---------------------------------------------------------------------------
// work list: items are BPI-block groups [BPI*m, BPI*m + BPI) of a line
// (line = b*H + h).  CTA c owns items [g0, g1) of the flattened (line, m)
// space, plus one left halo item (and, backward, one right halo item) when a
// boundary falls inside a line.  Items are walked with an incremental cursor.
// ---------------------------------------------------------------------------
struct Work {
  int first, g0, g1, last;  // global item ids gi in [first, last) (< 2^31, tc_supported)
};
// Range split of the item space.  SMs of a B200 differ by up to +-15% in sustained
// streaming rate, in a fixed pattern, so equal ranges finish when the
// slowest SM does.  When `weighted`, range r is sized for SM r (feedback from the
// per-SM item times of earlier launches of the op, g_spi) and a CTA claims the range
// of the SM it runs on (first free range if that is taken: every range is claimed
// exactly once, whatever the placement); results do not depend on the split.
constexpr int kMaxSM = 256;
struct Split {
  int weighted;
  int bnd[kMaxSM + 1];  // range r = items [bnd[r], bnd[r+1])
};
constexpr int kClaimSlots = 256;
__device__ unsigned g_claim[kClaimSlots][kMaxSM];  // {launch epoch} of the claimer, per range
__device__ float g_spi[9][kMaxSM];                 // ns per item of the last CTA on each SM, per op
__device__ __forceinline__ int claim_range(const Split& sp, uint32_t epoch) {
  if (!sp.weighted) return (int)blockIdx.x;
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  unsigned* cl = g_claim[epoch % kClaimSlots];
  const int n = (int)gridDim.x;
  if ((int)sm < n && atomicExch(&cl[sm], epoch) != epoch) return (int)sm;
  for (int r = 0; r < n; ++r)
    if (atomicExch(&cl[r], epoch) != epoch) return r;
  return -1;  // unreachable: as many ranges as CTAs
}
// HS > 1 (Cfg::GRP): the split is over "super-items" (one block of the HS heads of a
// group) and every range holds whole super-items; items are super * HS + head in group
template <bool BWD, int HS>
__device__ __forceinline__ Work work_of(const Split& sp, int r, int total, int nbi) {
  Work w;
  if (sp.weighted) {
    w.g0 = sp.bnd[r];
    w.g1 = sp.bnd[r + 1];
  } else {
    w.g0 = (int)((int64_t)r * total / gridDim.x);
    w.g1 = (int)(((int64_t)r + 1) * total / gridDim.x);
  }
  w.first = w.g0 - ((w.g0 < w.g1 && w.g0 % nbi != 0) ? 1 : 0);
  w.last = w.g1 + ((BWD && w.g0 < w.g1 && w.g1 % nbi != 0) ? 1 : 0);
  if (w.g0 >= w.g1) w.first = w.last = w.g0;
  w.first *= HS;
  w.g0 *= HS;
  w.g1 *= HS;
  w.last *= HS;
  return w;
}

// item gi = line * nbi + m (HS = 1); t0 = first block of the item.  HS > 1: gi =
// ((b * H/HS + gs) * nbi + m) * HS + hh, head h = gs * HS + hh (the HS heads of group gs
// for block m are consecutive items)
template <int HS>
struct Cursor {
  int gi, m, line;
  int b, h, gs, hh;
  __device__ __forceinline__ void set_line(int H) {
    h = gs * HS + hh;
    line = b * H + h;
  }
  __device__ __forceinline__ void init(int g, int nbi, int H) {
    gi = g;
    hh = g % HS;
    const int s = g / HS, sl = s / nbi, Gs = H / HS;
    m = s - sl * nbi;
    b = sl / Gs;
    gs = sl - b * Gs;
    set_line(H);
  }
  __device__ __forceinline__ void next(int nbi, int H) {
    ++gi;
    if (++hh == HS) {
      hh = 0;
      if (++m == nbi) {
        m = 0;
        if (++gs == H / HS) {
          gs = 0;
          ++b;
        }
      }
    }
    set_line(H);
  }
  __device__ __forceinline__ void step(int n, int nbi, int H) {
    for (int i = 0; i < n; ++i) next(nbi, H);
  }
};
template <>
struct Cursor<1> {
  int gi, m, line;
  int b, h;
  static constexpr int hh = 0;
  __device__ __forceinline__ void init(int g, int nbi, int H) {
    gi = g;
    line = g / nbi;
    m = g - line * nbi;
    b = line / H;
    h = line - b * H;
  }
  __device__ __forceinline__ void next(int nbi, int H) {
    ++gi;
    if (++m == nbi) {
      m = 0;
      ++line;
      if (++h == H) {
        h = 0;
        ++b;
      }
    }
  }
  __device__ __forceinline__ void step(int n, int nbi, int H) {  // n items forward
    gi += n;
    m += n;
    while (m >= nbi) {
      m -= nbi;
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
  __device__ __forceinline__ void init(int j) {
    s = (int)(j % NS);
    ph = (uint32_t)((j / NS) & 1);
  }
  __device__ __forceinline__ void next() {
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
  template <int N>  // N <= NS items forward
  __device__ __forceinline__ void step() {
    static_assert(N <= NS, "one wrap at most");
    s += N;
    if (s >= NS) {
      s -= NS;
      ph ^= 1;
    }
  }
  __device__ __forceinline__ void stepn(int n) {  // n < NS items forward
    s += n;
    if (s >= NS) {
      s -= NS;
      ph ^= 1;
    }
  }
  __device__ __forceinline__ void prev() {
    if (s == 0) {
      s = NS - 1;
      ph ^= 1;
    } else {
      --s;
    }
  }
};

// packed fp32x2 arithmetic (sm_100 FFMA2 / FMUL2): one instruction for two lanes of
// work; the builtins leave register pairing to ptxas
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) { return __fmul2_rn(a, b); }


// sigma(z) = 1/2 + tanh(z/2)/2 with the single-MUFU tanh.approx.f32 (relative error
// ~2^-11, below the bf16 rounding every TC output gets; R20) -- the layer
// mixer's bounding activation of the decay and key logits
__device__ __forceinline__ float sig_tc(float z) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * z));
  return fmaf(0.5f, t, 0.5f);
}
// 8 elements of u^ = sigma(zk) (.) v and k = sigma(zk) (into *kout when non-null, for
// the backward's epilogue), in packed bf16x2: k = 1/2 + tanh(zk/2)/2 with
// tanh.approx.bf16x2, then u^ = k v rounded once more (R20: |error of k| <=
// 2^-9, i.e. u^ within 2 bf16 roundings -- inside the 2e-2 tolerance of bf16 outputs)
__device__ __forceinline__ uint32_t sig_bf2(uint32_t z2) {
  const uint32_t half2 = 0x3F003F00u;  // (0.5, 0.5) in bf16x2
  uint32_t h, t, k;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(h) : "r"(z2), "r"(half2));
  asm("tanh.approx.bf16x2 %0, %1;" : "=r"(t) : "r"(h));
  asm("fma.rn.bf16x2 %0, %1, %2, %2;" : "=r"(k) : "r"(t), "r"(half2));
  return k;
}
__device__ __forceinline__ uint4 sigmul8(const uint4& zk, const uint4& v, uint4* kout = nullptr) {
  const uint4 k = make_uint4(sig_bf2(zk.x), sig_bf2(zk.y), sig_bf2(zk.z), sig_bf2(zk.w));
  if (kout) *kout = k;
  uint4 o;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(o.x) : "r"(k.x), "r"(v.x));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(o.y) : "r"(k.y), "r"(v.y));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(o.z) : "r"(k.z), "r"(v.z));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(o.w) : "r"(k.w), "r"(v.w));
  return o;
}
// 8 bf16 products, elementwise, one RNE rounding each (mul.rn.bf16x2)
__device__ __forceinline__ uint4 bmul8(const uint4& a, const uint4& b) {
  uint4 o;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(o.x) : "r"(a.x), "r"(b.x));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(o.y) : "r"(a.y), "r"(b.y));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(o.z) : "r"(a.z), "r"(b.z));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(o.w) : "r"(a.w), "r"(b.w));
  return o;
}
// pack two fp32 into bf16x2 (lo = first)
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---------------------------------------------------------------------------
// Epilogue fragment layout.  An epilogue warp (TMEM lane quarter wq) reads a
// block's 128 x 16 accumulator [channel lane][token column] in the m16n8
// fragment layout of tcgen05.ld.16x256b: lane l = 4 rr + qd holds
//     channels  c_k = 32 wq + rr + 8 k           (k = 0..3)
//     tokens    tk_m = 8 (m >> 1) + 2 qd + (m & 1)  (m = 0..3)
// as x[k][m].  Token pairs (m, m+1) of one channel pack into one bf16x2 word,
// which is exactly the element pair of an 8x8 b16 matrix fragment whose rows
// are channels: stmatrix/ldmatrix .trans move it to/from the swizzled token-row
// tile with no shuffles (matrix k = channels 32 wq + 8 k .. +7, tokens 8 tg ..
// +7; lane l supplies the address of row l & 7 of matrix l >> 3).
// ---------------------------------------------------------------------------
// x[k][m] <- TMEM columns col .. col+15 of lanes 32 wq .. 32 wq + 31 (taddr = lane
// quarter base | col).  Completes at tmem_wait_frag.
__device__ __forceinline__ void tmem_ld_frag(uint32_t taddr, float (&x)[4][4]) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                 "=r"(r[14]), "=r"(r[15])
               : "r"(taddr + (16u << 16)));
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // registers: (lane, col) = (rr, 2qd) (rr, 2qd+1) (rr+8, ..) x 2 col halves
    x[2 * h][0] = __uint_as_float(r[8 * h + 0]);
    x[2 * h][1] = __uint_as_float(r[8 * h + 1]);
    x[2 * h + 1][0] = __uint_as_float(r[8 * h + 2]);
    x[2 * h + 1][1] = __uint_as_float(r[8 * h + 3]);
    x[2 * h][2] = __uint_as_float(r[8 * h + 4]);
    x[2 * h][3] = __uint_as_float(r[8 * h + 5]);
    x[2 * h + 1][2] = __uint_as_float(r[8 * h + 6]);
    x[2 * h + 1][3] = __uint_as_float(r[8 * h + 7]);
  }
}
// wait for this thread's tcgen05.ld; the fragment is bound as an operand so no use
// of it can be scheduled above the wait
__device__ __forceinline__ void tmem_wait_frag(float (&x)[4][4]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(x[0][0]), "+f"(x[0][1]), "+f"(x[0][2]), "+f"(x[0][3]), "+f"(x[1][0]), "+f"(x[1][1]),
                 "+f"(x[1][2]), "+f"(x[1][3]), "+f"(x[2][0]), "+f"(x[2][1]), "+f"(x[2][2]), "+f"(x[2][3]),
                 "+f"(x[3][0]), "+f"(x[3][1]), "+f"(x[3][2]), "+f"(x[3][3])
               :
               : "memory");
}
// byte offset of this lane's stmatrix/ldmatrix row address inside a swizzled 4 KiB
// tile, token group tg = 0 (tg = 1 adds 1024 B): row (l & 7) of matrix k = l >> 3
template <int HS>
__device__ __forceinline__ uint32_t frag_row_off(int wq, int lane) {
  const int r = lane & 7, k = lane >> 3;
  return (uint32_t)((wq >> 1) * HS + r * 128 + (((4 * (wq & 1) + k) ^ r) << 4));
}
__device__ __forceinline__ void stsm_t(uint32_t p, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(p), "r"(r0),
               "r"(r1), "r"(r2), "r"(r3)
               : "memory");
}
__device__ __forceinline__ void ldsm_t(uint32_t p, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(p)
               : "memory");
}
// store x[k][m] (rounded once to bf16) into a swizzled tile; ro = frag_row_off
__device__ __forceinline__ void store_frag(uint32_t tile, uint32_t ro, const float (&x)[4][4]) {
#pragma unroll
  for (int tg = 0; tg < 2; ++tg)
    stsm_t(tile + ro + 1024 * tg, pack_bf2(x[0][2 * tg], x[0][2 * tg + 1]), pack_bf2(x[1][2 * tg], x[1][2 * tg + 1]),
           pack_bf2(x[2][2 * tg], x[2][2 * tg + 1]), pack_bf2(x[3][2 * tg], x[3][2 * tg + 1]));
}
// load a bf16 tile's elements in fragment order: t[k][tg] = bf16x2 (tokens 2qd+8tg, +1; channel c_k)
__device__ __forceinline__ void load_frag(uint32_t tile, uint32_t ro, uint32_t (&t)[2][4]) {
  ldsm_t(tile + ro, t[0]);
  ldsm_t(tile + ro + 1024, t[1]);
}
__device__ __forceinline__ float2 bf2f(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
// the value v held by lane (rr + 8k) for k = 0..3 (channel c_k of a 32x32b TMEM read)
__device__ __forceinline__ void chan4(float v, int rr, float (&o)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) o[k] = __shfl_sync(0xffffffffu, v, rr + 8 * k);
}
// aux arrays (g, r, gs) are stored per block in fragment token order: [qd][m]
__device__ __forceinline__ void load_aux(const float* p, float (&o)[4]) {
  const float4 x = *reinterpret_cast<const float4*>(p);
  o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w;
}
__device__ __forceinline__ int aux_perm(int i) { return 4 * ((i & 7) >> 1) + 2 * (i >> 3) + (i & 1); }

// ---------------------------------------------------------------------------
// the kernel
//
// Barriers (ring sizes in Cfg):
//   full[NI]     TMA bytes of the input stage landed            (producer, tx count)
//   prepped[NI]  L tiles (input stage) + g/r (work slot) + pre-gates written (prep)
//   inempty[NI]  input stage free: MMAs retired (SWR) / epilogue done (mixer)
//   mmad[NW]     tcgen05 MMAs of the item complete               (tcgen05.commit)
//   ready[NW]    MMAs of every item whose TMEM the epilogue reads are complete:
//                j-1, j (backward also j+1)                      (MMA warp)
//   wfree[NW]    work slot free: the item's epilogue and the neighbours that read
//                its TMEM / g are done (next; backward also previous) -- one
//                arrival per epilogue warp and user
//   ofull[NO]    outputs (and da partials) in the output slot    (each epilogue warp)
//   oempty[NO]   output slot free: TMA store has read it, da summed (store warp)
// The 4 warps of an epilogue group never synchronise with each other: each owns
// 32 channels (a TMEM lane quarter) and arrives on the barriers itself.
// ---------------------------------------------------------------------------
#ifndef SWR_PDL
// programmatic dependent launch: a launch may start its prologue (barrier init, TMEM
// allocation, range claim) on SMs the previous kernel has left and waits with
// griddepcontrol.wait before touching global memory.  Back to back the SWR step gets
// 124.5 -> 118.8 us (tools/ab_b2b.sh; with an L2 flush between steps it had measured 2%
// slower in round 1, when the flush kernel sat between the two)
#define SWR_PDL 1
#endif
#ifndef SWR_EPI_UNROLL
#define SWR_EPI_UNROLL 1
#endif
constexpr int kEpiUnroll = SWR_EPI_UNROLL;
template <int OP>
__global__ void __launch_bounds__((4 * Cfg<OP>::NG + Cfg<OP>::NPW + (Cfg<OP>::MIX ? 4 : 5)) * 32, 1)
    swr_tc_kernel(const __grid_constant__ Maps maps, const __grid_constant__ Split split, const Params p) {
  using C = Cfg<OP>;
  using S = Stage<OP>;
  constexpr int NI = C::NI, NW = C::NW, NO = C::NO, NG = C::NG, BPI = C::BPI;
  constexpr int kItemCols = BPI * C::COLS;
  // TMEM columns of a block: forward [w 0..15]; backward [lambda 0..15 | w 16..31], so
  // w is preceded by a valid column and can also be read shifted by one (w[i-1]).
  constexpr int kWo = C::BWD ? 16 : 0, kLo = 0, kWc = 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kPrepW0 = 4 * NG, kProdW = kPrepW0 + C::NPW, kMmaW = kProdW + 1, kStoreW = kMmaW + 1,
                kRetW = kStoreW + 1, kAProdW = C::MIX ? -1 : kRetW + 1;
  constexpr int NA = C::NA;

  // 1024-aligned base for the 128B-swizzle atoms.  Offset the __shared__ array
  // itself (not a uintptr_t round trip) so every access stays LDS/STS.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sin = smem + S::kInBase;
  uint8_t* sout = smem + S::kOutBase;
  uint8_t* work = smem + S::kWorkBase;
  uint8_t* sad = smem + S::kADBase;
  uint8_t* scratch = smem + S::kScratch;
  const uint32_t smem_s = su32(smem);
  // work slot s: transfer tiles at work + s*kWork, aux floats at auxf(s)
  auto auxf = [&](int s) { return reinterpret_cast<float*>(work + s * S::kWork + S::kAuxOff); };
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch);
  uint64_t* inempty = full + NI;
  uint64_t* afull = inempty + NI;
  uint64_t* aempty = afull + NA;
  uint64_t* prepped = aempty + NA;
  uint64_t* mmad = prepped + NW;
  uint64_t* ready = mmad + NW;
  uint64_t* wfree = ready + NW;
  uint64_t* ofull = wfree + NW;
  uint64_t* oempty = ofull + NO;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(oempty + NO);
  int* range_slot = reinterpret_cast<int*>(tmem_slot + 1);
  float* red = reinterpret_cast<float*>(scratch + 1024);  // [NO][4 warps][16*BPI] da partials

  constexpr int kTmemCols = (NW * kItemCols <= 32) ? 32 : (NW * kItemCols <= 64) ? 64
                          : (NW * kItemCols <= 128) ? 128 : (NW * kItemCols <= 256) ? 256 : 512;
  static_assert(NW * kItemCols <= 512, "TMEM budget");
  static_assert(NW >= 4 && NI >= 3 && NO >= 2, "ring depth (deadlock freedom)");
  // mbarrier waits are by phase parity, so a waiter must never be two phases ahead
  // of a barrier.  Prep warp j mod NPW waits afull[j mod NA] / wfree[j mod NW] (and,
  // mixer, full[j mod NI]) and arrives aempty[j mod NA] / prepped[j mod NW]; those
  // phases complete out of item order (TMA loads finish out of order), so each
  // stage and slot must always belong to the same prep warp, which then sees its
  // phases in order.  The epilogue's ready/oempty phases are produced in item order
  // by one thread; NO >= NG keeps a group (items j - NG, j) within one phase of oempty.
  static_assert(NA % C::NPW == 0 && NW % C::NPW == 0 && (!C::MIX || NI % C::NPW == 0),
                "prep warp <-> stage/slot ownership");
  static_assert(NO >= NG && NW >= NG, "epilogue group within one phase");
  // GRP: a group's consecutive items are up to (NG - 1) HS + 1 apart (the one-phase rule
  // above for that distance); the head's neighbour blocks are HS items away
  static_assert(C::HS == 1 || (BPI == 1 && C::MIX && C::BWD && NW > 2 * C::HS), "grouped walk");
  static_assert((2 * NI + 2 * NA + 4 * NW + 2 * NO) * 8 + 16 <= 1024 && NO * 4 * 16 * BPI * 4 <= 3072,
                "scratch budget");
  static_assert(S::kBytes + 1024 <= 227 * 1024, "shared memory budget");
  constexpr int kUsers = (C::BWD ? 3 : 2) * 4;  // users x epilogue warps

  if (threadIdx.x == 0) {
    trace_cta(p, 0);
    for (int s = 0; s < NI; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&inempty[s], C::MIX ? 4 : 1);
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < NW; ++s) {
      mbar_init(&prepped[s], 1);
      mbar_init(&mmad[s], 1);
      mbar_init(&ready[s], 1);
      mbar_init(&wfree[s], kUsers);
    }
    for (int s = 0; s < NO; ++s) {
      mbar_init(&ofull[s], 4);
      mbar_init(&oempty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *range_slot = claim_range(split, p.epoch);
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
  // Programmatic dependent launch: everything above (barrier init, TMEM allocation,
  // range claim) overlapped the previous kernel's tail; no global memory it may
  // write is touched before this wait.  The next kernel may start its own prologue
  // on SMs this grid frees (it waits for this grid's completion the same way).
#if SWR_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif

  const int nb = (int)p.nb, H = (int)p.H;   // sizes < 2^31 (tc_supported)
  const int nbi = (nb + BPI - 1) / BPI;       // items per line
  const int total = (int)p.B * H * nbi / C::HS;  // work units: items (HS = 1) / super-items
  const Work W = work_of<C::BWD, C::HS>(split, *range_slot, total, nbi);
  unsigned long long t_begin = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
  const int n_items = W.last - W.first;

  if (warp == kProdW) {
    // ===================== TMA producer =====================
    // SWR ops: the decay boxes come from their own producer warp, up to NA items
    // ahead, so the prep builds the transfer tiles while the d-tensor tiles are in
    // flight.  Mixer: the prep needs the tiles anyway; the decays are issued here,
    // just before the item's tiles.
    if (lane == 0 && n_items > 0) {
      Cursor<C::HS> cur;
      cur.init(W.first, nbi, H);
      Ring<NI> ri;
      Ring<NA> ra;
      ri.init(0);
      ra.init(0);
      for (int j = 0; j < n_items; ++j) {
        const int tt = (int)(cur.m * BPI * kEll);
        if constexpr (C::MIX) {
          mbar_wait(&aempty[ra.s], ra.ph ^ 1);
          mbar_expect_tx(&afull[ra.s], S::kAD);
          tma_load_3d(sad + ra.s * S::kAD, &maps.a, &afull[ra.s], cur.h & ~7, tt, cur.b);
          ra.next();
        }
        mbar_wait(&inempty[ri.s], ri.ph ^ 1);
        trace(p, j, 0);
        uint8_t* st = sin + ri.s * S::kIn;
        mbar_expect_tx(&full[ri.s], C::NT * S::kRegion);
#pragma unroll
        for (int x = 0; x < C::NT; ++x) {  // one box per 64-channel half: 16*BPI tokens
          uint8_t* dst = S::region(st, x);
          // layer mixer: q (x = 0) and k (x = 1) are read at the head's group
          const int hx = !C::LAYER ? cur.h : x == 0 ? cur.h / (int)p.hq : x == 1 ? cur.h / (int)p.hk : cur.h;
          tma_load_4d(dst, &maps.in[x], &full[ri.s], 0, hx, tt, cur.b);
          tma_load_4d(dst + S::kHS, &maps.in[x], &full[ri.s], 64, hx, tt, cur.b);
        }
        trace(p, j, 1);
        cur.next(nbi, H);
        ri.next();
      }
    }
  } else if (warp == kAProdW) {
    // ===================== decay producer (SWR ops) =====================
    if (lane == 0 && n_items > 0) {
      Cursor<C::HS> cur;
      cur.init(W.first, nbi, H);
      Ring<NA> ra;
      ra.init(0);
      for (int j = 0; j < n_items; ++j) {
        mbar_wait(&aempty[ra.s], ra.ph ^ 1);
        trace(p, j, 11);
        mbar_expect_tx(&afull[ra.s], S::kAD);
        tma_load_3d(sad + ra.s * S::kAD, &maps.a, &afull[ra.s], cur.h & ~7, (int)(cur.m * BPI * kEll), cur.b);
        cur.next(nbi, H);
        ra.next();
      }
    }
  } else if (warp == kMmaW) {
    // ===================== MMA issuer =====================
    // Blocks on prepped[] (which the prep arrives only after observing full[]),
    // issues the item's MMAs into its work slot's TMEM columns and commits them.
    if (lane == 0 && n_items > 0) {
      Ring<NI> ri;
      Ring<NW> rw;
      ri.init(0);
      rw.init(0);
      for (int j = 0; j < n_items; ++j) {
        mbar_wait(&prepped[rw.s], rw.ph);                  // transfer tiles (mixer: and pre-gates)
        if constexpr (!C::MIX) mbar_wait(&full[ri.s], ri.ph);  // operand tiles landed
        tc_fence_after();
        trace(p, j, 4);
        uint8_t* st = sin + ri.s * S::kIn;
#pragma unroll
        for (int k = 0; k < BPI; ++k) {
          const uint32_t d = tmem_base + (uint32_t)(rw.s * kItemCols + k * C::COLS);
          const uint32_t lt = su32(work + rw.s * S::kWork + 512 * k);
          const uint32_t lw = C::CYC ? lt + S::kLc : lt;
          umma_bf16(d + kWo, desc_A<S::kHS>(su32(S::tile(st, k, C::TU))), desc_Bmn(lw), kIdescBmn);  // w^T
          if constexpr (C::BWD)  // lambda^T
            umma_bf16(d + kLo, desc_A<S::kHS>(su32(S::tile(st, k, C::TG))), desc_Bk(lt), kIdescBk);
          if constexpr (C::WC)  // [w15, w0 .. w14]^T
            umma_bf16(d + kWc, desc_A<S::kHS>(su32(S::tile(st, k, C::TU))), desc_Bmn(lt + S::kLc), kIdescBmn);
        }
        umma_commit(&mmad[rw.s]);
        trace(p, j, 5);
        ri.next();
        rw.next();
      }
    }
    __syncwarp();
  } else if (warp == kRetW) {
    // ===================== MMA retire + readiness =====================
    // tcgen05 ops complete in issue order: retire items in order, which frees their
    // input stage (SWR: the operands are consumed), and mark an item ready once every
    // MMA its epilogue reads is complete: j-1, j (backward also j+1).
    if (lane == 0 && n_items > 0) {
      constexpr int kBack = C::BWD ? C::HS : 0;  // the next block of the head: HS items on
      Ring<NI> ri;
      Ring<NW> rw, rr;
      ri.init(0);
      rw.init(0);
      rr.init(0);
      for (int j = 0; j < n_items; ++j) {
        mbar_wait(&mmad[rw.s], rw.ph);
        tc_fence_before();
        if constexpr (!C::MIX) mbar_arrive(&inempty[ri.s]);  // operands consumed
        trace(p, j, 10);
        if (j - kBack >= 0) {
          mbar_arrive(&ready[rr.s]);
          trace(p, j - kBack, 6);
          rr.next();
        }
        ri.next();
        rw.next();
      }
      for (int jr = max(n_items - kBack, 0); jr < n_items; ++jr) {
        mbar_arrive(&ready[rr.s]);
        rr.next();
      }
    }
    __syncwarp();
  } else if (warp == kStoreW) {
    // ===================== TMA store, da sum, output-slot release =====================
    // lane 0 issues the TMA stores; backward: the warp sums the 4 epilogue warps'
    // da partials of the slot in a fixed order (deterministic) and writes da.  One
    // bulk group per item (empty for halo items); a slot is released once the NEXT
    // item's stores are issued and its own group has been read (wait_group.read 1),
    // so consecutive stores overlap instead of serialising on the SMEM read.
    if (n_items > 0) {
      Cursor<C::HS> cur;
      cur.init(W.first, nbi, H);
      Ring<NO> ro, rprev;
      ro.init(0);
      for (int j = 0; j < n_items; ++j) {
        SWR_DBG(j, n_items, ro.s, ro.ph);
        mbar_wait(&ofull[ro.s], ro.ph);
        const bool halo = cur.gi < W.g0 || cur.gi >= W.g1;
        if (lane == 0) {
          if (!halo && !C::EXACT1) {
            uint8_t* ot = sout + ro.s * S::kOut;
            const int tt = (int)(cur.m * BPI * kEll);
#pragma unroll
            for (int x = 0; x < C::NOUT; ++x) {  // rows past L are clipped by TMA
              // GRP: dq / dz_k (x = 0, 1) are the group sums, in the last head's slot
              if (C::GRP && x < 2 && cur.hh != C::HS - 1) continue;
              const int hx = (C::GRP && x < 2) ? cur.h / C::HS : cur.h;
              tma_store_4d(&maps.out[x], S::region(ot, x), 0, hx, tt, cur.b);
              tma_store_4d(&maps.out[x], S::region(ot, x) + S::kHS, 64, hx, tt, cur.b);
            }
          }
          bulk_commit();
          trace(p, j, 9);
        }
        if constexpr (C::BWD) {
          if (!halo) {
            const float* rb = red + ro.s * (4 * 16 * BPI);
            __nv_bfloat16* dA = (__nv_bfloat16*)p.da + (int64_t)cur.b * p.sa_b + (int64_t)cur.h * p.sa_h;
#pragma unroll
            for (int q0 = 0; q0 < 16 * BPI; q0 += 32) {
              const int q = q0 + lane;
              const int64_t n = (int64_t)cur.m * BPI * kEll + q;
              if (q < 16 * BPI && n < p.L) {
                const float sum = ((rb[q] + rb[16 * BPI + q]) + rb[32 * BPI + q]) + rb[48 * BPI + q];
                dA[n * p.sa_l] = __float2bfloat16_rn(sum);
              }
            }
          }
        }
        if (j >= 1) {  // release the previous item's slot once its stores have read it
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          if (lane == 0) mbar_arrive(&oempty[(j - 1) % NO]);
        }
        rprev = ro;
        cur.next(nbi, H);
        ro.next();
      }
      if (lane == 0) bulk_wait_all();
    }
  } else if (warp >= kPrepW0) {
    // ===================== prep: L tiles (Alg. 3), g, r, pre-gates =====================
    // prep warp pw owns items j = pw mod NPW; each 16-lane half builds one block
    const int pw = warp - kPrepW0;
    const int hf = lane >> 4, col = lane & 15;
    Cursor<C::HS> cur;
    if (pw < n_items) cur.init(W.first + pw, nbi, H);
    Ring<NI> ri;
    Ring<NA> ra;
    Ring<NW> rw;
    ri.init(pw);
    ra.init(pw);
    rw.init(pw);
    for (int j = pw; j < n_items; j += C::NPW) {
      // the transfer tiles need only the decays (loaded ahead) and a free work slot
      mbar_wait(&afull[ra.s], ra.ph);
      mbar_wait(&wfree[rw.s], rw.ph ^ 1);
      if (lane == 0) trace(p, j, 2);
      uint8_t* st = sin + ri.s * S::kIn;
      uint8_t* wt = work + rw.s * S::kWork;  // transfer tiles of this work slot
      float* gr = auxf(rw.s);               // [BPI][g 16 | r 16 | gs 16]
#pragma unroll
      for (int kb = 0; kb < BPI; kb += 2) {
        const int k = kb + hf;
        if (k < BPI) {
          const int t = cur.m * BPI + k;
          const int nval = (int)std::min<int64_t>(16, std::max<int64_t>(p.L - (int64_t)t * kEll, 0));  // valid tokens
          // lane col owns column col of L_t.  Alg. 3: tile a down the columns, pre-mask
          // the inclusive upper triangle with 1, column-wise cumulative product, zero
          // the strict upper triangle.  Products only, never ratios.
          const uint8_t* at = sad + ra.s * S::kAD + (k * kEll) * 16 + (cur.h & 7) * 2;
          float a[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            a[i] = (i < nval) ? __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(at + i * 16)) : 1.f;
          if constexpr (C::LAYER) {
            if (p.logit_a) {  // a = sigma(za); the padding keeps a = 1
#pragma unroll
              for (int i = 0; i < 16; ++i) a[i] = (i < nval) ? sig_tc(a[i]) : 1.f;
            }
            // sp = a (1 - a) = sigma'(za) for the logit gradient (token order)
            if (C::BWD && col == 0) {
#pragma unroll
              for (int i = 0; i < 16; ++i) gr[S::kAuxBlk * k + 48 + i] = a[i] * (1.f - a[i]);
            }
          }
          float Lc[16];
          float prod = 1.f;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i > col) prod *= a[i];
            Lc[i] = (i >= col) ? prod : 0.f;  // L[i][col]
          }
          // column col: two 16-byte stores (rows 0-7, rows 8-15), rounded once to bf16
          uint8_t* l = wt + 512 * k;
          uint4 lo, hi;
          lo.x = pack_bf2(Lc[0], Lc[1]);   lo.y = pack_bf2(Lc[2], Lc[3]);
          lo.z = pack_bf2(Lc[4], Lc[5]);   lo.w = pack_bf2(Lc[6], Lc[7]);
          hi.x = pack_bf2(Lc[8], Lc[9]);   hi.y = pack_bf2(Lc[10], Lc[11]);
          hi.z = pack_bf2(Lc[12], Lc[13]); hi.w = pack_bf2(Lc[14], Lc[15]);
          *reinterpret_cast<uint4*>(l + ltile_off(0, col)) = lo;
          *reinterpret_cast<uint4*>(l + ltile_off(8, col)) = hi;
          if constexpr (C::CYC || C::WC) {  // rows rotated by one: Lc[i][col] = L[(i-1) mod 16][col]
            uint8_t* lc = wt + S::kLc + 512 * k;
            uint4 clo, chi;
            clo.x = pack_bf2(Lc[15], Lc[0]); clo.y = pack_bf2(Lc[1], Lc[2]);
            clo.z = pack_bf2(Lc[3], Lc[4]);  clo.w = pack_bf2(Lc[5], Lc[6]);
            chi.x = pack_bf2(Lc[7], Lc[8]);  chi.y = pack_bf2(Lc[9], Lc[10]);
            chi.z = pack_bf2(Lc[11], Lc[12]); chi.w = pack_bf2(Lc[13], Lc[14]);
            *reinterpret_cast<uint4*>(lc + ltile_off(0, col)) = clo;
            *reinterpret_cast<uint4*>(lc + ltile_off(8, col)) = chi;
          }
          // aux arrays in the epilogue's fragment token order (aux_perm)
          if constexpr (C::BWD) gr[S::kAuxBlk * k + 16 + aux_perm(col)] = prod;  // r_t[j] = L[15][j]
          if (col == 0) {
            // g_t[i] = a_t[0] L_t[i][0] = a_t[0] ... a_t[i], fp32;
            // gs[i] = g_t[i-1] (gs[0] = 1)
            float g[17];
            g[0] = 1.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) g[i + 1] = a[0] * Lc[i];
            float4* gp = reinterpret_cast<float4*>(gr + S::kAuxBlk * k);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              gp[q] = make_float4(g[2 * q + 1], g[2 * q + 2], g[2 * q + 9], g[2 * q + 10]);
              gp[8 + q] = make_float4(g[2 * q], g[2 * q + 1], g[2 * q + 8], g[2 * q + 9]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&aempty[ra.s]);  // decays read
      if constexpr (C::MIX) {
        mbar_wait(&full[ri.s], ri.ph);
        // pre-gates in the swizzled tile layout (elementwise, layout-agnostic), each
        // rounded once to bf16: u^ = k (.) v; backward also G = dy (.) q.
        // A bf16 x bf16 product is exact in fp32, so the packed bf16x2 multiply (one
        // rounding of the exact product) equals fp32 multiply + one RNE rounding.
        uint4* K4 = reinterpret_cast<uint4*>(S::region(st, 1));
        const uint4* V4 = reinterpret_cast<const uint4*>(S::region(st, 2));
        uint4* U4 = reinterpret_cast<uint4*>(S::region(st, C::TU));
#pragma unroll 4
        for (int v = lane; v < S::kRegion / 16; v += 32) {
          if (C::LAYER && p.logit_k) {  // u^ = sigma(zk) (.) v
            if constexpr (C::BWD) {     // the epilogue reads k = sigma(zk) (bf16) over zk
              uint4 kb;
              U4[v] = sigmul8(K4[v], V4[v], &kb);
              K4[v] = kb;
            } else {
              U4[v] = sigmul8(K4[v], V4[v]);
            }
          } else
            U4[v] = bmul8(K4[v], V4[v]);
          if constexpr (C::BWD) {
            uint4* Q4 = reinterpret_cast<uint4*>(S::region(st, 0));  // G overwrites q
            const uint4* D4 = reinterpret_cast<const uint4*>(S::region(st, 3));
            Q4[v] = bmul8(D4[v], Q4[v]);
          }
        }
      }
      fence_proxy_async();  // this lane's generic-proxy writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&prepped[rw.s]);
        trace(p, j, 3);
      }
      cur.step(C::NPW, nbi, H);
      ri.template step<C::NPW>();
      ra.template step<C::NPW>();
      rw.template step<C::NPW>();
    }
  } else {
    // ===================== epilogue groups: fragment layout (see tmem_ld_frag) =====================
    // lane l = 4 rr + qd owns channels c_k = 32 wq + rr + 8k and tokens tk_m of every block;
    // token pairs (m, m+1) are packed fp32x2 lanes and one bf16x2 word of a fragment
    const int grp = warp >> 2;                       // epilogue group, items j = grp mod NG
    const int wq = warp & 3;                         // TMEM lane quarter
    const int qd = lane & 3, rr = lane >> 2;
    const int cb = 32 * wq + rr;                     // channel c_0
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t fro = frag_row_off<S::kHS>(wq, lane);
    const bool leader = (threadIdx.x & 127) == 0;   // trace only
    // group grp takes items j = grp mod NG (HS = 1); GRP: the super-items grp mod NG,
    // i.e. the HS consecutive items (heads of one group, one block) of each
    const int j0 = grp * C::HS;
    Cursor<C::HS> cur;
    if (j0 < n_items) cur.init(W.first + j0, nbi, H);
    Ring<NI> ri;
    Ring<NW> rw;
    Ring<NO> ro;
    ri.init(j0);
    rw.init(j0);
    ro.init(j0);
    // GRP: the head's dq and dz_k terms summed over the group's heads (fp32, head order)
    float acc_q[4][4], acc_k[4][4];
    (void)acc_q;
    (void)acc_k;
    for (int j = j0; j < n_items;) {
      Ring<NW> rp = rw, rn = rw;  // work slots of the head's previous / next block: items j -+ HS
#pragma unroll
      for (int i = 0; i < C::HS; ++i) {
        rp.prev();
        rn.next();
      }
      const int t0 = cur.m * BPI;
      const bool halo = cur.gi < W.g0 || cur.gi >= W.g1;
      const int nblk = min(BPI, nb - t0);  // valid blocks of this item
      const uint32_t st = smem_s + S::kInBase + ri.s * S::kIn;   // shared-window addresses
      const uint32_t ot = smem_s + S::kOutBase + ro.s * S::kOut;
      const float* gr = auxf(rw.s);
      const int co = cur.line * kD + cb;              // carry / mu index of c_0 (< 2^31)
      const uint32_t tslot = tmem_base + lane_base + (uint32_t)(rw.s * kItemCols);
      const bool first_item = t0 == 0, last_item = t0 + nblk == nb;
      mbar_wait(&ready[rw.s], rw.ph);
      // lanes may leave the polling loop apart; converge before the .sync.aligned
      // tcgen05.ld / stmatrix / ldmatrix below
      __syncwarp();
      tc_fence_after();
      if (leader) trace(p, j, 7);
      // 1) neighbour reads first, so the neighbours' work slots are released early:
      //    carrier entering block t0: v = w_{t0-1}[15], the last block of item j-1;
      //    backward: mu of the item's last block from block 0 of item j+1
      float v[4] = {0.f, 0.f, 0.f, 0.f}, mu_last[4] = {0.f, 0.f, 0.f, 0.f};
      if (!halo) {
        if (first_item) {  // v_{-1}
          if (p.carry_in) {
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = p.carry_in[co + 8 * k];
          }
        } else if constexpr (C::EXACT) {  // s_{t0-1}: the exact state entering the item
          const float* S = p.ex_S + ((int64_t)cur.line * nb + t0 - 1) * kD;
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] = S[cb + 8 * k];
        } else {
          // w[15] of the previous item's last block (CYC: stored in its column 0)
          float x = tmem_ld1(tmem_base + lane_base +
                             (uint32_t)(rp.s * kItemCols + (BPI - 1) * C::COLS + kWo + (C::CYC ? 0 : 15)));
          tmem_wait_f(x);
          chan4(x, rr, v);
        }
        if constexpr (C::BWD) {
          if (last_item) {
            if (p.mu_in) {
#pragma unroll
              for (int k = 0; k < 4; ++k) mu_last[k] = p.mu_in[co + 8 * k];
            }
          } else {  // mu_t = a_{t+1}[0] lambda_{t+1}[0]
            float l0 = tmem_ld1(tmem_base + lane_base + (uint32_t)(rn.s * kItemCols + kLo));
            tmem_wait_f(l0);
            chan4(auxf(rn.s)[0] * l0, rr, mu_last);  // g[0] = a[0]
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (j >= C::HS) mbar_arrive(&wfree[rp.s]);                       // as "next" of item j-HS
        if (C::BWD && j + C::HS < n_items) mbar_arrive(&wfree[rn.s]);  // as "previous" of item j+HS
      }
      SWR_DBG(j, cur.hh, ro.s, ro.ph);
      mbar_wait(&oempty[ro.s], ro.ph ^ 1);
      __syncwarp();
      float* rb = red + ro.s * (4 * 16 * BPI);  // this slot's da partials [4 lane quarters][16*BPI tokens]
      // 2) the item's blocks, in order (the carrier passes block to block in registers)
      if (!halo) {
#pragma unroll kEpiUnroll
        for (int kb = 0; kb < nblk; ++kb) {
          const float* ga = gr + S::kAuxBlk * kb;  // [g 16 | r 16 | gs 16], fragment order
          const uint32_t tb = tslot + kb * C::COLS;
          if constexpr (!C::BWD) {
            float w[4][4];
            tmem_ld_frag(tb + kWo, w);
            float gg[4];
            load_aux(ga + 4 * qd, gg);
            tmem_wait_frag(w);
            float out[4][4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // Pass II: x~ = w + g v, packed token pairs
              const float2 v2 = make_float2(v[k], v[k]);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float2 o = f2fma(make_float2(gg[2 * h], gg[2 * h + 1]), v2, make_float2(w[k][2 * h], w[k][2 * h + 1]));
                out[k][2 * h] = o.x;
                out[k][2 * h + 1] = o.y;
              }
            }
            if constexpr (C::MIX) {  // post-gate with residual: y = q x~ + v
              uint32_t tq[2][4], tv[2][4];
              load_frag(S::tile(st, kb, 0), fro, tq);
              load_frag(S::tile(st, kb, 2), fro, tv);
#pragma unroll
              for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const float2 o = f2fma(bf2f(tq[h][k]), make_float2(out[k][2 * h], out[k][2 * h + 1]), bf2f(tv[h][k]));
                  out[k][2 * h] = o.x;
                  out[k][2 * h + 1] = o.y;
                }
            }
            if constexpr (C::EXACT1) {  // v_t = w_t[15] per channel, c_t = g_t[15] per line
              if (qd == 3) {
                float* V = const_cast<float*>(p.ex_S) + ((int64_t)cur.line * nb + t0 + kb) * kD;
#pragma unroll
                for (int k = 0; k < 4; ++k) V[cb + 8 * k] = w[k][3];
                if (wq == 0 && rr == 0) p.ex_C[(int64_t)cur.line * nb + t0 + kb] = gg[3];
              }
            } else {
              store_frag(S::tile(ot, kb, 0), fro, out);
            }
            if (!C::EXACT && !C::EXACT1 && t0 + kb == nb - 1 && p.carry_out && qd == 3) {
#pragma unroll
              for (int k = 0; k < 4; ++k) p.carry_out[co + 8 * k] = w[k][3];  // w_t[15]
            }
            // next carrier: B2P v_t = w_t[15]; exact: the state at token 15
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __shfl_sync(0xffffffffu, C::EXACT ? out[k][3] : w[k][3], lane | 3);
          } else {
            // lambda and w[i-1] of the block.  SWR (CYC): the rotated tile puts w[i-1] at
            // token i and w[15] at token 0.  Mixer: w[i] in place (needed for dq), w[i-1]
            // by shuffles inside the lane quad (tcgen05.ld.16x256b needs 8-column alignment).
            float lam[4][4], w[4][4];
            tmem_ld_frag(tb + kLo, lam);
            tmem_ld_frag(tb + kWo, w);
            float mu[4] = {mu_last[0], mu_last[1], mu_last[2], mu_last[3]};
            if (kb + 1 < nblk) {  // next block inside this item: mu_t = a_{t+1}[0] lambda_{t+1}[0]
              float l0 = tmem_ld1(tb + C::COLS + kLo);
              tmem_wait_f(l0);
              chan4(ga[S::kAuxBlk] * l0, rr, mu);
            }
            float rv[4], sv[4];
            load_aux(ga + 16 + 4 * qd, rv);
            load_aux(ga + 32 + 4 * qd, sv);  // gs = g shifted by one
            float wc[4][4];
            if constexpr (C::WC) tmem_ld_frag(tb + kWc, wc);
            tmem_wait_frag(lam);
            tmem_wait_frag(w);
            if constexpr (C::WC) tmem_wait_frag(wc);
            float wsh[4][4], vnext[4] = {0.f, 0.f, 0.f, 0.f};  // wsh[k][m] = w[tk_m - 1], w[-1] = 0
            if constexpr (C::CYC || C::WC) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float (&wr)[4] = C::WC ? wc[k] : w[k];  // the rotated product
                vnext[k] = __shfl_sync(0xffffffffu, wr[0], lane & ~3);  // token 0 of qd 0: w[15]
                wsh[k][0] = qd == 0 ? 0.f : wr[0];
                wsh[k][1] = wr[1];
                wsh[k][2] = wr[2];
                wsh[k][3] = wr[3];
              }
            } else {
              const int src = (lane & ~3) | ((lane + 3) & 3);  // lane - 1 inside the quad (qd 0 <- qd 3)
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float x0 = __shfl_sync(0xffffffffu, w[k][1], src);                    // token 2qd - 1
                const float x2 = __shfl_sync(0xffffffffu, qd == 3 ? w[k][1] : w[k][3], src);  // token 7 + 2qd
                wsh[k][0] = qd == 0 ? 0.f : x0;
                wsh[k][1] = w[k][0];
                wsh[k][2] = x2;
                wsh[k][3] = w[k][2];
              }
            }
            // du = lambda + r mu;  da[i] = sum_c lambda x~[i-1] + r mu w[i-1]
            //                           = sum_c du w[i-1] + g[i-1] sum_c lambda v
            // (both channel sums of the thread as packed FMA chains over k)
            float du[4][4];
            float2 dw[2], lv[2];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 v2 = make_float2(v[k], v[k]), mu2 = make_float2(mu[k], mu[k]);
#pragma unroll
              for (int h = 0; h < 2; ++h) {  // token pairs (2h, 2h+1)
                const float2 lam2 = make_float2(lam[k][2 * h], lam[k][2 * h + 1]);
                const float2 wp = make_float2(wsh[k][2 * h], wsh[k][2 * h + 1]);
                const float2 d2 = f2fma(make_float2(rv[2 * h], rv[2 * h + 1]), mu2, lam2);
                dw[h] = k == 0 ? f2mul(d2, wp) : f2fma(d2, wp, dw[h]);
                lv[h] = k == 0 ? f2mul(lam2, v2) : f2fma(lam2, v2, lv[h]);
                du[k][2 * h] = d2.x;
                du[k][2 * h + 1] = d2.y;
              }
            }
            if (t0 + kb == 0 && p.mu_out && qd == 0) {
#pragma unroll
              for (int k = 0; k < 4; ++k) p.mu_out[co + 8 * k] = ga[0] * lam[k][0];  // a_0[0] lambda_0[0]
            }
            // da: the thread's 4-channel sums per token, then a transpose-reduce over the
            // 8 lanes sharing qd (lane bits 2..4); fixed order, no atomics
            float s[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float2 s2 = f2fma(make_float2(sv[2 * h], sv[2 * h + 1]), lv[h], dw[h]);
              s[2 * h] = s2.x;
              s[2 * h + 1] = s2.y;
            }
            const bool u16 = lane & 16, u8 = lane & 8;
            const float a0 = (u16 ? s[2] : s[0]) + __shfl_xor_sync(0xffffffffu, u16 ? s[0] : s[2], 16);
            const float a1 = (u16 ? s[3] : s[1]) + __shfl_xor_sync(0xffffffffu, u16 ? s[1] : s[3], 16);
            float b = (u8 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, u8 ? a0 : a1, 8);
            b += __shfl_xor_sync(0xffffffffu, b, 4);
            if ((lane & 4) == 0) {  // lane holds m = 2 u16 + u8: token 8 u16 + 2 qd + u8
              const int tok = (u16 ? 8 : 0) + 2 * qd + (u8 ? 1 : 0);
              if (C::LAYER && p.logit_a) b *= ga[48 + tok];  // dza = da sigma'(za)
              rb[wq * (16 * BPI) + kb * 16 + tok] = b;
            }
            if constexpr (!C::MIX) {
              store_frag(S::tile(ot, kb, 0), fro, du);
            } else {
              float gg[4];
              load_aux(ga + 4 * qd, gg);
              uint32_t tdy[2][4], tk[2][4], tv[2][4];
              load_frag(S::tile(st, kb, 3), fro, tdy);
              load_frag(S::tile(st, kb, 1), fro, tk);
              load_frag(S::tile(st, kb, 2), fro, tv);
              float o[4][4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {  // dq = dy x~,  x~ = w + g v
                const float2 v2 = make_float2(v[k], v[k]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const float2 x2 = f2fma(make_float2(gg[2 * h], gg[2 * h + 1]), v2, make_float2(w[k][2 * h], w[k][2 * h + 1]));
                  const float2 q2 = f2mul(bf2f(tdy[h][k]), x2);
                  o[k][2 * h] = q2.x; o[k][2 * h + 1] = q2.y;
                }
              }
              if constexpr (C::GRP) {  // dq of the group: sum over its heads, stored by the last
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                  for (int m = 0; m < 4; ++m) acc_q[k][m] = cur.hh == 0 ? o[k][m] : acc_q[k][m] + o[k][m];
                if (cur.hh == C::HS - 1) store_frag(S::tile(ot, kb, 0), fro, acc_q);
              } else {
                store_frag(S::tile(ot, kb, 0), fro, o);
              }
#pragma unroll
              for (int k = 0; k < 4; ++k) {  // dv = du^ k + dy ; dk = du^ v
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const float2 d2 = make_float2(du[k][2 * h], du[k][2 * h + 1]);
                  const float2 kf = bf2f(tk[h][k]);  // layer mixer: k = sigma(zk), written by the prep
                  const float2 dv2 = f2fma(d2, kf, bf2f(tdy[h][k]));
                  float2 dk2 = f2mul(d2, bf2f(tv[h][k]));
                  if (C::GRP) {  // group sum first; sigma'(zk) of the group's zk at the last head
                    dk2.x = cur.hh == 0 ? dk2.x : acc_k[k][2 * h] + dk2.x;
                    dk2.y = cur.hh == 0 ? dk2.y : acc_k[k][2 * h + 1] + dk2.y;
                    acc_k[k][2 * h] = dk2.x;
                    acc_k[k][2 * h + 1] = dk2.y;
                  }
                  if (C::LAYER && p.logit_k && (!C::GRP || cur.hh == C::HS - 1))  // dzk = dk sigma'(zk), sigma' = k (1 - k)
                    dk2 = f2mul(dk2, make_float2(kf.x * (1.f - kf.x), kf.y * (1.f - kf.y)));
                  o[k][2 * h] = dv2.x; o[k][2 * h + 1] = dv2.y;
                  du[k][2 * h] = dk2.x; du[k][2 * h + 1] = dk2.y;
                }
              }
              store_frag(S::tile(ot, kb, 2), fro, o);
              if (!C::GRP || cur.hh == C::HS - 1) store_frag(S::tile(ot, kb, 1), fro, du);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)  // v_t = w_t[15]
              v[k] = (C::CYC || C::WC) ? vnext[k] : __shfl_sync(0xffffffffu, w[k][3], lane | 3);
          }
        }
      }
      // 3) this warp's outputs (and da partials) are in the output slot: hand them to
      //    the store warp; release the work slot (and, mixer, the input stage)
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (leader) trace(p, j, 8);
        mbar_arrive(&ofull[ro.s]);
        mbar_arrive(&wfree[rw.s]);                                 // self
        if (j >= n_items - C::HS) mbar_arrive(&wfree[rw.s]);       // no next item
        if (C::BWD && j < C::HS) mbar_arrive(&wfree[rw.s]);        // no previous item
        if constexpr (C::MIX) mbar_arrive(&inempty[ri.s]);
      }
      if constexpr (C::HS == 1) {
        j += NG;
        cur.step(NG, nbi, H);
        ri.template step<NG>();
        rw.template step<NG>();
        ro.template step<NG>();
      } else {  // the super-item's next head, else the group's next super-item
        constexpr int kAdv = (NG - 1) * C::HS + 1;
        static_assert(kAdv <= NI && kAdv <= NW && kAdv <= NO, "one wrap at most");
        const int adv = cur.hh == C::HS - 1 ? kAdv : 1;
        j += adv;
        cur.step(adv, nbi, H);
        ri.init(j);
        rw.init(j);
        ro.init(j);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    trace_cta(p, 1);
#if SWR_TRACE
    if (p.trace != nullptr) p.trace[16 * p.trace_n + 4 * blockIdx.x + 3] = (unsigned long long)(W.g1 - W.g0);
#endif
    if (split.weighted && W.g1 > W.g0) {  // this SM's time per item, for the next split
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      if (sm < kMaxSM) g_spi[OP][sm] = (float)(t_end - t_begin) / (float)(W.g1 - W.g0);
    }
  }
  if (warp == kMmaW) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// Host side of the weighted split (see Split): per op, the SM rates learned from
// g_spi.  After a launch, g_spi[op] is copied to pinned memory on a private stream
// that waits for the launch (so the caller's stream never waits for the copy); a
// later launch folds the copy in once it has completed (never a host sync).  Skipped
// while the caller's stream is being captured into a graph.
struct Balance {
  std::mutex mu;
  std::vector<float> rate;  // items per ns, per SM (0 = unknown)
  float* host = nullptr;    // pinned readback buffer
  cudaEvent_t ev = nullptr, done = nullptr;
  cudaStream_t side = nullptr;
  bool pending = false;
  uint64_t launches = 0;

  // fills the split for this launch (q.epoch is already set); true if a readback
  // should follow it
  bool plan(Params& q, Split& sp, int grid, int sms, int64_t total, cudaStream_t st) {
    (void)q;
    sp.weighted = 0;
    if (grid != sms || sms > kMaxSM) return false;
    std::lock_guard<std::mutex> lock(mu);
    if ((int)rate.size() != sms) rate.assign(sms, 0.f);
    if (pending && cudaEventQuery(ev) == cudaSuccess) {
      for (int s = 0; s < sms; ++s)
        if (host[s] > 0.f) rate[s] = rate[s] > 0.f ? 0.7f * rate[s] + 0.3f / host[s] : 1.f / host[s];
      pending = false;
    }
    double sum = 0.0;
    bool known = true;
    for (int s = 0; s < sms; ++s) {
      known = known && rate[s] > 0.f;
      sum += rate[s];
    }
    if (known) {
      sp.weighted = 1;
      double acc = 0.0;
      sp.bnd[0] = 0;
      for (int s = 0; s < sms; ++s) {
        acc += rate[s];
        sp.bnd[s + 1] = (int)std::llround(acc / sum * (double)total);
        if (sp.bnd[s + 1] < sp.bnd[s]) sp.bnd[s + 1] = sp.bnd[s];
      }
      sp.bnd[sms] = (int)total;
    } else {
      // uniform ranges by SM id until every SM has reported (CTA placement then learns)
      sp.weighted = 1;
      for (int s = 0; s <= sms; ++s) sp.bnd[s] = (int)((int64_t)s * total / sms);
    }
    ++launches;
    // refresh the table from every 8th launch (each readback costs the host a few
    // CUDA calls; the rates move slowly)
    return !pending && (launches < 8 || launches % 8 == 0);
  }
  void request(int op, int sms, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(mu);
    if (pending) return;
    if (host == nullptr && cudaMallocHost(reinterpret_cast<void**>(&host), kMaxSM * sizeof(float)) != cudaSuccess) {
      host = nullptr;
      return;
    }
    if (ev == nullptr && (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
                          cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess ||
                          cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess)) {
      ev = nullptr;
      return;
    }
    if (cudaEventRecord(done, st) != cudaSuccess || cudaStreamWaitEvent(side, done, 0) != cudaSuccess) return;
    if (cudaMemcpyFromSymbolAsync(host, g_spi, sms * sizeof(float), (size_t)op * kMaxSM * sizeof(float),
                                  cudaMemcpyDeviceToHost, side) != cudaSuccess)
      return;
    if (cudaEventRecord(ev, side) == cudaSuccess) pending = true;
  }
};
constexpr int kMaxDev = 64;
static Balance g_balance[kMaxDev][9];  // per device (SM rates are a property of the GPU), per op

// Claim slots of the weighted split, per device.  A weighted launch claims its ranges
// in g_claim[epoch % kClaimSlots]; a slot may only be reused once the launch that used
// it last has completed, otherwise two in-flight launches would share claim words and a
// range could be processed twice or not at all.  Each weighted launch records an event
// on its stream; if the slot's event has not completed (more than kClaimSlots launches
// in flight), the launch takes the uniform split by CTA index instead, which uses no
// claims (bitwise the same results).  Under CUDA-graph capture the launch is replayed
// with the same parameters, so captured launches always take the uniform split.
struct Claims {
  std::mutex mu;
  uint32_t next = 0;
  cudaEvent_t ev[kClaimSlots] = {};
  bool used[kClaimSlots] = {};

  // epoch for the launch and whether it may use the claim slot (weighted split)
  bool acquire(cudaStream_t st, uint32_t* epoch) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    const bool capturing = cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone;
    std::lock_guard<std::mutex> lock(mu);
    do {
      *epoch = ++next;
    } while (*epoch == 0);
    if (capturing) return false;
    const int s = (int)(*epoch % kClaimSlots);
    if (used[s] && cudaEventQuery(ev[s]) != cudaSuccess) {
      (void)cudaGetLastError();  // cudaErrorNotReady is not an error of this call
      return false;
    }
    return true;
  }
  // after a weighted launch: mark its slot busy until the stream passes this point
  void release(cudaStream_t st, uint32_t epoch) {
    std::lock_guard<std::mutex> lock(mu);
    const int s = (int)(epoch % kClaimSlots);
    if (ev[s] == nullptr && cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming) != cudaSuccess) {
      ev[s] = nullptr;
      return;
    }
    if (cudaEventRecord(ev[s], st) == cudaSuccess) used[s] = true;
  }
};
static Claims g_claims[kMaxDev];

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

// Encoded tensor maps, cached per calling thread: a training step calls the same
// ops on the same (caching-allocator) buffers, so the key -- pointer, dims, strides,
// box rows -- repeats and the ~1 us host-side encode is skipped.
struct MapKey {
  const void* ptr;
  uint64_t dims[4], strides[3];
  uint32_t rows, kind;
};
struct MapCache {
  static constexpr int N = 32;
  MapKey key[N];
  CUtensorMap map[N];
  int used = 0, next = 0;
  const CUtensorMap* find(const MapKey& k) const {
    for (int i = 0; i < used; ++i)
      if (std::memcmp(&key[i], &k, sizeof(MapKey)) == 0) return &map[i];
    return nullptr;
  }
  void put(const MapKey& k, const CUtensorMap& m) {
    key[next] = k;
    map[next] = m;
    next = (next + 1) % N;
    if (used < N) ++used;
  }
};
static thread_local MapCache g_maps;

static bool encode_cached(CUtensorMap* m, const void* ptr, CUtensorMapDataType ty, int rank, const cuuint64_t* dims,
                          const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle sw, uint32_t kind) {
  MapKey k;
  std::memset(&k, 0, sizeof(k));
  k.ptr = ptr;
  for (int i = 0; i < rank; ++i) k.dims[i] = dims[i];
  for (int i = 0; i + 1 < rank; ++i) k.strides[i] = strides[i];
  k.rows = box[rank - 2];
  k.kind = kind;
  if (const CUtensorMap* c = g_maps.find(k)) {
    *m = *c;
    return true;
  }
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (encoder()(m, ty, rank, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  g_maps.put(k, *m);
  return true;
}

}  // namespace tc

// a bf16 tensor map without swizzle, cached like the tensor-core family's (for the
// staged narrow-head kernels, swr_narrow.cu); kind separates maps of different boxes
bool tma_encode_bf16(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box, uint32_t kind) {
  if (tc::encoder() == nullptr || rank < 2 || rank > 4) return false;
  cuuint64_t d[4], s[3];
  cuuint32_t bx[4];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i + 1 < rank; ++i) s[i] = strides[i];
  return tc::encode_cached(m, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, d, s, bx, CU_TENSOR_MAP_SWIZZLE_NONE, kind);
}

namespace tc {
// which: 0 = a [B, L, H, D] d-tensor with the strides sx; 1 / 2 = the layer mixer's
// group-shared q / k (and dq / dk) [B, L, G, D] with their own strides; 3 = a per-head
// scratch [B, L, H, D], contiguous
static bool map_dtensor(CUtensorMap* m, const void* ptr, const Params& p, int rows, int which = 0) {
  const int64_t G = which == 1 ? p.H / p.hq : which == 2 ? p.H / p.hk : p.H;
  const int64_t sh = which == 1 ? p.sq_h : which == 2 ? p.sk_h : which == 3 ? p.D : p.sx_h;
  const int64_t sl = which == 1 ? p.sq_l : which == 2 ? p.sk_l : which == 3 ? p.H * p.D : p.sx_l;
  const int64_t sb = which == 1 ? p.sq_b : which == 2 ? p.sk_b : which == 3 ? p.L * p.H * p.D : p.sx_b;
  cuuint64_t dims[4] = {(cuuint64_t)p.D, (cuuint64_t)G, (cuuint64_t)p.L, (cuuint64_t)p.B};
  cuuint64_t strides[3] = {(cuuint64_t)sh * 2, (cuuint64_t)sl * 2, (cuuint64_t)sb * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)rows, 1};
  return encode_cached(m, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, 0);
}

static bool map_decay(CUtensorMap* m, const void* ptr, const Params& p, int bpi) {
  cuuint64_t dims[3] = {(cuuint64_t)p.H, (cuuint64_t)p.L, (cuuint64_t)p.B};
  cuuint64_t strides[2] = {(cuuint64_t)p.sa_l * 2, (cuuint64_t)p.sa_b * 2};
  cuuint32_t box[3] = {8, (cuuint32_t)(16 * bpi), 1};
  return encode_cached(m, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE, 1);
}

template <int OP>
static cudaError_t launch_op(const Params& p, cudaStream_t st, int sms) {
  Maps maps;
  std::memset(&maps, 0, sizeof(maps));
  const void* ins[4] = {nullptr, nullptr, nullptr, nullptr};
  const void* outs[3] = {nullptr, nullptr, nullptr};
  int nin = 0, nout = 0;
  switch (OP) {
    case 0: case 6: case 7: ins[0] = p.u; outs[0] = (OP == 7) ? p.u : p.x; nin = 1; nout = 1; break;
    case 1: ins[0] = p.u; ins[1] = p.dx; outs[0] = p.du; nin = 2; nout = 1; break;
    case 2: case 4: ins[0] = p.q; ins[1] = p.k; ins[2] = p.v; outs[0] = p.y; nin = 3; nout = 1; break;
    default:
      ins[0] = p.q; ins[1] = p.k; ins[2] = p.v; ins[3] = p.dy;
      outs[0] = p.dq; outs[1] = p.dk; outs[2] = p.dv; nin = 4; nout = 3;
  }
  // layer mixer: q / k (inputs 0, 1) and dq / dk (outputs 0, 1) use the group strides
  auto kind = [](int i) { return (OP >= 4 && i < 2) ? i + 1 : 0; };
  for (int i = 0; i < nin; ++i)
    if (!map_dtensor(&maps.in[i], ins[i], p, 16 * Cfg<OP>::BPI, kind(i))) return cudaErrorNotSupported;
  // layer backward with shared groups: per-head dq / dk into the scratch (summed afterwards);
  // OP 8 sums the pairs in the kernel and stores the group tensors directly
  const bool scr[3] = {OP == 5 && p.hq > 1, OP == 5 && p.hk > 1, false};
  if (scr[0]) outs[0] = p.gq;
  if (scr[1]) outs[1] = p.gk;
  for (int i = 0; i < nout; ++i)
    if (!map_dtensor(&maps.out[i], outs[i], p, 16 * Cfg<OP>::BPI, scr[i] ? 3 : (OP == 5 || OP == 8) ? kind(i) : 0))
      return cudaErrorNotSupported;
  if (!map_decay(&maps.a, p.a, p, Cfg<OP>::BPI)) return cudaErrorNotSupported;

  constexpr int smem = smem_bytes<OP>();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) dev = -1;
  static std::atomic<bool> attr_set[kMaxDev];  // the attribute is per device (per context)
  if (dev < 0 || !attr_set[dev].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(swr_tc_kernel<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0) attr_set[dev].store(true, std::memory_order_release);
  }
  // work units of the split: items, or for HS > 1 super-items (a block of a group's heads)
  const int64_t total = p.B * p.H * ((p.nb + Cfg<OP>::BPI - 1) / Cfg<OP>::BPI) / Cfg<OP>::HS;
  const int grid = (int)std::min<int64_t>(sms, std::max<int64_t>(total, 1));
  constexpr int threads = (4 * Cfg<OP>::NG + Cfg<OP>::NPW + (Cfg<OP>::MIX ? 4 : 5)) * 32;
  Params q = p;
  Split sp;
  sp.weighted = 0;
  Balance* bal = dev >= 0 ? &g_balance[dev][OP] : nullptr;
  bool readback = false;
  q.epoch = 1;
  if (bal != nullptr && g_claims[dev].acquire(st, &q.epoch)) readback = bal->plan(q, sp, grid, sms, total, st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = SWR_PDL ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, swr_tc_kernel<OP>, maps, sp, q);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess && sp.weighted) {
    g_claims[dev].release(st, q.epoch);
    (void)cudaGetLastError();
  }
  if (e == cudaSuccess && readback) {
    bal->request(OP, sms, st);
    (void)cudaGetLastError();  // a failed readback only skips a table refresh; keep it out of the error state
  }
  return e;
}

}  // namespace tc

// layer backward with q and k shared by pairs of heads: group sums inside the kernel (Cfg<8>)
bool tc_layer_pairs(const Params& p) { return p.hq == 2 && p.hk == 2; }

bool tc_supported(int op, bool bf16, const Params& p) {
  if (!bf16 || p.D != 128) return false;
  // layer mixer backward with shared groups: needs the caller's per-head scratch
  if (op == 5 && !tc_layer_pairs(p) && ((p.hq != 1 && p.gq == nullptr) || (p.hk != 1 && p.gk == nullptr)))
    return false;
  if (tc::encoder() == nullptr) return false;
  auto a16 = [](const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  // decays must be TMA-addressable: heads contiguous, 16-byte token/batch strides
  if (p.sa_h != 1 || (p.sa_l * 2) % 16 != 0 || (p.sa_b * 2) % 16 != 0 || !a16(p.a)) return false;
  // 32-bit item / carry indexing in the kernel
  if (p.B * p.H > (1 << 22) || p.B * p.H * p.nb >= (int64_t(1) << 31) || p.L > (1 << 30)) return false;
  return true;
}

// dst[b, l, g, :] = sum over the group's hpg heads (in head order, fp32) of the per-head
// scratch src[b, l, g*hpg + j, :], rounded once to bf16; a thread per 8 channels
__global__ void __launch_bounds__(256) group_sum_bf16(const __nv_bfloat16* __restrict__ src,
                                                      __nv_bfloat16* __restrict__ dst, int64_t B, int64_t L,
                                                      int64_t H, int64_t D, int64_t hpg, int64_t s_b, int64_t s_l,
                                                      int64_t s_h) {
  const int64_t G = H / hpg, nv = D / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * L * G * nv) return;
  const int64_t cv = i % nv, g = (i / nv) % G, bl = i / (nv * G), b = bl / L, l = bl % L;
  const uint4* s4 = reinterpret_cast<const uint4*>(src + (bl * H + g * hpg) * D) + cv;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int64_t j = 0; j < hpg; ++j) {
    const uint4 w = __ldg(s4 + j * nv);
    const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc[2 * q] += __uint_as_float(x[q] << 16);
      acc[2 * q + 1] += __uint_as_float(x[q] & 0xffff0000u);
    }
  }
  uint4 o;
  o.x = tc::pack_bf2(acc[0], acc[1]);
  o.y = tc::pack_bf2(acc[2], acc[3]);
  o.z = tc::pack_bf2(acc[4], acc[5]);
  o.w = tc::pack_bf2(acc[6], acc[7]);
  *reinterpret_cast<uint4*>(dst + b * s_b + l * s_l + g * s_h + 8 * cv) = o;
}

static cudaError_t group_sum(const void* src, void* dst, const Params& p, int64_t hpg, int64_t sb, int64_t sl,
                             int64_t sh, cudaStream_t st) {
  const int64_t n = p.B * p.L * (p.H / hpg) * (p.D / 8);
  group_sum_bf16<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((const __nv_bfloat16*)src, (__nv_bfloat16*)dst, p.B,
                                                             p.L, p.H, p.D, hpg, sb, sl, sh);
  return cudaGetLastError();
}

cudaError_t launch_tc(int op, const Params& p, cudaStream_t st, int sms, int* launches) {
  *launches = 0;
  cudaError_t e;
  switch (op) {
    case 0: e = tc::launch_op<0>(p, st, sms); break;
    case 1: e = tc::launch_op<1>(p, st, sms); break;
    case 2: e = tc::launch_op<2>(p, st, sms); break;
    case 3: e = tc::launch_op<3>(p, st, sms); break;
    case 4: e = tc::launch_op<4>(p, st, sms); break;
    case 5: e = tc_layer_pairs(p) ? tc::launch_op<8>(p, st, sms) : tc::launch_op<5>(p, st, sms); break;
    case 6: e = tc::launch_op<6>(p, st, sms); break;
    default: e = tc::launch_op<7>(p, st, sms); break;
  }
  if (e == cudaSuccess) *launches = 1;
  if (op == 5 && tc_layer_pairs(p)) return e;
  if (e == cudaSuccess && op == 5 && p.hq > 1) {
    e = group_sum(p.gq, p.dq, p, p.hq, p.sq_b, p.sq_l, p.sq_h, st);
    if (e == cudaSuccess) ++*launches;
  }
  if (e == cudaSuccess && op == 5 && p.hk > 1) {
    e = group_sum(p.gk, p.dk, p, p.hk, p.sk_b, p.sk_l, p.sk_h, st);
    if (e == cudaSuccess) ++*launches;
  }
  return e;
}

}  // namespace swr
