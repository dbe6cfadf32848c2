/*
 * swr.h -- C ABI of libswr.so: the Sliding Window Recurrence (SWR) operator of
 * arXiv 2512.13921 computed by the Block Two-Pass (B2P) algorithm on NVIDIA
 * B200 (sm_100a), forward and backward, and the Phalanx double-gated mixer
 * that wraps it.
 *
 * Citations are /root/reference/PAPER.md line numbers ("P:n") with the
 * section / equation / algorithm they fall in.
 *
 * ------------------------------------------------------------------------
 * The operation
 * ------------------------------------------------------------------------
 * Per (batch b, head h) the decays a in R^L are shared by the D channels of
 * the head ("the same set of recurrence coefficients is shared across
 * all d feature dimensions").  Tokens are grouped in blocks of ell = 16
 * (P:1486), aligned to token 0.  For block t with local decays a_t[0..15]:
 *
 *   L_t[i][j] = a_t[j+1] * ... * a_t[i]   (i >= j, else 0)     P:591-597, Alg. 3
 *   g_t[i]    = a_t[0] * ... * a_t[i]
 *   Pass I :  w_t = L_t u_t ,  v_t = w_t[15]                    Alg. 4
 *   Pass II:  x~_t = w_t + g_t (x) v_{t-1},  v_{-1} = carry_in or 0   Alg. 4
 *
 * i.e. x~ = L~ u with the jagged-window operator L~ = blockdiag(L_t) + G Z_b R
 * (Eq. truncated_factorization, Eq. block_bidiagonal).
 * Each block's output depends only on its own inputs and those of its
 * immediate predecessor.
 *
 * Phalanx mixer:  u^ = k (.) v ;  x~ = L~ u^ ;  y = q (.) x~ + v.
 *
 * Backward (the paper gives none; reading R12): the exact gradient
 * of the jagged operator, du = L~^T dx, da from reverse mode, and
 * mu_out = dLoss/dcarry_in.
 *
 * ------------------------------------------------------------------------
 * Conventions shared by every entry point
 * ------------------------------------------------------------------------
 * Pointers  : DEVICE pointers owned by the caller.  The library never
 *             allocates or frees device memory the caller sees.
 * State     : no state changes any result.  What the library does keep:
 *             - per calling thread: the kernel-family selector (swr_set_path)
 *               and the family of the thread's last call (swr_last_path);
 *             - a process-wide launch counter (swr_launch_count, diagnostics);
 *             - for the tensor-core kernels (bf16, D = 128), per device and op,
 *               a table of per-SM item rates that sizes each SM's share of the
 *               work (the "weighted split"): module-static device
 *               arrays, refreshed by an asynchronous device->pinned-host copy on
 *               a library-private stream that waits on the caller's stream and
 *               never blocks it, plus one event per claim slot (256 per device)
 *               marking when a launch's range claims are retired.  A launch
 *               whose claim slot is still in flight (more than 256 tensor-core
 *               launches queued) or that is being captured into a CUDA graph
 *               takes the uniform split instead.  Outputs are bit-identical for
 *               any split.
 *             Thread-safe.
 * Layout    : every "d-tensor" (u, x, dx, du, q, k, v, y, dy, dq, dk, dv) is
 *             [B, L, H, D] with D contiguous (stride 1) and element strides
 *             (sx_b, sx_l, sx_h); all d-tensors of one call share those strides.
 *             Decays a and their gradient da are [B, L, H] with strides
 *             (sa_b, sa_l, sa_h).  carry_in / carry_out / mu_in / mu_out are
 *             fp32 [B, H, D], contiguous.
 * Dtype     : one storage dtype (SWR_F32 or SWR_BF16) for every d-tensor, a and
 *             da; arithmetic is fp32 throughout ("accumulates ... using
 *             fp32"); each output is rounded once (RNE) to the storage dtype.
 * Length    : any L >= 0.  A partial last block behaves as if padded with
 *             u = 0 and a = 1 (causality makes the real outputs exact);
 *             carry_out is then the local state at token L-1.  L == 0 is a
 *             no-op that zero-fills carry_out / mu_out.
 * Asynchrony: every call enqueues on `stream` (a cudaStream_t; NULL = legacy
 *             default stream) and returns without synchronising.  Launch
 *             errors are returned as SWR_ERR_CUDA; faults inside a kernel
 *             surface at the caller's next synchronisation.
 * Graphs    : every call may be captured into a CUDA graph (any capture mode).
 *             A captured tensor-core launch neither reads nor refreshes the
 *             per-SM rate table and splits the work uniformly by CTA index, so
 *             replays are safe; outputs are bit-identical to eager calls
 *             (tests/test_graph.py).
 * Validation: done before any launch; on error nothing is launched.
 *   SWR_ERR_NULL   a required pointer is NULL
 *   SWR_ERR_SHAPE  B, L or H < 0, D not in {16, 32, 64, 128}, B > 65535 or
 *                  H > 262140 (grid limits)
 *   SWR_ERR_STRIDE a d-tensor stride is negative or not a multiple of 16 bytes
 *                  (8 bf16 / 4 fp32 elements), a decay stride is negative, or
 *                  any stride is 0 over a dimension of size > 1 (outputs would
 *                  overlap)
 *   SWR_ERR_ALIGN  a d-tensor or carry pointer is not 16-byte aligned, or a
 *                  decay pointer is not aligned to its element size
 *   SWR_ERR_DTYPE  unknown dtype
 *   SWR_ERR_CUDA   a CUDA launch/runtime error (see swr_last_cuda_error)
 *   SWR_ERR_ARCH   the current device is not sm_100 (B200)
 *   SWR_ERR_UNSUPPORTED  SWR_PATH_TC is selected and the call is outside the
 *                  tensor-core envelope (bf16, D = 128, heads contiguous and
 *                  16-byte token / batch strides in a) -- no silent fallback
 */
#ifndef SWR_H_
#define SWR_H_

#include <stdint.h>

#if defined(__GNUC__)
#define SWR_API __attribute__((visibility("default")))
#else
#define SWR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SWR_OK = 0,
  SWR_ERR_NULL = 1,
  SWR_ERR_SHAPE = 2,
  SWR_ERR_STRIDE = 3,
  SWR_ERR_ALIGN = 4,
  SWR_ERR_DTYPE = 5,
  SWR_ERR_CUDA = 6,
  SWR_ERR_ARCH = 7,
  SWR_ERR_UNSUPPORTED = 8
} swr_status;

typedef enum { SWR_F32 = 0, SWR_BF16 = 1 } swr_dtype;

/* Kernel family used by swr_fwd / swr_bwd / phalanx_mix / phalanx_mix_bwd
 * (per calling thread, default AUTO; the other entry points have one family).
 * SWR_PATH_FFMA: per-thread fp32 recurrences on CUDA cores (any dtype / D).
 * SWR_PATH_TC  : tcgen05 tensor-core Pass I with TMEM accumulators and
 *                TMA-staged tiles (bf16, D == 128 only; any other call returns
 *                SWR_ERR_UNSUPPORTED).
 * SWR_PATH_AUTO: the faster one for the call, as measured. */
typedef enum { SWR_PATH_AUTO = 0, SWR_PATH_FFMA = 1, SWR_PATH_TC = 2 } swr_path;

typedef struct {
  int64_t B, L, H, D;       /* batch, sequence length, heads, head dim (d = D/h of P:1555) */
  int64_t sx_b, sx_l, sx_h; /* element strides of every [B,L,H,D] d-tensor; D is contiguous */
  int64_t sa_b, sa_l, sa_h; /* element strides of the [B,L,H] decay tensor (and da)        */
} swr_shape;

/* Forward SWR: x = L~ u.
 *   u         [B,L,H,D] input (u^ of the mixer)               required
 *   a         [B,L,H]   decays a_i^eta                       required
 *   x         [B,L,H,D] output x~ (may not alias u)                   required
 *   carry_in  [B,H,D] fp32, nullable: carrier v_{-1} entering block 0 (the
 *             x_0 fold of P:116 for block 0; the segment checkpoint of P:1526).
 *             Only block 0 sees it.  NULL = 0.
 *   carry_out [B,H,D] fp32, nullable: local end state of the last block,
 *             v_b = w_b[15] -- the carry_in of the next segment. */
SWR_API swr_status swr_fwd(const void* u, const void* a, void* x, const float* carry_in,
                   float* carry_out, swr_shape s, swr_dtype dt, void* stream);

/* Backward SWR.  Given dx = dLoss/dx:
 *   du     [B,L,H,D] = L~^T dx (+ the mu_in term)                     required
 *   da     [B,L,H]   dLoss/da                                         required
 *   carry_in  same value given to swr_fwd (nullable = 0)
 *   mu_in  [B,H,D] fp32, nullable: dLoss/dcarry_out from the next segment
 *   mu_out [B,H,D] fp32, nullable: dLoss/dcarry_in = a[0] * lambda_0[0]
 * No buffer may alias another. */
SWR_API swr_status swr_bwd(const void* u, const void* a, const void* dx, void* du, void* da,
                   const float* carry_in, const float* mu_in, float* mu_out, swr_shape s,
                   swr_dtype dt, void* stream);

/* Phalanx mixer forward: y = q (.) SWR(k (.) v) + v.
 * q, k, v, a, y required; carries as in swr_fwd (for u^ = k (.) v). */
SWR_API swr_status phalanx_mix(const void* q, const void* k, const void* v, const void* a, void* y,
                       const float* carry_in, float* carry_out, swr_shape s, swr_dtype dt,
                       void* stream);

/* Phalanx mixer backward: dq = dy (.) x~, dk = du^ (.) v, dv = du^ (.) k + dy, da,
 * where du^ = SWR backward of G = dy (.) q.  x~ is recomputed, never stored.
 * q, k, v, a, dy, dq, dk, dv, da required; carries as in swr_bwd. */
SWR_API swr_status phalanx_mix_bwd(const void* q, const void* k, const void* v, const void* a,
                           const void* dy, void* dq, void* dk, void* dv, void* da,
                           const float* carry_in, const float* mu_in, float* mu_out,
                           swr_shape s, swr_dtype dt, void* stream);

/* ------------------------------------------------------------------------
 * The Phalanx layer around the mixer
 * ------------------------------------------------------------------------
 * The mixer fed directly by the featurization:
 *   a = sigma(za)   the recurrence coefficient, sigmoid-bounded
 *   k = sigma(zk)   the key-like gate
 * with q and k shared by groups of heads ("we apply group sharing separately to K
 * and Q projections, such that within each group, multiple heads share the same
 * gate parameters"; 8 groups): q is [B, L, Gq, D], zk is
 * [B, L, Gk, D], and head h reads group h / (H / Gq) of q and h / (H / Gk) of k
 * (contiguous head groups, R18).  Then, per head,
 *   y = q_g (.) SWR_a(k_g (.) v) + v
 * and the backward returns the gradients of the logits and of the group tensors:
 *   dza = da (.) a (1 - a),  dzk = (sum over the group's heads of du^ (.) v) (.) k (1 - k),
 *   dq  = sum over the group's heads of dy (.) x~,  dv = du^ (.) k + dy.
 * The sums over heads are formed in a fixed head order (deterministic).
 * sigma is evaluated in fp32 (e^-z by ex2, then an IEEE reciprocal). */
typedef struct {
  int64_t Gq, Gk;            /* groups of q and of k; each divides H (Gq = Gk = H: no sharing) */
  int64_t sq_b, sq_l, sq_h;  /* element strides of q and dq, [B, L, Gq, D], D contiguous      */
  int64_t sk_b, sk_l, sk_h;  /* element strides of zk and dzk, [B, L, Gk, D], D contiguous    */
  int32_t logit_a;           /* nonzero: za holds logits, a = sigma(za); else za is a itself  */
  int32_t logit_k;           /* nonzero: zk holds logits, k = sigma(zk); else zk is k itself  */
  void* workspace;           /* nullable device scratch for the tensor-core backward with     */
  int64_t workspace_bytes;   /* shared groups (phalanx_layer_workspace_bytes); unused forward */
} swr_layer;

/* Scratch the layer backward needs to run on the tensor cores when heads share q or k:
 * per-head dq / dk (bf16 [B, L, H, D] each, for the groups of q resp. k that are shared),
 * summed over each group by a second kernel in a fixed head order.  0 when no scratch is
 * needed -- no sharing, or q and k both shared by pairs of heads (H / Gq = H / Gk = 2,
 * the paper's 8 groups at H = 16: the kernel walks each pair together and sums in
 * registers) -- or the call is outside the tensor-core envelope; without it such a call
 * runs on the CUDA-core family (AUTO) or is refused (SWR_PATH_TC). */
SWR_API int64_t phalanx_layer_workspace_bytes(swr_shape s, swr_layer g, swr_dtype dt);

/* Layer mixer forward.  v, y [B,L,H,D] with the strides of s; za [B,L,H] with the
 * decay strides of s; q, zk as described by g; carries as in phalanx_mix.
 * Errors as above, plus SWR_ERR_SHAPE when Gq or Gk does not divide H and
 * SWR_ERR_STRIDE / SWR_ERR_ALIGN for the group tensors' strides / pointers. */
SWR_API swr_status phalanx_layer_mix(const void* q, const void* zk, const void* v, const void* za,
                             void* y, const float* carry_in, float* carry_out, swr_shape s,
                             swr_layer g, swr_dtype dt, void* stream);

/* Layer mixer backward.  dq [B,L,Gq,D] and dzk [B,L,Gk,D] with the strides of g
 * (the group sums), dv [B,L,H,D], dza [B,L,H]; carries as in phalanx_mix_bwd.
 * The tensor-core kernels (bf16, D = 128) take shared groups when g.workspace holds
 * phalanx_layer_workspace_bytes(s, g, dt) bytes (16-byte aligned; none for pairs of
 * heads); else the CUDA-core kernels form the group sums inside one CTA: H / Gq and
 * H / Gk must be powers of two and at most 256 / (D / 4) (64 at D = 16, 8 at D = 128),
 * else SWR_ERR_UNSUPPORTED.  All group sums run in a fixed head order (deterministic). */
SWR_API swr_status phalanx_layer_mix_bwd(const void* q, const void* zk, const void* v,
                                 const void* za, const void* dy, void* dq, void* dzk, void* dv,
                                 void* dza, const float* carry_in, const float* mu_in,
                                 float* mu_out, swr_shape s, swr_layer g, swr_dtype dt,
                                 void* stream);

/* Recurrence-mode decoding (the paper decodes Phalanx "in
 * recurrence mode"): one new token per (b, h).  The state is
 *   w_state [B,H,D] fp32  local state of the current block, w_t[i]
 *   v_state [B,H,D] fp32  carrier of the previous block, v_{t-1} = w_{t-1}[15]
 *   g_state [B,H]   fp32  decay product since the block start, g_t[i]
 * all contiguous and updated in place.  For the token at sequence position pos
 * (i = pos mod 16, the same for every (b, h)):
 *   i == 0:  v <- w,  g <- a,      w <- u        (L_t excludes a_t[0])
 *   else  :  g <- g a, w <- a w + u
 *   x = w + g v                                   (Pass II)
 * -- B2P's forward evaluated one token at a time: decoding a sequence from pos 0
 * gives bitwise the outputs of swr_fwd on the CUDA-core path.  Before pos 0 set
 * w_state to carry_in (or 0); v_state and g_state need no initialisation.
 * u, x [B,H,D] with element strides (s.sx_b, s.sx_h), D contiguous, 16-byte
 * aligned; a [B,H] with strides (s.sa_b, s.sa_h).  s.L must be 1 (s.sx_l and
 * s.sa_l are ignored); pos >= 0 (else SWR_ERR_SHAPE).  Other errors as above. */
SWR_API swr_status swr_decode_step(const void* u, const void* a, void* x, float* w_state,
                           float* v_state, float* g_state, int64_t pos, swr_shape s,
                           swr_dtype dt, void* stream);

/* Phalanx mixer decode step: u^ = k (.) v into the step above, y = q (.) x~ + v. */
SWR_API swr_status phalanx_mix_decode_step(const void* q, const void* k, const void* v,
                           const void* a, void* y, float* w_state, float* v_state,
                           float* g_state, int64_t pos, swr_shape s, swr_dtype dt,
                           void* stream);

/* Exact full-range recurrence: x_n = a_n x_{n-1} + u_n over
 * the whole sequence (Eq. 2.1, x_{-1} = carry_in) -- the operator B2P truncates --
 * computed as Alg. 2: per-block local solves give the carrier system
 * s_t = c_t s_{t-1} + v_t, resolved across CTAs by a decoupled look-back
 * over published chunk aggregates / inclusive prefixes.  bf16, D = 128 (the tensor-core
 * envelope): the scan writes every block's exact carrier, then the B2P forward's
 * tensor-core Pass I runs with s_{t-1} in place of v_{t-1} (two launches); otherwise
 * one CUDA-core pass re-runs each chunk from its entering state (one launch).  Plus a
 * memset of the look-back flags.  The last bits of x may differ between runs (the
 * look-back's summation order depends on timing); within the tolerances.
 *   u, a, x, carry_in as in swr_fwd; carry_out = x at token L-1 (the full state).
 *   workspace  device memory of >= 2 * swr_exact_workspace_bytes(s) bytes, 16-byte
 *              aligned, caller-owned scratch (no allocation here); too small ->
 *              SWR_ERR_SHAPE, NULL with a non-empty problem -> SWR_ERR_NULL. */
SWR_API int64_t swr_exact_workspace_bytes(swr_shape s);
SWR_API swr_status swr_exact_fwd(const void* u, const void* a, void* x, const float* carry_in,
                         float* carry_out, void* workspace, int64_t workspace_bytes,
                         swr_shape s, swr_dtype dt, void* stream);

/* Backward of swr_exact_fwd (reverse mode of Eq. 2.1): du_n = lambda_n with
 * lambda_n = dx_n + a_{n+1} lambda_{n+1}, da_n = sum_c lambda_n x_{n-1} (x_{-1} =
 * carry_in), mu_out = a_0 lambda_0 = dLoss/dcarry_in; mu_in = dLoss/dcarry_out enters
 * at token L-1.  Blockwise: per-block local solves give the forward carriers s_t and
 * the reverse carriers mu_{t-1} = a_t[0] (l_t[0] + r_t[0] mu_t), resolved by decoupled
 * look-back scans from 1024 blocks per line on (three launches) and by per-line serial
 * chains below (five launches); then a reconstruction pass forms du and da.
 * Workspace >= 3 * swr_exact_workspace_bytes(s).  Arguments otherwise as swr_bwd. */
SWR_API swr_status swr_exact_bwd(const void* u, const void* a, const void* dx, void* du, void* da,
                         const float* carry_in, const float* mu_in, float* mu_out,
                         void* workspace, int64_t workspace_bytes, swr_shape s, swr_dtype dt,
                         void* stream);

/* Uniform-window recurrence (Sec. uniform_window P:1104-1113,
 * Eq. banded_L): x = (I + AZ + ... + (AZ)^{k-1}) u, i.e. every token sees its k most
 * recent inputs, x_n = sum_{j<k} (a_{n-j+1} ... a_n) u_{n-j}, with no carry.  The
 * paper's "theoretical baseline" next to the jagged window.  k a power of two in
 * [1, 32] (else SWR_ERR_SHAPE); u, a, x as in swr_fwd.  CUDA cores, one launch. */
SWR_API swr_status swr_uniform_fwd(const void* u, const void* a, void* x, int k, swr_shape s,
                           swr_dtype dt, void* stream);

/* Human-readable name of a status code (static storage). */
SWR_API const char* swr_strerror(swr_status st);

/* Text of the last CUDA error seen by this thread (static storage, "" if none). */
SWR_API const char* swr_last_cuda_error(void);

/* Select the kernel family for calls made by this thread.  Returns the
 * thread's previous value. */
SWR_API swr_path swr_set_path(swr_path p);

/* Number of kernels this library has launched since load, all threads (for
 * bench.py's "gpu_launches"), and the family that served this thread's most
 * recent call (1 = FFMA, 2 = TC, 0 = none). */
SWR_API int64_t swr_launch_count(void);
SWR_API int swr_last_path(void);

/* Diagnostics (effective only in a library built with -DSWR_TRACE=1, e.g.
 * tools/build_var.sh trace -DSWR_TRACE=1; the product build compiles it out):
 * when `buf` (device memory, >= 16 * n + 4 * gridDim uint64) is non-NULL, the
 * tensor-core kernels of CTA 0 record a clock64 timestamp (SM cycles) per pipeline
 * event for each of their first n items (slot = 16 * item + event; events are
 * listed in paper_2512_13921_b200/csrc/swr_tc.cu), and every CTA its start/end
 * %globaltimer, SM id and range size at 16 * n + 4 * cta.  NULL disables it. */
SWR_API void swr_set_trace(unsigned long long* buf, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* SWR_H_ */
