// swr_api.cu -- the C ABI of libswr.so (declared in include/swr.h): argument
// validation, kernel-family dispatch, launch accounting.  No allocation, no
// host synchronisation, no torch types.
#include <atomic>
#include <cstdio>
#include <cstring>

#include "../../include/swr.h"
#include "swr_common.cuh"

namespace swr {
cudaError_t launch_ffma(int op, bool bf16, const Params& p, cudaStream_t st, int sms);
// tensor-core family (swr_tc.cu); returns cudaErrorNotSupported when the call
// is outside its envelope so the caller can fall back to FFMA.
cudaError_t launch_tc(int op, const Params& p, cudaStream_t st, int sms, int* launches);
bool tc_supported(int op, bool bf16, const Params& p);
cudaError_t launch_decode(bool mix, bool bf16, const DecParams& p, cudaStream_t st);
cudaError_t launch_exact(bool bf16, Params p, void* workspace, cudaStream_t st, int sms);
cudaError_t launch_exact_lb(bool bf16, Params p, void* workspace, cudaStream_t st);
cudaError_t launch_exact_carriers(bool bf16, Params p, void* workspace, cudaStream_t st, const float** carriers,
                                  bool stashed);
void exact_stash(const Params& p, void* workspace, float** V, float** C);
cudaError_t launch_exact_bwd(bool bf16, Params p, void* workspace, cudaStream_t st, int sms);
cudaError_t launch_uniform(bool bf16, Params p, int k, cudaStream_t st, int sms);
bool ffma_layer_supported(const Params& p);
}  // namespace swr

namespace {

std::atomic<int64_t> g_launches{0};        // diagnostics: kernels launched since load
thread_local int g_path = SWR_PATH_AUTO;    // per calling thread (swr_set_path)
thread_local int g_last_path = 0;           // family of this thread's last call
std::atomic<unsigned long long*> g_trace{nullptr};
std::atomic<int64_t> g_trace_n{0};
thread_local char g_cuda_err[256] = "";

constexpr int kMaxDev = 64;
std::atomic<int> g_sms[kMaxDev];   // 0 = unknown
std::atomic<int> g_major[kMaxDev];

swr_status cuda_fail(cudaError_t e) {
  snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return SWR_ERR_CUDA;
}

swr_status device_info(int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  if (dev < 0 || dev >= kMaxDev) return SWR_ERR_ARCH;
  int n = g_sms[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    int major = 0;
    e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return cuda_fail(e);
    g_major[dev].store(major);
    g_sms[dev].store(n);
  }
  if (g_major[dev].load() != 10) return SWR_ERR_ARCH;  // sm_100 (B200) only
  *sms = n;
  return SWR_OK;
}

bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

swr_status validate(const swr_shape& s, swr_dtype dt, const void* const* dtens, int nd,
                    const void* const* atens, int na, const void* const* carries, int nc) {
  if (dt != SWR_F32 && dt != SWR_BF16) return SWR_ERR_DTYPE;
  if (s.B < 0 || s.L < 0 || s.H < 0) return SWR_ERR_SHAPE;
  if (!(s.D == 16 || s.D == 32 || s.D == 64 || s.D == 128)) return SWR_ERR_SHAPE;
  const bool empty = s.B == 0 || s.L == 0 || s.H == 0;  // empty tensors may carry NULL pointers
  if (!empty) {
    for (int i = 0; i < nd; ++i)
      if (!dtens[i]) return SWR_ERR_NULL;
    for (int i = 0; i < na; ++i)
      if (!atens[i]) return SWR_ERR_NULL;
  }
  // grid limits: B is grid.z; H / (heads per CTA >= 4) is grid.y of the CUDA-core kernels
  if (s.B > 65535 || s.H > 65535 * 4) return SWR_ERR_SHAPE;
  const int64_t vec = (dt == SWR_BF16) ? 8 : 4;  // elements per 16 bytes
  if (s.sx_b < 0 || s.sx_l < 0 || s.sx_h < 0 || s.sa_b < 0 || s.sa_l < 0 || s.sa_h < 0)
    return SWR_ERR_STRIDE;
  if (s.sx_b % vec || s.sx_l % vec || s.sx_h % vec) return SWR_ERR_STRIDE;
  // a zero stride over a dimension of size > 1 makes output elements overlap
  // (several (b, l, h) lines would write the same addresses of x / du / da)
  if ((s.B > 1 && (s.sx_b == 0 || s.sa_b == 0)) || (s.L > 1 && (s.sx_l == 0 || s.sa_l == 0)) ||
      (s.H > 1 && (s.sx_h == 0 || s.sa_h == 0)))
    return SWR_ERR_STRIDE;
  for (int i = 0; i < nd; ++i)
    if (!aligned16(dtens[i])) return SWR_ERR_ALIGN;
  const uintptr_t esz = (dt == SWR_BF16) ? 2 : 4;
  for (int i = 0; i < na; ++i)
    if (reinterpret_cast<uintptr_t>(atens[i]) % esz) return SWR_ERR_ALIGN;
  for (int i = 0; i < nc; ++i)
    if (!aligned16(carries[i])) return SWR_ERR_ALIGN;
  return SWR_OK;
}

swr::Params make_params(const swr_shape& s) {
  swr::Params p;
  std::memset(&p, 0, sizeof(p));
  p.B = s.B;
  p.L = s.L;
  p.H = s.H;
  p.D = s.D;
  p.sx_b = s.sx_b;
  p.sx_l = s.sx_l;
  p.sx_h = s.sx_h;
  p.sa_b = s.sa_b;
  p.sa_l = s.sa_l;
  p.sa_h = s.sa_h;
  p.nb = (s.L + swr::kEll - 1) / swr::kEll;
  p.hq = p.hk = 1;
  p.sq_b = p.sk_b = s.sx_b;
  p.sq_l = p.sk_l = s.sx_l;
  p.sq_h = p.sk_h = s.sx_h;
  p.trace = g_trace.load();
  p.trace_n = g_trace_n.load();
  return p;
}

// Empty problem: zero-fill the fp32 carries the caller asked for.
swr_status empty_call(const swr_shape& s, float* carry_out, float* mu_out, cudaStream_t st) {
  const size_t bytes = sizeof(float) * (size_t)(s.B * s.H * s.D);
  if (bytes == 0) return SWR_OK;
  if (carry_out) {
    cudaError_t e = cudaMemsetAsync(carry_out, 0, bytes, st);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  if (mu_out) {
    cudaError_t e = cudaMemsetAsync(mu_out, 0, bytes, st);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  return SWR_OK;
}

swr_status dispatch(int op, swr_dtype dt, const swr::Params& p, cudaStream_t st) {
  int sms = 0;
  swr_status stt = device_info(&sms);
  if (stt != SWR_OK) return stt;
  const bool bf16 = dt == SWR_BF16;
  const int path = g_path;
  const bool tc_ok = swr::tc_supported(op, bf16, p);
  if (path == SWR_PATH_TC && !tc_ok) return SWR_ERR_UNSUPPORTED;  // forced, no silent fallback
  if (path != SWR_PATH_FFMA && tc_ok) {
    int launches = 0;
    cudaError_t e = swr::launch_tc(op, p, st, sms, &launches);
    if (e == cudaSuccess) {
      g_launches += launches;
      g_last_path = SWR_PATH_TC;
      return SWR_OK;
    }
    if (e != cudaErrorNotSupported || path == SWR_PATH_TC) return cuda_fail(e);
  }
  if (op == 5 && !swr::ffma_layer_supported(p)) return SWR_ERR_UNSUPPORTED;
  cudaError_t e = swr::launch_ffma(op, bf16, p, st, sms);
  if (e != cudaSuccess) return cuda_fail(e);
  g_launches += 1;
  g_last_path = SWR_PATH_FFMA;
  return SWR_OK;
}

}  // namespace

extern "C" {

swr_status swr_fwd(const void* u, const void* a, void* x, const float* carry_in, float* carry_out,
                   swr_shape s, swr_dtype dt, void* stream) {
  const void* dt_[] = {u, x};
  const void* at_[] = {a};
  const void* ct_[] = {carry_in, carry_out};
  swr_status st = validate(s, dt, dt_, 2, at_, 1, ct_, 2);
  if (st != SWR_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (s.B == 0 || s.H == 0 || s.L == 0) return empty_call(s, carry_out, nullptr, cs);
  swr::Params p = make_params(s);
  p.u = u;
  p.a = a;
  p.x = x;
  p.carry_in = carry_in;
  p.carry_out = carry_out;
  return dispatch(0, dt, p, cs);
}

swr_status swr_bwd(const void* u, const void* a, const void* dx, void* du, void* da,
                   const float* carry_in, const float* mu_in, float* mu_out, swr_shape s,
                   swr_dtype dt, void* stream) {
  const void* dt_[] = {u, dx, du};
  const void* at_[] = {a, da};
  const void* ct_[] = {carry_in, mu_in, mu_out};
  swr_status st = validate(s, dt, dt_, 3, at_, 2, ct_, 3);
  if (st != SWR_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (s.B == 0 || s.H == 0 || s.L == 0) return empty_call(s, nullptr, mu_out, cs);
  swr::Params p = make_params(s);
  p.u = u;
  p.a = a;
  p.dx = dx;
  p.du = du;
  p.da = da;
  p.carry_in = carry_in;
  p.mu_in = mu_in;
  p.mu_out = mu_out;
  return dispatch(1, dt, p, cs);
}

swr_status phalanx_mix(const void* q, const void* k, const void* v, const void* a, void* y,
                       const float* carry_in, float* carry_out, swr_shape s, swr_dtype dt,
                       void* stream) {
  const void* dt_[] = {q, k, v, y};
  const void* at_[] = {a};
  const void* ct_[] = {carry_in, carry_out};
  swr_status st = validate(s, dt, dt_, 4, at_, 1, ct_, 2);
  if (st != SWR_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (s.B == 0 || s.H == 0 || s.L == 0) return empty_call(s, carry_out, nullptr, cs);
  swr::Params p = make_params(s);
  p.q = q;
  p.k = k;
  p.v = v;
  p.a = a;
  p.y = y;
  p.carry_in = carry_in;
  p.carry_out = carry_out;
  return dispatch(2, dt, p, cs);
}

swr_status phalanx_mix_bwd(const void* q, const void* k, const void* v, const void* a,
                           const void* dy, void* dq, void* dk, void* dv, void* da,
                           const float* carry_in, const float* mu_in, float* mu_out,
                           swr_shape s, swr_dtype dt, void* stream) {
  const void* dt_[] = {q, k, v, dy, dq, dk, dv};
  const void* at_[] = {a, da};
  const void* ct_[] = {carry_in, mu_in, mu_out};
  swr_status st = validate(s, dt, dt_, 7, at_, 2, ct_, 3);
  if (st != SWR_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (s.B == 0 || s.H == 0 || s.L == 0) return empty_call(s, nullptr, mu_out, cs);
  swr::Params p = make_params(s);
  p.q = q;
  p.k = k;
  p.v = v;
  p.a = a;
  p.dy = dy;
  p.dq = dq;
  p.dk = dk;
  p.dv = dv;
  p.da = da;
  p.carry_in = carry_in;
  p.mu_in = mu_in;
  p.mu_out = mu_out;
  return dispatch(3, dt, p, cs);
}

}  // extern "C"

namespace {
// the group description of a layer call: groups divide H; q / k group tensors with
// D contiguous, 16-byte strides, no zero stride over a dimension of size > 1
swr_status validate_layer(const swr_shape& s, const swr_layer& g, swr_dtype dt, const void* const* qt, int nq,
                          const void* const* kt, int nk) {
  if (g.Gq <= 0 || g.Gk <= 0 || (s.H > 0 && (s.H % g.Gq || s.H % g.Gk))) return SWR_ERR_SHAPE;
  const int64_t vec = (dt == SWR_BF16) ? 8 : 4;
  auto strides_ok = [&](int64_t sb, int64_t sl, int64_t sh, int64_t G) {
    if (sb < 0 || sl < 0 || sh < 0 || sb % vec || sl % vec || sh % vec) return false;
    return !((s.B > 1 && sb == 0) || (s.L > 1 && sl == 0) || (G > 1 && sh == 0));
  };
  if (!strides_ok(g.sq_b, g.sq_l, g.sq_h, g.Gq) || !strides_ok(g.sk_b, g.sk_l, g.sk_h, g.Gk)) return SWR_ERR_STRIDE;
  const bool empty = s.B == 0 || s.L == 0 || s.H == 0;
  for (int i = 0; i < nq; ++i) {
    if (!empty && !qt[i]) return SWR_ERR_NULL;
    if (!aligned16(qt[i])) return SWR_ERR_ALIGN;
  }
  for (int i = 0; i < nk; ++i) {
    if (!empty && !kt[i]) return SWR_ERR_NULL;
    if (!aligned16(kt[i])) return SWR_ERR_ALIGN;
  }
  return SWR_OK;
}

void set_layer(swr::Params& p, const swr_shape& s, const swr_layer& g) {
  p.logit_a = g.logit_a != 0;
  p.logit_k = g.logit_k != 0;
  p.hq = s.H / g.Gq;
  p.hk = s.H / g.Gk;
  p.sq_b = g.sq_b;
  p.sq_l = g.sq_l;
  p.sq_h = g.sq_h;
  p.sk_b = g.sk_b;
  p.sk_l = g.sk_l;
  p.sk_h = g.sk_h;
}
}  // namespace

extern "C" {

int64_t phalanx_layer_workspace_bytes(swr_shape s, swr_layer g, swr_dtype dt) {
  if (dt != SWR_BF16 || s.D != 128 || s.B <= 0 || s.L <= 0 || s.H <= 0 || g.Gq <= 0 || g.Gk <= 0) return 0;
  if (s.H % g.Gq || s.H % g.Gk) return 0;
  if (s.H / g.Gq == 2 && s.H / g.Gk == 2) return 0;  // pairs of heads: group sums in the kernel
  const int64_t per = s.B * s.L * s.H * s.D * 2;
  return (g.Gq < s.H ? per : 0) + (g.Gk < s.H ? per : 0);
}

swr_status phalanx_layer_mix(const void* q, const void* zk, const void* v, const void* za, void* y,
                             const float* carry_in, float* carry_out, swr_shape s, swr_layer g, swr_dtype dt,
                             void* stream) {
  const void* dt_[] = {v, y};
  const void* at_[] = {za};
  const void* ct_[] = {carry_in, carry_out};
  swr_status st = validate(s, dt, dt_, 2, at_, 1, ct_, 2);
  if (st != SWR_OK) return st;
  const void* qt_[] = {q};
  const void* kt_[] = {zk};
  st = validate_layer(s, g, dt, qt_, 1, kt_, 1);
  if (st != SWR_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (s.B == 0 || s.H == 0 || s.L == 0) return empty_call(s, carry_out, nullptr, cs);
  swr::Params p = make_params(s);
  set_layer(p, s, g);
  p.q = q;
  p.k = zk;
  p.v = v;
  p.a = za;
  p.y = y;
  p.carry_in = carry_in;
  p.carry_out = carry_out;
  return dispatch(4, dt, p, cs);
}

swr_status phalanx_layer_mix_bwd(const void* q, const void* zk, const void* v, const void* za, const void* dy,
                                 void* dq, void* dzk, void* dv, void* dza, const float* carry_in,
                                 const float* mu_in, float* mu_out, swr_shape s, swr_layer g, swr_dtype dt,
                                 void* stream) {
  const void* dt_[] = {v, dy, dv};
  const void* at_[] = {za, dza};
  const void* ct_[] = {carry_in, mu_in, mu_out};
  swr_status st = validate(s, dt, dt_, 3, at_, 2, ct_, 3);
  if (st != SWR_OK) return st;
  const void* qt_[] = {q, dq};
  const void* kt_[] = {zk, dzk};
  st = validate_layer(s, g, dt, qt_, 2, kt_, 2);
  if (st != SWR_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (s.B == 0 || s.H == 0 || s.L == 0) return empty_call(s, nullptr, mu_out, cs);
  swr::Params p = make_params(s);
  set_layer(p, s, g);
  const int64_t need = phalanx_layer_workspace_bytes(s, g, dt);
  if (need > 0 && g.workspace != nullptr && g.workspace_bytes >= need) {
    if (!aligned16(g.workspace)) return SWR_ERR_ALIGN;
    const int64_t per = s.B * s.L * s.H * s.D;  // bf16 elements of one per-head scratch
    uint8_t* w = reinterpret_cast<uint8_t*>(g.workspace);
    if (p.hq > 1) {
      p.gq = w;
      w += per * 2;
    }
    if (p.hk > 1) p.gk = w;
  }
  p.q = q;
  p.k = zk;
  p.v = v;
  p.a = za;
  p.dy = dy;
  p.dq = dq;
  p.dk = dzk;
  p.dv = dv;
  p.da = dza;
  p.carry_in = carry_in;
  p.mu_in = mu_in;
  p.mu_out = mu_out;
  return dispatch(5, dt, p, cs);
}

}  // extern "C"

namespace {
swr_status decode_call(bool mix, const void* u, const void* vv, const void* q, const void* a, void* x,
                       float* w_state, float* v_state, float* g_state, int64_t pos, swr_shape s,
                       swr_dtype dt, void* stream) {
  if (s.L != 1 || pos < 0) return SWR_ERR_SHAPE;
  s.sx_l = 0;  // one token: the sequence strides are not used
  s.sa_l = 0;
  const void* dt_[] = {u, x, vv, q};
  const void* at_[] = {a};
  const void* ct_[] = {w_state, v_state};
  swr_status st = validate(s, dt, dt_, mix ? 4 : 2, at_, 1, ct_, 2);
  if (st != SWR_OK) return st;
  if (s.B == 0 || s.H == 0) return SWR_OK;
  if (!w_state || !v_state || !g_state) return SWR_ERR_NULL;
  if (reinterpret_cast<uintptr_t>(g_state) % 4) return SWR_ERR_ALIGN;
  int sms = 0;
  st = device_info(&sms);
  if (st != SWR_OK) return st;
  swr::DecParams p;
  std::memset(&p, 0, sizeof(p));
  p.u = u;
  p.v = vv;
  p.q = q;
  p.a = a;
  p.x = x;
  p.w = w_state;
  p.vc = v_state;
  p.g = g_state;
  p.B = s.B;
  p.H = s.H;
  p.D = s.D;
  p.sx_b = s.sx_b;
  p.sx_h = s.sx_h;
  p.sa_b = s.sa_b;
  p.sa_h = s.sa_h;
  p.pos = pos;
  cudaError_t e = swr::launch_decode(mix, dt == SWR_BF16, p, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  g_launches += 1;
  g_last_path = SWR_PATH_FFMA;
  return SWR_OK;
}
}  // namespace

extern "C" {

swr_status swr_decode_step(const void* u, const void* a, void* x, float* w_state, float* v_state,
                           float* g_state, int64_t pos, swr_shape s, swr_dtype dt, void* stream) {
  return decode_call(false, u, nullptr, nullptr, a, x, w_state, v_state, g_state, pos, s, dt, stream);
}

swr_status phalanx_mix_decode_step(const void* q, const void* k, const void* v, const void* a, void* y,
                                   float* w_state, float* v_state, float* g_state, int64_t pos,
                                   swr_shape s, swr_dtype dt, void* stream) {
  return decode_call(true, k, v, q, a, y, w_state, v_state, g_state, pos, s, dt, stream);
}

int64_t swr_exact_workspace_bytes(swr_shape s) {
  if (s.B <= 0 || s.H <= 0 || s.L <= 0 || s.D <= 0) return 0;
  const int64_t nb = (s.L + swr::kEll - 1) / swr::kEll;
  return (int64_t)sizeof(float) * (s.B * s.H * nb * s.D + (s.B * s.H * nb + 3) / 4 * 4);
}

swr_status swr_exact_fwd(const void* u, const void* a, void* x, const float* carry_in, float* carry_out,
                         void* workspace, int64_t workspace_bytes, swr_shape s, swr_dtype dt,
                         void* stream) {
  const void* dt_[] = {u, x};
  const void* at_[] = {a};
  const void* ct_[] = {carry_in, carry_out, workspace};
  swr_status st = validate(s, dt, dt_, 2, at_, 1, ct_, 3);
  if (st != SWR_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (s.B == 0 || s.H == 0 || s.L == 0) return empty_call(s, carry_out, nullptr, cs);
  if (!workspace) return SWR_ERR_NULL;
  if (workspace_bytes < 2 * swr_exact_workspace_bytes(s)) return SWR_ERR_SHAPE;
  int sms = 0;
  st = device_info(&sms);
  if (st != SWR_OK) return st;
  swr::Params p = make_params(s);
  p.u = u;
  p.a = a;
  p.x = x;
  p.carry_in = carry_in;
  p.carry_out = carry_out;
#ifndef SWR_EXACT_3STAGE  // 1: the round-1 three-launch forward (local, carrier chain, output)
  cudaError_t e;
  int launches = 1;
  const bool bf16 = dt == SWR_BF16;
  if (g_path != SWR_PATH_FFMA && swr::tc_supported(6, bf16, p)) {
    // tensor cores: the look-back scan's per-block carriers, then the B2P forward's
    // Pass I with the exact carrier (swr_tc.cu Cfg<6>)
    // pass 1 (tensor cores): every block's local end state v_t and decay product c_t;
    // the look-back scan over them; pass 2 (tensor cores): x with the exact carriers
    float *V = nullptr, *C = nullptr;
    swr::exact_stash(p, workspace, &V, &C);
    swr::Params q1 = p;
    q1.ex_S = V;
    q1.ex_C = C;
    q1.carry_out = nullptr;
    int t1 = 0, t2 = 0;
    e = swr::launch_tc(7, q1, cs, sms, &t1);
    const float* carriers = nullptr;
    if (e == cudaSuccess) e = swr::launch_exact_carriers(bf16, p, workspace, cs, &carriers, true);
    if (e == cudaSuccess) {
      swr::Params q = p;
      q.ex_S = carriers;
      q.carry_out = nullptr;  // written by the scan (the exact final state)
      e = swr::launch_tc(6, q, cs, sms, &t2);
    }
    launches = t1 + 1 + t2;
    g_last_path = SWR_PATH_TC;
  } else {
    if (g_path == SWR_PATH_TC) return SWR_ERR_UNSUPPORTED;
    e = swr::launch_exact_lb(bf16, p, workspace, cs);
    g_last_path = SWR_PATH_FFMA;
  }
#else
  cudaError_t e = swr::launch_exact(dt == SWR_BF16, p, workspace, cs, sms);
  const int launches = 3;
  g_last_path = SWR_PATH_FFMA;
#endif
  if (e != cudaSuccess) return cuda_fail(e);
  g_launches += launches;
  return SWR_OK;
}

swr_status swr_exact_bwd(const void* u, const void* a, const void* dx, void* du, void* da,
                         const float* carry_in, const float* mu_in, float* mu_out, void* workspace,
                         int64_t workspace_bytes, swr_shape s, swr_dtype dt, void* stream) {
  const void* dt_[] = {u, dx, du};
  const void* at_[] = {a, da};
  const void* ct_[] = {carry_in, mu_in, mu_out, workspace};
  swr_status st = validate(s, dt, dt_, 3, at_, 2, ct_, 4);
  if (st != SWR_OK) return st;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (s.B == 0 || s.H == 0 || s.L == 0) return empty_call(s, nullptr, mu_out, cs);
  if (!workspace) return SWR_ERR_NULL;
  if (workspace_bytes < 3 * swr_exact_workspace_bytes(s)) return SWR_ERR_SHAPE;
  int sms = 0;
  st = device_info(&sms);
  if (st != SWR_OK) return st;
  swr::Params p = make_params(s);
  p.u = u;
  p.a = a;
  p.dx = dx;
  p.du = du;
  p.da = da;
  p.carry_in = carry_in;
  p.mu_in = mu_in;
  p.mu_out = mu_out;
  cudaError_t e = swr::launch_exact_bwd(dt == SWR_BF16, p, workspace, cs, sms);
  if (e != cudaSuccess) return cuda_fail(e);
#ifndef SWR_EXACT_3STAGE
  g_launches += (p.nb >= 1024) ? 3 : 5;  // launch_exact_bwd: look-back scans from 1024 blocks on
#else
  g_launches += 5;
#endif
  g_last_path = SWR_PATH_FFMA;
  return SWR_OK;
}

swr_status swr_uniform_fwd(const void* u, const void* a, void* x, int k, swr_shape s, swr_dtype dt,
                           void* stream) {
  const void* dt_[] = {u, x};
  const void* at_[] = {a};
  swr_status st = validate(s, dt, dt_, 2, at_, 1, nullptr, 0);
  if (st != SWR_OK) return st;
  if (k < 1 || k > 32 || (k & (k - 1)) != 0) return SWR_ERR_SHAPE;
  if (s.B == 0 || s.H == 0 || s.L == 0) return SWR_OK;
  int sms = 0;
  st = device_info(&sms);
  if (st != SWR_OK) return st;
  swr::Params p = make_params(s);
  p.u = u;
  p.a = a;
  p.x = x;
  cudaError_t e = swr::launch_uniform(dt == SWR_BF16, p, k, reinterpret_cast<cudaStream_t>(stream), sms);
  if (e != cudaSuccess) return cuda_fail(e);
  g_launches += 1;
  g_last_path = SWR_PATH_FFMA;
  return SWR_OK;
}

const char* swr_strerror(swr_status st) {
  switch (st) {
    case SWR_OK: return "SWR_OK";
    case SWR_ERR_NULL: return "SWR_ERR_NULL: a required pointer is NULL";
    case SWR_ERR_SHAPE: return "SWR_ERR_SHAPE: B/L/H < 0 or D not in {16,32,64,128}";
    case SWR_ERR_STRIDE: return "SWR_ERR_STRIDE: negative stride or d-tensor stride not a multiple of 16 bytes";
    case SWR_ERR_ALIGN: return "SWR_ERR_ALIGN: pointer misaligned (16 B for d-tensors/carries, element size for decays)";
    case SWR_ERR_DTYPE: return "SWR_ERR_DTYPE: unknown dtype";
    case SWR_ERR_CUDA: return "SWR_ERR_CUDA: CUDA error (see swr_last_cuda_error)";
    case SWR_ERR_ARCH: return "SWR_ERR_ARCH: current device is not sm_100 (B200)";
    case SWR_ERR_UNSUPPORTED: return "SWR_ERR_UNSUPPORTED: SWR_PATH_TC forced for a call outside the tensor-core envelope (bf16, D = 128, TMA-addressable decays), or a layer backward whose head groups do not fit one CTA";
  }
  return "unknown swr_status";
}

const char* swr_last_cuda_error(void) { return g_cuda_err; }

swr_path swr_set_path(swr_path p) {
  const int prev = g_path;
  g_path = (int)p;
  return (swr_path)prev;
}

int64_t swr_launch_count(void) { return g_launches.load(); }

int swr_last_path(void) { return g_last_path; }

void swr_set_trace(unsigned long long* buf, int64_t n) {
  g_trace_n.store(buf ? n : 0);
  g_trace.store(buf);
}

}  // extern "C"
