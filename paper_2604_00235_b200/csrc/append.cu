// K0 — KV append with in-kernel RoPE, and the step's rotated queries.
//
// Reference: engine.py:434-437 (rotate k_pre[j] at position m, append to the
// store), kvstore.py:105-119 (single rounding through the storage dtype),
// attention.py:212-232 (interleaved pairs, angle t*omega_j in float64) and
// engine.py:460 (q_rot = R_m q_pre[h]).  The position m and the angles are
// shared by the key and the g queries of one kv head, so one CTA per
// (request, kv head) computes each sin/cos once in fp64 and rotates all of
// them.  Rotated queries go to the workspace in the math dtype.
#include "common.cuh"

namespace mac {

template <int MODE>
__global__ void __launch_bounds__(256) append_rope_kernel(MacDecodeParams p, int32_t* __restrict__ mpos,
                                                          typename Traits<MODE>::acc_t* __restrict__ qrot,
                                                          int rotate_only, int plan) {
  using kv_t = typename Traits<MODE>::kv_t;
  using acc_t = typename Traits<MODE>::acc_t;
  const int b = blockIdx.x / p.n_kv_heads;
  const int kvh = blockIdx.x % p.n_kv_heads;
  const int g = p.n_q_heads / p.n_kv_heads;
  const int d = p.head_dim, dv = p.head_dim_v, half = d / 2;
  // append: the step's token goes to m = seq_lens + 1; rotate_only: attend at m = seq_lens
  const int m = p.seq_lens[b] + (rotate_only ? 0 : 1);
  const int t_local = m - p.kv_offset;        // position inside this shard's cache
  if (threadIdx.x == 0) mpos[b] = m;
  bool store_kv = !rotate_only && t_local >= 1 && (p.kv_limit <= 0 || t_local <= p.kv_limit);
  if (store_kv && !kv_fits(p.pages_per_seq, t_local, p.page_size)) {
    store_kv = false;
    if (threadIdx.x == 0) atomicOr(ws_ptr<unsigned>(p, workspace_layout(p).ctr_off) + 2, 1u);
  }
  int64_t row = 0;
  if (store_kv) row = kv_row(p.page_table, p.pages_per_seq, b, t_local, p.page_size, p.n_kv_heads, kvh);
  kv_t* kc = static_cast<kv_t*>(p.k_cache);
  kv_t* vc = static_cast<kv_t*>(p.v_cache);
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    double s, c;
    sincos((double)m * p.rope_freqs[j], &s, &c);
    if (store_kv) {
      int64_t ki = ((int64_t)b * p.n_kv_heads + kvh) * d + 2 * j;
      double x0 = load_in(p.k_pre, ki, p.in_dtype), x1 = load_in(p.k_pre, ki + 1, p.in_dtype);
      kc[row * d + 2 * j] = from_f64<kv_t>(x0 * c - x1 * s);
      kc[row * d + 2 * j + 1] = from_f64<kv_t>(x0 * s + x1 * c);
    }
    for (int hl = 0; hl < g; ++hl) {
      int h = kvh * g + hl;
      int64_t qi = ((int64_t)b * p.n_q_heads + h) * d + 2 * j;
      double x0 = load_in(p.q_pre, qi, p.in_dtype), x1 = load_in(p.q_pre, qi + 1, p.in_dtype);
      qrot[qi] = (acc_t)(x0 * c - x1 * s);
      qrot[qi + 1] = (acc_t)(x0 * s + x1 * c);
    }
  }
  if (plan && threadIdx.x == 0) {  // full-attention modes: every head reads [1, m]
    int* lo = ws_ptr<int>(p, workspace_layout(p).lo_off);
    for (int hl = 0; hl < g; ++hl) lo[b * p.n_q_heads + kvh * g + hl] = 1;
    plan_group(p, b, kvh, m, 1);
  }
  if (store_kv) {
    for (int e = threadIdx.x; e < dv; e += blockDim.x) {
      int64_t vi = ((int64_t)b * p.n_kv_heads + kvh) * dv + e;
      vc[row * dv + e] = from_f64<kv_t>(load_in(p.v_in, vi, p.in_dtype));
    }
  }
}

template <int MODE>
cudaError_t launch_append(const MacDecodeParams& p, cudaStream_t st, int rotate_only, int plan) {
  Workspace w = workspace_layout(p);
  char* ws = static_cast<char*>(p.workspace);
  int threads = p.head_dim / 2;
  threads = threads < 32 ? 32 : (threads > 256 ? 256 : ((threads + 31) / 32) * 32);
  append_rope_kernel<MODE><<<p.batch * p.n_kv_heads, threads, 0, st>>>(
      p, reinterpret_cast<int32_t*>(ws + w.mpos_off),
      reinterpret_cast<typename Traits<MODE>::acc_t*>(ws + w.qrot_off), rotate_only, plan);
  return cudaGetLastError();
}

template cudaError_t launch_append<MAC_MODE_F32>(const MacDecodeParams&, cudaStream_t, int, int);
template cudaError_t launch_append<MAC_MODE_BF16>(const MacDecodeParams&, cudaStream_t, int, int);
template cudaError_t launch_append<MAC_MODE_F64>(const MacDecodeParams&, cudaStream_t, int, int);

}  // namespace mac
