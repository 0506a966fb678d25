// Bulk KV append for prefill: n tokens per request at positions seq_lens+1 ..
// seq_lens+n, RoPE'd in-kernel (fp64 angles), then seq_lens += n.
//
// Same per-token math as the decode append (engine.py:434-437, attention.py:
// 212-232, kvstore.py:105-119), for a prompt at once.  The reference has no
// prefill (its store fills one decode step at a time); this is the bulk half of
// the caller (engine.py BatchDecodeEngine.prefill) appends
// all but the last min(n, W) prompt tokens here and runs the last W as
// forced-miss decode steps, which leaves the exact all-miss ring state
// (summary AS[1, t-r] under q_t for every ring slot).
//
// One warp per (request, token, kv head): lanes split the d/2 rotation pairs
// and the d_v value elements.  Inputs are token-major [B, n, Hkv, d].
#include "common.cuh"

namespace mac {

template <int MODE>
__global__ void __launch_bounds__(256) prefill_kv_kernel(MacDecodeParams p, int n_tokens) {
  using kv_t = typename Traits<MODE>::kv_t;
  const int lane = threadIdx.x & 31;
  const int64_t row_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int Hkv = p.n_kv_heads, d = p.head_dim, dv = p.head_dim_v;
  if (row_id >= (int64_t)p.batch * n_tokens * Hkv) return;
  const int kvh = (int)(row_id % Hkv);
  const int t = (int)((row_id / Hkv) % n_tokens);
  const int b = (int)(row_id / ((int64_t)Hkv * n_tokens));
  const int pos = p.seq_lens[b] + 1 + t;
  const int local = pos - p.kv_offset;
  if (local < 1 || (p.kv_limit > 0 && local > p.kv_limit)) return;
  if (!kv_fits(p.pages_per_seq, local, p.page_size)) {
    if (lane == 0) atomicOr(ws_ptr<unsigned>(p, workspace_layout(p).ctr_off) + 2, 1u);
    return;
  }
  const int64_t row = kv_row(p.page_table, p.pages_per_seq, b, local, p.page_size, Hkv, kvh);
  const int64_t src = (((int64_t)b * n_tokens + t) * Hkv + kvh);
  kv_t* kc = static_cast<kv_t*>(p.k_cache);
  kv_t* vc = static_cast<kv_t*>(p.v_cache);
  for (int j = lane; j < d / 2; j += 32) {
    double s, c;
    sincos((double)pos * p.rope_freqs[j], &s, &c);
    const double x0 = load_in(p.k_pre, src * d + 2 * j, p.in_dtype);
    const double x1 = load_in(p.k_pre, src * d + 2 * j + 1, p.in_dtype);
    kc[row * d + 2 * j] = from_f64<kv_t>(x0 * c - x1 * s);
    kc[row * d + 2 * j + 1] = from_f64<kv_t>(x0 * s + x1 * c);
  }
  for (int e = lane; e < dv; e += 32) vc[row * dv + e] = from_f64<kv_t>(load_in(p.v_in, src * dv + e, p.in_dtype));
}

__global__ void advance_seq_lens_kernel(int32_t* seq_lens, int batch, int n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) seq_lens[b] += n;
}

template <int MODE>
cudaError_t launch_prefill_kv(const MacDecodeParams& p, int n_tokens, cudaStream_t st) {
  const int64_t rows = (int64_t)p.batch * n_tokens * p.n_kv_heads;
  const int64_t blocks = (rows + 7) / 8;
  if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
  prefill_kv_kernel<MODE><<<(unsigned)blocks, 256, 0, st>>>(p, n_tokens);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  advance_seq_lens_kernel<<<(p.batch + 127) / 128, 128, 0, st>>>(p.seq_lens, p.batch, n_tokens);
  return cudaGetLastError();
}

template cudaError_t launch_prefill_kv<MAC_MODE_F32>(const MacDecodeParams&, int, cudaStream_t);
template cudaError_t launch_prefill_kv<MAC_MODE_BF16>(const MacDecodeParams&, int, cudaStream_t);
template cudaError_t launch_prefill_kv<MAC_MODE_F64>(const MacDecodeParams&, int, cudaStream_t);

}  // namespace mac
