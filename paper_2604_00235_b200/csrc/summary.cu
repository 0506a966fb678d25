// The reference's summary algebra and query matcher as standalone device calls — the public
// building blocks of `attnreuse` (attention.py:75-232, matching.py:141-175) over plain arrays
// instead of the engine's paged cache and slot-aligned rings:
//
//   mac_summarize     summarize / attend_full (attention.py:75-116, 182-189) for many query
//                     rows at once, each over its own key range [lo, hi] of a key set, the query
//                     optionally rotated at position t first — which also makes it the batched
//                     causal oracle_outputs (engine.py:542-572: row t over [1, t])
//   mac_remove_summaries  remove() down-date with its guards (attention.py:138-172)
//   mac_rope_rotate   rope_rotate (attention.py:212-232), per-row positions
//   mac_match_rows    match_query (matching.py:141-175) over rings with explicit positions
//
// All math is f64 like the reference (inputs f32 or f64, rounded copies of the reference's
// own storage), so these calls agree with it to f64 reduction-order roundoff.  The merge of
// summaries is mac_merge_partials (merge.cu).
#include "common.cuh"

namespace mac {

namespace {
template <typename T> __device__ __forceinline__ double ld(const void* p, int64_t i) {
  return (double)static_cast<const T*>(p)[i];
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

constexpr int SUM_WARPS = 8;
constexpr int SUM_MAX_DV = 256;  // acc elements per lane: d_v / 32 <= 8
}  // namespace

// one CTA per query row; each warp runs an online softmax over a strided subset of the row's
// keys (lanes split the dims), then the warps' (max, Z, S) merge in shared memory
template <typename T>
__global__ void __launch_bounds__(SUM_WARPS * 32) summarize_kernel(MacSummarizeParams p) {
  const int row = blockIdx.x;  // set * q_per_set + i
  const int set = row / p.q_per_set;
  const int kset = set / p.sets_per_kv;
  const int d = p.head_dim, dv = p.head_dim_v;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double qs[1024];
  __shared__ double wm[SUM_WARPS], wz[SUM_WARPS];
  __shared__ double ws[SUM_WARPS][SUM_MAX_DV];
  // the query, rotated at t (attention.py:212-232: pair j by t * freqs[j], fp64 angles)
  const int64_t qoff = (int64_t)row * d;
  const double t = p.rope_t ? (double)p.rope_t[row] : 0.0;
  for (int j = threadIdx.x; j < d / 2; j += blockDim.x) {
    const double x0 = ld<T>(p.q, qoff + 2 * j), x1 = ld<T>(p.q, qoff + 2 * j + 1);
    if (p.rope_t) {
      double s, c;
      sincos(t * p.rope_freqs[j], &s, &c);
      qs[2 * j] = x0 * c - x1 * s;
      qs[2 * j + 1] = x0 * s + x1 * c;
    } else {
      qs[2 * j] = x0;
      qs[2 * j + 1] = x1;
    }
  }
  __syncthreads();
  const int lo = p.lo ? p.lo[row] : 1;
  const int hi = p.hi ? p.hi[row] : p.n_keys;
  const double scale = 1.0 / sqrt((double)d);
  const int64_t kbase = (int64_t)kset * p.n_keys;
  double M = -CUDART_INF, Z = 0.0, S[SUM_MAX_DV / 32];
#pragma unroll
  for (int e = 0; e < SUM_MAX_DV / 32; ++e) S[e] = 0.0;
  for (int k = lo - 1 + warp; k < hi; k += SUM_WARPS) {
    double dot = 0.0;
    for (int j = lane; j < d; j += 32) dot += ld<T>(p.keys, (kbase + k) * d + j) * qs[j];
    const double l = warp_sum(dot) * scale;
    const double nm = fmax(M, l);
    const double a = exp(M - nm), w = exp(l - nm);  // M = -inf on the first key: a = 0
    Z = Z * a + w;
#pragma unroll
    for (int e = 0; e < SUM_MAX_DV / 32; ++e) {
      const int c = lane + 32 * e;
      if (c < dv) S[e] = S[e] * a + w * ld<T>(p.values, (kbase + k) * dv + c);
    }
    M = nm;
  }
  if (lane == 0) {
    wm[warp] = M;
    wz[warp] = Z;
  }
#pragma unroll
  for (int e = 0; e < SUM_MAX_DV / 32; ++e) {
    const int c = lane + 32 * e;
    if (c < dv) ws[warp][c] = S[e];
  }
  __syncthreads();
  double GM = -CUDART_INF;
  for (int w = 0; w < SUM_WARPS; ++w) GM = fmax(GM, wm[w]);
  double GZ = 0.0;
  for (int w = 0; w < SUM_WARPS; ++w)
    if (wm[w] != -CUDART_INF) GZ += wz[w] * exp(wm[w] - GM);
  for (int c = threadIdx.x; c < dv; c += blockDim.x) {
    double a = 0.0;
    for (int w = 0; w < SUM_WARPS; ++w)
      if (wm[w] != -CUDART_INF) a += ws[w][c] * exp(wm[w] - GM);
    p.out_acc[(int64_t)row * dv + c] = GZ > 0.0 ? a / GZ : 0.0;  // empty range: the empty summary
  }
  if (threadIdx.x == 0) p.out_lse[row] = GZ > 0.0 ? GM + log(GZ) : -CUDART_INF;
}

// remove(a, band) per row (attention.py:138-172); counts are checked by the caller, the mass
// guards here: status 0 ok, 1 cancellation (|diff| < eps), 2 mass exceeded (diff < -eps)
__global__ void remove_kernel(int n_rows, int dv, const double* a_acc, const double* a_lse, const double* b_acc,
                              const double* b_lse, double eps, double* out_acc, double* out_lse, int32_t* status) {
  const int row = blockIdx.x;
  const double al = a_lse[row], bl = b_lse[row];
  const double diff = al - bl;
  const int st = diff < -eps ? 2 : (diff < eps ? 1 : 0);
  const double lse = st ? -CUDART_INF : bl + log(expm1(diff));
  for (int c = threadIdx.x; c < dv; c += blockDim.x) {
    const int64_t i = (int64_t)row * dv + c;
    out_acc[i] = st ? 0.0 : a_acc[i] * exp(al - lse) - b_acc[i] * exp(bl - lse);
  }
  if (threadIdx.x == 0) {
    out_lse[row] = lse;
    status[row] = st;
  }
}

// rope_rotate (attention.py:212-232): row i rotated by t[i] (f64 angles)
__global__ void rope_rotate_kernel(int n_rows, int d, const double* x, const double* t, const double* freqs,
                                   double* out) {
  const int64_t n = (int64_t)n_rows * (d / 2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / (d / 2)), j = (int)(i % (d / 2));
    const double x0 = x[(int64_t)row * d + 2 * j], x1 = x[(int64_t)row * d + 2 * j + 1];
    double s, c;
    sincos(t[row] * freqs[j], &s, &c);
    out[(int64_t)row * d + 2 * j] = x0 * c - x1 * s;
    out[(int64_t)row * d + 2 * j + 1] = x0 * s + x1 * c;
  }
}

// match_query (matching.py:141-175) for one ring per CTA: sq = |q|^2 + |c|^2 - 2 q.c in f64
// with the ring's cached norms, clamped at 0, Δmax filter, optional post-RoPE frame change of
// the candidates (matching.py:129-138, 165-168), argmin with ties to the larger position,
// hit iff best < thr_sq strictly
__global__ void __launch_bounds__(256) match_rows_kernel(MacMatchRowsParams p) {
  const int s = blockIdx.x;
  const int d = p.head_dim;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double qs[1024];
  __shared__ double bd[32];
  __shared__ long long bp[32];
  __shared__ int ns[32];
  for (int j = threadIdx.x; j < d; j += blockDim.x) qs[j] = p.q[(int64_t)s * d + j];
  __syncthreads();
  double qq = 0.0;
  for (int j = lane; j < d; j += 32) qq += qs[j] * qs[j];
  qq = warp_sum(qq);  // float(q @ q)
  const int m = p.m[s], n = p.n_live[s];
  double best = CUDART_INF;
  long long bpos = -1;
  int scanned = 0;
  for (int i = warp; i < n; i += nw) {
    const long long pos = p.ring_pos[(int64_t)s * p.capacity + i];
    if (p.delta_max > 0 && (long long)m - pos > p.delta_max) continue;
    const double* c = p.ring_q + ((int64_t)s * p.capacity + i) * d;
    double dot = 0.0;
    if (p.post_rope) {  // R(pos - m) c, same pairing as rope_rotate
      const double delta = (double)(pos - m);
      for (int j = lane; j < d / 2; j += 32) {
        double sn, cs;
        sincos(delta * p.rope_freqs[j], &sn, &cs);
        const double c0 = c[2 * j], c1 = c[2 * j + 1];
        dot += (c0 * cs - c1 * sn) * qs[2 * j] + (c0 * sn + c1 * cs) * qs[2 * j + 1];
      }
    } else {
      for (int j = lane; j < d; j += 32) dot += c[j] * qs[j];
    }
    dot = warp_sum(dot);
    double sq = qq + p.ring_sqnorm[(int64_t)s * p.capacity + i] - 2.0 * dot;
    sq = sq < 0.0 ? 0.0 : sq;
    ++scanned;
    if (sq < best || (sq == best && pos > bpos)) {
      best = sq;
      bpos = pos;
    }
  }
  if (lane == 0) {
    bd[warp] = best;
    bp[warp] = bpos;
    ns[warp] = scanned;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double B = CUDART_INF;
    long long P = -1;
    int N = 0;
    for (int w = 0; w < nw; ++w) {
      N += ns[w];
      if (bp[w] >= 0 && (bd[w] < B || (bd[w] == B && bp[w] > P))) {
        B = bd[w];
        P = bp[w];
      }
    }
    const bool hit = N > 0 && B < p.thr_sq;
    p.out_hit[s] = hit;
    p.out_pos[s] = hit ? (int32_t)P : -1;
    p.out_dist[s] = N > 0 ? B : CUDART_INF;
    p.out_scanned[s] = N;
  }
}

}  // namespace mac

using namespace mac;

extern "C" int mac_summarize(const MacSummarizeParams* p, void* stream) {
  if (!p || !p->q || !p->keys || !p->values || !p->out_acc || !p->out_lse) return MAC_ERR_NULL;
  if (p->n_sets < 0 || p->q_per_set < 0 || p->n_keys < 0 || p->sets_per_kv < 1 || p->head_dim < 2 ||
      p->head_dim % 2 || p->head_dim > 1024 || p->head_dim_v < 1 || p->head_dim_v > SUM_MAX_DV)
    return MAC_ERR_SHAPE;
  if (p->rope_t && !p->rope_freqs) return MAC_ERR_NULL;
  const int rows = p->n_sets * p->q_per_set;
  if (rows == 0) return MAC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->dtype == MAC_DT_F64) summarize_kernel<double><<<rows, SUM_WARPS * 32, 0, st>>>(*p);
  else if (p->dtype == MAC_DT_F32) summarize_kernel<float><<<rows, SUM_WARPS * 32, 0, st>>>(*p);
  else return MAC_ERR_DTYPE;
  return (int)cudaGetLastError();
}

extern "C" int mac_remove_summaries(int32_t n_rows, int32_t head_dim_v, const double* a_acc, const double* a_lse,
                                    const double* band_acc, const double* band_lse, double eps_cancel,
                                    double* out_acc, double* out_lse, int32_t* status, void* stream) {
  if (!a_acc || !a_lse || !band_acc || !band_lse || !out_acc || !out_lse || !status) return MAC_ERR_NULL;
  if (n_rows < 0 || head_dim_v < 1) return MAC_ERR_SHAPE;
  if (n_rows == 0) return MAC_OK;
  remove_kernel<<<n_rows, 128, 0, static_cast<cudaStream_t>(stream)>>>(n_rows, head_dim_v, a_acc, a_lse, band_acc,
                                                                      band_lse, eps_cancel, out_acc, out_lse, status);
  return (int)cudaGetLastError();
}

extern "C" int mac_rope_rotate(int32_t n_rows, int32_t head_dim, const double* x, const double* t,
                               const double* rope_freqs, double* out, void* stream) {
  if (!x || !t || !rope_freqs || !out) return MAC_ERR_NULL;
  if (n_rows < 0 || head_dim < 2 || head_dim % 2) return MAC_ERR_SHAPE;
  if (n_rows == 0) return MAC_OK;
  const int64_t n = (int64_t)n_rows * (head_dim / 2);
  const int grid = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
  rope_rotate_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(n_rows, head_dim, x, t, rope_freqs, out);
  return (int)cudaGetLastError();
}

extern "C" int mac_match_rows(const MacMatchRowsParams* p, void* stream) {
  if (!p || !p->q || !p->ring_q || !p->ring_sqnorm || !p->ring_pos || !p->n_live || !p->m || !p->out_hit ||
      !p->out_pos || !p->out_dist || !p->out_scanned)
    return MAC_ERR_NULL;
  if (p->n_rings < 0 || p->capacity < 1 || p->head_dim < 2 || p->head_dim % 2 || p->head_dim > 1024)
    return MAC_ERR_SHAPE;
  if (p->post_rope && !p->rope_freqs) return MAC_ERR_NULL;
  if (p->n_rings == 0) return MAC_OK;
  match_rows_kernel<<<p->n_rings, 256, 0, static_cast<cudaStream_t>(stream)>>>(*p);
  return (int)cudaGetLastError();
}
