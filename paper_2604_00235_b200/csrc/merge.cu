// Cross-shard log-domain merge of (acc, lse) partials (attention.py:119-135),
// the exchange step of the KV-sharded miss path: after an all-gather of every
// rank's [rows, d_v + 1] partial, each row is merged over the G shards.
#include "common.cuh"

namespace mac {

template <typename T>
__global__ void merge_partials_kernel(MacMergeParams p) {
  const int row = blockIdx.x;
  const T* acc = static_cast<const T*>(p.part_acc);
  const T* lse = static_cast<const T*>(p.part_lse);
  const int dv = p.head_dim_v;
  double mx = -CUDART_INF;
  for (int g = 0; g < p.n_parts; ++g) mx = fmax(mx, (double)lse[(int64_t)g * p.n_rows + row]);
  double L = mx;
  if (mx != -CUDART_INF) {
    double s = 0.0;
    for (int g = 0; g < p.n_parts; ++g) {
      double l = (double)lse[(int64_t)g * p.n_rows + row];
      if (l != -CUDART_INF) s += exp(l - mx);
    }
    L = mx + log(s);
  }
  for (int e = threadIdx.x; e < dv; e += blockDim.x) {
    double a = 0.0;
    if (L != -CUDART_INF)
      for (int g = 0; g < p.n_parts; ++g) {
        double l = (double)lse[(int64_t)g * p.n_rows + row];
        if (l != -CUDART_INF) a += (double)acc[((int64_t)g * p.n_rows + row) * dv + e] * exp(l - L);
      }
    static_cast<T*>(p.out_acc)[(int64_t)row * dv + e] = (T)a;
  }
  if (threadIdx.x == 0) static_cast<T*>(p.out_lse)[row] = (T)L;
}

cudaError_t launch_merge_partials(const MacMergeParams& p, cudaStream_t st) {
  if (p.dtype == MAC_DT_F64) merge_partials_kernel<double><<<p.n_rows, 128, 0, st>>>(p);
  else merge_partials_kernel<float><<<p.n_rows, 128, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace mac
