// Development probe (not part of the product): achievable HBM read bandwidth for
// short streams on this B200, to calibrate the roofline of the ~90-270 MB hit-path
// kernels.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/stream_probe.cu -o tools/stream_probe
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

__global__ void read_ldg(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
// unrolled: each thread loads U vectors per iteration (contiguous chunks per CTA)
template <int U>
__global__ void read_ldg_unroll(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  size_t per_cta = (n + gridDim.x - 1) / gridDim.x;
  size_t b = blockIdx.x * per_cta, e = min(n, b + per_cta);
  for (size_t i = b + threadIdx.x; i < e; i += (size_t)blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      v[u] = j < e ? __ldcs(p + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void flush_write(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(i, 0, 0, 0);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t big = (size_t)1 << 30;  // 1 GiB buffer
  uint4 *buf, *fl;
  unsigned* out;
  cudaMalloc(&buf, big);
  cudaMalloc(&fl, (size_t)512 << 20);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, big);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  size_t sizes[] = {(size_t)87 << 20, (size_t)268 << 20, (size_t)1 << 30};
  for (int flushmode = 0; flushmode < 3; ++flushmode) {
    for (size_t bytes : sizes) {
      size_t n = bytes / 16;
      for (int cfg = 0; cfg < 6; ++cfg) {
        float best = 1e9, sum = 0;
        for (int it = 0; it < 6; ++it) {
          if (flushmode == 1) flush_write<<<sms * 8, 256>>>(fl, ((size_t)512 << 20) / 16);
          if (flushmode == 2) read_ldg<<<sms * 8, 256>>>(fl, ((size_t)512 << 20) / 16, out);
          cudaEventRecord(a);
          switch (cfg) {
            case 0: read_ldg<<<sms * 8, 256>>>(buf, n, out); break;
            case 1: read_ldg<<<sms * 16, 256>>>(buf, n, out); break;
            case 2: read_ldg_unroll<4><<<sms * 4, 256>>>(buf, n, out); break;
            case 3: read_ldg_unroll<8><<<sms * 2, 256>>>(buf, n, out); break;
            case 4: read_ldg_unroll<8><<<sms * 4, 256>>>(buf, n, out); break;
            case 5: read_ldg_unroll<16><<<sms * 2, 256>>>(buf, n, out); break;
          }
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (it > 0) { best = ms < best ? ms : best; sum += ms; }
        }
        printf("flush=%s bytes=%zuMB cfg=%d best=%.1fus avg=%.1fus -> %.0f GB/s (avg %.0f)\n",
               flushmode == 0 ? "none " : (flushmode == 1 ? "write" : "read "), bytes >> 20, cfg, best * 1e3,
               sum / 5 * 1e3, bytes / (best * 1e-3) / 1e9, bytes / (sum / 5 * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
