// Probe: latency of one scattered 512-byte read per warp (1024 warps) as a function of
// the footprint the reads are scattered over (2 MB .. 2 GB), after a 256 MB streaming
// write that evicts L2 — the access pattern of the complete kernel's cached-summary
// reads (one ring slot per head, heads 512 KB apart).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tlb_probe tools/tlb_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void scatter_read(const float4* __restrict__ buf, size_t n_slots, size_t stride_f4, float* out, int salt) {
  const int lane = threadIdx.x & 31;
  const unsigned w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const size_t slot = ((size_t)(w * 2654435761u + salt * 40503u)) % n_slots;
  const float4 v = buf[slot * stride_f4 + lane];
  float s = v.x + v.y + v.z + v.w;
  if (s == 12345.f) out[w] = s;
}

__global__ void flush(float* f, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) f[i] = 0.f;
}

int main() {
  const size_t big = 2ull << 30;
  float4* buf;
  float *out, *fl;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 0, big);
  cudaMalloc(&out, 1 << 20);
  const size_t fl_n = (256ull << 20) / 4;
  cudaMalloc(&fl, fl_n * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t foots[] = {2ull << 20, 16ull << 20, 64ull << 20, 256ull << 20, 512ull << 20, 2ull << 30};
  for (size_t f : foots) {
    for (int mode = 0; mode < 2; ++mode) {  // 0: slots 512 KB apart (head stride), 1: 512 B apart (dense)
      const size_t stride_f4 = mode == 0 ? (512 << 10) / 16 : 512 / 16;
      const size_t n_slots = f / (stride_f4 * 16);
      if (n_slots < 1) continue;
      float best = 1e9f, sum = 0.f;
      const int reps = 20;
      for (int r = 0; r < reps; ++r) {
        flush<<<1184, 256>>>(fl, fl_n);
        cudaEventRecord(a);
        scatter_read<<<256, 128>>>(buf, n_slots, stride_f4, out, r);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
        sum += ms;
      }
      printf("footprint %6zu MB  %s  slots %8zu  best %.2f us  mean %.2f us\n", f >> 20,
             mode == 0 ? "head-stride" : "dense      ", n_slots, best * 1e3, sum / reps * 1e3);
    }
  }
  return 0;
}
