// Development probe: the ring scan's access pattern.  1024 heads x 1024 rows of 256 B
// (256 MiB, the C3 query ring); read the first P bytes of every row (P = 64 or 128) with the
// scan's CTA shape (256 threads, 8 16-byte loads per lane, 4 CTAs per SM) either
//   strided: row-major [head][row][256 B], P bytes of each row (the current layout), or
//   planar:  the same bytes stored contiguously per head ([head][plane][row][P]).
// Prints the best / mean kernel time of each, after an L2-evicting write.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/prefix_probe tools/prefix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int LPR, bool PLANAR>
__global__ void __launch_bounds__(256, 4) scan(const uint4* __restrict__ ring, int rows_per_cta, unsigned* out) {
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = 1024;
  const int nsplit = W / rows_per_cta;
  const int bh = blockIdx.x / nsplit, split = blockIdx.x % nsplit;
  const int sub = lane % LPR, quad = lane / LPR;
  const int row0 = split * rows_per_cta;
  uint4 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int slot = row0 + k * 8 * RPW + warp * RPW + quad;
    const size_t idx = PLANAR ? ((size_t)bh * 16 * W + (size_t)slot * LPR + sub)  // head block of 16*W uint4
                              : ((size_t)bh * W + slot) * 16 + sub;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(ring + idx));
  }
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  if (acc == 0x9e3779b9u) out[0] = acc;
}

__global__ void flush(uint4* f, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    f[i] = make_uint4((unsigned)i, 0, 0, 0);
}

template <int LPR, bool PLANAR>
void run(const uint4* ring, unsigned* out, uint4* fl, size_t fl_n, const char* name) {
  const int rows_per_cta = 8 * 8 * (32 / LPR);
  const int grid = 1024 * (1024 / rows_per_cta);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f, sum = 0.f;
  for (int r = 0; r < 12; ++r) {
    flush<<<1184, 256>>>(fl, fl_n);
    cudaEventRecord(a);
    scan<LPR, PLANAR><<<grid, 256>>>(ring, rows_per_cta, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
  }
  const double mb = 1024.0 * 1024 * LPR * 16 / 1e6;
  printf("%-28s %6.1f MB  best %6.2f us  mean %6.2f us  (%.2f TB/s best)\n", name, mb, best * 1e3, sum / 10 * 1e3,
         mb / (best * 1e3) * 1e-6 * 1e6 / 1e6);
}

int main() {
  uint4 *ring, *fl;
  unsigned* out;
  const size_t ring_bytes = (size_t)256 << 20;
  cudaMalloc(&ring, ring_bytes);
  cudaMemset(ring, 1, ring_bytes);
  cudaMalloc(&out, 4);
  const size_t fl_n = ((size_t)256 << 20) / 16;
  cudaMalloc(&fl, fl_n * 16);
  run<8, false>(ring, out, fl, fl_n, "strided 128 B of 256 B rows");
  run<4, false>(ring, out, fl, fl_n, "strided 64 B of 256 B rows");
  run<8, true>(ring, out, fl, fl_n, "planar 128 B rows");
  run<4, true>(ring, out, fl, fl_n, "planar 64 B rows");
  return 0;
}
