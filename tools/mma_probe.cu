// Development probe (not part of the product): legacy mma.sync m16n8k16 bf16 throughput and
// latency on this part, and FFMA2 throughput, to size the amend kernel's inner loop.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(float* c, const unsigned* a, unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <int CHAINS>
__global__ void mma_loop(float* out, int iters, long long* cyc) {
  unsigned a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u};
  float c[CHAINS][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) mma(c[k], a, (unsigned)i, (unsigned)k);
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
  int iters = 4096;
  for (int warps : {1, 2, 4, 8, 16}) {
    for (int chains : {1, 8}) {
      long long h = 0;
      if (chains == 1) mma_loop<1><<<1, 32 * warps>>>(out, iters, cyc); else mma_loop<8><<<1, 32 * warps>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      double per = (double)h / (iters * chains);
      printf("warps/SM=%2d chains=%d : %.2f cycles per HMMA per warp  -> SM rate %.3f HMMA/cycle\n", warps, chains, per, warps / per);
    }
  }
  return 0;
}
