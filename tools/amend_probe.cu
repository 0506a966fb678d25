// Development probe (not part of the product): HBM throughput of the amend kernel's load
// pattern with no math — paged bf16 K/V ([page][Hkv=8][16][128], 4 KB per (page, kv head)),
// 256 GQA groups x `span` tokens at the end of 128K-token requests — to separate the
// pattern's memory ceiling from the kernel's per-warp compute latency.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/amend_probe.cu -o tools/amend_probe
// Modes: cp.async 1-warp CTAs with ST stages of 16-token K+V sub-tiles (the amend's
// structure), and a 256-thread LDG.128 kernel over the same sub-tiles.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int HKV = 8, PS = 16, D = 128;

__device__ __forceinline__ void cp16(unsigned s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}

// sub-tile j of the virtual work: group = j / nsub_g, sub-tile within the group's span
// layout 0: [page][Hkv][16][d] (4 KB per (page, kv head), pages 32 KB apart);
// layout 1: [Hkv][page][16][d] (a kv head's pages contiguous)
__device__ int g_layout = 0;
__device__ __forceinline__ long long subtile_row(int j, int nsub_g, int pps, int first_page) {
  const int grp = j / nsub_g, k = j % nsub_g;
  const int b = grp / HKV, kvh = grp % HKV;
  const long long page = (long long)b * pps + first_page + k;
  if (g_layout) return ((long long)kvh * 32 * pps + page) * PS;
  return (page * HKV + kvh) * PS;
}

template <int ST>
__global__ void __launch_bounds__(32) cp_kernel(const uint4* K, const uint4* V, int nsub_total, int nsub_g, int pps,
                                                int first_page, int per_warp, unsigned* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x;
  const unsigned sm = (unsigned)__cvta_generic_to_shared(smem);
  const int j0 = blockIdx.x * per_warp, j1 = min(nsub_total, j0 + per_warp);
  unsigned acc = 0;
  auto issue = [&](int j, int stage) {
    const long long row = subtile_row(j, nsub_g, pps, first_page);
    const char* kg = reinterpret_cast<const char*>(K) + row * 256;
    const char* vg = reinterpret_cast<const char*>(V) + row * 256;
    const unsigned ks = sm + stage * 8192, vs = ks + 4096;
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      cp16(ks + rr * 512 + lane * 16, kg + rr * 512 + lane * 16);
      cp16(vs + rr * 512 + lane * 16, vg + rr * 512 + lane * 16);
    }
  };
  for (int i = 0; i < ST; ++i) {
    if (j0 + i < j1) issue(j0 + i, i);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int j = j0; j < j1; ++j) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 1));
    __syncwarp();
    const int stage = (j - j0) % ST;
    acc ^= *reinterpret_cast<const unsigned*>(smem + stage * 8192 + lane * 4);
    __syncwarp();
    if (j + ST < j1) issue(j + ST, stage);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// 256 threads, each sub-tile (8 KB K+V) read by 2 warps with LDG.128 x 4 per thread
__global__ void __launch_bounds__(256) ldg_kernel(const uint4* K, const uint4* V, int nsub_total, int nsub_g, int pps,
                                                  int first_page, unsigned* out) {
  unsigned acc = 0;
  const int w = (blockIdx.x * 256 + threadIdx.x) >> 6, l = threadIdx.x & 63;
  for (int j = w; j < nsub_total; j += (gridDim.x * 256) >> 6) {
    const long long row = subtile_row(j, nsub_g, pps, first_page);
    const uint4* kg = K + row * 16;
    const uint4* vg = V + row * 16;
    uint4 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { a[u] = __ldcs(kg + l + 64 * u); b[u] = __ldcs(vg + l + 64 * u); }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= a[u].x ^ b[u].y;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void flush_write(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4((unsigned)i, 0, 0, 0);
}

int main() {
  const int B = 32, ctx = 131072, pps = ctx / PS;
  const size_t tok_bytes = (size_t)B * pps * HKV * PS * D * 2;  // 8.6 GB per tensor
  uint4 *K, *V, *fl;
  unsigned* out;
  if (cudaMalloc(&K, tok_bytes) || cudaMalloc(&V, tok_bytes)) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&fl, (size_t)256 << 20);
  cudaMalloc(&out, 4);
  cudaMemset(K, 1, tok_bytes);
  cudaMemset(V, 1, tok_bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int spans[] = {672, 256};
  for (int layout = 0; layout < 2; ++layout) {
  cudaMemcpyToSymbol(g_layout, &layout, sizeof(int));
  printf("layout %s\n", layout ? "[Hkv][page][16][d]" : "[page][Hkv][16][d]");
  for (int span : spans) {
    const int nsub_g = span / 16, groups = B * HKV, nsub_total = nsub_g * groups;
    const int first_page = pps - nsub_g;
    const double bytes = (double)nsub_total * 8192;
    for (int mode = 0; mode < 7; ++mode) {
      float best = 1e9f, sum = 0.f;
      const int reps = 8;
      for (int it = 0; it < reps; ++it) {
        flush_write<<<148 * 8, 256>>>(fl, ((size_t)256 << 20) / 16);
        cudaEventRecord(a);
        int warps = 0, st = 0;
        switch (mode) {
          case 0: warps = 888; st = 4; break;
          case 1: warps = 888; st = 6; break;
          case 2: warps = 148 * 12; st = 4; break;
          case 3: warps = 148 * 16; st = 2; break;
          case 4: warps = 148 * 16; st = 4; break;
          default: break;
        }
        if (mode < 5) {
          const int per = (nsub_total + warps - 1) / warps;
          const int sm = st * 8192;
          if (st == 2) { cudaFuncSetAttribute(cp_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); cp_kernel<2><<<warps, 32, sm>>>(K, V, nsub_total, nsub_g, pps, first_page, per, out); }
          if (st == 4) { cudaFuncSetAttribute(cp_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); cp_kernel<4><<<warps, 32, sm>>>(K, V, nsub_total, nsub_g, pps, first_page, per, out); }
          if (st == 6) { cudaFuncSetAttribute(cp_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); cp_kernel<6><<<warps, 32, sm>>>(K, V, nsub_total, nsub_g, pps, first_page, per, out); }
        } else {
          ldg_kernel<<<mode == 5 ? 148 * 4 : 148 * 8, 256>>>(K, V, nsub_total, nsub_g, pps, first_page, out);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 0) { best = ms < best ? ms : best; sum += ms; }
      }
      const char* names[] = {"cp.async 888 warps x4 st", "cp.async 888 warps x6 st", "cp.async 1776 warps x4 st",
                             "cp.async 2368 warps x2 st", "cp.async 2368 warps x4 st", "ldg 592x256", "ldg 1184x256"};
      printf("span %4d  %.1f MB  %-28s best %6.1f us (%5.0f GB/s)  avg %6.1f us\n", span, bytes / 1e6, names[mode],
             best * 1e3, bytes / (best * 1e-3) / 1e9, sum / (reps - 1) * 1e3);
    }
  }
  }
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
