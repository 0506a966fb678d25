// tcgen05 (UMMA) descriptor probe (development tool): one CTA issues the two MMA shapes the
// tensor-core ring build uses and checks them against a host GEMM.
//   S  = A[128 x 128] . B[64 x 128]^T   A, B K-major, SWIZZLE_128B (two 64-element atoms each),
//        two MMA chains accumulated (hi + lo operands), fp32 accumulator in TMEM
//   O  = P[128 x 64] . V[64 x 128]      P K-major SWIZZLE_128B, V MN-major SWIZZLE_128B
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe tools/umma_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2604_00235_b200/csrc/umma.cuh"

using namespace mac::umma;

// element (r, k) of a K-major SW128 tile with R rows: 64-element atoms of R x 128 B
__device__ __host__ inline uint32_t kmaj_off(int r, int k, int R) {
  return (uint32_t)((k >> 6) * R * 128 + r * 128 + ((((k & 63) >> 3) ^ (r & 7)) << 4) + (k & 7) * 2);
}
// element (kk, n) of an MN-major SW128 tile with K rows: 64-element N atoms of K x 128 B
__device__ __host__ inline uint32_t mnmaj_off(int kk, int n, int K) {
  return (uint32_t)((n >> 6) * K * 128 + kk * 128 + ((((n & 63) >> 3) ^ (kk & 7)) << 4) + (n & 7) * 2);
}

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* A2, const __nv_bfloat16* B, const __nv_bfloat16* P,
                      const __nv_bfloat16* V, float* S_out, float* O_out, float* O2_out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* sA = sm;              // 32 KB
  unsigned char* sA2 = sm + 32768;     // 32 KB
  unsigned char* sB = sm + 65536;      // 16 KB
  unsigned char* sP = sm + 81920;      // 16 KB
  unsigned char* sV = sm + 98304;      // 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 128; i += blockDim.x) {
    const int r = i / 128, k = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(sA + kmaj_off(r, k, 128)) = A[i];
    *reinterpret_cast<__nv_bfloat16*>(sA2 + kmaj_off(r, k, 128)) = A2[i];
  }
  for (int i = tid; i < 64 * 128; i += blockDim.x) {
    const int r = i / 128, k = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(sB + kmaj_off(r, k, 64)) = B[i];
    const int kk = i / 128, n = i % 128;  // V[kk][n]
    *reinterpret_cast<__nv_bfloat16*>(sV + mnmaj_off(kk, n, 64)) = V[i];
  }
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    *reinterpret_cast<__nv_bfloat16*>(sP + kmaj_off(r, k, 128)) = P[i];
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), 512);
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t idS = instr_desc_bf16(128, 64, false, false);
    for (int ks = 0; ks < 8; ++ks) {  // hi chain then lo chain into the same accumulator
      const uint32_t koff = (ks >> 2) * 128 * 128 + (ks & 3) * 32;
      const uint32_t boff = (ks >> 2) * 64 * 128 + (ks & 3) * 32;
      mma_bf16(tm, sdesc_kmajor_sw128(smem_u32(sA) + koff), sdesc_kmajor_sw128(smem_u32(sB) + boff), idS, ks > 0);
    }
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t koff = (ks >> 2) * 128 * 128 + (ks & 3) * 32;
      const uint32_t boff = (ks >> 2) * 64 * 128 + (ks & 3) * 32;
      mma_bf16(tm, sdesc_kmajor_sw128(smem_u32(sA2) + koff), sdesc_kmajor_sw128(smem_u32(sB) + boff), idS, true);
    }
    const uint32_t idO = instr_desc_bf16(128, 128, false, true);
    for (int ks = 0; ks < 4; ++ks)
      mma_bf16(tm + 128, sdesc_kmajor_sw128(smem_u32(sP) + ks * 32),
               sdesc_mnmajor_sw128(smem_u32(sV) + ks * 2048, 64 * 128), idO, ks > 0);
    mma_commit(smem_u32(&bar));
  }
  mbar_wait_parity(smem_u32(&bar), 0);
  tc_fence_after();
  {  // P row -> TMEM columns 384.. (two bf16 per column), then O2 = P[tmem] . V
    const int row = warp * 32 + lane;
    uint32_t pv[32];
    for (int c = 0; c < 32; ++c) {
      __nv_bfloat162 t2;
      t2.x = P[row * 64 + 2 * c];
      t2.y = P[row * 64 + 2 * c + 1];
      pv[c] = *reinterpret_cast<uint32_t*>(&t2);
    }
    tmem_st32(tm + ((uint32_t)(warp * 32) << 16) + 384, pv);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idO = instr_desc_bf16(128, 128, false, true);
    for (int ks = 0; ks < 4; ++ks)
      mma_bf16_ta(tm + 256, tm + 384 + ks * 8, sdesc_mnmajor_sw128(smem_u32(sV) + ks * 2048, 64 * 128), idO, ks > 0);
    mma_commit(smem_u32(&bar));
  }
  mbar_wait_parity(smem_u32(&bar), 1);
  tc_fence_after();
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  uint32_t v[32];
  for (int c = 0; c < 64; c += 32) {
    tmem_ld32(tm + lane_base + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) S_out[(warp * 32 + lane) * 64 + c + j] = __uint_as_float(v[j]);
  }
  for (int c = 0; c < 128; c += 32) {
    tmem_ld32(tm + 128 + lane_base + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) O_out[(warp * 32 + lane) * 128 + c + j] = __uint_as_float(v[j]);
  }
  for (int c = 0; c < 128; c += 32) {
    tmem_ld32(tm + 256 + lane_base + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) O2_out[(warp * 32 + lane) * 128 + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  const int nA = 128 * 128, nB = 64 * 128, nP = 128 * 64, nV = 64 * 128;
  std::vector<__nv_bfloat16> A(nA), A2(nA), B(nB), P(nP), V(nV);
  std::vector<float> fA(nA), fA2(nA), fB(nB), fP(nP), fV(nV);
  srand(1);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  auto fill = [&](std::vector<__nv_bfloat16>& h, std::vector<float>& f, float s) {
    for (size_t i = 0; i < h.size(); ++i) { h[i] = __float2bfloat16(rnd() * s); f[i] = __bfloat162float(h[i]); }
  };
  fill(A, fA, 1.f); fill(A2, fA2, 1.f / 256); fill(B, fB, 1.f); fill(P, fP, 1.f); fill(V, fV, 1.f);
  __nv_bfloat16 *dA, *dA2, *dB, *dP, *dV;
  float *dS, *dO, *dO2;
  cudaMalloc(&dA, nA * 2); cudaMalloc(&dA2, nA * 2); cudaMalloc(&dB, nB * 2); cudaMalloc(&dP, nP * 2);
  cudaMalloc(&dV, nV * 2); cudaMalloc(&dS, 128 * 64 * 4); cudaMalloc(&dO, 128 * 128 * 4); cudaMalloc(&dO2, 128 * 128 * 4);
  cudaMemcpy(dA, A.data(), nA * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dA2, A2.data(), nA * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), nB * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), nP * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), nV * 2, cudaMemcpyHostToDevice);
  const int smem = 114688 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dA, dA2, dB, dP, dV, dS, dO, dO2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> S(128 * 64), O(128 * 128), O2(128 * 128);
  cudaMemcpy(O2.data(), dO2, O2.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0, ns = 0, no = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 64; ++j) {
      double r = 0;
      for (int k = 0; k < 128; ++k) r += (double)fA[i * 128 + k] * fB[j * 128 + k] + (double)fA2[i * 128 + k] * fB[j * 128 + k];
      es = fmax(es, fabs(r - S[i * 64 + j]));
      ns = fmax(ns, fabs(r));
    }
  for (int i = 0; i < 128; ++i)
    for (int n = 0; n < 128; ++n) {
      double r = 0;
      for (int kk = 0; kk < 64; ++kk) r += (double)fP[i * 64 + kk] * fV[kk * 128 + n];
      eo = fmax(eo, fabs(r - O[i * 128 + n]));
      eo = fmax(eo, fabs(r - O2[i * 128 + n]));
      no = fmax(no, fabs(r));
    }
  printf("S max abs err %.3e (max |S| %.2f)  O max abs err %.3e (max |O| %.2f)\n", es, ns, eo, no);
  printf("%s\n", (es < 1e-3 && eo < 1e-3) ? "UMMA PROBE OK" : "UMMA PROBE FAILED");
  return (es < 1e-3 && eo < 1e-3) ? 0 : 1;
}
