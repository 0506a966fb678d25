// tcgen05 (UMMA) probe for the tensor-core amend (development tool): one CTA issues the two
// transposed MMA shapes amend_tc.cu uses and checks them against a host GEMM.
//   S^T = K[64 x 128] . Qc[N_S x 128]^T    M = 128 (rows 64..127 read past the 64-token tile:
//        don't-care), N_S = 8, A = the K tile as TMA lands it (two 64-dim SW128 atoms 64 rows
//        apart), B = Qc K-major SW128
//   O^T = V[64 x 128]^T . P[N_O x 64]^T    M = 128 dims, N_O = 16 / 32, K = 64 tokens,
//        A = the V tile as TMA lands it read MN-major (M atoms of 64 dims, LBO = 8 KiB),
//        B = P K-major SW128 (one 64-token atom)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe2 tools/umma_probe2.cu
#include <cuda_bf16.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2604_00235_b200/csrc/umma.cuh"

using namespace mac::umma;

constexpr int T = 64, D = 128, NS = 8;

// (token, dim) of a 64-token K or V tile: two 64-dim SW128 atoms of 64 rows x 128 B
__device__ __host__ inline uint32_t tile_off(int t, int d) {
  return (uint32_t)((d >> 6) * (T * 128) + t * 128 + ((((d & 63) >> 3) ^ (t & 7)) << 4) + (d & 7) * 2);
}
// (row n, k) of a K-major SW128 operand with R rows and 64-element atoms R*128 bytes apart
__device__ __host__ inline uint32_t kmaj_off(int n, int k, int R) {
  return (uint32_t)((k >> 6) * R * 128 + n * 128 + ((((k & 63) >> 3) ^ (n & 7)) << 4) + (k & 7) * 2);
}

template <int NO>
__global__ void probe(const __nv_bfloat16* K, const __nv_bfloat16* Q, const __nv_bfloat16* V, const __nv_bfloat16* P,
                      float* S_out, float* O_out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* sK = sm;                // 16 KB (+ 16 KB slack the M = 128 rows read)
  unsigned char* sV = sm + 32768;        // 16 KB
  unsigned char* sQ = sm + 49152;        // 2 KB
  unsigned char* sP = sm + 53248;        // NO * 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 32768 / 2; i += blockDim.x) reinterpret_cast<__nv_bfloat16*>(sK)[i] = __float2bfloat16(0.f);
  __syncthreads();
  for (int i = tid; i < T * D; i += blockDim.x) {
    const int t = i / D, d = i % D;
    *reinterpret_cast<__nv_bfloat16*>(sK + tile_off(t, d)) = K[i];
    *reinterpret_cast<__nv_bfloat16*>(sV + tile_off(t, d)) = V[i];
  }
  for (int i = tid; i < NS * D; i += blockDim.x) {
    const int n = i / D, d = i % D;
    *reinterpret_cast<__nv_bfloat16*>(sQ + kmaj_off(n, d, NS)) = Q[i];
  }
  for (int i = tid; i < NO * T; i += blockDim.x) {
    const int n = i / T, k = i % T;
    *reinterpret_cast<__nv_bfloat16*>(sP + kmaj_off(n, k, NO)) = P[i];
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(smem_u32(&tmem_base), 128);
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t idS = instr_desc_bf16(128, NS, false, false);
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t a = smem_u32(sK) + (ks >> 2) * (T * 128) + (ks & 3) * 32;
      const uint32_t b = smem_u32(sQ) + (ks >> 2) * (NS * 128) + (ks & 3) * 32;
      mma_bf16(tm, sdesc_kmajor_sw128(a), sdesc_kmajor_sw128(b), idS, ks > 0);
    }
    const uint32_t idO = instr_desc_bf16(128, NO, true, false);
    for (int ks = 0; ks < T / 16; ++ks)
      mma_bf16(tm + 32, sdesc_mnmajor_sw128(smem_u32(sV) + ks * 2048, T * 128),
               sdesc_kmajor_sw128(smem_u32(sP) + ks * 32), idO, ks > 0);
    mma_commit(smem_u32(&bar));
  }
  mbar_wait_parity(smem_u32(&bar), 0);
  tc_fence_after();
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const int row = warp * 32 + lane;
  uint32_t v[8];
  tmem_ld8(tm + lane_base, v);
  tmem_wait_ld();
  for (int j = 0; j < NS; ++j) S_out[row * NS + j] = __uint_as_float(v[j]);
  for (int c = 0; c < NO; c += 8) {
    tmem_ld8(tm + lane_base + 32 + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) O_out[row * NO + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 128);
}

template <int NO>
static int run() {
  std::vector<__nv_bfloat16> K(T * D), Q(NS * D), V(T * D), P(NO * T);
  std::vector<float> fK(T * D), fQ(NS * D), fV(T * D), fP(NO * T);
  srand(7 + NO);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  auto fill = [&](std::vector<__nv_bfloat16>& h, std::vector<float>& f) {
    for (size_t i = 0; i < h.size(); ++i) { h[i] = __float2bfloat16(rnd()); f[i] = __bfloat162float(h[i]); }
  };
  fill(K, fK); fill(Q, fQ); fill(V, fV); fill(P, fP);
  __nv_bfloat16 *dK, *dQ, *dV, *dP;
  float *dS, *dO;
  cudaMalloc(&dK, K.size() * 2); cudaMalloc(&dQ, Q.size() * 2); cudaMalloc(&dV, V.size() * 2);
  cudaMalloc(&dP, P.size() * 2); cudaMalloc(&dS, 128 * NS * 4); cudaMalloc(&dO, 128 * NO * 4);
  cudaMemcpy(dK, K.data(), K.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Q.data(), Q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 53248 + 4096 + 1024;
  cudaFuncSetAttribute(probe<NO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<NO><<<1, 128, smem>>>(dK, dQ, dV, dP, dS, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("kernel error: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> S(128 * NS), O(128 * NO);
  cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0;
  for (int t = 0; t < T; ++t)
    for (int n = 0; n < NS; ++n) {
      double r = 0;
      for (int d = 0; d < D; ++d) r += (double)fK[t * D + d] * fQ[n * D + d];
      es = fmax(es, fabs(r - S[t * NS + n]));
    }
  for (int d = 0; d < D; ++d)
    for (int n = 0; n < NO; ++n) {
      double r = 0;
      for (int k = 0; k < T; ++k) r += (double)fV[k * D + d] * fP[n * T + k];
      eo = fmax(eo, fabs(r - O[d * NO + n]));
    }
  const bool ok = es < 1e-3 && eo < 1e-3;
  printf("N_O=%d  S^T max abs err %.3e  O^T max abs err %.3e  %s\n", NO, es, eo, ok ? "OK" : "FAILED");
  return ok ? 0 : 1;
}

int main() {
  const int rc = run<16>() | run<32>() | run<8>();
  printf("%s\n", rc == 0 ? "UMMA PROBE2 OK" : "UMMA PROBE2 FAILED");
  return rc;
}
