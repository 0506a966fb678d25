// K2 fast path — the persistent amend kernel (bf16 K/V, d = d_v = 128, GQA
// group g <= 8, tensor cores), launched after the front kernel with
// programmatic dependent launch.  The per-item math and its design notes live
// in amend_mma.cuh.  (A variant that ran concurrently with the front kernel on
// a second stream, polling the plan as groups were decided, measured equal at
// 5-8 warps/SM and slower below: profiles/r01/SUMMARY.md.)
#include <stdio.h>
#include <stdlib.h>

#include "amend_mma.cuh"

namespace mac {

#ifdef MAC_TIMELINE
// per-CTA amend trace (development builds): t_waited, t_end (globaltimer ns), items, tokens,
// end of the first item, tokens of the first item
__device__ unsigned long long g_amend_trace[4096 * 8];
#endif

bool amend_tma_supported(const MacDecodeParams& p);
int amend_tma_grid(cudaError_t* err);
cudaError_t launch_amend_tma(const MacDecodeParams& p, cudaStream_t st, int nb);
#ifdef MAC_DEV_KNOBS
bool amend_tc_supported(const MacDecodeParams& p);
int amend_tc_grid(const MacDecodeParams& p, cudaError_t* err);
cudaError_t launch_amend_tc(const MacDecodeParams& p, cudaStream_t st, int nb);
#endif

bool amend_mma_supported(const MacDecodeParams& p) {
  const int g = p.n_q_heads / p.n_kv_heads;
  return p.storage == MAC_MODE_BF16 && p.head_dim == 128 && p.head_dim_v == 128 && g >= 1 && g <= 8 &&
         p.page_size % 16 == 0;
}

template <int ST, int MINB>  // cp.async stages per warp, min resident warps per SM (register budget)
__global__ void __launch_bounds__(32, MINB) amend_mma_kernel(MacDecodeParams p, int nb) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x;
  const uint32_t sm = smem_u32(smem);
  TL_MARK(p, TL_AMEND_IN);
#ifdef MAC_TIMELINE
  unsigned long long tr_in, tr_band_end = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_in));
#endif
  if (nb > 0) {
    // Split band (common.cuh band_items): the band items need only what the front kernel
    // (the verify kernel's predecessor, complete before any of this grid launched) wrote —
    // this step's KV row, rotated queries and positions — so they stream while the verify
    // kernel still decides the heads.  Static assignment, one item per warp at C3.
    const int G = p.batch * p.n_kv_heads;
    const int* mpos = ws_ptr<const int>(p, workspace_layout(p).mpos_off);
    for (int i = blockIdx.x; i < G * nb; i += gridDim.x) {
      const int grp = i / nb, c = i - grp * nb;
      const int m = (int)__reduce_max_sync(0xffffffffu, (unsigned)__ldcg(mpos + grp / p.n_kv_heads));
      const BandItems bi = band_items(m, p.band, nb);
      if (c >= bi.n) continue;
      const int t0 = bi.t0 + c * bi.len;
      amend_mma_item<ST, true>(p, make_int4(grp, c, t0, min(m, t0 + bi.len - 1)), sm, []() {});
    }
  }
#ifdef MAC_TIMELINE
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_band_end));
#endif
  // programmatic dependent launch: wait for the front kernel's plan before touching it
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  TL_MARK(p, TL_AMEND_WAITED);
  // and let the complete kernel's grid launch as amend warps retire
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const Workspace w = workspace_layout(p);
  unsigned int* ctr = ws_ptr<unsigned int>(p, w.ctr_off);
  int4* list = ws_ptr<int4>(p, w.list_off);
  // Every per-item scalar is passed through __reduce_max_sync: REDUX lands in a uniform
  // register, so ptxas can prove the warp converged and the shuffles stay plain SHFL
  // (values only known to be equal across lanes otherwise compile to slow
  // WARPSYNC.COLLECTIVE sequences).
  const unsigned n_items = __reduce_max_sync(0xffffffffu, __ldcg(ctr));
  // Items are claimed one at a time, after the previous one: claiming the next item at the
  // start of the current one (to prefetch its plan entry) let early warps hoard two items
  // while late ones found the list empty (C3: 58.6 -> 54.1 us per step).
#ifdef MAC_TIMELINE
  unsigned long long tr_t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_t0));
  unsigned tr_items = 0, tr_tokens = 0, tr_first_tok = 0;
  unsigned long long tr_first = 0;
#endif
  unsigned next = 0;
  if (lane == 0) next = atomicAdd(ctr + 1, 1u);
  next = __reduce_max_sync(0xffffffffu, next);
  int4 next_it = next < n_items ? __ldcg(list + next) : make_int4(0, 0, 0, 0);
  for (;;) {
    if (next >= n_items) break;
    int4 it = next_it;
    it.x -= 1;
    amend_mma_item<ST, false>(p, it, sm, []() {});
    unsigned nx = 0;
    if (lane == 0) nx = atomicAdd(ctr + 1, 1u);
    next = __reduce_max_sync(0xffffffffu, nx);
    if (next < n_items) next_it = __ldcg(list + next);
#ifdef MAC_TIMELINE
    if (tr_items == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_first));
      tr_first_tok = (unsigned)(it.w - it.z + 1);
    }
    tr_items++;
    tr_tokens += (unsigned)(it.w - it.z + 1);
#endif
  }
#ifdef MAC_TIMELINE
  if (lane == 0 && blockIdx.x < 4096) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    g_amend_trace[blockIdx.x * 8 + 0] = tr_t0;
    g_amend_trace[blockIdx.x * 8 + 1] = t1;
    g_amend_trace[blockIdx.x * 8 + 2] = tr_items;
    g_amend_trace[blockIdx.x * 8 + 3] = tr_tokens;
    g_amend_trace[blockIdx.x * 8 + 4] = tr_first;
    g_amend_trace[blockIdx.x * 8 + 5] = tr_first_tok;
    g_amend_trace[blockIdx.x * 8 + 6] = tr_in;
    g_amend_trace[blockIdx.x * 8 + 7] = (nb > 0 && (int)blockIdx.x < p.batch * p.n_kv_heads * nb) ? tr_band_end : 0;
  }
#endif
  TL_MARK(p, TL_AMEND_OUT);
  // the work counters are returned to zero by the complete kernel (after this grid)
}

// Variants (stages, min warps per SM); development builds (-DMAC_DEV_KNOBS) select one with
// MAC_AMEND_VARIANT.
struct AmendVariant {
  void (*fn)(MacDecodeParams, int);
  int smem;
};
static const AmendVariant kAmendVariants[] = {
    {amend_mma_kernel<4, 7>, 4 * 2 * TILE_BYTES},  // 0: the hit step
    {amend_mma_kernel<3, 8>, 3 * 2 * TILE_BYTES},  // 1: full spans
#ifdef MAC_DEV_KNOBS
    {amend_mma_kernel<6, 4>, 6 * 2 * TILE_BYTES},
    {amend_mma_kernel<2, 8>, 2 * 2 * TILE_BYTES},
#endif
};
constexpr int kAmendN = (int)(sizeof(kAmendVariants) / sizeof(kAmendVariants[0]));

// full_spans: every group reads [1, m] (full-attention decode and its miss path), where
// the 3-stage / 8-warps-per-SM variant measured best (C3: 2.41 vs 2.53 ms); the hit path's
// short spans prefer 4 stages at 6 warps per SM (81.0 vs 84.5 us).  MAC_AMEND_VARIANT
// overrides both.
static int amend_variant(bool full_spans) {
#ifdef MAC_DEV_KNOBS
  static int forced = -2;
  if (forced == -2) {
    const char* env = getenv("MAC_AMEND_VARIANT");
    forced = env ? atoi(env) : -1;
    if (forced >= kAmendN) forced = -1;
  }
  if (forced >= 0) return forced;
#endif
  return full_spans ? 1 : 0;
}

// resident warps of a variant's persistent grid (sets the smem attribute on first use)
static int amend_grid_full(int vi, cudaError_t* err) {
  static int grid_full[kAmendN] = {};
  if (!grid_full[vi]) {
    const AmendVariant& v = kAmendVariants[vi];
    cudaError_t e = cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v.smem);
    if (e != cudaSuccess) { if (err) *err = e; return 0; }
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v.fn, 32, v.smem);
#ifdef MAC_DEV_KNOBS
    if (const char* env = getenv("MAC_AMEND_PER_SM")) per_sm = atoi(env) > 0 ? atoi(env) : per_sm;
#endif
    grid_full[vi] = sms * (per_sm < 1 ? 1 : per_sm);
  }
  return grid_full[vi];
}

// Which kernel runs the hit step's amend.  With fewer GQA groups than SMs (C2: B = 8, 8 KV heads)
// each group's items are long and few, and the one-warp kernel streams an item at ~5 GB/s per
// warp (its 2-stage lookahead covers one DRAM round trip per 32 tokens), so the TMA kernel
// (amend_tma.cu: a producer warp keeps four 32-token stages in flight per CTA, two consumer
// warps share each item) ends the C2 amend 6 us earlier; with many groups (C3: 256) the one-warp
// kernel's 6-7 independent warps per SM win (in-step timelines, profiles/r02/SUMMARY.md).  Steps
// the engine expects to miss (match_mode 1 / 2) also take the TMA kernel: a missing head's group
// reads its whole context in a few long items, which the one-warp kernel streams slowly (C3
// geometry at 16K with 2% misses: 118 vs 170 us per step).  Development builds can force either
// with MAC_AMEND_TMA=0 / 1, and pick the TMA kernel's other geometries with 2-4 (amend_tma.cu).
static bool hit_amend_tma(const MacDecodeParams& p) {
  bool want = p.batch * p.n_kv_heads < 148 || p.match_mode != 0;
#ifdef MAC_DEV_KNOBS
  static int forced = -2;
  if (forced == -2) {
    const char* env = getenv("MAC_AMEND_TMA");
    forced = env ? atoi(env) : -1;
  }
  if (forced >= 0) want = forced >= 1;
#endif
  return want && p.n_shards == 0 && amend_tma_supported(p);
}

bool amend_uses_tma(const MacDecodeParams& p) { return hit_amend_tma(p); }

// Whether a CTA-cooperative amend (hit_amend_tma) runs on the tcgen05 kernel (amend_tc.cu,
// development builds only, MAC_AMEND_TC=1) rather than the mma.sync one (amend_tma.cu).
static bool coop_amend_tc(const MacDecodeParams& p) {
#ifdef MAC_DEV_KNOBS
  static int forced = -2;
  if (forced == -2) {
    const char* env = getenv("MAC_AMEND_TC");
    forced = env ? atoi(env) : -1;
  }
  return forced >= 1 && amend_tc_supported(p);
#else
  (void)p;
  return false;
#endif
}
// CTAs of the cooperative amend's persistent grid
static int coop_amend_grid(const MacDecodeParams& p) {
#ifdef MAC_DEV_KNOBS
  if (coop_amend_tc(p)) return amend_tc_grid(p, nullptr);
#endif
  (void)p;
  return amend_tma_grid(nullptr);
}

// Band items per GQA group for the split band (common.cuh band_items), 0 when the step does
// not split it: the hit step of the fast path only — the two-pass front (whose verify kernel
// the band overlaps, and which guarantees the append finished before this grid launches),
// one KV shard, r > 0.  The one-warp amend: as many items per group as its grid has warps per
// group (1..4); the TMA-fed amend: one.  In development builds MAC_BAND_SPLIT=0 turns it off, =n forces n items.  The verify
// kernel's plan and this launch call it with the same parameters, so they always agree.
int band_split(const MacDecodeParams& p) {
#ifdef MAC_DEV_KNOBS
  static int forced = -2;
  if (forced == -2) {
    const char* env = getenv("MAC_BAND_SPLIT");
    forced = env ? atoi(env) : -1;
  }
#else
  const int forced = -1;
#endif
  if (forced == 0 || !amend_mma_supported(p) || !front_two_pass(p) || p.kv_offset != 0 || p.kv_limit != 0 ||
      p.band <= 0)
    return 0;
  const int G = p.batch * p.n_kv_heads;
  // the TMA-fed amend: one band item per group (C2: 33.3 vs 34.2 us with 4; dense-mode steps at
  // 16K 0.5 / 2 / 10 % misses 71.5 / 86.7 / 179.8 vs 71.8 / 87.8 / 180.1; r02 same-box sweeps)
  int nb = forced > 0 ? forced : (hit_amend_tma(p) ? 1 : amend_grid_full(amend_variant(false), nullptr) / G);
  if (nb > 4 && forced < 0) nb = 4;
  if (nb > p.max_chunks - 1) nb = p.max_chunks - 1;
  return nb < 1 ? 0 : nb;
}

// piece items per group with the split band: the persistent grid's warps per group (>= 1)
// (encoded for plan_chunking: the TMA amend's CTAs take items of up to 512 tokens, two per CTA)
int piece_target(const MacDecodeParams& p) {
  const int G = p.batch * p.n_kv_heads;
  if (hit_amend_tma(p)) {
    const int t = 2 * coop_amend_grid(p) / G;
    int subs = 32;  // longest item: 32 sub-tiles of 16 tokens
#ifdef MAC_DEV_KNOBS
    if (const char* env = getenv("MAC_TMA_MAXSUB")) subs = atoi(env) > 0 ? atoi(env) : subs;
#endif
    return (t < 1 ? 1 : (t > 0xffff ? 0xffff : t)) | (subs << 16);
  }
  const int t = amend_grid_full(amend_variant(false), nullptr) / G;
  return t < 1 ? 1 : t;
}

cudaError_t launch_amend_mma_bf16(const MacDecodeParams& p, cudaStream_t st, bool full_spans) {
  // the KV-sharded path (n_shards > 0: one very long request, the miss path) is long-span work
  // too: the full-span variant streams it faster (C4, one 512K request: 0.457 -> 0.421 ms)
  const int vi = amend_variant(full_spans || p.n_shards > 0);
  const AmendVariant& v = kAmendVariants[vi];
  cudaError_t err = cudaSuccess;
  const int gfull = amend_grid_full(vi, &err);
  if (err != cudaSuccess) return err;
  const int nb = full_spans ? 0 : band_split(p);
  if (!full_spans && hit_amend_tma(p)) {
#ifdef MAC_DEV_KNOBS
    if (coop_amend_tc(p)) return launch_amend_tc(p, st, nb);
#endif
    return launch_amend_tma(p, st, nb);
  }
  const long cap = (long)p.batch * p.n_kv_heads * p.max_chunks;
  const int grid = (int)(gfull < cap ? gfull : cap);
  // programmatic dependent launch: the grid is set up while the front kernel drains
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = v.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, v.fn, p, nb);
}

}  // namespace mac

#ifdef MAC_TIMELINE
// development builds only: copy the per-CTA amend trace ([n][8] u64) to host memory
extern "C" int mac_timeline_amend(void* host_out, int n) {
  return (int)cudaMemcpyFromSymbol(host_out, mac::g_amend_trace, (size_t)n * 8 * sizeof(unsigned long long));
}
#endif
