// C-ABI entry points (include/macattn.h): validation, dispatch, step sequencing.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace mac {
template <int MODE> cudaError_t launch_append(const MacDecodeParams&, cudaStream_t, int, int);
template <int MODE> cudaError_t launch_match_generic(const MacDecodeParams&, cudaStream_t);
template <int MODE> cudaError_t launch_amend_generic(const MacDecodeParams&, cudaStream_t);
template <int MODE> cudaError_t launch_complete(const MacDecodeParams&, cudaStream_t, int);
cudaError_t launch_front_bf16(const MacDecodeParams&, cudaStream_t, bool do_match, bool do_append, int rotate_only,
                              int plan, int passes);
cudaError_t launch_amend_mma_bf16(const MacDecodeParams&, cudaStream_t, bool full_spans);
bool amend_mma_supported(const MacDecodeParams&);
bool match_fast_supported(const MacDecodeParams&);
bool front_fast_supported(const MacDecodeParams&);
cudaError_t launch_merge_partials(const MacMergeParams&, cudaStream_t);
template <int MODE> cudaError_t launch_prefill_kv(const MacDecodeParams&, int, cudaStream_t);
bool ring_build_supported(const MacDecodeParams&);
cudaError_t launch_ring_build(const MacDecodeParams&, const MacRingBuildParams&, cudaStream_t, int use_tc);
template <int MODE> cudaError_t launch_step_stats(const MacDecodeParams&, double*, double*, cudaStream_t);
template <int MODE> cudaError_t launch_mass_bound(const MacDecodeParams&, const MacMassBoundParams&, cudaStream_t);
}  // namespace mac

using namespace mac;

static int validate(const MacDecodeParams* p, bool need_ring) {
  if (!p) return MAC_ERR_NULL;
  if (p->batch < 1 || p->n_q_heads < 1 || p->n_kv_heads < 1 || p->n_q_heads % p->n_kv_heads) return MAC_ERR_SHAPE;
  if (p->head_dim < 2 || p->head_dim % 2 || p->head_dim > 1024 || p->head_dim_v < 1 || p->head_dim_v > 1024)
    return MAC_ERR_SHAPE;
  if (p->n_q_heads / p->n_kv_heads > 64) return MAC_ERR_SHAPE;
  if (p->window < 1 || p->band < 0 || p->max_chunks < 1 || p->min_chunk < 1 || p->kv_offset < 0) return MAC_ERR_SHAPE;
  if (p->storage < MAC_MODE_F32 || p->storage > MAC_MODE_F64) return MAC_ERR_DTYPE;
  if (p->in_dtype < MAC_DT_F32 || p->in_dtype > MAC_DT_F64) return MAC_ERR_DTYPE;
  if (p->page_size < 1 || p->pages_per_seq < 1) return MAC_ERR_PAGING;
  if (!p->seq_lens || !p->page_table || !p->k_cache || !p->v_cache || !p->rope_freqs || !p->q_pre || !p->k_pre ||
      !p->v_in || !p->out || !p->full_lse || !p->workspace)
    return MAC_ERR_NULL;
  if (need_ring && (!p->ring_q || !p->ring_acc || !p->ring_lse || !p->match_hit || !p->use_hit || !p->match_pos ||
                    !p->match_dist || !p->match_scanned || !p->band_mass))
    return MAC_ERR_NULL;
  if (p->kv_limit < 0) return MAC_ERR_SHAPE;
  if (p->workspace_bytes < workspace_layout(*p).total) return MAC_ERR_WORKSPACE;
  return MAC_OK;
}

enum : int {
  STAGE_APPEND = 1,         // append K/V at m = seq_lens + 1, rotate q
  STAGE_MATCH = 2,          // ring match + decision + plan (both passes of the two-pass match)
  STAGE_AMEND = 4,          // split-KV partials over the plan
  STAGE_COMPLETE = 8,       // merge, output, ring write-back
  STAGE_COMPLETE_FULL = 16, // merge and output only (full-attention modes)
  STAGE_ROTATE = 32,        // rotate q at m = seq_lens, no append
  STAGE_PLAN_FULL = 64,     // plan every group as [1, m] in the append stage
  STAGE_EXPORT = 128,       // this KV shard's (piece, band) partials -> shard_out
  STAGE_SHARDS = 256,       // merge the gathered shard partials, output, ring write-back
  STAGE_SCAN_ONLY = 512,    // with STAGE_MATCH: pass 1 only (profiling)
  STAGE_VERIFY_ONLY = 1024  // with STAGE_MATCH: pass 2 only (profiling)
};

template <int MODE>
static cudaError_t run_step(const MacDecodeParams& p, cudaStream_t st, int mask) {
  cudaError_t e = cudaSuccess;
  const bool app = mask & (STAGE_APPEND | STAGE_ROTATE);
  const int rot = (mask & STAGE_ROTATE) ? 1 : 0, plan = (mask & STAGE_PLAN_FULL) ? 1 : 0;
  if (MODE == MAC_MODE_BF16 && front_fast_supported(p)) {
    const bool fast_match = (mask & STAGE_MATCH) && match_fast_supported(p);
    const int passes = (mask & STAGE_SCAN_ONLY) ? 1 : ((mask & STAGE_VERIFY_ONLY) ? 2 : 3);
    if (app || fast_match) {
      e = launch_front_bf16(p, st, fast_match, app && passes != 2, rot, plan, passes);
      if (e) return e;
    }
    if ((mask & STAGE_MATCH) && !fast_match) { e = launch_match_generic<MODE>(p, st); if (e) return e; }
  } else {
    if (app) { e = launch_append<MODE>(p, st, rot, plan); if (e) return e; }
    if (mask & STAGE_MATCH) { e = launch_match_generic<MODE>(p, st); if (e) return e; }
  }
  const bool fast_amend = MODE == MAC_MODE_BF16 && amend_mma_supported(p);
  if (mask & STAGE_AMEND) {
    if (fast_amend) e = launch_amend_mma_bf16(p, st, plan != 0);
    else e = launch_amend_generic<MODE>(p, st);
    if (e) return e;
  }
  {
    if (mask & STAGE_COMPLETE) { e = launch_complete<MODE>(p, st, 0); if (e) return e; }
    if (mask & STAGE_COMPLETE_FULL) { e = launch_complete<MODE>(p, st, 1); if (e) return e; }
    if (mask & STAGE_EXPORT) { e = launch_complete<MODE>(p, st, 2); if (e) return e; }
    if (mask & STAGE_SHARDS) { e = launch_complete<MODE>(p, st, 3); if (e) return e; }
  }
  return e;
}

static int dispatch(const MacDecodeParams* p, void* stream, int stage_mask, bool need_ring) {
  int v = validate(p, need_ring);
  if (v) return v;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (p->storage) {
    case MAC_MODE_F32: e = run_step<MAC_MODE_F32>(*p, st, stage_mask); break;
    case MAC_MODE_BF16: e = run_step<MAC_MODE_BF16>(*p, st, stage_mask); break;
    default: e = run_step<MAC_MODE_F64>(*p, st, stage_mask); break;
  }
  return (int)e;
}

extern "C" {

int mac_abi_version(void) { return MACATTN_ABI_VERSION; }
size_t mac_params_size(void) { return sizeof(MacDecodeParams); }

const char* mac_error_string(int code) {
  switch (code) {
    case MAC_OK: return "ok";
    case MAC_ERR_NULL: return "macattn: a required pointer is NULL";
    case MAC_ERR_SHAPE: return "macattn: head counts / dims / window / band out of range";
    case MAC_ERR_DTYPE: return "macattn: unknown storage mode or input dtype";
    case MAC_ERR_WORKSPACE: return "macattn: workspace smaller than mac_workspace_bytes()";
    case MAC_ERR_PAGING: return "macattn: invalid page geometry";
    default: return cudaGetErrorString((cudaError_t)code);
  }
}

size_t mac_workspace_bytes(const MacDecodeParams* p) { return p ? workspace_layout(*p).total : 0; }
size_t mac_overflow_flag_offset(const MacDecodeParams* p) { return p ? workspace_layout(*p).ctr_off + 8 : 0; }

#ifdef MAC_TIMELINE
// development builds only (not in macattn.h): byte offset of the timeline stamps in the workspace
size_t mac_timeline_offset(const MacDecodeParams* p) { return p ? workspace_layout(*p).tl_off : 0; }
#endif

int mac_amend_variant(const MacDecodeParams* p) {
  return (p && p->storage == MAC_MODE_BF16 && amend_mma_supported(*p)) ? 1 : 0;
}

int mac_match_path(const MacDecodeParams* p) {
  if (!p || validate(p, false)) return -1;
  int path = 0;
  if (p->storage == MAC_MODE_BF16 && match_fast_supported(*p) && front_two_pass(*p)) {
    path |= MAC_PATH_TWO_PASS;
    path |= verify_per_group(*p) ? MAC_PATH_VERIFY_GROUP : MAC_PATH_VERIFY_HEAD;
    if (dense_deferred(*p)) path |= MAC_PATH_DENSE_KERNEL;
  }
  if (p->storage == MAC_MODE_BF16 && amend_mma_supported(*p)) {
    path |= MAC_PATH_AMEND_MMA;
    if (amend_uses_tma(*p)) path |= MAC_PATH_AMEND_TMA;
  }
  const int nb = (p->storage == MAC_MODE_BF16) ? band_split(*p) : 0;
  return path | (nb << 8);
}

int mac_append_kv(const MacDecodeParams* p, void* stream) { return dispatch(p, stream, STAGE_APPEND, false); }
int mac_match(const MacDecodeParams* p, void* stream) { return dispatch(p, stream, STAGE_MATCH, true); }
int mac_match_scan(const MacDecodeParams* p, void* stream) {
  return dispatch(p, stream, STAGE_MATCH | STAGE_SCAN_ONLY, true);
}
int mac_match_verify(const MacDecodeParams* p, void* stream) {
  return dispatch(p, stream, STAGE_MATCH | STAGE_VERIFY_ONLY, true);
}
int mac_amend(const MacDecodeParams* p, void* stream) { return dispatch(p, stream, STAGE_AMEND, true); }
int mac_complete(const MacDecodeParams* p, void* stream) { return dispatch(p, stream, STAGE_COMPLETE, true); }
int mac_decode_step(const MacDecodeParams* p, void* stream) {
  return dispatch(p, stream, STAGE_APPEND | STAGE_MATCH | STAGE_AMEND | STAGE_COMPLETE, true);
}

int mac_full_decode(const MacDecodeParams* p, void* stream) {
  if (!p) return MAC_ERR_NULL;
  MacDecodeParams q = *p;
  q.force_miss = 1;
  q.band = 0;  // no prefix/band split: one summary over [1, m]
  return dispatch(&q, stream, STAGE_APPEND | STAGE_PLAN_FULL | STAGE_AMEND | STAGE_COMPLETE_FULL, false);
}

int mac_attend_full(const MacDecodeParams* p, void* stream) {
  if (!p) return MAC_ERR_NULL;
  MacDecodeParams q = *p;
  q.force_miss = 1;
  q.band = 0;
  return dispatch(&q, stream, STAGE_ROTATE | STAGE_PLAN_FULL | STAGE_AMEND | STAGE_COMPLETE_FULL, false);
}

int mac_shard_partial(const MacDecodeParams* p, void* stream) {
  if (!p) return MAC_ERR_NULL;
  if (!p->shard_out) return MAC_ERR_NULL;
  return dispatch(p, stream, STAGE_APPEND | STAGE_MATCH | STAGE_AMEND | STAGE_EXPORT, true);
}

int mac_shard_complete(const MacDecodeParams* p, void* stream) {
  if (!p) return MAC_ERR_NULL;
  if (!p->shard_parts) return MAC_ERR_NULL;
  if (p->n_shards < 1) return MAC_ERR_SHAPE;
  return dispatch(p, stream, STAGE_SHARDS, true);
}

int mac_prefill_kv(const MacDecodeParams* p, int32_t n_tokens, void* stream) {
  const int v = validate(p, false);
  if (v) return v;
  if (n_tokens < 0) return MAC_ERR_SHAPE;
  if (n_tokens == 0) return MAC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (p->storage) {
    case MAC_MODE_F32: return (int)launch_prefill_kv<MAC_MODE_F32>(*p, n_tokens, st);
    case MAC_MODE_BF16: return (int)launch_prefill_kv<MAC_MODE_BF16>(*p, n_tokens, st);
    default: return (int)launch_prefill_kv<MAC_MODE_F64>(*p, n_tokens, st);
  }
}

int mac_build_ring(const MacDecodeParams* p, const MacRingBuildParams* rb, void* stream) {
  const int v = validate(p, true);
  if (v) return v;
  if (!rb) return MAC_ERR_NULL;
  if (!ring_build_supported(*p)) return MAC_ERR_SHAPE;
  if (rb->n_rows < 0 || rb->n_rows > p->window || rb->n_chunks < 1) return MAC_ERR_SHAPE;
  if (rb->n_chunks > 1 && !rb->part) return MAC_ERR_NULL;
  if (rb->n_rows == 0) return MAC_OK;
  if (rb->variant < 0 || rb->variant > 2) return MAC_ERR_SHAPE;
  return (int)launch_ring_build(*p, *rb, static_cast<cudaStream_t>(stream), rb->variant == 0 ? -1 : (rb->variant == 2 ? 1 : 0));
}

int mac_step_stats(const MacDecodeParams* p, double* head_stats, double* group_stats, void* stream) {
  if (!p || !head_stats || !group_stats) return MAC_ERR_NULL;
  if (p->batch < 1 || p->n_q_heads < 1 || p->n_kv_heads < 1 || p->n_q_heads % p->n_kv_heads || p->band < 0)
    return MAC_ERR_SHAPE;
  if (p->storage < MAC_MODE_F32 || p->storage > MAC_MODE_F64) return MAC_ERR_DTYPE;
  if (!p->seq_lens || !p->match_hit || !p->use_hit || !p->match_pos || !p->match_scanned || !p->band_mass)
    return MAC_ERR_NULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (p->storage) {
    case MAC_MODE_F32: return (int)launch_step_stats<MAC_MODE_F32>(*p, head_stats, group_stats, st);
    case MAC_MODE_BF16: return (int)launch_step_stats<MAC_MODE_BF16>(*p, head_stats, group_stats, st);
    default: return (int)launch_step_stats<MAC_MODE_F64>(*p, head_stats, group_stats, st);
  }
}

int mac_mass_bound(const MacDecodeParams* p, const MacMassBoundParams* mb, void* stream) {
  if (!p || !mb) return MAC_ERR_NULL;
  if (p->n_kv_heads < 1 || p->head_dim < 1 || (mb->rotate && p->head_dim % 2) || p->head_dim > 256 || p->head_dim_v < 1 ||
      p->head_dim_v > 256 || mb->band < 0 || mb->n_items < 0 || p->kv_offset != 0)
    return MAC_ERR_SHAPE;
  if (p->storage < MAC_MODE_F32 || p->storage > MAC_MODE_F64) return MAC_ERR_DTYPE;
  if (p->page_size < 1 || p->pages_per_seq < 1) return MAC_ERR_PAGING;
  if (!p->page_table || !p->k_cache || !p->v_cache || (mb->rotate && !p->rope_freqs)) return MAC_ERR_NULL;
  if (mb->n_items == 0) return MAC_OK;
  if (!mb->item_req || !mb->item_kv_head || !mb->item_m || !mb->item_p || !mb->q_m || !mb->q_p || !mb->out)
    return MAC_ERR_NULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (p->storage) {
    case MAC_MODE_F32: return (int)launch_mass_bound<MAC_MODE_F32>(*p, *mb, st);
    case MAC_MODE_BF16: return (int)launch_mass_bound<MAC_MODE_BF16>(*p, *mb, st);
    default: return (int)launch_mass_bound<MAC_MODE_F64>(*p, *mb, st);
  }
}

int mac_merge_partials(const MacMergeParams* p, void* stream) {
  if (!p) return MAC_ERR_NULL;
  if (p->n_parts < 1 || p->n_rows < 1 || p->head_dim_v < 1) return MAC_ERR_SHAPE;
  if (p->dtype != MAC_DT_F32 && p->dtype != MAC_DT_F64) return MAC_ERR_DTYPE;
  if (!p->part_acc || !p->part_lse || !p->out_acc || !p->out_lse) return MAC_ERR_NULL;
  return (int)launch_merge_partials(*p, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
