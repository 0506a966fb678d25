/*
 * macattn.h — C-ABI of the B200-native MAC-Attention decode path.
 *
 * The reference (`attnreuse`, /root/reference/pkg/src/attnreuse) is an
 * in-process Python API with no FFI; the entry points below are what a
 * binding of its hot path would call.  Each replaces one piece of
 * `DecodeEngine.decode_step` (engine.py:410-539):
 *
 *   mac_append_kv     engine.py:434-437   rotate k at position m, append K/V
 *                     (+ attention.py:212-232 rope_rotate, kvstore.py:105-119 append)
 *                     and rotate the step's queries (engine.py:460)
 *   mac_match         matching.py:141-175 match_query over the pre-RoPE ring,
 *                     engine.py:449-459   with the roi / refresh gates
 *   mac_amend         engine.py:464-470,484-493  split-KV partial summaries over
 *                     [lo, m] cut at m-r (attention.py:75-116 summarize)
 *   mac_complete      engine.py:471-479,486-502  cached(p) (+) piece (+) band merge
 *                     (attention.py:119-135), output, band mass, and the ring
 *                     write-back rectify_append (engine.py:374-402)
 *   mac_decode_step   the four above, in stream order (one decode_step call)
 *   mac_full_decode   append + exact attention over [1, m] (attention.py:182-189
 *                     attend_full): the full-attention decode baseline
 *   mac_attend_full   exact attention of R_m q over the stored [1, m], m = seq_lens
 *                     (no append): the per-step fidelity oracle (engine.py:507-509)
 *   mac_merge_partials  log-domain merge of per-shard (acc, lse) partials
 *                     (attention.py:119-135 merge) for the KV-sharded miss path
 *   mac_prefill_kv    bulk KV append of a prompt (engine.py:434-437 applied to n tokens)
 *   mac_shard_partial / mac_shard_complete  decode_step split around the one
 *                     cross-GPU exchange of the KV-sharded path (all-gather of
 *                     per-shard (piece, band) summaries, then the merge)
 *   mac_step_stats    DecodeMetrics.record_hit / record_miss (engine.py:188-205)
 *                     and group_kv_span (engine.py:66-77, :525-528) accumulated
 *                     on the device per head after a step
 *   mac_mass_bound    mass_bound_check (engine.py:246-281), offline, over the
 *                     paged cache
 *   mac_build_ring    the ring entries of the last n prompt positions from the
 *                     cached KV in one GEMM-form pass (what n forced-miss decode steps
 *                     write, engine.py:374-402 + 484-499)
 *
 * The reference's public building blocks on plain device arrays (f64 math):
 *   mac_summarize     summarize / attend_full (attention.py:75-116,182-189) for many
 *                     query rows, each over its own key range, q optionally rotated
 *                     at t first: also the batched causal oracle_outputs
 *                     (engine.py:542-572)
 *   mac_remove_summaries  remove() and its guards (attention.py:138-172)
 *   mac_rope_rotate   rope_rotate (attention.py:212-232)
 *   mac_match_rows    match_query (matching.py:141-175) over QueryRing arrays
 *
 * Conventions: plain device pointers and sizes, no allocation inside, every
 * launch is stream-ordered and graph-capturable (no host synchronisation).
 * Return value 0 on success, a MAC_ERR_* code for a rejected parameter set,
 * or a cudaError_t value (< 1000) from the launch.
 */
#ifndef MACATTN_H_
#define MACATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MACATTN_ABI_VERSION 14
/* dims of the planar query-ring copy the two-pass scan streams (ring_qp) */
#define MAC_PLANAR_DIMS 8

/* storage modes: dtype of the K/V cache and the query ring; summaries are
 * f32 in MAC_MODE_F32/BF16 and f64 in MAC_MODE_F64 (engine.py:152-153 allows
 * f32|f64; bf16 is the B200 serving storage) */
enum { MAC_MODE_F32 = 0, MAC_MODE_BF16 = 1, MAC_MODE_F64 = 2 };
/* element dtypes of the per-step inputs q_pre / k_pre / v */
enum { MAC_DT_F32 = 0, MAC_DT_BF16 = 1, MAC_DT_F64 = 2 };
/* matching.py:25-26 */
enum { MAC_MATCH_PRE_ROPE = 0, MAC_MATCH_POST_ROPE = 1 };
/* engine.py:41-42 */
enum { MAC_DOWNDATE_SPLIT = 0, MAC_DOWNDATE_REMOVE = 1 };

enum {
  MAC_OK = 0,
  MAC_ERR_NULL = 1001,      /* a required pointer is NULL */
  MAC_ERR_SHAPE = 1002,     /* head counts / dims / window / band out of range */
  MAC_ERR_DTYPE = 1003,     /* unknown storage mode or input dtype */
  MAC_ERR_WORKSPACE = 1004, /* workspace smaller than mac_workspace_bytes() */
  MAC_ERR_PAGING = 1005     /* page geometry invalid */
};

typedef struct MacDecodeParams {
  /* ---- geometry -------------------------------------------------------- */
  int32_t batch;         /* B requests */
  int32_t n_q_heads;     /* Hq */
  int32_t n_kv_heads;    /* Hkv, Hq % Hkv == 0 (engine.py:138-139) */
  int32_t head_dim;      /* d, even (engine.py:132-133) */
  int32_t head_dim_v;    /* d_v */
  int32_t window;        /* W, ring capacity (engine.py:115) */
  int32_t band;          /* r (engine.py:116) */
  int32_t page_size;     /* tokens per KV page (kvstore.py:76) */
  int32_t pages_per_seq; /* row stride of page_table */
  int32_t storage;       /* MAC_MODE_* */
  int32_t in_dtype;      /* MAC_DT_* of q_pre / k_pre / v_in */
  int32_t max_chunks;    /* split-KV partial slots per (request, kv head) */
  int32_t min_chunk;     /* minimum tokens per split */
  int32_t kv_offset;     /* tokens of this request held by earlier KV shards (0 unless sharded) */
  int32_t kv_limit;      /* tokens this KV shard holds (positions kv_offset+1 .. kv_offset+kv_limit);
                            0: unbounded (the tail shard, or no sharding) */
  int32_t n_shards;      /* partials in shard_parts (mac_shard_complete) */
  int32_t span_chunks;   /* splits of a span planned without the split band (full attention, the
                            one-pass miss path); 0 or >= max_chunks: max_chunks.  The split band's
                            long (miss) pieces use every slot: 0 < span_chunks < max_chunks leaves
                            full attention at its best split while a hit step's few missing groups
                            spread over the whole amend grid */
  /* ---- match rule (matching.py:58-64, 141-175; engine.py:452-459) ----- */
  double thr_sq;         /* (sqrt(2d)(1 - tau_layer))^2 */
  int32_t delta_max;     /* <= 0: off */
  int32_t match_space;   /* MAC_MATCH_* */
  int32_t refresh_every; /* 0: off */
  int32_t roi_gate;      /* break_even_gate (engine.py:57-63) */
  double roi_b_kv;
  double roi_b_q;
  int32_t downdate;      /* MAC_DOWNDATE_* */
  int32_t force_miss;    /* 1: every head takes the miss path */
  double eps_cancel;     /* remove() guard (attention.py:142) */
  /* ---- persistent state (device) --------------------------------------- */
  int32_t* seq_lens;          /* [B] tokens stored before this step; the step stores m = seq_lens+1 */
  const int32_t* page_table;  /* [B, pages_per_seq] physical page ids */
  void* k_cache;              /* [num_pages, Hkv, page_size, d]   post-RoPE keys, storage dtype */
  void* v_cache;              /* [num_pages, Hkv, page_size, d_v] values, storage dtype */
  void* ring_q;               /* [B, Hq, W, d]   pre-RoPE queries, storage dtype */
  void* ring_acc;             /* [B, Hq, W, d_v] prefix summary acc (f32 | f64) */
  void* ring_lse;             /* [B, Hq, W]      prefix summary lse (-inf: empty) */
  void* ring_qp;              /* optional [B, Hq, W, MAC_PLANAR_DIMS] bf16: dims 0..7 of every
                                 ring_q row, contiguous per head (32 B per row), kept in step by
                                 the ring write-back; pass 1 of the two-pass scan of the bf16
                                 d = 128 path streams it (NULL: it reads the strided row prefixes
                                 of ring_q) */
  const double* rope_freqs;   /* [d/2] omega_j = base^(-2j/d) (attention.py:208-209) */
  /* ---- per-step inputs (device) ---------------------------------------- */
  const void* q_pre;          /* [B, Hq, d]   pre-RoPE queries */
  const void* k_pre;          /* [B, Hkv, d]  pre-RoPE keys */
  const void* v_in;           /* [B, Hkv, d_v] values */
  /* ---- per-step outputs (device) --------------------------------------- */
  void* out;                  /* [B, Hq, d_v] attention output (f32 | f64) */
  int32_t* match_hit;         /* [B, Hq] raw match decision (MatchResult.hit) */
  int32_t* use_hit;           /* [B, Hq] decision after the gates (reuse taken) */
  int32_t* match_pos;         /* [B, Hq] p, -1 on a raw miss */
  double* match_dist;         /* [B, Hq] best squared distance, +inf if nothing scanned */
  int32_t* match_scanned;     /* [B, Hq] candidates scanned */
  void* full_lse;             /* [B, Hq] lse of the full summary (f32 | f64) */
  void* band_mass;            /* [B, Hq] rho = exp(band.lse - full.lse) (f32 | f64) */
  void* cached_acc;           /* optional [B, Hq, d_v]: summary reused at p (NULL: not written) */
  void* cached_lse;           /* optional [B, Hq] */
  int32_t* fallbacks;         /* optional [B, Hq]: 1 when remove() fell back to the split prefix */
  void* out_bf16;             /* optional [B, Hq, d_v] bf16: the output narrowed, written by the bf16
                                 d = 128 complete beside `out` — e.g. the device alias of a pinned
                                 host buffer, so the step's result reaches the host with no copy */
  /* ---- KV-sharded miss path ------------------------------ */
  void* shard_out;            /* [B, Hq, 2, d_v+1] this shard's (piece, band) partials: acc..., lse */
  const void* shard_parts;    /* [n_shards, B, Hq, 2, d_v+1] every shard's partials, rank order */
  /* ---- scratch --------------------------------------------------------- */
  void* workspace;
  size_t workspace_bytes;
  /* ---- match-scan choice (bf16 d = 128 path) ------------------------------ */
  int32_t match_mode;         /* 0: by geometry (two-pass scan + verify for rings of 512..1024 rows
                                 and enough heads); 1: one-pass scan; 2: two-pass with the full
                                 walks of heads without a near-repeat spread over the GPU
                                 (dense_kernel; per-group verify geometry, else as 0).  Both take the argmin of an fp32
                                 sum of squares, associated differently: only a near-tie below
                                 fp32 resolution can resolve differently (pin the mode for
                                 bitwise reproducible decisions) */
  int32_t* feedback;          /* optional int32[2] (e.g. a pinned host buffer's device alias):
                                 {heads that missed, heads} over the steps since the last
                                 publication, stored at the start of every 8th step (the complete
                                 kernel counts, the append warps publish) */
  int32_t inputs_host;        /* 1: q_pre / k_pre / v_in are device aliases of pinned host memory
                                 (zero-copy).  On the two-pass bf16 d = 128 path the step reads
                                 them over the host link once: the scan its MAC_PLANAR_DIMS query dims, the
                                 append warps the rest, staging q in the workspace for the later
                                 kernels — no separate input copy before the step */
} MacDecodeParams;

/* Per-shard (acc, lse) partial merge for the KV-sharded miss path. */
typedef struct MacMergeParams {
  int32_t n_parts;       /* G partials per row */
  int32_t n_rows;        /* rows (request x head) */
  int32_t head_dim_v;
  int32_t dtype;         /* MAC_DT_F32 | MAC_DT_F64 */
  const void* part_acc;  /* [G, n_rows, d_v] normalised acc */
  const void* part_lse;  /* [G, n_rows] lse (-inf: empty) */
  void* out_acc;         /* [n_rows, d_v] */
  void* out_lse;         /* [n_rows] */
} MacMergeParams;

/* Per-head decision statistics accumulated by mac_step_stats (f64 counters, summed
 * over the batch): head_stats is [Hq, MAC_STAT_COUNT], group_stats [Hkv, MAC_GSTAT_COUNT].
 * Fields follow DecodeMetrics (engine.py:167-186). */
enum {
  MAC_STAT_STEPS = 0,      /* decisions */
  MAC_STAT_HITS = 1,       /* reuses taken (use_hit) */
  MAC_STAT_FORCED = 2,     /* raw hits the gates turned into misses */
  MAC_STAT_FALLBACKS = 3,  /* remove() fell back to the split prefix */
  MAC_STAT_SKIP_SUM = 4,   /* sum of (p - r)+ / m over hits */
  MAC_STAT_KV_READ = 5,    /* tokens read: m - (p - r)+ on a hit, m on a miss */
  MAC_STAT_KV_FULL = 6,    /* tokens of full attention: m */
  MAC_STAT_GAP_SUM = 7,    /* sum of m - p over hits */
  MAC_STAT_RHO_SUM = 8,    /* sum of the band mass rho */
  MAC_STAT_CANDIDATES = 9, /* ring rows scanned */
  MAC_STAT_COUNT = 10
};
enum { MAC_GSTAT_KV_TOKENS = 0, MAC_GSTAT_KV_TOTAL = 1, MAC_GSTAT_COUNT = 2 };

/* Items of mac_mass_bound: one hit each, keys / values [1, p] of (request, kv head)
 * read from the paged cache described by the MacDecodeParams. */
typedef struct MacMassBoundParams {
  int32_t n_items;
  int32_t band;                 /* r */
  int32_t rotate;               /* 1: q_m / q_p are pre-RoPE, rotated at m / p in-kernel; 0: post-RoPE */
  const int32_t* item_req;      /* [n] request (page_table row) */
  const int32_t* item_kv_head;  /* [n] */
  const int32_t* item_m;        /* [n] position of the current query */
  const int32_t* item_p;        /* [n] hit position p >= 1 */
  const double* q_m;            /* [n, d] current query */
  const double* q_p;            /* [n, d] the ring query stored at p */
  double* out;                  /* [n, 2] (lhs, rhs) of engine.py:246-281 */
} MacMassBoundParams;

/* summarize (attention.py:75-116) for n_sets * q_per_set query rows.  Query set s reads key
 * set s / sets_per_kv (GQA); row i of a set covers keys [lo, hi] (1-based, inclusive; an
 * empty range gives the empty summary acc = 0, lse = -inf).  Scale 1/sqrt(head_dim). */
typedef struct MacSummarizeParams {
  int32_t n_sets;
  int32_t q_per_set;
  int32_t n_keys;           /* rows per key set */
  int32_t sets_per_kv;      /* query sets per key set (>= 1) */
  int32_t head_dim;         /* d, even, <= 1024 */
  int32_t head_dim_v;       /* d_v <= 256 */
  int32_t dtype;            /* MAC_DT_F32 | MAC_DT_F64 of q / keys / values */
  const void* q;            /* [n_sets, q_per_set, d] */
  const void* keys;         /* [n_sets / sets_per_kv, n_keys, d] */
  const void* values;       /* [n_sets / sets_per_kv, n_keys, d_v] */
  const int32_t* lo;        /* optional [n_sets * q_per_set] first key; NULL: 1 */
  const int32_t* hi;        /* optional [n_sets * q_per_set] last key; NULL: n_keys */
  const int32_t* rope_t;    /* optional [n_sets * q_per_set]: rotate q at this position first */
  const double* rope_freqs; /* [d/2], needed with rope_t */
  double* out_acc;          /* [n_sets * q_per_set, d_v] */
  double* out_lse;          /* [n_sets * q_per_set] */
} MacSummarizeParams;

/* match_query (matching.py:141-175) for n_rings independent rings of explicit positions. */
typedef struct MacMatchRowsParams {
  int32_t n_rings;
  int32_t capacity;         /* rows per ring (stride) */
  int32_t head_dim;
  int32_t delta_max;        /* <= 0: off */
  int32_t post_rope;        /* 1: candidates rotated by R(pos - m) first (matching.py:165-168) */
  double thr_sq;            /* threshold(d, tau)^2; hit iff best < thr_sq */
  const double* rope_freqs; /* [d/2], needed with post_rope */
  const double* q;          /* [n_rings, d] */
  const double* ring_q;     /* [n_rings, capacity, d] */
  const double* ring_sqnorm;/* [n_rings, capacity] cached |c|^2 (matching.py:109) */
  const int64_t* ring_pos;  /* [n_rings, capacity] */
  const int32_t* n_live;    /* [n_rings] live rows (the first n_live of each ring) */
  const int32_t* m;         /* [n_rings] current position */
  int32_t* out_hit;
  int32_t* out_pos;         /* -1 on a miss */
  double* out_dist;         /* +inf when nothing was scanned */
  int32_t* out_scanned;
} MacMatchRowsParams;

/* mac_build_ring: positions seq_lens[b] - n_rows + 1 .. seq_lens[b] of every request, whose K/V
 * is already in the paged cache; q_pre is [B, n_rows, Hq, d] (their pre-RoPE queries, in_dtype). */
typedef struct MacRingBuildParams {
  int32_t n_rows;     /* 1 .. min(window, seq_lens[b]) */
  int32_t n_chunks;   /* key splits per row block (>= 1); > 1 needs `part` */
  void* part;         /* [B, n_rows, Hq, n_chunks, d_v + 1] f32 scratch (NULL when n_chunks == 1) */
  int32_t variant;    /* 0: tcgen05 kernel where supported (else mma.sync), 1: mma.sync, 2: tcgen05 */
} MacRingBuildParams;

int mac_abi_version(void);
size_t mac_params_size(void);
const char* mac_error_string(int code);
/* bytes of scratch the decode entry points need for this geometry */
size_t mac_workspace_bytes(const MacDecodeParams* p);
/* byte offset in the workspace of a sticky uint32 flag that an append sets when a token has no
 * page in its request's page_table row (the token is then not stored); 0 while every append fit */
size_t mac_overflow_flag_offset(const MacDecodeParams* p);
/* which kernel family mac_amend would launch: 0 generic CUDA-core, 1 bf16 tensor-core (mma) */
int mac_amend_variant(const MacDecodeParams* p);

/* which kernels mac_decode_step launches for this parameter set (host-side decision, no launch):
 * a bit set of MAC_PATH_* plus, in bits 8-15, the split-band items per GQA group (0: the band
 * rides in the plan); -1 for an invalid parameter set.  Tests use it to prove which path ran. */
enum {
  MAC_PATH_TWO_PASS = 1,      /* two-pass match: planar scan + verify kernel */
  MAC_PATH_VERIFY_GROUP = 2,  /* verify: one CTA per GQA group */
  MAC_PATH_VERIFY_HEAD = 4,   /* verify: one CTA per head */
  MAC_PATH_AMEND_MMA = 8,     /* bf16 d = 128 tensor-core amend (else the generic CUDA-core amend) */
  MAC_PATH_DENSE_KERNEL = 16, /* match_mode 2: heads with no near-repeat are walked by dense_kernel */
  MAC_PATH_AMEND_TMA = 32     /* the hit step's amend is the TMA-fed kernel (few GQA groups) */
};
int mac_match_path(const MacDecodeParams* p);

int mac_append_kv(const MacDecodeParams* p, void* stream);
int mac_match(const MacDecodeParams* p, void* stream);
/* mac_match as its two passes (profiling; the bf16 d=128 path with >= 148 GQA groups):
 * the ring scan (first-half distances) and the verification + decision + plan.  Where
 * the match runs in one pass, mac_match_scan is the whole match and mac_match_verify is
 * a no-op. */
int mac_match_scan(const MacDecodeParams* p, void* stream);
int mac_match_verify(const MacDecodeParams* p, void* stream);
int mac_amend(const MacDecodeParams* p, void* stream);
int mac_complete(const MacDecodeParams* p, void* stream);
int mac_decode_step(const MacDecodeParams* p, void* stream);
int mac_full_decode(const MacDecodeParams* p, void* stream);
int mac_attend_full(const MacDecodeParams* p, void* stream);
int mac_merge_partials(const MacMergeParams* p, void* stream);
/* KV-sharded step, half 1: append (stored only by the shard holding position m),
 * match, plan clamped to this shard's tokens, amend, and the per-head (piece,
 * band) partials of this shard into shard_out.  Rings and seq_lens untouched. */
int mac_shard_partial(const MacDecodeParams* p, void* stream);
/* half 2, after the caller gathered every shard's shard_out into shard_parts:
 * cached(p) (+) pieces (+) bands in rank order, output, rho, ring write-back,
 * seq_lens advance.  Every shard computes the same result. */
int mac_shard_complete(const MacDecodeParams* p, void* stream);
/* prefill, bulk half: append n_tokens tokens per request at positions seq_lens+1 ..
 * seq_lens+n_tokens (k_pre / v_in are token-major [B, n_tokens, Hkv, d]), keys RoPE'd
 * in-kernel, then seq_lens += n_tokens.  No ring work (the reference fills rings one
 * decode step at a time, engine.py:374-402; see BatchDecodeEngine.prefill). */
int mac_prefill_kv(const MacDecodeParams* p, int32_t n_tokens, void* stream);
/* after a decode step: add its per-head decisions (match_hit, use_hit, match_pos,
 * match_scanned, band_mass, fallbacks, seq_lens = m) into head_stats / group_stats.
 * Only the fields listed are read; the step's other buffers may be NULL. */
int mac_step_stats(const MacDecodeParams* p, double* head_stats, double* group_stats, void* stream);
/* mass_bound_check for n_items hits; p supplies the cache geometry (storage, dims,
 * page_table, k_cache, v_cache, rope_freqs); d, d_v <= 256; no KV sharding. */
int mac_mass_bound(const MacDecodeParams* p, const MacMassBoundParams* mb, void* stream);
/* step I/O without the copy engines (StepGraph): the device alias of a pinned host
 * buffer (cudaHostGetDevicePointer), and a stream-ordered copy kernel between device and
 * pinned-host aliases, same dtype or f32 -> bf16 (MAC_DT_*); pointers 16-byte aligned,
 * n_elems * element size a multiple of 16 (of 8 elements when narrowing). */
int mac_host_alias(void* host, void** device_alias);
int mac_io_copy(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, size_t n_elems, void* stream);

int mac_summarize(const MacSummarizeParams* p, void* stream);
/* remove(a, band) row-wise in f64; status[row]: 0 ok, 1 CancellationError (|a.lse - band.lse|
 * < eps_cancel), 2 MassExceededError (band.lse > a.lse + eps_cancel).  Token-count checks
 * (attention.py:156-162) are the caller's. */
int mac_remove_summaries(int32_t n_rows, int32_t head_dim_v, const double* a_acc, const double* a_lse,
                         const double* band_acc, const double* band_lse, double eps_cancel, double* out_acc,
                         double* out_lse, int32_t* status, void* stream);
/* out[i] = R(t[i]) x[i] for n_rows rows of head_dim (interleaved pairs, f64 angles) */
int mac_rope_rotate(int32_t n_rows, int32_t head_dim, const double* x, const double* t, const double* rope_freqs,
                    double* out, void* stream);
int mac_match_rows(const MacMatchRowsParams* p, void* stream);
/* Ring entries (ring_q, ring_qp, ring_acc, ring_lse) of the last rb->n_rows positions of every
 * request from the cached KV: slot (t-1) % W <- (q_t, AS[1, t-r] under R_t q_t).  bf16 d = 128
 * storage with 8 % (Hq / Hkv) == 0, page_size % 16 == 0, unsharded (else MAC_ERR_SHAPE: callers
 * then run forced-miss decode steps).  Tensor-core pass; no seq_lens change. */
int mac_build_ring(const MacDecodeParams* p, const MacRingBuildParams* rb, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MACATTN_H_ */
