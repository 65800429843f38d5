/*
 * sals.h — C ABI of the B200-native SALS decode-attention hot path
 * (Sparse Attention in Latent Space, arXiv 2510.24273).
 *
 * Citations: "P:n" = line n of the paper's LaTeX; "S:n" = SPEC.md.
 *
 * Conventions shared by every entry point
 *  - Tensor arguments are DEVICE pointers (cudaMalloc / torch CUDA storage)
 *    owned by the caller, row-major, 16-byte aligned, contiguous.  The
 *    decode path allocates nothing and keeps no state between calls (the
 *    exceptions: the opaque communicator of sals_comm_init, owned by the
 *    caller, and the thread-local cuBLAS / cuSOLVER handles the prefill and
 *    calibration calls create on first use).
 *  - `stream` is a cudaStream_t passed as void*.  Every call only enqueues
 *    work on that stream (no host synchronisation), so all calls are CUDA-graph
 *    capturable.  Kernels are launched with programmatic dependent launch.
 *  - Argument errors are detected on the host and returned synchronously with
 *    nothing enqueued.  Launch failures return SALS_ERR_CUDA; asynchronous
 *    device faults surface at the caller's next synchronisation.
 *    sals_last_error() returns a thread-local message for the last failure.
 *  - Element type of U, q, k_new, v_new, caches and out is cfg->dtype
 *    (SALS_F32 or SALS_BF16); accumulation is always fp32.
 *  - Notation: B = batch, s_b = tokens of request b INCLUDING the
 *    token being decoded (positions 0..s_b-1, query at s_b-1), n_q / n_kv query
 *    / KV heads, G = n_q/n_kv (query head h reads KV head h/G), d = head_dim,
 *    D = n_kv*d (the paper's "nd"), r = rank, r* = score_rank, k = top_k.
 */
#ifndef SALS_H_
#define SALS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SALS_OK = 0,
  SALS_ERR_INVALID_ARGUMENT = 1,   /* shape / pointer / range violation */
  SALS_ERR_UNSUPPORTED = 2,        /* shape outside the kernels' limits (see each call) */
  SALS_ERR_WORKSPACE_TOO_SMALL = 3,
  SALS_ERR_CUDA = 4,
  SALS_ERR_NCCL = 5                /* NCCL missing or a collective failed (sals_decode_sharded) */
} sals_status;

typedef enum { SALS_F32 = 0, SALS_BF16 = 1 } sals_dtype;

/* RoPE pairing (the paper is silent): HALF rotates (i, i+d/2) (HF
 * rotate_half), INTERLEAVED rotates (2i, 2i+1). */
typedef enum { SALS_ROPE_HALF = 0, SALS_ROPE_INTERLEAVED = 1 } sals_rope_style;

/* Reconstruction + attention path.  AUTO picks TCGEN05 when the selected-row
 * reconstruction is a real dense contraction (bf16, B*k >= 128 rows,
 * d in {64,128,256}, D % 256 == 0), SIMT otherwise. */
typedef enum { SALS_PATH_AUTO = 0, SALS_PATH_SIMT = 1, SALS_PATH_TCGEN05 = 2 } sals_path;

/* The problem statement of Algorithm 1: heads, head_dim, rank r,
 * score rank r*, budget k, RoPE base, GQA grouping. */
typedef struct {
  int32_t num_q_heads;    /* n_q; n_q % n_kv == 0 (contiguous GQA groups)            */
  int32_t num_kv_heads;   /* n_kv                                                     */
  int32_t head_dim;       /* d: even, one of 16, 32, 64, 128, 256                     */
  int32_t rank;           /* r: 1 <= r <= D, r % 8 == 0 (P:358 U_r in R^{nd x r})     */
  int32_t score_rank;     /* r*: 1 <= r* <= r, r* % 8 == 0; paper: r* = r/2   */
  int32_t top_k;          /* k >= 1 (Alg. 1 line 5)                                   */
  int32_t sink;           /* x: first x positions always selected; 0 = pure Alg. 1 */
  int32_t recent;         /* z: last z positions always selected; sink + recent <= k  */
  float   rope_base;      /* theta base of RoPE (model config; the paper never states it) */
  int32_t rope_style;     /* sals_rope_style                                          */
  int32_t dtype;          /* sals_dtype of every tensor argument                      */
  float   softmax_scale;  /* 0 => 1/sqrt(head_dim) (Alg. 1 line 8)             */
  int32_t path;           /* sals_path                                                */
  int32_t v_bits;         /* value cache format: 0 or 16 = dtype
                             values; 4 or 2 = channel-wise group quantised (groups of 32
                             channels of one token, asymmetric min/max grid, bf16 scale / zero),
                             bf16 + head_dim 128 + the tcgen05 path only.  Row layout per
                             token: for every KV head, d*v_bits/8 code bytes (4-bit: two
                             channels per byte, low nibble first; 2-bit: four, lowest bits
                             first) then d/32 (bf16 scale, bf16 zero) pairs.  v = zero + scale*code */
} sals_config;

/* Bytes of one token's row of the value cache (D * sizeof(dtype), or the
 * quantised layout above).  0 on invalid arguments. */
size_t sals_v_row_bytes(const sals_config* cfg);
/* Bytes of a value cache of `batch` requests x `cap` rows.  With v_bits 4 / 2
 * and recent = w > 0 the high-precision recent window ("tokens in the
 * most recent window are compressed by only 50%", aligned with the forced recent
 * window of the selection) follows the rows: a ring [batch, w, n_kv * 144] of
 * 8-bit rows (128 code bytes + 4 (bf16 scale, bf16 zero) per head), slot
 * pos % w; the decode reads positions >= s_b - w from it.  Not with the sharded
 * calls. */
size_t sals_v_cache_bytes(const sals_config* cfg, int32_t batch, int64_t cap);
/* The ring sits at byte offset batch * cap * sals_v_row_bytes(cfg) of the value
 * cache, so with v_bits 4 / 2 and recent > 0, sals_append_latent, sals_decode and
 * sals_append_decode must be called with the `batch` the cache was allocated for
 * (a call on the first B' < B requests would address another ring). */

/* Bytes of device workspace sals_decode needs for `batch` requests of at most
 * `max_seq_len` tokens.  0 on invalid arguments. */
size_t sals_workspace_bytes(const sals_config* cfg, int32_t batch, int32_t max_seq_len);

/*
 * sals_append_latent — Algorithm 1 lines 2-3 for the new token (
 * Eq. 1): k~ = U^T k_new (fp32 accumulate, rounded to dtype) is
 * written to latent_cache[b, d_pos[b], :], and v_new[b] to v_cache[b, d_pos[b], :].
 *   U            [D, r]       column-orthonormal projection, columns in
 *                             descending-eigenvalue order
 *   k_new        [B, D]       PRE-RoPE keys of the new token
 *   v_new        [B, D]       values of the new token
 *   d_pos        [B] int32    device: slot (= absolute position) of the new token, 0 <= pos < cap
 *   latent_cache [B, cap, r]  written in place (row d_pos[b] only)
 *   v_cache      [B, cap, D]  written in place (row d_pos[b] only); with cfg->v_bits 4 / 2:
 *                [B, cap, sals_v_row_bytes(cfg)] bytes, v_new quantised into the row
 * Must precede sals_decode of the same step on the same stream (Alg. 1 appends
 * before scoring).
 */
sals_status sals_append_latent(const sals_config* cfg, const void* U, const void* k_new,
                               const void* v_new, int32_t batch, const int32_t* d_pos,
                               void* latent_cache, void* v_cache, int64_t cap, void* stream);

/*
 * sals_decode — Algorithm 1 lines 2 and 4-9 for a batch of
 * independent requests:
 *   q~ = U[:, :r*]^T q_bar          q_bar = sum of the query heads of a KV group
 *                                   (reading R1; = q for MHA)
 *   p'_j = q~ . K~[b, j, :r*]        j < s_b
 *   C_b = [0,x) u [s_b-z, s_b) u TopK over [x, s_b-z) of k-x-z tokens, ties to
 *         the lower index; all s_b tokens when s_b <= k   (line 5)
 *   K_C = K~[b, C_b, :] U^T, reshaped to [|C|, n_kv, d]      (line 6)
 *   q^R = RoPE_{s_b-1}(q), K^R_C = RoPE_j(K_C) at the original positions j
 *   y = softmax(q^R K^R_C^T * scale) V[b, C_b]                (lines 7-9, Eq. 6)
 *   U            [D, r]
 *   q            [B, n_q*d]       PRE-RoPE queries of the decoded token
 *   latent_cache [B, cap, r]      rows 0..s_b-1 valid (append already done)
 *   v_cache      [B, cap, D]      (or [B, cap, sals_v_row_bytes(cfg)] bytes with cfg->v_bits 4 / 2)
 *   d_seq_len    [B] int32        device: s_b, 1 <= s_b <= min(cap, max_seq_len)
 *   max_seq_len  host upper bound of every s_b (sizes grids; no device read)
 *   out          [B, n_q*d]       attention output y
 *   sel_idx_out  [B, k] int32 or NULL: C_b ascending, -1 padded past min(k, s_b)
 *   scores_out   [B, max_seq_len] fp32 or NULL: p' (debug / parity)
 *   workspace    >= sals_workspace_bytes(cfg, batch, max_seq_len) bytes, 256-B aligned
 * Limits (SALS_ERR_UNSUPPORTED): max_seq_len <= 380928 (16-CTA top-k cluster), batch <= 65535,
 * n_q/n_kv <= 8.
 */
sals_status sals_decode(const sals_config* cfg, const void* U, const void* q,
                        const void* latent_cache, const void* v_cache, int64_t cap,
                        int32_t batch, const int32_t* d_seq_len, int32_t max_seq_len,
                        void* out, int32_t* sel_idx_out, float* scores_out,
                        void* workspace, size_t ws_bytes, void* stream);

/*
 * sals_append_latent_bulk -- prefill: Eq. 1 / Alg. 1 line 3
 * for n_tokens consecutive tokens of every request at once:
 *   latent_cache[b, start + i, :] = U^T k[b, i, :],  v_cache[b, start + i, :] = v[b, i, :]
 *   k, v    [B, n_tokens, D]  PRE-RoPE keys / values (device)
 *   start   host: slot of token 0 (the same for every request), start + n_tokens <= cap
 * bf16 with D and r multiples of 64: the in-build tcgen05 GEMM (TMA-fed, fp32
 * accumulation in TMEM, rounded to bf16 in the epilogue), written straight into
 * the cache rows; other shapes / fp32: cuBLAS (fp32 accumulate) with a cuBLAS
 * handle created on the calling thread's first call per device.
 * Value rows: copied as dtype, or with cfg->v_bits 4 / 2 (bf16, head_dim 128)
 * quantised per token exactly as sals_append_latent does (R15: codes, bf16 scale
 * and zero), and with recent = w > 0 the LAST w tokens of the block also written
 * into the 8-bit recent-window ring (slot pos % w; call with the cache's
 * allocation batch, as for the other calls).
 */
sals_status sals_append_latent_bulk(const sals_config* cfg, const void* U, const void* k, const void* v,
                                    int32_t batch, int32_t n_tokens, int64_t start, void* latent_cache,
                                    void* v_cache, int64_t cap, void* stream);

/*
 * sals_calibrate -- offline calibration of the latent basis (
 * Sec. 4.2): C = K^T K over the stacked pre-RoPE calibration keys,
 * C = U S U^T, U_r = the leading r = cfg->rank eigenvectors.
 *   K            [n_rows, D] device, dtype (heads merged: D = n_kv * d)
 *   U_out        [D, r] device, dtype: columns in descending eigenvalue order
 *                (so the first r* columns span the score subspace), each column
 *                signed so that its largest-magnitude component is positive
 *   eigvals_out  [D] fp32 device or NULL: eigenvalues of C, descending
 *   workspace    >= sals_calibrate_workspace_bytes(cfg) bytes (D^2 fp32 + solver)
 * Gram matrix on cuBLAS (fp32 accumulate), eigensolver cuSOLVER syevd (fp32);
 * library-owned cuBLAS / cuSOLVER handles per calling thread.  Synchronises
 * internally (cuSOLVER); not for the decode hot path.
 */
size_t sals_calibrate_workspace_bytes(const sals_config* cfg);
sals_status sals_calibrate(const sals_config* cfg, const void* K, int64_t n_rows, void* U_out, float* eigvals_out,
                           void* workspace, size_t ws_bytes, void* stream);

/*
 * sals_append_decode -- sals_append_latent followed by sals_decode for the same
 * step in ONE call (Alg. 1 lines 2-9): the new token's latent row
 * (k~ = U^T k_new) and value row are written at slot d_seq_len[b] - 1, and the
 * append's projection shares one launch with the query projection (U is read
 * once for both).  Arguments as for the two calls; latent_cache and v_cache are
 * written (row d_seq_len[b] - 1 only).  The cache rows it writes are identical to
 * sals_append_latent(..., d_pos = d_seq_len - 1, ...)'s; the decode that follows is
 * sals_decode's arithmetic, except that for D > 2048 the shared launch splits the
 * query projection over a different cluster shape (fp32 summation order of q~ and
 * hence of the scores may differ in the last bits; the selection then agrees except
 * inside the tie band).  Parity against the oracle is tested for this call itself.
 */
sals_status sals_append_decode(const sals_config* cfg, const void* U, const void* k_new, const void* v_new,
                               const void* q, void* latent_cache, void* v_cache, int64_t cap, int32_t batch,
                               const int32_t* d_seq_len, int32_t max_seq_len, void* out, int32_t* sel_idx_out,
                               float* scores_out, void* workspace, size_t ws_bytes, void* stream);

/*
 * sals_decode_profile — profiling only: runs sals_decode `iters` times with a
 * CUDA event after every stage kernel and SYNCHRONISES the stream after each
 * run; writes the mean milliseconds of each stage to stage_ms[6] =
 * {query projection + query RoPE, latent scoring, top-k, reconstruct(+fused
 * attention on the tcgen05 path), SIMT flash attention, LSE merge} (0 for a
 * stage the chosen path does not launch).  Events between kernels serialise
 * the chain (no programmatic overlap), so the sum exceeds a sals_decode.
 */
sals_status sals_decode_profile(const sals_config* cfg, const void* U, const void* q,
                                const void* latent_cache, const void* v_cache, int64_t cap,
                                int32_t batch, const int32_t* d_seq_len, int32_t max_seq_len,
                                void* out, void* workspace, size_t ws_bytes, int32_t iters,
                                float* stage_ms, void* stream);

/*
 * Dense full-KV comparator built in the same library (the "vs dense" baseline
 * of the north star; FlashAttention-2 is the paper's).
 * sals_dense_append: k_cache[b, pos] = RoPE_pos(k_new[b]) (post-RoPE cache),
 * v_cache[b, pos] = v_new[b].
 * sals_dense_decode: y = softmax(RoPE_{s-1}(q) K[0:s]^T * scale) V[0:s],
 * flash-decode split over the sequence with a log-sum-exp merge.
 */
sals_status sals_dense_append(const sals_config* cfg, const void* k_new, const void* v_new,
                              int32_t batch, const int32_t* d_pos, void* k_cache, void* v_cache,
                              int64_t cap, void* stream);
size_t sals_dense_workspace_bytes(const sals_config* cfg, int32_t batch, int32_t max_seq_len);
sals_status sals_dense_decode(const sals_config* cfg, const void* q, const void* k_cache,
                              const void* v_cache, int64_t cap, int32_t batch,
                              const int32_t* d_seq_len, int32_t max_seq_len, void* out,
                              void* workspace, size_t ws_bytes, void* stream);

/*
 * Sequence-sharded decode — the three device phases around the
 * two exchanges.  Rank p holds the contiguous positions
 * [shard_start, shard_start + local_len_b) of every request b; ranks are in
 * ascending position order.  The caller (one process per GPU) all-gathers
 * between the phases over NCCL:
 *  1. sals_shard_candidates: local q~, p' over the shard, and the local top
 *     min(k-x-z, n_ranked) of the ranked range [x, s_b-z) with GLOBAL indices,
 *     ascending index order, padded with (idx -1, score -inf) to k entries.
 *       cand_score [B, k] fp32, cand_idx [B, k] int32 (outputs)
 *     It also leaves the rotated query q^R in `workspace`, which phase 3 reads:
 *     sals_shard_attend must be given the SAME workspace, unmodified in between
 *     (sals_decode_sharded does this itself).
 *  2. (caller) all-gather of the SCORES only -> cand_all_score [P, B, k] in rank
 *     order.  The indices stay local: since the shards are contiguous and every
 *     list is ascending, the gathered order (rank, position) IS the global index
 *     order, which is all the tie-break (lower index first, R5) needs.
 *  3. sals_shard_attend(..., cand_all_score, cand_idx = this rank's phase-1
 *     indices, world, rank, ...): the exact global TopK of Alg. 1 line 5
 *     over the union -- the (k-x-z)-th largest score T by a radix select over
 *     the P*k gathered scores and the quota of ties at T, ranks in order -- fused
 *     with this rank's owned list (owned sinks | its candidates above T and its
 *     share of the ties | owned recents), then reconstruct + RoPE + attention
 *     over the owned tokens -> partial (m, l, o) per (b, query head):
 *       partial [B, n_q, d+2] fp32: m (log2 domain), l, o[d]
 *  4. (caller) all-gather -> partial_all [P, B, n_q, d+2].
 *  5. sals_merge_partials: log-sum-exp merge -> out [B, n_q*d] (every rank).
 * With P = 1 the result equals sals_decode's (bit-identical selection).
 *   d_local_len [B] int32 device, d_seq_len [B] int32 device (global s_b).
 */
/* Inspection: byte offsets, inside a workspace of sals_workspace_bytes /
 * sals_shard_workspace_bytes(cfg, batch, max_seq_len (max_local_len), ...), of the
 * selection list [B, k] int32 (sals_decode: selected positions, ascending, -1
 * padded; sals_shard_attend: the owned LOCAL rows, ascending) and its counts [B]
 * int32, valid after the call that wrote them completes. */
sals_status sals_workspace_selection_offsets(const sals_config* cfg, int32_t batch, int32_t max_seq_len,
                                             size_t* off_sel, size_t* off_count);
sals_status sals_shard_candidates(const sals_config* cfg, const void* U, const void* q,
                                  const void* latent_shard, int64_t cap_local, int32_t batch,
                                  int64_t shard_start, const int32_t* d_local_len,
                                  int32_t max_local_len, const int32_t* d_seq_len,
                                  float* cand_score, int32_t* cand_idx,
                                  void* workspace, size_t ws_bytes, void* stream);
sals_status sals_shard_attend(const sals_config* cfg, const void* U, const void* q,
                              const void* latent_shard, const void* v_shard, int64_t cap_local,
                              int32_t batch, int64_t shard_start, const int32_t* d_local_len,
                              int32_t max_local_len, const int32_t* d_seq_len,
                              const float* cand_all_score, const int32_t* cand_idx,
                              int32_t world, int32_t rank, float* partial, void* workspace,
                              size_t ws_bytes, void* stream);
sals_status sals_merge_partials(const sals_config* cfg, const float* partial_all, int32_t world,
                                int32_t batch, void* out, void* stream);
size_t sals_shard_workspace_bytes(const sals_config* cfg, int32_t batch, int32_t max_local_len,
                                  int32_t world);

/*
 * The whole sequence-sharded layer-step in one call: the
 * three phases above around two in-place NCCL all-gathers on `stream`, then
 * the merge; `out` [B, n_q*d] is identical on every rank.  One process (or
 * thread) per GPU, every rank calls with the same cfg / batch / max_local_len.
 *  - sals_comm_unique_id: writes an ncclUniqueId (128 bytes) to HOST memory;
 *    rank 0 creates it and the caller broadcasts it (e.g. torch.distributed).
 *  - sals_comm_init: blocking collective over `world` ranks; *comm receives an
 *    opaque handle owned by the caller until sals_comm_destroy.  Returns
 *    SALS_ERR_NCCL when libnccl.so.2 cannot be loaded (resolved at run time:
 *    the copy already in the process if any) or initialisation fails.
 *  - sals_decode_sharded: arguments as sals_shard_candidates / _attend (rank p
 *    holds global positions [shard_start, shard_start + local_len_b) of every
 *    request); workspace of sals_decode_sharded_workspace_bytes(cfg, B,
 *    max_local_len, world) bytes holds the phases' workspace plus the gathered
 *    candidate scores [P, B, k] fp32, this rank's candidate indices [B, k] int32
 *    and the gathered partials [P, B, n_q, d+2] fp32.
 *    With world = 1 the result equals sals_decode's.  The quantised values'
 *    recent window is not sharded (SALS_ERR_UNSUPPORTED).
 */
sals_status sals_comm_unique_id(void* id_out);
sals_status sals_comm_init(const void* nccl_unique_id, int32_t world, int32_t rank, void** comm);
sals_status sals_comm_destroy(void* comm);
size_t sals_decode_sharded_workspace_bytes(const sals_config* cfg, int32_t batch, int32_t max_local_len,
                                           int32_t world);
sals_status sals_decode_sharded(const sals_config* cfg, void* comm, const void* U, const void* q,
                                const void* latent_shard, const void* v_shard, int64_t cap_local,
                                int32_t batch, int64_t shard_start, const int32_t* d_local_len,
                                int32_t max_local_len, const int32_t* d_seq_len, void* out,
                                void* workspace, size_t ws_bytes, void* stream);
/* The sharded layer-step with the new token's append (Alg. 1 lines 2-3)
 * in the same call, as sals_append_decode is for one GPU: every rank passes
 * k_new / v_new [B, D]; the rank whose shard holds the newest position of request b
 * (shard_start + d_local_len[b] - 1 == d_seq_len[b] - 1, its last local row) writes
 * U^T k_new and v_new into that row inside the query projection's launch (one read
 * of U), the others write nothing.  d_local_len / d_seq_len already count the new
 * token.  Equivalent to sals_append_latent(pos = d_local_len - 1) on that rank
 * followed by sals_decode_sharded; same workspace, errors and limits. */
sals_status sals_append_decode_sharded(const sals_config* cfg, void* comm, const void* U, const void* k_new,
                                       const void* v_new, const void* q, void* latent_shard, void* v_shard,
                                       int64_t cap_local, int32_t batch, int64_t shard_start,
                                       const int32_t* d_local_len, int32_t max_local_len,
                                       const int32_t* d_seq_len, void* out, void* workspace, size_t ws_bytes,
                                       void* stream);

const char* sals_status_string(sals_status s);
const char* sals_last_error(void);
/* Number of kernel launches enqueued by the calling thread since the last reset
 * (bench.py's gpu_launches count). */
uint64_t sals_launch_count(int32_t reset);
/* Profiling only: restrict the calling thread's sals_decode / sals_append_latent
 * to a subset of their kernels so a benchmark can time one stage in isolation
 * (its inputs are whatever the previous full call left in the workspace).
 * Bit 0 query projection + query RoPE, 1 latent scoring, 2 top-k,
 * 3 reconstruct (+ fused attention on the tcgen05 path), 4 SIMT flash
 * attention, 5 LSE merge, 6 sals_append_latent.  0xffffffff (the default)
 * runs everything.  Returns the previous mask. */
uint32_t sals_profile_stage_mask(uint32_t mask);

#ifdef __cplusplus
}
#endif
#endif /* SALS_H_ */
