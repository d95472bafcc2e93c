/*
 * maestro_b200.h -- C ABI of the B200-native section-graph executor hot path.
 *
 * Plain pointers and sizes only (no torch types).  Every pointer named d_* is
 * device memory; `stream` is a cudaStream_t passed as void*.  Every call is
 * stream-ordered, never allocates, never synchronises, and returns 0 or a
 * CUDA error code (launch failure).  Domain errors found on the device (the
 * reference's exceptions) are folded into one device error word
 * `int64 d_err` = min over errors of (priority << 32 | code << 24 | index),
 * INT64_MAX when clean (maestro_error_reset).  Priority reproduces the
 * reference's raise order: sample construction (K1, by batch index) before
 * duplicate ids before activation errors (by LPT position) before fan-out
 * violations (by merge order).  The host shim decodes the word into the
 * reference's exception classes (MAESTRO_E_* map 1:1 to maestro/errors.py;
 * see paper_2605_10501_b200/errors.py DEVICE_CODES).
 *
 * The reference has no C/C++ interface: its boundary is a set of Python
 * functions (/root/reference/pkg/src/maestro/scheduling.py, workload.py,
 * simulator.py, mq.py).  Each entry point below names the reference function
 * it replaces; INTEGRATION.md shows the ctypes binding a maintainer would add.
 */
#ifndef MAESTRO_B200_H
#define MAESTRO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MAESTRO_MAX_SECTIONS 16
#define MAESTRO_MAX_BITS 32
#define MAESTRO_MAX_DP 64
#define MAESTRO_MAX_BATCH 4096      /* per step (partition stages it in smem) */
#define MAESTRO_MAX_RANK_SAMPLES 1023 /* per critical rank (one thread per insertion slot) */

/* device error codes (errors.py class per code) */
#define MAESTRO_E_OK 0
#define MAESTRO_E_NEGATIVE_TIME 1       /* NegativeTime         workload.py:164-177 */
#define MAESTRO_E_BOTH_ACTIVATED 2      /* BothActivated        workload.py:310-316 */
#define MAESTRO_E_ACTIVATION 3          /* ActivationError      workload.py:323-328,351-355 */
#define MAESTRO_E_INVALID_DIMS 4        /* InvalidDims          costs.py:116-117 */
#define MAESTRO_E_FANOUT_MISMATCH 5     /* FanoutMismatch       scheduling.py:219,275-279 */
#define MAESTRO_E_EMPTY_BATCH 6         /* EmptyBatch           scheduling.py:217,324 */
#define MAESTRO_E_INCONSISTENT 7        /* InconsistentSchedule scheduling.py:327 */
#define MAESTRO_E_FANOUT_VIOLATION 8    /* FanoutViolation      scheduling.py:361-365 */

#define MAESTRO_POLICY_INTERLEAVED 0      /* ExecPolicy.INTERLEAVED      scheduling.py:42 */
#define MAESTRO_POLICY_ALL_FWD_THEN_BWD 1 /* ExecPolicy.ALL_FWD_THEN_BWD scheduling.py:43 */

/* Lowered section graph (SectionGraph.tables in workload.py mirror). */
typedef struct {
  int32_t n_sections;
  int32_t n_bits;                              /* submodule names, sorted; bit b = name b */
  int32_t critical;                            /* section index of the critical section */
  int32_t n_up, n_down;                        /* candidate auxiliaries per side */
  int32_t n_aux;                               /* auxiliaries in merge order */
  int32_t sub_owner[MAESTRO_MAX_BITS];         /* bit -> owning section */
  int32_t side[MAESTRO_MAX_SECTIONS];          /* 0 upstream, 1 critical, 2 downstream */
  int32_t up_cand[MAESTRO_MAX_SECTIONS];
  int32_t down_cand[MAESTRO_MAX_SECTIONS];
  int32_t neighbor[MAESTRO_MAX_SECTIONS];      /* toward-critical hop, -1 for critical */
  int32_t merge_order[MAESTRO_MAX_SECTIONS];   /* auxiliaries by (hops, id) */
  int32_t dp[MAESTRO_MAX_SECTIONS];
  int32_t fanout[MAESTRO_MAX_SECTIONS];
  int32_t mbs[MAESTRO_MAX_SECTIONS];
  uint32_t sec_bits[MAESTRO_MAX_SECTIONS];     /* submodule bits owned by each section */
  int32_t crit_bit;                            /* bit of the critical section's own id */
  int32_t par_up;                              /* NOT IN REF: 1 = a sample may activate several
                                                  upstream sections (parallel resources):
                                                  t_f_bc/t_b_ac = max over them, the sample joins
                                                  each one's order; 0 = reference behaviour */
} maestro_graph_t;

/* Reset a device error word to "no error" (INT64_MAX). */
int maestro_error_reset(int64_t* d_err, void* stream);

/* K1 -- per-sample 6-tuples from token counts (costs.py:105-123,182-200 summed per side as
 * derive_batch does, costs.py:276-286).  d_tokens[n_bits][B] = tokens the sample occupies
 * in submodule b (0 = not activated; the critical section's id bit carries its length).
 * d_cost[n_bits][8] rows = (flops_per_token_fwd, effective_rate, bwd_fwd_ratio,
 * forward_only, mbs, pp, dp, owner).  Outputs phase-major d_times[6][B] and the
 * activation bitmask d_act[B] (non-critical bits with tokens > 0). */
int maestro_sample_times(const maestro_graph_t* g, const double* d_cost, const int32_t* d_tokens,
                         int32_t B, double* d_times, uint32_t* d_act, int64_t* d_err, void* stream);

/* K2 -- activation resolution (workload.py:297-355) + partition_batch (scheduling.py:202-264).
 * Outputs: d_up/d_down[B] resolved section or -1; d_lpt[B] LPT order; d_part[B] the
 * per-rank lists in assignment order, rank r at d_part_off[r] .. d_part_off[r+1]. */
int maestro_partition(const maestro_graph_t* g, const double* d_times, const int32_t* d_ids,
                      const uint32_t* d_act, int32_t B, int32_t* d_up, int32_t* d_down,
                      int32_t* d_lpt, int32_t* d_part, int32_t* d_part_off, int64_t* d_err,
                      void* stream);

/* K3 -- schedule_rank (scheduling.py:162-199) for every critical rank, one CTA per rank.
 * d_orders[B] receives the per-rank orders at the same offsets as d_part.  d_metrics[3*dp]
 * = (makespan, critical_busy, critical_span) of each final order (rank_metrics,
 * scheduling.py:81-152); d_evals[dp] = calculate_makespan evaluations (EvalCounter). */
int maestro_wavefront(const double* d_times, int32_t B, const int32_t* d_part,
                      const int32_t* d_part_off, int32_t dp, int32_t policy, int32_t* d_orders,
                      double* d_metrics, int64_t* d_evals, void* stream);

/* rank_metrics (scheduling.py:81-152) of one given order: d_out[3] = (makespan,
 * critical_busy, critical_span).  Also serves calculate_makespan (scheduling.py:155-159). */
int maestro_rank_metrics(const double* d_times, int32_t B, const int32_t* d_order, int32_t n,
                         int32_t policy, double* d_out, void* stream);

/* K4 -- build_schedule's auxiliary pass (scheduling.py:347-371): for each auxiliary in
 * merge order, rank q's order = merge_fanout (scheduling.py:267-285) of its neighbour's
 * ranks [q*f, (q+1)*f) filtered to activating samples.  d_orders[n_sections][B],
 * d_sec_off[n_sections][MAESTRO_MAX_DP+1]; the critical slots must already hold K3's
 * output (maestro_build_schedule does that). */
int maestro_fanout_merge(const maestro_graph_t* g, int32_t B, const int32_t* d_up,
                         const int32_t* d_down, int32_t* d_orders, int32_t* d_sec_off,
                         int64_t* d_err, void* stream);

/* K1..K4 in one stream-ordered call: build_schedule (scheduling.py:309-373) from
 * 6-tuples.  d_work must hold maestro_schedule_workspace(B, dp) bytes. */
int64_t maestro_schedule_workspace(int32_t B, int32_t dp_critical);
int maestro_build_schedule(const maestro_graph_t* g, const double* d_times, const int32_t* d_ids,
                           const uint32_t* d_act, int32_t B, int32_t policy, int32_t* d_orders,
                           int32_t* d_sec_off, double* d_metrics, int64_t* d_evals, void* d_work,
                           int64_t* d_err, void* stream);

/* K5 -- varlen pack of one section rank's order (not in the reference).
 * d_tok_off[k] = exclusive prefix of d_len over the order (offset of order[k] in the rank's
 * packed token stream); consecutive groups of `mbs` samples form micro-batches:
 * d_mb[k] = k / mbs, d_mb_start[m] = first token of micro-batch m, d_mb_tokens[m] its token
 * count, d_cu[m*(mbs+1) + j] its cu_seqlens (relative).  d_len[B] = length per batch index. */
int maestro_varlen_pack(const int32_t* d_order, int32_t n, const int32_t* d_len, int32_t mbs,
                        int32_t* d_mb, int32_t* d_tok_off, int32_t* d_mb_tokens, int32_t* d_cu,
                        int32_t* d_mb_start, void* stream);

/* Gather the token ids of the ordered samples into the packed stream:
 * d_out[d_tok_off[k] + j] = d_ids[d_order[k] * ld + j], j < d_len[d_order[k]]. */
int maestro_pack_tokens(const int32_t* d_ids, int32_t ld, const int32_t* d_order, const int32_t* d_len,
                        const int32_t* d_tok_off, int32_t n, int32_t* d_out, void* stream);

/* K5b -- handoff (scatter) indices between a producer section's row buffer and the consumer
 * (critical) rank's packed stream (north_star item 2).  d_up_order[nu]: the
 * producer's order (its row buffer holds d_rows[i] rows per sample, in that order);
 * d_crit_order[n] / d_tok_off[n]: the consumer order and its varlen_pack offsets; mbs its
 * micro-batch size; d_rows[B] / d_dst_off[B] per sample id: rows exchanged (0 = none) and their
 * offset inside the sample's sequence.  Out: d_pos[n+1] = exclusive scan of d_rows over the
 * consumer order; for position k (sample i) and r < d_rows[i], at index d_pos[k] + r:
 * d_src_rows = producer-buffer row, d_dst_rows = row inside consumer micro-batch k / mbs
 * (d_tok_off[k] - d_tok_off[(k/mbs)*mbs] + d_dst_off[i] + r).  d_scratch: B int32.  A sample with
 * rows in the consumer order but absent from the producer order sets InconsistentSchedule. */
int maestro_handoff_index(const int32_t* d_up_order, int32_t nu, const int32_t* d_crit_order, int32_t n,
                          const int32_t* d_tok_off, int32_t mbs, const int32_t* d_rows, const int32_t* d_dst_off,
                          int32_t B, int32_t* d_scratch, int32_t* d_pos, int32_t* d_src_rows, int32_t* d_dst_rows,
                          int64_t* d_err, void* stream);

/* K6 -- row scatter of encoder outputs into the packed token stream and its backward.
 * fwd: dst[dst_row[k], :] = src[src_row[k], :]  (bf16, d multiple of 8)
 * bwd: dsrc[r, :] = sum over k in seg[r]..seg[r+1] of ddst[seg_dst[k], :] (fp32 accumulate). */
int maestro_scatter_rows_fwd(const void* d_src, void* d_dst, const int32_t* d_src_row,
                             const int32_t* d_dst_row, int32_t n_rows, int32_t d, void* stream);
/* K6 over one micro-batch of a K5b handoff index: the pairs [d_pos[k0], d_pos[k1]) (read on
 * device); max_rows >= d_pos[k1] - d_pos[k0] sizes the grid; accumulate != 0: dst += src (bf16,
 * fp32 sum rounded once). */
int maestro_scatter_rows_range(const void* d_src, void* d_dst, const int32_t* d_src_row, const int32_t* d_dst_row,
                               const int32_t* d_pos, int32_t k0, int32_t k1, int32_t max_rows, int32_t d,
                               int32_t accumulate, void* stream);
int maestro_gather_rows_bwd(const void* d_ddst, void* d_dsrc, const int32_t* d_seg,
                            const int32_t* d_seg_dst, int32_t n_src_rows, int32_t d, void* stream);


/* ---------------------------------------------------------------- section compute
 * Not in the reference (paper prose only: PAPER.md:56,88,93,250,270-271).  bf16 operands,
 * fp32 accumulation.  All pointers are device memory; row pitches are in elements. */

/* K7 -- C[m,n] (+)= sum_k A(m,k) B(n,k) on tcgen05/TMEM.  A(m,k) = A[m*lda+k] (a_mn = 0) or
 * A[k*lda+m] (a_mn = 1); likewise B.  epi: 0 store bf16, 1 store fp32, 2 accumulate into fp32
 * (small-output shapes split K and use fp32 reductions).  N, lda, ldb, ldc multiples of 8. */
int maestro_gemm_bf16(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t lda,
                      int32_t ldb, int32_t ldc, int32_t a_mn, int32_t b_mn, int32_t epi, void* stream);

/* K7 + fused RoPE epilogue: C = A B^T (bf16, K-major A/B); every head_dim-column head (64 or 128)
 * in columns [0, rope_cols) is rotated (rotate-half) at position pos[row].  cos_sin is
 * position-tiled: [ceil(P/32)][head_dim/2 freqs][32 positions] of (cos, sin) fp32 pairs
 * (transformer.rope_table). */
int maestro_gemm_bf16_rope(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t lda,
                           int32_t ldb, int32_t ldc, const int32_t* pos, const void* cos_sin, int32_t rope_cols,
                           int32_t head_dim, void* stream);

/* K7 + fused residual epilogue: C = R + A B^T (bf16; the sum is formed in fp32 and rounded
 * once).  Used by the attention-output and down projections to write the residual stream. */
int maestro_gemm_bf16_residual(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t lda,
                               int32_t ldb, int32_t ldc, const void* R, int32_t ldr, void* stream);
/* K7 + fused SwiGLU epilogue: C = A B^T is the gate/up activation with gate/up rows of B
 * interleaved in 32-row blocks ([g_0..g_31, u_0..u_31, g_32..]); S[m, f] = silu(g_f) * u_f.
 * C may be NULL (forward-only sections): then only S is written. */
int maestro_gemm_bf16_swiglu(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t lda,
                             int32_t ldb, int32_t ldc, void* S, int32_t lds, void* stream);

/* K8 -- varlen GQA attention, head_dim dh: q [T,H,dh], k/v [T,Hk,dh] (pitched), cu [nseq+1];
 * out [T,H,dh] bf16, lse [H,T] fp32 (natural LSE of the scaled scores).  Forward: dh 64 or 128;
 * backward: dh 64 or 128. */
int64_t maestro_attn_workspace(int32_t T, int32_t nseq);
/* Per-micro-batch work plan (query-tile and KV-tile lists, heavy-first) built once from cu and
 * passed to every layer's attn_fwd / attn_bwd; plan == NULL builds it per call in the workspace. */
int64_t maestro_attn_plan_size(int32_t T, int32_t nseq);
int maestro_attn_plan(const int32_t* cu, int32_t nseq, int32_t T, void* plan, void* stream);
int maestro_attn_fwd(const void* q, const void* k, const void* v, const int32_t* cu, int32_t nseq, int32_t T,
                     int32_t H, int32_t Hk, int32_t head_dim, int32_t ldq, int32_t ldk, int32_t ldv, void* out,
                     int32_t ldo, float* lse, float softmax_scale, int32_t causal, const void* plan, void* workspace,
                     void* stream);
int64_t maestro_attn_bwd_workspace(int32_t T, int32_t nseq, int32_t H, int32_t head_dim);
int maestro_attn_bwd(const void* dout, int32_t lddo, const void* q, const void* k, const void* v, const void* o,
                     int32_t ldo, const float* lse, const int32_t* cu, int32_t nseq, int32_t T, int32_t H,
                     int32_t Hk, int32_t head_dim, int32_t ldq, int32_t ldk, int32_t ldv, void* dq, int32_t lddq,
                     void* dk, int32_t lddk, void* dv, int32_t lddv, float softmax_scale, int32_t causal,
                     const int32_t* rope_pos, const void* rope_cos_sin, const void* plan, void* workspace,
                     void* stream);
/* (rope_pos/rope_cos_sin (position-tiled table, as above) non-null: dQ and dK are returned through the inverse RoPE rotation,
 * i.e. w.r.t. the pre-rotation projections.) */

/* fp64 CUDA-core probe (scheduler roofline denominators): mode 0 = add throughput over
 * blocks x 256 threads x 8 independent chains x iters adds; mode 1 = one dependent chain of iters adds. */
int maestro_fp64_probe(double* out, int32_t mode, int32_t iters, int32_t blocks, void* stream);

/* Upper bound on the SMs the persistent kernels (GEMM, attention) size their grids to; 0 = all.
 * Executors whose NCCL point-to-point kernels run concurrently with compute reserve a few SMs so
 * that a static persistent tile schedule never waits on a CTA that cannot become resident. */
int maestro_set_sm_budget(int32_t n_sms);

/* Programmatic dependent launch of the step kernels (GEMM, attention, losses, norms, ...): 1 on
 * (default; MAESTRO_PDL=0 starts it off), 0 off.  Returns the previous setting. */
int maestro_set_pdl(int32_t on);

/* One-sided NVLink handoff (mq.PeerTransport): receiver-owned slot ring + per-slot flags exported
 * by CUDA IPC; sends are copy-engine copies into the peer slot followed by a stream memory write of
 * the slot flag, receives are stream waits on the flag -- no kernel spins on another GPU. */
int maestro_device_alloc(int64_t bytes, void** dev_ptr_out);
int maestro_device_free(void* dev_ptr);
int maestro_ipc_get_handle(const void* dev_ptr, void* handle_out /* 64 bytes */);
int maestro_ipc_open_handle(const void* handle /* 64 bytes */, void** dev_ptr_out);
int maestro_ipc_close(void* dev_ptr);
int maestro_stream_wait_geq(void* stream, const void* dev_addr, uint32_t value);
int maestro_stream_write(void* stream, void* dev_addr, uint32_t value);
int maestro_copy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* Reshard data mover (mq.py:163-174, 460-469): dst[box] = src[box] for an N-d box (ndim <= 6,
 * strides in elements, elem_bytes 1/2/4/8).  Used by apply_plan and Endpoint.pull to gather
 * fragments into a receiver's shard and by push_tensor to slice a sender's shard. */
int maestro_box_copy(const void* src, const int64_t* src_strides, void* dst, const int64_t* dst_strides,
                     const int64_t* shape, int32_t ndim, int32_t elem_bytes, void* stream);

/* K9 -- fused full-vocab KL(softmax(t/tau) || softmax(s/tau)) per token (d_loss[T]) and
 * ds = grad_scale * dKL/ds (bf16, may alias s).  Teacher head colocated per workload.py:471-514. */
int maestro_kd_loss_fwd_bwd(const void* d_t, const void* d_s, void* d_ds, float* d_loss, int32_t T, int32_t V,
                            int32_t ldt, int32_t lds, int32_t ldd, float grad_scale, float inv_tau, void* stream);

/* Next-token cross entropy (VLM backbone loss) with ignore index label < 0. */
int maestro_ce_loss_fwd_bwd(const void* d_s, const int32_t* d_labels, void* d_ds, float* d_loss, int32_t T,
                            int32_t V, int32_t lds, int32_t ldd, float grad_scale, void* stream);

/* Memory-bound block kernels. */
int maestro_add_rmsnorm_fwd(const void* x, const void* a, void* h, void* y, const void* w, float* rstd, int32_t T,
                            int32_t d, float eps, void* stream);
int maestro_rmsnorm_bwd(const void* dy, const void* h, const void* w, const float* rstd, const void* dres,
                        void* dx, float* dw, int32_t T, int32_t d, void* stream);
/* In-place rotate-half RoPE; cos_sin position-tiled [ceil(P/32)][dh/2][32][2] (see maestro_gemm_bf16_rope);
 * dh a multiple of 16, row pitch ld a multiple of 8 elements. */
int maestro_rope(void* qk, const int32_t* pos, const void* cos_sin, int32_t T, int32_t n_heads, int32_t dh,
                 int32_t ld, int32_t backward, void* stream);
int maestro_positions(const int32_t* cu, int32_t nseq, int32_t* pos, void* stream);
/* gu layout: gate/up interleaved in 32-column blocks (see maestro_gemm_bf16_swiglu) */
int maestro_swiglu_fwd(const void* gu, void* out, int32_t T, int32_t F, void* stream);
int maestro_swiglu_bwd(const void* dout, const void* gu, void* dgu, int32_t T, int32_t F, void* stream);
int maestro_embed_fwd(const void* table, const int32_t* ids, void* out, int32_t T, int32_t d, void* stream);
int maestro_embed_bwd(const void* dout, const int32_t* ids, float* dtable, int32_t T, int32_t d, void* stream);
/* dst[c * ld_dst + r] = src[r * ld_src + c] (bf16; rows, cols, pitches multiples of 8).  Keeps the
   K-major weight copies the dgrad GEMM reads (see FlatParams.refresh_transposed). */
int maestro_transpose_bf16(const void* src, void* dst, int32_t rows, int32_t cols, int32_t ld_src, int32_t ld_dst,
                           void* stream);
/* Several transposes in one launch.  desc: device int64[n][8] = {src ptr, dst ptr, rows, cols,
   ld_src, ld_dst, first tile, tiles along cols}; tiles are 64 x 64, numbered consecutively over
   the matrices (first tile ascending); total_tiles = sum of ceil(rows/64) * ceil(cols/64). */
int maestro_transpose_bf16_batched(const int64_t* desc, int32_t n, int32_t total_tiles, void* stream);
int maestro_adamw(float* p, const float* g, float* m, float* v, void* pb, int64_t n, float lr, float b1, float b2,
                  float eps, float wd, int32_t step, float gscale, void* stream);

#ifdef __cplusplus
}
#endif
#endif
