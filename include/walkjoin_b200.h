/*
 * walkjoin_b200.h -- C ABI of the B200 walk -> RPE -> join hot path.
 *
 * Every entry point takes DEVICE pointers owned by the caller, plain sizes
 * and a cudaStream_t (passed as void*), launches asynchronously on that
 * stream and returns WJ_OK or an error code; wj_last_error() gives the
 * message of the last failure on the calling host thread.  Nothing is
 * allocated inside and there is no global mutable state, so the library is
 * safe to drive from several host threads on different streams.
 *
 * Each function names the reference interface it replaces
 * (/root/reference/pkg/src/walkjoin/<file>:<line>).  The reference binds its
 * numba kernels from Python; INTEGRATION.md shows the ctypes stub a
 * maintainer adds to call these instead.
 */
#ifndef WALKJOIN_B200_H
#define WALKJOIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WJ_ABI_VERSION 1

#define WJ_OK 0
#define WJ_ERR_ARG 1          /* bad argument (maps to ValueError) */
#define WJ_ERR_CUDA 2         /* CUDA launch/runtime failure */
#define WJ_ERR_UNSUPPORTED 3  /* shape outside the kernels' envelope */

/* dense element types for wj_join / wj_gather_rpe */
#define WJ_F32 0
#define WJ_F64 1
#define WJ_BF16 2
#define WJ_F16 3

typedef void *wj_stream_t; /* cudaStream_t */

int wj_abi_version(void);
const char *wj_last_error(void);

/* Walk sampling for anchors [lo, hi): walks_out[(u-lo), M, L+1] int32.
 * Replaces _kernels.sample_all_walks (_kernels.py:69-74) as driven by
 * sampler.preprocess (sampler.py:114-115).  Bit-exact with the reference
 * splitmix64 stream: walk j step i of u draws mix64(S0(u) + (j*L+i)*G).
 * idxptr is int32 (idxptr_bytes=4, requires 2E < 2^31) or int64 (8).
 * fix_flags: [hi-lo] uint8 scratch, zeroed by the caller; anchors whose
 * walks hit a mid-walk dead end (only possible in a non-symmetric CSR) are
 * flagged and re-sampled sequentially on device by a second launch. */
int wj_sample_walks(const void *idxptr, int idxptr_bytes, const int32_t *indices, int64_t n_nodes,
                    int64_t lo, int64_t hi, int32_t num_walks, int32_t num_steps, uint64_t seed,
                    int32_t *walks_out, uint8_t *fix_flags, wj_stream_t stream);

/* Typed / metapath walks (no reference implementation exists --
 * SPEC.md:121-124 leaves typed walks open -- so the semantics are ours,
 * chosen so that the homogeneous special case IS wj_sample_walks): step i
 * of walk j from anchor u follows an edge of type metapath[(i-1) % P]
 * (negative = any edge), uniform among the current node's edges of that type
 * in CSR order, with the reference's draw mix64(S0(u) + (j*L+i)*G); with no
 * such edge the walk stays put for that step.  metapath is a HOST array of
 * P <= 32 entries (copied into the launch); type_off [n*T+1] int64 /
 * typed_indices [2E] int32 come from the grouping below (NULL allowed when every
 * entry is negative).  With metapath {-1} on the reference's symmetric CSR
 * the walks equal wj_sample_walks bit for bit. */
int wj_sample_walks_typed(const void *idxptr, int idxptr_bytes, const int32_t *indices, const int64_t *type_off,
                          const int32_t *typed_indices, int32_t num_types, const int8_t *metapath,
                          int32_t metapath_len, int64_t n_nodes, int64_t lo, int64_t hi, int32_t num_walks,
                          int32_t num_steps, uint64_t seed, int32_t *walks_out, wj_stream_t stream);

/* Edge-type grouping of a CSR for the typed sampler: typed_indices_out [2E]
 * = each node's neighbours grouped by edge type (edge_types [2E] uint8,
 * aligned with indices; CSR order kept inside a type), type_off_out
 * [n*T + 1] = start of node c's type-t group.  1 <= num_types <= 64. */
int wj_typed_csr(const void *idxptr, int idxptr_bytes, const int32_t *indices, const uint8_t *edge_types,
                 int64_t n_nodes, int32_t num_types, int64_t *type_off_out, int32_t *typed_indices_out,
                 wj_stream_t stream);

/* One anchor from an explicit stream state; writes the end state.
 * Replaces _kernels.sample_node_walks (_kernels.py:53-66) as used by
 * sampler.sample_walks (sampler.py:61-76). */
int wj_sample_node_walks(const void *idxptr, int idxptr_bytes, const int32_t *indices, int64_t u,
                         int32_t num_walks, int32_t num_steps, uint64_t state, int32_t *out,
                         uint64_t *end_state_out, wj_stream_t stream);

/* Distinct landings per anchor (counts_out[k] = |V_{lo+k}|).
 * Replaces _kernels.count_distinct_all (_kernels.py:87-101), sampler.py:117-121. */
int wj_rpe_count(const int32_t *walks, int64_t n_anchors, int32_t num_walks, int32_t num_steps,
                 int64_t n_nodes, int32_t *counts_out, wj_stream_t stream);

/* Per-anchor RPE index: sorted unique landing ids (uniq_x), packed positional
 * count vector (uniq_key: count of step c in bits [c*cb, (c+1)*cb), cb =
 * bits(M)), first-appearance flat position (uniq_first) and, per walk slot,
 * the index of its node in the anchor's unique list (slot_idx[k, M*(L+1)]).
 * Entries of anchor k live at [offsets[k], offsets[k+1]).
 * Replaces _kernels.fill_distinct_all (_kernels.py:104-126), sampler.py:122-128. */
int wj_rpe_fill(const int32_t *walks, int64_t n_anchors, int32_t num_walks, int32_t num_steps,
                int64_t n_nodes, const int64_t *offsets, int32_t *uniq_x, uint64_t *uniq_key,
                uint16_t *uniq_first, uint16_t *slot_idx, wj_stream_t stream);

/* Global interning, phase 1: insert every entry's packed vector into an
 * open-addressing table (table_keys zeroed, table_order set to all-ones,
 * table_cap a power of two) keeping the minimum scan order
 * ((anchor_base+k) << 16 | first).  *overflow_flag becomes nonzero if the
 * table fills.  Phase 2 (rank by first occurrence) is host plumbing; phase 3
 * is wj_intern_assign.  Together they replace the sequential
 * _kernels.intern_rows (_kernels.py:137-171) / store.intern_vectors
 * (store.py:107-121) and reproduce its ids exactly. */
int wj_intern_insert(const uint64_t *uniq_key, const uint16_t *uniq_first, const int64_t *offsets,
                     int64_t n_anchors, int64_t anchor_base, uint64_t *table_keys,
                     uint64_t *table_order, int64_t table_cap, int32_t *overflow_flag,
                     wj_stream_t stream);

/* Global interning, phase 3: uniq_id[e] = table_ids[slot of uniq_key[e]]. */
int wj_intern_assign(const uint64_t *uniq_key, int64_t n_entries, const uint64_t *table_keys,
                     const int32_t *table_ids, int64_t table_cap, int32_t *uniq_id,
                     wj_stream_t stream);

/* Query-level join fused with densify.  queries [B, A] int64.  Any of the
 * three outputs may be NULL:
 *   walk_nodes_out [B, A*M, L+1] int32          (_kernels.py:231-233)
 *   rpe_ids_out    [B, A*M*(L+1), A] int32      (_kernels.py:237-245)
 *   dense_out      [B, A*M*(L+1), row_stride] of dense_dtype; columns
 *                  [0, A*(L+1)) get table[rpe_id] (pipeline.py:178)
 * table_keys [table_len] packed count vectors (id order, row 0 = 0).
 * Replaces joiner.join_batch_arrays (joiner.py:53-71) + _kernels.join_fill
 * (_kernels.py:209-245) + the densify of pipeline._dense_batch
 * (pipeline.py:169-182). */
int wj_join(const int64_t *queries, int64_t n_batch, int32_t arity, const int32_t *walks,
            const int64_t *offsets, const int32_t *uniq_x, const int32_t *uniq_id,
            const uint16_t *slot_idx, int32_t num_walks, int32_t num_steps, int32_t max_unique,
            const uint64_t *table_keys, int64_t table_len, int32_t *walk_nodes_out,
            int32_t *rpe_ids_out, void *dense_out, int32_t dense_dtype, int64_t row_stride,
            wj_stream_t stream);

/* Join fused with the encoder's first layer.  For every query b computes,
 * without materialising the [A*M*(L+1), A*(L+1)] input or its [rows, H]
 * hidden activations,
 *   pooled_out[b, h] = sum_r relu(z_r[h]) * d_r[h]
 *   s_out[b, c, h]   = sum_r x_r[c] * 1[z_r[h] > 0] * d_r[h]   (may be NULL)
 *   msum_out[b, h]   = sum_r 1[z_r[h] > 0] * d_r[h]           (may be NULL)
 * with z_r = x_r W1 + b1 (w1 [A*(L+1), hidden] fp32, row-major), x_r the
 * joined RPE row of walk slot r and d_r a Bernoulli(keep_prob) dropout draw
 * from a counter-based stream keyed by (seed, *step, b, virtual landing,
 * unit) (keep_prob = 1: no dropout).  *step is read on the device so a
 * captured CUDA graph advances it itself.  cross (nullable) holds the
 * query's cross RPE ids computed by wj_join_cross; then the kernel does no
 * searches, while NULL makes it search the sorted lists itself.  voff / vcnt / vslots are the
 * store's virtual-landing index (wj_vindex_count / wj_vindex_fill) and
 * table_rows_f16 the fp16 table rows (wj_table_rows_f16); with them,
 * hidden = 64, A*(L+1) <= 15, L+1 <= 8 and M <= 2048 run the tensor-core
 * kernel (encode_mma.cu); otherwise (or if any of the four is NULL) the SIMT
 * kernel (wj_join_encode_simt) runs.  keep_prob = 1 with M*(L+1) <= 1024
 * runs the tensor-core kernel's no-dropout variant (no random stream; one
 * row per distinct landing weighted by its row count): the same outputs, bit
 * for bit, as every row kept.  An empty batch (n_batch = 0) only checks the
 * shape against the kernels' envelope (WJ_ERR_UNSUPPORTED outside it).
 * Replaces _kernels.join_fill +
 * pipeline._dense_batch + the first layer of encoder.forward/backward
 * (_kernels.py:209-245, pipeline.py:169-182, encoder.py:150-161,224-232). */
int wj_join_encode(const int64_t *queries, int64_t n_batch, int32_t arity, const int64_t *offsets,
                   const int32_t *uniq_x, const int32_t *uniq_id, const int32_t *cross, const int64_t *voff,
                   const int32_t *vcnt, const uint16_t *vslots, const uint16_t *table_rows_f16,
                   int32_t num_walks, int32_t num_steps, int32_t max_unique,
                   const uint64_t *table_keys, int64_t table_len, const float *w1, const float *b1,
                   int32_t hidden, float keep_prob, uint64_t seed, const int64_t *step,
                   float *pooled_out, float *s_out, float *msum_out, wj_stream_t stream);

/* Cross RPE ids of every distinct landing of every query anchor:
 * cross_out [B, A, A-1, max_unique] int32, entry [b, a, jj, l] = RPE id of
 * the l-th landing (sorted order) of anchor a relative to the jj-th other
 * anchor of query b, 0 if absent; entries l >= U_a are left untouched.  The
 * per-landing form of the rpe_ids columns _kernels.join_fill writes per walk
 * slot (_kernels.py:237-245).  A in {2, 3}. */
int wj_join_cross(const int64_t *queries, int64_t n_batch, int32_t arity, const int64_t *offsets,
                  const int32_t *uniq_x, const int32_t *uniq_id, int32_t max_unique, int32_t *cross_out,
                  wj_stream_t stream);

/* Virtual-landing index of a store (the encoder input layout; no reference
 * counterpart -- it describes the rows pipeline._dense_batch builds,
 * pipeline.py:169-182).  n_l = row sum of landing l's count vector = its
 * number of rows in anchor u's block.  Count pass: vcnt_out[2u] =
 * sum_l floor(n_l/2), vcnt_out[2u+1] = sum_l (n_l & 1).  Fill pass (voff =
 * exclusive cumsum of vcnt[2u] + vcnt[2u+1], [n+1] int64): vslots_out
 * [voff[u], voff[u] + vcnt[2u]) = l repeated floor(n_l/2) times, then every
 * l with odd n_l once (uint16 landing indices into u's sorted list). */
int wj_vindex_count(const int64_t *offsets, const int32_t *uniq_id, int64_t n_anchors,
                    const uint64_t *table_keys, int32_t num_walks, int32_t num_steps,
                    int32_t *vcnt_out, wj_stream_t stream);
int wj_vindex_fill(const int64_t *offsets, const int32_t *uniq_id, int64_t n_anchors,
                   const uint64_t *table_keys, int32_t num_walks, int32_t num_steps,
                   const int64_t *voff, const int32_t *vcnt, uint16_t *vslots_out,
                   wj_stream_t stream);

/* fp16 rows of the RPE table: rows_out [table_len, 8] halves, counts of
 * table row i in columns [0, L+1), zeros after (L+1 <= 8, M <= 2048: exact).
 * The same vectors as store.table (store.py:33-46). */
int wj_table_rows_f16(const uint64_t *table_keys, int64_t table_len, int32_t num_walks,
                      int32_t num_steps, uint16_t *rows_out, wj_stream_t stream);

/* Same contract on CUDA cores only (hidden in {32, 64, 128}, A*(L+1) <= 16);
 * its dropout stream differs from wj_join_encode's tensor-core kernel. */
int wj_join_encode_simt(const int64_t *queries, int64_t n_batch, int32_t arity,
                        const int64_t *offsets, const int32_t *uniq_x, const int32_t *uniq_id,
                        int32_t num_walks, int32_t num_steps, int32_t max_unique,
                        const uint64_t *table_keys, int64_t table_len, const float *w1,
                        const float *b1, int32_t hidden, float keep_prob, uint64_t seed,
                        const int64_t *step, float *pooled_out, float *s_out, float *msum_out,
                        wj_stream_t stream);

/* Encoder tail on the wj_join_encode outputs (hidden = 64): W2 layer on the
 * pooled encodings (pm = pooled * scale), 2-layer classifier, BCE and the
 * full backward.  params is the flat fp32 parameter vector laid out by
 * offsets9 = {w1, b1, w2, b2, u1, c1, u2, c2, total}.  logits_out (may be
 * NULL) gets the [B] logits.  Training (labels != NULL) launches exactly
 * partial_rows CTAs: CTA i reduces queries [i*q, (i+1)*q), q = ceil(B /
 * partial_rows) (best: partial_rows = ceil(B / 16)), in a fixed order into
 * partial[i, 0:total] and its loss partial into partial[i, total] (partial
 * 8-byte aligned: rows are written with 8-B stores).  work is
 * unused (may be NULL).  step_inc (nullable) is incremented by one when the
 * tail is done (the graph-resident step counter wj_join_encode and wj_adam
 * read).  The [16 x 64] x [64 x 64] products run on the tensor cores in
 * 3-pass TF32.  Replaces encoder.forward / bce_loss /
 * backward after layer 1 (encoder.py:159-233). */
int wj_encoder_tail(const float *pooled, const float *s, const float *msum, const float *labels,
                    int64_t n_batch, int32_t aw, int32_t hidden, const float *params,
                    const int32_t *offsets9, float scale, float *logits_out, float *partial,
                    int32_t partial_rows, float *work, int64_t *step_inc, wj_stream_t stream);

/* Deterministic reduction of the partial gradients + bias-corrected Adam
 * with t = *step (encoder.py:236-249).  grad_out / loss_out may be NULL. */
int wj_adam(float *params, float *m, float *v, const float *partial, int32_t partial_rows,
            int32_t n_params, float lr, float beta1, float beta2, float eps, const int64_t *step,
            float *grad_out, float *loss_out, wj_stream_t stream);

/* Scoring of queries that share their first anchor (the test protocol: a
 * positive followed by its negatives (u, v_i); pipeline.py:185-198): same
 * pooled / S / msum as wj_join_encode at keep_prob = 1, bit for bit, with u's
 * alone rows and their tile sums built once per run of equal first anchors
 * in a CTA's contiguous range of queries.  Arity 2, hidden 64. */
int wj_score_shared(const int64_t *queries, int64_t n_batch, const int64_t *offsets, const int32_t *uniq_x,
                    const int32_t *uniq_id, const uint16_t *table_rows_f16, int32_t num_walks, int32_t num_steps,
                    int32_t max_unique, const float *w1, const float *b1, float *pooled_out, float *s_out,
                    float *msum_out, wj_stream_t stream);

/* Step executor: one fused training step per wj_stepper_run -- replaces
 * the body of train()'s batch loop after the batch is drawn
 * (pipeline.py:302-305: _dense_batch -> forward -> bce_loss -> backward ->
 * adam_step; encoder.py:126-249) --
 * wj_join_encode -> wj_encoder_tail -> wj_adam with every static argument
 * (the store's index, flat params / Adam moments at offsets9, work buffers
 * pooled [B_max, 64], s_out [B_max, A*(L+1), 64], msum [B_max, 64],
 * partial [partial_rows_max, n_params + 1], the device step counter,
 * tail_scale = 1 / (keep_prob * A * M * (L+1)) as wj_encoder_tail takes it,
 * sched: NULL, or two zeroed int32 in device memory owned by this stepper --
 * the join+encode kernel then grabs queries dynamically from a counter
 * there and resets it when done) fixed
 * at creation.  All three launches are programmatic-dependent, so
 * consecutive runs on one stream form a single PDL chain: the next step's
 * join+encode kernel stages its first query while this step's tail and Adam
 * finish.  queries [B, A] int64 / labels [B] fp32 may be device memory or
 * mapped pinned host memory (read by the kernels directly; the caller keeps
 * them unchanged until the step completes); loss_out (device or mapped
 * host, may be NULL) receives the step's mean BCE.  Same math and dropout
 * stream as the three separate calls (the TrainStep graph).  groups (device,
 * from wj_group_queries, needs sched) makes the join+encode kernel schedule
 * groups of identical queries: a group stages, merges and builds its rows
 * once and runs tiles + reduction per member -- same outputs. */
typedef struct wj_stepper wj_stepper;
int wj_stepper_create(const int64_t *offsets, const int32_t *uniq_x, const int32_t *uniq_id, const int64_t *voff,
                      const int32_t *vcnt, const uint16_t *vslots, const uint16_t *table_rows_f16, int32_t arity,
                      int32_t num_walks, int32_t num_steps, int32_t max_unique, float *params, float *adam_m,
                      float *adam_v, const int32_t *offsets9, float keep_prob, float tail_scale, uint64_t seed,
                      float lr, float beta1,
                      float beta2, float eps, int64_t *step, float *pooled, float *s_out, float *msum,
                      float *partial, int32_t partial_rows_max, int32_t *sched, wj_stepper **out);
int wj_stepper_run(wj_stepper *stepper, const int64_t *queries, const float *labels, int64_t n_batch,
                   const int32_t *groups, int64_t n_groups, float *loss_out, wj_stream_t stream);
/* The step's join+encode kernel alone, exactly as wj_stepper_run launches
 * it (same plan, scheduling and buffers; the step counter is not advanced):
 * for timing the production kernel in isolation. */
int wj_stepper_encode(wj_stepper *stepper, const int64_t *queries, int64_t n_batch, const int32_t *groups,
                      int64_t n_groups, wj_stream_t stream);
/* Data parallel: the step split around the gradient exchange.
 * wj_stepper_grads = join+encode + tail + fixed-order sum of the partial
 * rows into grad_out [n_params + 1] (gradients | loss); the caller
 * all-reduces (averages) it over ranks, then wj_stepper_apply runs Adam on
 * it (and writes the loss to loss_out, device or mapped host, may be NULL). */
int wj_stepper_grads(wj_stepper *stepper, const int64_t *queries, const float *labels, int64_t n_batch,
                     const int32_t *groups, int64_t n_groups, float *grad_out, wj_stream_t stream);
int wj_stepper_apply(wj_stepper *stepper, const float *grad, float *loss_out, wj_stream_t stream);
/* Batch-sharded data parallel (one reference mini-batch over P
 * ranks): rank r runs queries [b_offset, b_offset + n_batch) of a global batch
 * of b_global queries whose single-GPU tail rows of per_cta queries are rows
 * [b_offset / per_cta, + rows): join+encode with the global dropout keys, the
 * tail with the global 1/B into partial_out [rows, n_params + 1].  Gathering
 * every rank's rows in order and applying them (wj_stepper_apply_rows) is
 * bit-identical to wj_stepper_run on the whole batch. */
int wj_stepper_grads_shard(wj_stepper *stepper, const int64_t *queries, const float *labels, int64_t n_batch,
                           const int32_t *groups, int64_t n_groups, int64_t b_offset, int64_t b_global,
                           int32_t per_cta, int32_t rows, float *partial_out, wj_stream_t stream);
int wj_stepper_apply_rows(wj_stepper *stepper, const float *partial, int32_t rows, float *loss_out,
                          wj_stream_t stream);
int wj_stepper_destroy(wj_stepper *stepper);

/* Fixed-order column sums out[c] = sum_r partial[r, c] of a [rows, n_cols]
 * partial buffer (the data-parallel step reduces locally, all-reduces the
 * [n_params + 1] result over ranks, then runs wj_adam on it as one row). */
int wj_sum_partials(const float *partial, int32_t partial_rows, int32_t n_cols, float *out,
                    wj_stream_t stream);

/* Densify ids: out[i, :] = table[rpe_ids[i], :] (table [T, width] int32).
 * Replaces joiner.gather_rpe (joiner.py:96-104); *bad_flag set if an id is
 * out of range (the reference raises ValueError). */
int wj_gather_rpe(const int32_t *rpe_ids, int64_t n_ids, const int32_t *table, int64_t table_len,
                  int32_t width, void *out, int32_t dtype, int32_t *bad_flag, wj_stream_t stream);

/* Export the reference per-node dictionaries bit-exactly (dict_keys
 * pre-filled with -1, dict_vals with 0; cap_offsets from
 * store.dict_capacities).  Replaces _kernels.build_dicts
 * (_kernels.py:174-188), sampler.py:133-138. */
int wj_export_dicts(const int64_t *offsets, const int32_t *uniq_x, const int32_t *uniq_id,
                    const uint16_t *uniq_first, const uint16_t *slot_idx, int64_t n_anchors,
                    int32_t num_walks, int32_t num_steps, const int64_t *cap_offsets,
                    int32_t *dict_keys, int32_t *dict_vals, wj_stream_t stream);

/* Reference store-file (SURL v1) node records as 4-byte words (store.py:
 * 167-193, 204-264): record u at word rec_off[u] = capacity, walks[u]
 * (walk_words = M*(L+1) int32), dict_keys, dict_vals of node u (capacity =
 * dict_offsets[u+1] - dict_offsets[u]).  pack writes the records of n_nodes
 * nodes; unpack reads walks (and, when dict_keys_out != NULL, the dicts)
 * back.  The host writes / parses the header, table and id map. */
int wj_surl_pack(const int32_t *walks, int64_t n_nodes, int32_t walk_words, const int64_t *dict_offsets,
                 const int32_t *dict_keys, const int32_t *dict_vals, const int64_t *rec_off, int32_t *out,
                 wj_stream_t stream);
int wj_surl_unpack(const int32_t *records, int64_t n_nodes, int32_t walk_words, const int64_t *rec_off,
                   const int64_t *dict_offsets, int32_t *walks_out, int32_t *dict_keys_out,
                   int32_t *dict_vals_out, wj_stream_t stream);

/* Point lookups out[i] = RPE id of x[i] relative to anchor u[i] (0 if
 * absent).  Replaces store.get_rpe_id / _kernels.dict_get_one
 * (store.py:160-164, _kernels.py:203-206). */
int wj_lookup(const int64_t *u, const int64_t *x, int64_t count, const int64_t *offsets,
              const int32_t *uniq_x, const int32_t *uniq_id, int32_t *out, wj_stream_t stream);


/* ---- Host-side training mini-batch planner (no device state) -------------
 * Replaces the per-batch Python of train() (pipeline.py:292-304):
 * sample_minibatch (pipeline.py:77-129, BFS over query-sharing neighbours)
 * and sample_negatives (pipeline.py:132-166, in-seed rejection negatives)
 * or the fixed-pool draw (pipeline.py:298-300), on numpy's PCG64 stream:
 * with the Generator state copied in (wj_planner_set_rng: state hi/lo,
 * inc hi/lo, has_uint32, uinteger) each wj_planner_next returns exactly the
 * reference's batch and leaves the same state (wj_planner_get_rng).
 * The handle owns HOST memory (node -> query index, positive-tuple hash
 * set); it is the one object in this ABI that allocates, and one handle
 * must not be driven from two threads at once.  arity <= 4, node ids < 2^31.
 * positives [n_pos, arity], filter_tuples [n_filter, arity] (the canonical
 * positive set, pipeline.py:278-280), neg_pool [n_pool, arity] or NULL. */
typedef struct wj_planner wj_planner;
int wj_planner_create(const int64_t *positives, int64_t n_pos, int32_t arity, const int64_t *filter_tuples,
                      int64_t n_filter, int64_t num_nodes, int32_t batch_capacity, int32_t batch_size,
                      int32_t k_neg, const int64_t *neg_pool, int64_t n_pool, wj_planner **out);
int wj_planner_destroy(wj_planner *planner);
int wj_planner_set_rng(wj_planner *planner, const uint64_t *words6);
int wj_planner_get_rng(const wj_planner *planner, uint64_t *words6);
/* One batch: queries_out [cap, arity] (positives first, then negatives),
 * labels_out [cap] (1 / 0, may be NULL); n_queries 0 = empty batch. */
int wj_planner_next(wj_planner *planner, int64_t *queries_out, float *labels_out, int64_t cap,
                    int64_t *n_queries_out, int64_t *n_pos_out, int64_t *n_seeds_out);
/* Units of identical queries (same anchor tuple, same order) of a batch:
 * groups_out [(2 + arity) n + 2] int32 = [G | start[0..G] | order[0..n) |
 * tuple[0..G)[arity]] (each unit's anchors; node ids < 2^31); each tuple's
 * queries in batch order, cut into units of <= max_group members (0 = no
 * cap), larger units first (stable: first occurrence).  Host only; the
 * reference's in-seed negatives (pipeline.py:132-166) repeat tuples (~28 %
 * of a C3 batch).  The
 * producer thread of wj_planner_start_epoch uses max_group = 4. */
int wj_group_queries(const int64_t *queries, int64_t n, int32_t arity, int32_t max_group, int32_t *groups_out,
                     int64_t *n_groups_out);

/* One epoch of train()'s batch loop (pipeline.py:287-305) on a producer
 * thread, ahead of the consumer: batches until the positives consumed reach
 * n_pos or a batch is empty, written in order into a caller-owned ring of
 * n_slots slots (ring_queries [n_slots, cap, arity], ring_labels
 * [n_slots, cap], e.g. pinned host memory; ring_groups [n_slots, (2+arity)*cap + 2]
 * or NULL receives each batch's wj_group_queries).  wj_planner_acquire spins until
 * the next batch is ready and returns its slot (-1 at the end of the epoch,
 * after which the rng state is the reference's end-of-epoch state);
 * wj_planner_release hands a slot back once its contents have been copied.
 * wj_planner_stop abandons the epoch (the rng state is then ahead). */
int wj_planner_start_epoch(wj_planner *planner, int64_t *ring_queries, float *ring_labels, int32_t *ring_groups,
                           int32_t n_slots, int64_t cap);
int wj_planner_acquire(wj_planner *planner, int32_t *slot_out, int64_t *n_queries_out, int64_t *n_pos_out);
int wj_planner_release(wj_planner *planner, int32_t slot);
int wj_planner_stop(wj_planner *planner);

/* ---- Native training epoch (replaces train()'s batch loop body,
 * pipeline.py:287-310, when planner and step executor are native) ----------
 * After wj_planner_start_epoch on the pinned ring (ring_q [n_slots, cap,
 * arity], ring_g [n_slots, (2+arity)*cap + 2]): for every batch of the epoch
 * (or the first max_steps; max_steps < 0: all), copy it H2D on copy_stream
 * one batch ahead into a device ring (dev_q [dev_depth, cap, arity], dev_g
 * [dev_depth, (2+arity)*cap + 2]), then wj_stepper_run on stream with labels
 * dev_labels + cap - n_pos (dev_labels = cap ones then cap zeros) and the
 * loss into loss_out[k] (device or pinned host).  Planner slots are handed
 * back once copied; steps_done receives the number of steps launched and
 * h2d_bytes (nullable) the bytes copied host -> device (batches issued).  The
 * caller stops the planner if max_steps ended the loop before the epoch. */
int wj_train_epoch(wj_stepper *stepper, wj_planner *planner, const int64_t *ring_q, const int32_t *ring_g,
                   int32_t n_slots, int64_t cap, int32_t arity, int64_t *dev_q, int32_t *dev_g, int32_t dev_depth,
                   const float *dev_labels, float *loss_out, int64_t max_steps, wj_stream_t stream,
                   wj_stream_t copy_stream, int64_t *steps_done, int64_t *h2d_bytes);

/* Host -> device copy of a large pageable host array (the graph CSR of a
 * host-input preprocess; replaces the torch/driver pageable copy inside
 * reference-facing sampler.preprocess(graph) -> sampler.py:94-151): the
 * array is split over `threads` workers, each staging its part through its
 * own pinned double buffer on its own stream.  Synchronous: every byte is on
 * the device when it returns. */
int wj_upload(void *dst, const void *src, int64_t bytes, int32_t threads);

#ifdef __cplusplus
}
#endif

#endif /* WALKJOIN_B200_H */
