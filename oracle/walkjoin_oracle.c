/*
 * walkjoin_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load the library built from it.
 * The product package never imports, links or calls it.
 *
 * Every function restates one numba kernel of the reference
 * (/root/reference/pkg/src/walkjoin/_kernels.py, cited as K:line).  The
 * reference parallelises with numba `prange`; this restatement uses OpenMP
 * with the same disjoint-slot write discipline, so output is independent of
 * the thread count exactly as in the reference (K:5-8).
 *
 * Pinned against the reference itself: tests/golden/make_golden.py runs the
 * reference (with the SURVEY Appendix A numba shim) and commits fixtures;
 * tests/test_oracle_golden.py checks this file against them.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define WJ_GOLDEN 0x9E3779B97F4A7C15ULL

/* K:22-27 splitmix64 finalizer */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline void set_threads(int threads) {
#ifdef _OPENMP
    if (threads < 1) threads = 1;
    omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

/* K:47-50 start state of node u's walk stream */
uint64_t wjo_node_stream_state(uint64_t seed, int64_t u) {
    return mix64(seed + WJ_GOLDEN * ((uint64_t)u + 1ULL));
}

/* K:53-66 M walks of L steps from u; returns the end state.  K:36-39 is the
 * multiply-shift draw ((z >> 32) * deg) >> 32. */
uint64_t wjo_sample_node_walks(const int64_t *idxptr, const int32_t *indices, int64_t u,
                               int64_t num_walks, int64_t num_steps, uint64_t state,
                               int32_t *out) {
    const int64_t width = num_steps + 1;
    for (int64_t j = 0; j < num_walks; ++j) {
        int64_t cur = u;
        out[j * width] = (int32_t)cur;
        for (int64_t i = 1; i <= num_steps; ++i) {
            int64_t deg = idxptr[cur + 1] - idxptr[cur];
            if (deg > 0) {
                state += WJ_GOLDEN;
                uint64_t z = mix64(state);
                int64_t off = (int64_t)(((z >> 32) * (uint64_t)deg) >> 32);
                cur = indices[idxptr[cur] + off];
            }
            out[j * width + i] = (int32_t)cur;
        }
    }
    return state;
}

/* K:69-74 */
void wjo_sample_all_walks(const int64_t *idxptr, const int32_t *indices, int64_t n,
                          int64_t num_walks, int64_t num_steps, uint64_t seed, int32_t *walks,
                          int threads) {
    set_threads(threads);
    const int64_t block = num_walks * (num_steps + 1);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t u = 0; u < n; ++u) {
        wjo_sample_node_walks(idxptr, indices, u, num_walks, num_steps,
                              wjo_node_stream_state(seed, u), walks + u * block);
    }
}

/* K:69-74 restricted to an explicit anchor list (bench.py samples the
 * anchors of one batch, or a contiguous shard, with their own streams). */
void wjo_sample_nodes(const int64_t *idxptr, const int32_t *indices, const int64_t *nodes,
                      int64_t count, int64_t num_walks, int64_t num_steps, uint64_t seed,
                      int32_t *walks, int threads) {
    set_threads(threads);
    const int64_t block = num_walks * (num_steps + 1);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t k = 0; k < count; ++k) {
        const int64_t u = nodes[k];
        wjo_sample_node_walks(idxptr, indices, u, num_walks, num_steps,
                              wjo_node_stream_state(seed, u), walks + k * block);
    }
}

/* K:77-84 linear probe in a local table */
static inline int64_t probe_local(const int64_t *keys, int64_t x, int64_t cap_mask) {
    int64_t h = (int64_t)(mix64((uint64_t)x) & (uint64_t)cap_mask);
    for (;;) {
        int64_t k = keys[h];
        if (k == -1 || k == x) return h;
        h = (h + 1) & cap_mask;
    }
}

/* K:87-101 number of distinct ids per walk block */
void wjo_count_distinct_all(const int32_t *walks, int64_t n, int64_t block, int64_t local_cap,
                            int64_t *counts_out, int threads) {
    set_threads(threads);
#pragma omp parallel
    {
        int64_t *keys = (int64_t *)malloc(sizeof(int64_t) * local_cap);
#pragma omp for schedule(dynamic, 256)
        for (int64_t u = 0; u < n; ++u) {
            for (int64_t t = 0; t < local_cap; ++t) keys[t] = -1;
            int64_t k = 0;
            const int32_t *flat = walks + u * block;
            for (int64_t t = 0; t < block; ++t) {
                int64_t x = flat[t];
                int64_t h = probe_local(keys, x, local_cap - 1);
                if (keys[h] == -1) {
                    keys[h] = x;
                    ++k;
                }
            }
            counts_out[u] = k;
        }
        free(keys);
    }
}

/* K:104-126 distinct ids in first-appearance order + positional counts */
void wjo_fill_distinct_all(const int32_t *walks, int64_t n, int64_t num_walks, int64_t width,
                           const int64_t *offsets, int64_t local_cap, int32_t *nodes_out,
                           int32_t *vecs_out, int threads) {
    set_threads(threads);
    const int64_t block = num_walks * width;
#pragma omp parallel
    {
        int64_t *keys = (int64_t *)malloc(sizeof(int64_t) * local_cap);
        int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * local_cap);
#pragma omp for schedule(dynamic, 256)
        for (int64_t u = 0; u < n; ++u) {
            for (int64_t t = 0; t < local_cap; ++t) keys[t] = -1;
            const int64_t base = offsets[u];
            int64_t k = 0;
            const int32_t *w = walks + u * block;
            for (int64_t j = 0; j < num_walks; ++j) {
                for (int64_t i = 0; i < width; ++i) {
                    int64_t x = w[j * width + i];
                    int64_t h = probe_local(keys, x, local_cap - 1);
                    if (keys[h] == -1) {
                        keys[h] = x;
                        slot[h] = k;
                        nodes_out[base + k] = (int32_t)x;
                        for (int64_t c = 0; c < width; ++c) vecs_out[(base + k) * width + c] = 0;
                        ++k;
                    }
                    vecs_out[(base + slot[h]) * width + i] += 1;
                }
            }
        }
        free(keys);
        free(slot);
    }
}

/* K:129-134 */
static inline uint64_t hash_row(const int32_t *row, int64_t width) {
    uint64_t h = WJ_GOLDEN;
    for (int64_t c = 0; c < width; ++c) h = mix64(h ^ ((uint64_t)(int64_t)row[c] + WJ_GOLDEN));
    return h;
}

/* K:137-171 sequential scan-order dedup; returns the unique count.  ids_out
 * gets 0-based ids (store.py:121 adds one). */
int64_t wjo_intern_rows(const int32_t *vecs, int64_t n_rows, int64_t width, int32_t *ids_out,
                        int64_t *reps_out) {
    int64_t cap = 1;
    while (cap < 2 * n_rows + 2) cap <<= 1;
    const int64_t mask = cap - 1;
    int64_t *table = (int64_t *)malloc(sizeof(int64_t) * cap);
    if (!table) return -1;
    for (int64_t t = 0; t < cap; ++t) table[t] = -1;
    int64_t n_unique = 0;
    for (int64_t r = 0; r < n_rows; ++r) {
        const int32_t *row = vecs + r * width;
        int64_t h = (int64_t)(hash_row(row, width) & (uint64_t)mask);
        for (;;) {
            int64_t s = table[h];
            if (s == -1) {
                table[h] = r;
                ids_out[r] = (int32_t)n_unique;
                reps_out[n_unique] = r;
                ++n_unique;
                break;
            }
            if (memcmp(vecs + s * width, row, sizeof(int32_t) * width) == 0) {
                ids_out[r] = ids_out[s];
                break;
            }
            h = (h + 1) & mask;
        }
    }
    free(table);
    return n_unique;
}

/* K:174-188 packed per-node open addressing; keys_out pre-filled with -1 */
void wjo_build_dicts(const int32_t *nodes_flat, const int32_t *vals_flat,
                     const int64_t *item_offsets, const int64_t *cap_offsets, int64_t n,
                     int32_t *keys_out, int32_t *vals_out, int threads) {
    set_threads(threads);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t u = 0; u < n; ++u) {
        const int64_t base = cap_offsets[u];
        const int64_t mask = cap_offsets[u + 1] - base - 1;
        for (int64_t t = item_offsets[u]; t < item_offsets[u + 1]; ++t) {
            int64_t x = nodes_flat[t];
            int64_t h = (int64_t)(mix64((uint64_t)x) & (uint64_t)mask);
            while (keys_out[base + h] != -1) h = (h + 1) & mask;
            keys_out[base + h] = (int32_t)x;
            vals_out[base + h] = vals_flat[t];
        }
    }
}

/* K:191-200 */
static inline int32_t dict_get(const int32_t *keys, const int32_t *vals, int64_t base, int64_t mask,
                               int64_t x) {
    int64_t h = (int64_t)(mix64((uint64_t)x) & (uint64_t)mask);
    for (;;) {
        int64_t k = keys[base + h];
        if (k == x) return vals[base + h];
        if (k == -1) return 0;
        h = (h + 1) & mask;
    }
}

/* K:203-206 */
int32_t wjo_dict_get_one(const int32_t *keys, const int32_t *vals, const int64_t *cap_offsets,
                         int64_t u, int64_t x) {
    const int64_t base = cap_offsets[u];
    return dict_get(keys, vals, base, cap_offsets[u + 1] - base - 1, x);
}

/* K:209-245 walk concatenation + query-level RPE-id buffer */
void wjo_join_fill(const int32_t *walks, int64_t num_walks, int64_t width, const int32_t *dict_keys,
                   const int32_t *dict_vals, const int64_t *cap_offsets, const int64_t *queries,
                   int64_t n_batch, int64_t arity, int32_t *walk_nodes_out, int32_t *rpe_ids_out,
                   int threads) {
    set_threads(threads);
    const int64_t block = num_walks * width;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t task = 0; task < n_batch * arity; ++task) {
        const int64_t b = task / arity, j = task % arity;
        const int64_t anchor = queries[b * arity + j];
        int32_t *wn = walk_nodes_out + (b * arity + j) * block;
        memcpy(wn, walks + anchor * block, sizeof(int32_t) * block);
        const int64_t base = cap_offsets[anchor];
        const int64_t mask = cap_offsets[anchor + 1] - base - 1;
        int32_t *ri = rpe_ids_out + b * (arity * block) * arity;
        for (int64_t a = 0; a < arity; ++a) {
            const int32_t *src = walks + queries[b * arity + a] * block;
            const int64_t r0 = a * block;
            for (int64_t t = 0; t < block; ++t)
                ri[(r0 + t) * arity + j] = dict_get(dict_keys, dict_vals, base, mask, src[t]);
        }
    }
}

/* pipeline.py:178 / joiner.py:103-104 densify: table[rpe_ids] -> float64 */
void wjo_densify(const int32_t *table, int64_t width, const int32_t *rpe_ids, int64_t n_ids,
                 double *out, int threads) {
    set_threads(threads);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_ids; ++t) {
        const int32_t *v = table + (int64_t)rpe_ids[t] * width;
        for (int64_t c = 0; c < width; ++c) out[t * width + c] = (double)v[c];
    }
}

/* Typed / metapath walks.  NO reference implementation exists
 * (SPEC.md:121-124 leaves typed walks open), so this restates OUR definition
 * (include/walkjoin_b200.h, wj_sample_walks_typed) straight from the CSR and
 * the per-entry edge types, without the device's type-grouped layout: step i
 * of walk j from u follows an edge of type metapath[(i-1) % P] (negative =
 * any), the idx-th such edge of the current node in CSR order with
 * idx = umulhi32(mix64(S0(u) + (j*L+i)*G), count); none -> stay.  Its
 * homogeneous special case is pinned to the reference sampler (K:53-74) by
 * tests/test_typed_walks.py; the typed semantics are "parity unpinned". */
void wjo_sample_typed(const int64_t *idxptr, const int32_t *indices, const uint8_t *etype,
                      const int8_t *metapath, int64_t P, int64_t n, int64_t num_walks,
                      int64_t num_steps, uint64_t seed, int32_t *walks, int threads) {
    set_threads(threads);
    const int64_t width = num_steps + 1;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t u = 0; u < n; ++u) {
        const uint64_t s0 = wjo_node_stream_state(seed, u);
        int32_t *out = walks + u * num_walks * width;
        for (int64_t j = 0; j < num_walks; ++j) {
            int64_t cur = u;
            out[j * width] = (int32_t)cur;
            for (int64_t i = 1; i <= num_steps; ++i) {
                const int t = metapath[(i - 1) % P];
                int64_t cnt = 0;
                for (int64_t e = idxptr[cur]; e < idxptr[cur + 1]; ++e) cnt += (t < 0 || etype[e] == t);
                if (cnt > 0) {
                    const uint64_t z = mix64(s0 + (uint64_t)(j * num_steps + i) * WJ_GOLDEN);
                    int64_t k = (int64_t)(((z >> 32) * (uint64_t)cnt) >> 32);
                    for (int64_t e = idxptr[cur]; e < idxptr[cur + 1]; ++e) {
                        if (t < 0 || etype[e] == t) {
                            if (k == 0) {
                                cur = indices[e];
                                break;
                            }
                            --k;
                        }
                    }
                }
                out[j * width + i] = (int32_t)cur;
            }
        }
    }
}
