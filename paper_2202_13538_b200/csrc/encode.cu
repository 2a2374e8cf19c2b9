// Join fused with the encoder's first layer (forward + the statistics its
// backward needs), sm_100a.
//
// Reference: joiner.join_batch_arrays + pipeline._dense_batch + encoder
// forward/backward (joiner.py:53-71, pipeline.py:169-182, encoder.py:
// 126-233).  The reference materialises, per query, a [A*M*(L+1), A*(L+1)]
// float64 matrix X, multiplies it by W1 ([rows, 64] hidden), applies ReLU and
// dropout, and its backward forms dW1 = X^T dZ1.  Two exact identities make
// that matrix unnecessary:
//
//  * every row of X is determined by the walked node's RPE ids: the rows of
//    anchor a's block that land on the same node x are identical, so X has
//    only U_a distinct rows per block, with multiplicity n_x = (row sum of
//    x's count vector relative to a);
//  * the downstream layers only see the row MEAN of a1 (mean commutes with
//    the affine W2 layer), and the backward only needs
//      pooled[h] = sum_r relu(z_r[h]) * d_r[h],
//      S[c][h]   = sum_r x_r[c] * 1[z_r[h] > 0] * d_r[h],
//      msum[h]   = sum_r 1[z_r[h] > 0] * d_r[h]
//    (dW1 = sum_b S_b * g_b / keep, db1 = sum_b msum_b * g_b / keep with
//    g_b = dhq_b W2^T / rows).
//
// So one CTA per query resolves the distinct landings against every query
// anchor (as the join kernel), and for each distinct landing computes
// z = b1 + x W1 once (x is sparse: a handful of non-zero counts), draws the
// n_x * H dropout bits of its rows from a counter-based splitmix64 stream,
// and accumulates pooled / S / msum in registers (one warp lane per 2 hidden
// units).  Nothing of size [rows, *] ever touches memory.
#include "common.cuh"

namespace wj {

constexpr int kEncWarps = 8;

struct EncArgs {
    const int64_t *queries;
    int64_t n_batch;
    const int64_t *offsets;
    const int32_t *ux;
    const int32_t *uid;
    int W, P, max_u;
    const uint64_t *tkeys;
    int64_t tlen;
    int stage_table;
    int cb;
    const float *w1;  // [A*W, H]
    const float *b1;  // [H]
    uint32_t keep_thr;  // keep if u16 < keep_thr; 65536 = no dropout
    uint64_t seed;
    const int64_t *step;  // device counter (read per launch: CUDA-graph safe)
    float *pooled;      // [B, H]
    float *s_out;       // [B, A*W, H] or null
    float *msum;        // [B, H] or null
};

__device__ __forceinline__ int ub_int(const int *a, int n, int v) {  // first i with a[i] > v
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int lb_s(const int32_t *a, int n, int32_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// A query anchors, AW = A * (L+1) input columns, HU = hidden units per lane
//
// Per query (one CTA, 8 warps) and per anchor block a:
//  1. pre-pass, one thread per distinct landing l: its RPE ids against every
//     query anchor, the non-zero entries of x_l (u16: c << 12 | count), the
//     row count n_l, and a CTA-wide exclusive scan of (n_l, nnz_l);
//  2. the block's P virtual rows are split evenly over the warps; a warp
//     walks the landings of its row range: z = b1 + x W1 over the non-zero
//     entries, kept counts from the dropout stream (one splitmix64 word per
//     (row group, lane) covers 4/HU rows x HU units), then pooled / msum in
//     registers and S in the warp's shared-memory accumulator.
template <int A, int AW, int HU>
__global__ void __launch_bounds__(kEncWarps * 32) join_encode_kernel(EncArgs g) {
    constexpr int H = HU * 32;
    constexpr int NV = 2 + AW;  // per-warp accumulators: pooled, msum, S[AW]
    constexpr int RPW = 4 / HU > 0 ? 4 / HU : 1;  // rows per random word
    constexpr int NT = kEncWarps * 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int P = g.P, mu = g.max_u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *w1s = reinterpret_cast<float *>(smem_raw);     // [AW][H]
    float *b1s = w1s + AW * H;                             // [H]
    float *sacc = b1s + H;                                 // [warps][NV][H]
    int64_t *qa = reinterpret_cast<int64_t *>(sacc + kEncWarps * NV * H);  // [4]
    int *un = reinterpret_cast<int *>(qa + 4);             // [4]
    unsigned long long *wsum = reinterpret_cast<unsigned long long *>(un + 4);  // [warps + 1]
    int32_t *sx = reinterpret_cast<int32_t *>(wsum + kEncWarps + 2);  // [A][mu]
    int32_t *sid = sx + A * mu;                            // [A][mu]
    int32_t *cross = sid + A * mu;                         // [A][A-1][mu]
    int2 *loc = reinterpret_cast<int2 *>(cross + A * (A - 1) * mu + 2);  // [mu + 1] {rowoff, nzoff}
    uint16_t *nz = reinterpret_cast<uint16_t *>(loc + mu + 1);            // [mu * AW]
    uint64_t *tks = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(nz + (size_t)mu * AW) + 15) & ~uintptr_t(15));
    const uint64_t cmask = (1ULL << g.cb) - 1;
    const uint64_t skey = mix64(g.seed + kGolden * ((uint64_t)(g.step ? *g.step : 0) + 1ULL));
    const bool dropout = g.keep_thr < 65536u;
    float *my = sacc + warp * NV * H;

    for (int i = threadIdx.x; i < AW * H; i += NT) w1s[i] = g.w1[i];
    for (int i = threadIdx.x; i < H; i += NT) b1s[i] = g.b1[i];
    if (g.stage_table)
        for (int64_t i = threadIdx.x; i < g.tlen; i += NT) tks[i] = g.tkeys[i];

    for (int64_t b = blockIdx.x; b < g.n_batch; b += gridDim.x) {
        if (threadIdx.x < A) {
            const int64_t q = g.queries[b * A + threadIdx.x];
            qa[threadIdx.x] = q;
            un[threadIdx.x] = (int)(g.offsets[q + 1] - g.offsets[q]);
        }
        for (int i = lane; i < NV * H; i += 32) my[i] = 0.f;
        __syncthreads();
#pragma unroll
        for (int a = 0; a < A; ++a) {
            const int64_t lo = g.offsets[qa[a]];
            for (int i = threadIdx.x; i < un[a]; i += NT) {
                sx[a * mu + i] = __ldg(g.ux + lo + i);
                sid[a * mu + i] = __ldg(g.uid + lo + i);
            }
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < A; ++a) {
#pragma unroll
            for (int jj = 0; jj < A - 1; ++jj) {
                const int j = jj < a ? jj : jj + 1;
                const int nj = un[j];
                const int32_t *xj = sx + j * mu;
                int32_t *dst = cross + (a * (A - 1) + jj) * mu;
                for (int k = threadIdx.x; k < un[a]; k += NT) {
                    const int32_t x = sx[a * mu + k];
                    const int pos = lb_s(xj, nj, x);
                    dst[k] = (pos < nj && xj[pos] == x) ? sid[j * mu + pos] : 0;
                }
            }
        }

        float pooled[HU], msum[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) pooled[u] = msum[u] = 0.f;

        for (int a = 0; a < A; ++a) {
            const int U = un[a];
            __syncthreads();  // cross ready; previous block's loc/nz consumers done
            // ---- pre-pass: thread t owns landings [t*per, (t+1)*per)
            const int per = (U + NT - 1) / NT;
            const int l0 = threadIdx.x * per;
            const int l1 = min(l0 + per, U);
            unsigned long long tot = 0;  // (nnz << 32) | rows
            for (int l = l0; l < l1; ++l) {
                int rows = 0, cntnz = 0;
#pragma unroll
                for (int j = 0; j < A; ++j) {
                    const int id = (j == a) ? sid[a * mu + l]
                                            : cross[(a * (A - 1) + (j < a ? j : j - 1)) * mu + l];
                    const uint64_t key = g.stage_table ? tks[id] : __ldg(g.tkeys + id);
#pragma unroll
                    for (int c = 0; c < AW / A; ++c) {
                        const uint32_t v = (uint32_t)((key >> (g.cb * c)) & cmask);
                        cntnz += v != 0;
                        if (j == a) rows += (int)v;
                    }
                }
                tot += ((unsigned long long)cntnz << 32) | (unsigned)rows;
            }
            // CTA exclusive scan of the per-thread totals
            unsigned long long incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long t = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long run = 0;
                for (int w = 0; w < kEncWarps; ++w) {
                    const unsigned long long t = wsum[w];
                    wsum[w] = run;
                    run += t;
                }
                wsum[kEncWarps] = run;
            }
            __syncthreads();
            unsigned long long pos = wsum[warp] + incl - tot;
            for (int l = l0; l < l1; ++l) {
                int rows = 0;
                int e = (int)(pos >> 32);
                loc[l] = make_int2((int)(unsigned)pos, e);
#pragma unroll
                for (int j = 0; j < A; ++j) {
                    const int id = (j == a) ? sid[a * mu + l]
                                            : cross[(a * (A - 1) + (j < a ? j : j - 1)) * mu + l];
                    const uint64_t key = g.stage_table ? tks[id] : __ldg(g.tkeys + id);
#pragma unroll
                    for (int c = 0; c < AW / A; ++c) {
                        const uint32_t v = (uint32_t)((key >> (g.cb * c)) & cmask);
                        if (v) nz[e++] = (uint16_t)(((j * (AW / A) + c) << 12) | v);
                        if (j == a) rows += (int)v;
                    }
                }
                pos += ((unsigned long long)(e - (int)(pos >> 32)) << 32) + (unsigned)rows;
            }
            if (threadIdx.x == 0) {
                const unsigned long long t = wsum[kEncWarps];
                loc[U] = make_int2((int)(unsigned)t, (int)(t >> 32));
            }
            __syncthreads();
            // ---- rows of this warp
            const int r_beg = (int)((int64_t)P * warp / kEncWarps);
            const int r_end = (int)((int64_t)P * (warp + 1) / kEncWarps);
            if (r_beg >= r_end) continue;
            int l;
            {
                int lo_ = 0, hi_ = U + 1;  // first l with loc[l].x > r_beg, minus one
                while (lo_ < hi_) {
                    const int mid = (lo_ + hi_) >> 1;
                    if (loc[mid].x <= r_beg)
                        lo_ = mid + 1;
                    else
                        hi_ = mid;
                }
                l = lo_ - 1;
            }
            int r = r_beg;
            const uint64_t qkey = mix64(skey ^ mix64(((uint64_t)b << 3) | (uint64_t)a));
            int2 cur = loc[l];
            int64_t word_idx = -1;
            uint64_t rnd = 0;
            while (r < r_end) {
                const int2 nxt = loc[l + 1];
                const int cnt = min(nxt.x, r_end) - r;
                float z[HU];
#pragma unroll
                for (int u = 0; u < HU; ++u) z[u] = b1s[u * 32 + lane];
                for (int e = cur.y; e < nxt.y; ++e) {
                    const uint32_t ent = nz[e];
                    const float v = (float)(ent & 0xFFFu);
                    const float *wrow = w1s + (ent >> 12) * H + lane;
#pragma unroll
                    for (int u = 0; u < HU; ++u) z[u] = fmaf(v, wrow[u * 32], z[u]);
                }
                float kept[HU];
                if (!dropout) {
#pragma unroll
                    for (int u = 0; u < HU; ++u) kept[u] = (float)cnt;
                } else {
                    int kc[HU];
#pragma unroll
                    for (int u = 0; u < HU; ++u) kc[u] = 0;
                    for (int row = r; row < r + cnt; ++row) {
                        const int64_t wi = row / RPW;
                        if (wi != word_idx) {
                            word_idx = wi;
                            rnd = mix64(qkey + (((uint64_t)wi << 5) | (uint64_t)lane) * kGolden);
                        }
                        const int s0 = (row - (int)wi * RPW) * HU;
#pragma unroll
                        for (int u = 0; u < HU; ++u)
                            kc[u] += ((uint32_t)(rnd >> (16 * (s0 + u))) & 0xFFFFu) < g.keep_thr;
                    }
#pragma unroll
                    for (int u = 0; u < HU; ++u) kept[u] = (float)kc[u];
                }
                float gk[HU];
#pragma unroll
                for (int u = 0; u < HU; ++u) {
                    const bool pz = z[u] > 0.f;
                    gk[u] = pz ? kept[u] : 0.f;
                    pooled[u] = fmaf(pz ? z[u] : 0.f, kept[u], pooled[u]);
                    msum[u] += gk[u];
                }
                for (int e = cur.y; e < nxt.y; ++e) {
                    const uint32_t ent = nz[e];
                    const float v = (float)(ent & 0xFFFu);
                    float *srow = my + (2 + (ent >> 12)) * H + lane;
#pragma unroll
                    for (int u = 0; u < HU; ++u) srow[u * 32] = fmaf(v, gk[u], srow[u * 32]);
                }
                r += cnt;
                ++l;
                cur = nxt;
            }
        }
        // ---- CTA reduction of the per-warp accumulators, one store per value
#pragma unroll
        for (int u = 0; u < HU; ++u) {
            my[u * 32 + lane] = pooled[u];
            my[H + u * 32 + lane] = msum[u];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < NV * H; i += NT) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kEncWarps; ++w) s += sacc[w * NV * H + i];
            const int v = i / H, h = i - v * H;
            if (v == 0)
                g.pooled[b * H + h] = s;
            else if (v == 1) {
                if (g.msum) g.msum[b * H + h] = s;
            } else if (g.s_out) {
                g.s_out[(b * AW + (v - 2)) * (int64_t)H + h] = s;
            }
        }
        __syncthreads();
    }
}

using EncKernel = void (*)(EncArgs);

template <int A, int AW>
static EncKernel pick_hu(int hu) {
    switch (hu) {
        case 1: return join_encode_kernel<A, AW, 1>;
        case 2: return join_encode_kernel<A, AW, 2>;
        case 4: return join_encode_kernel<A, AW, 4>;
        default: return nullptr;
    }
}

static EncKernel pick(int A, int W, int hu) {
#define WJ_CASE(a, w) \
    if (A == a && W == w) return pick_hu<a, a * w>(hu);
    WJ_CASE(1, 2) WJ_CASE(1, 3) WJ_CASE(1, 4) WJ_CASE(1, 5)
    WJ_CASE(2, 2) WJ_CASE(2, 3) WJ_CASE(2, 4) WJ_CASE(2, 5) WJ_CASE(2, 6) WJ_CASE(2, 7) WJ_CASE(2, 8)
    WJ_CASE(3, 2) WJ_CASE(3, 3) WJ_CASE(3, 4) WJ_CASE(3, 5)
    WJ_CASE(4, 3) WJ_CASE(4, 4) WJ_CASE(4, 5)
#undef WJ_CASE
    return nullptr;
}

}  // namespace wj

extern "C" int wj_join_encode_simt(const int64_t *queries, int64_t n_batch, int32_t arity,
                              const int64_t *offsets, const int32_t *uniq_x,
                              const int32_t *uniq_id, int32_t num_walks, int32_t num_steps,
                              int32_t max_unique, const uint64_t *table_keys, int64_t table_len,
                              const float *w1, const float *b1, int32_t hidden, float keep_prob,
                              uint64_t seed, const int64_t *step, float *pooled_out, float *s_out,
                              float *msum_out, wj_stream_t stream) {
    using namespace wj;
    if (arity < 1 || num_walks < 1 || num_steps < 1 || !(keep_prob > 0.f) || keep_prob > 1.f) {
        set_error("bad arity / shape / keep_prob");
        return WJ_ERR_ARG;
    }
    const int W = num_steps + 1;
    if (hidden % 32 || hidden < 32 || hidden > 128 || hidden == 96) {
        set_error("hidden=%d: the fused encoder supports 32, 64, 128", hidden);
        return WJ_ERR_UNSUPPORTED;
    }
    EncKernel k = pick(arity, W, hidden / 32);
    if (!k) {
        set_error("fused join+encode not instantiated for arity %d, L+1=%d", arity, W);
        return WJ_ERR_UNSUPPORTED;
    }
    if ((int64_t)num_walks * W > 65535) {
        set_error("M*(L+1) too large");
        return WJ_ERR_UNSUPPORTED;
    }
    EncArgs g;
    g.queries = queries;
    g.n_batch = n_batch;
    g.offsets = offsets;
    g.ux = uniq_x;
    g.uid = uniq_id;
    g.W = W;
    g.P = num_walks * W;
    g.max_u = max_unique < 1 ? 1 : max_unique;
    g.tkeys = table_keys;
    g.tlen = table_len;
    g.cb = bits_for((uint64_t)num_walks);
    g.w1 = w1;
    g.b1 = b1;
    const double thr = (double)keep_prob * 65536.0;
    g.keep_thr = keep_prob >= 1.f ? 65536u : (uint32_t)(thr + 0.5);
    g.seed = seed;
    g.step = step;
    g.pooled = pooled_out;
    g.s_out = s_out;
    g.msum = msum_out;
    const int AW = arity * W, H = hidden;
    size_t base = (size_t)(AW * H + H + kEncWarps * (2 + AW) * H) * 4 + 64 + 8 * (kEncWarps + 2) +
                  (size_t)arity * g.max_u * 8 + (size_t)arity * (arity - 1) * g.max_u * 4 + 8 +
                  (size_t)(g.max_u + 1) * 8 + (size_t)g.max_u * AW * 2 + 32;
    const size_t limit = 200 * 1024;
    g.stage_table = (base + (size_t)table_len * 8 <= limit && table_len <= 8192) ? 1 : 0;
    const size_t smem = base + (g.stage_table ? (size_t)table_len * 8 : 0);
    if (smem > limit) {
        set_error("join_encode needs %zu B of shared memory", smem);
        return WJ_ERR_UNSUPPORTED;
    }
    if (n_batch == 0) return WJ_OK;  // an empty batch probes the envelope
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        set_error("join_encode smem attribute: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kEncWarps * 32, smem);
    int64_t blocks = n_batch;
    const int64_t cap = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1) * 8;
    if (blocks > cap) blocks = cap;
    k<<<(unsigned)blocks, kEncWarps * 32, smem, (cudaStream_t)stream>>>(g);
    return check_launch("wj_join_encode");
}
