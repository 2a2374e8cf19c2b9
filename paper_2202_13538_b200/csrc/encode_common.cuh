// Shared pieces of the two join+encode kernels (encode_mma.cu: mma.sync
// tiles; encode_tc.cu: tcgen05 tiles): kernel arguments, per-query metadata,
// the fp16 landing-row splice, the merge-path cross ids and the row build.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"

namespace wj {

constexpr int kWS = 24;       // halves per staged W^T row (48 B: conflict-free ldmatrix)
constexpr int kRedS = 17;     // floats per unit in the reduction buffer (16 S^T cols + pad)
constexpr int kRowB = 32;     // bytes per landing row [x | 1 | 0..] (16 halves)
constexpr int kWtBytes = 2 * 64 * kWS * 2;
constexpr int kRowU = 4;      // landings per thread per batch in the row build
constexpr int kMetaQ = 16;    // queries whose metadata a CTA loads at once
struct QMeta {
    int64_t lo, vo;  // first entry of the anchor's sorted list / of its virtual landings
    int u, v2, v1;   // list length, 2-row and 1-row virtual landings
};
constexpr int kHdrBytes = (kMetaQ * 3 * (int)sizeof(QMeta) + 16 + 64 + 16 + 15) & ~15;  // meta | wscale[4] | wred[16] | next_b

struct EncMmaArgs {
    const int64_t *queries;
    int64_t n_batch;
    const int64_t *offsets;
    const int32_t *ux;
    const int32_t *uid;
    const int64_t *voff;
    const int32_t *vcnt;
    const uint16_t *vslots;
    const uint4 *trow;  // [tlen] fp16 count rows (8 halves)
    int mu, lcap, xr_bytes;
    const int32_t *cross;  // [B][A][A-1][mu] cross RPE ids (wj_join_cross) or null: search in-kernel
    const float *w1;  // [AW, 64]
    const float *b1;  // [64]
    uint32_t t11, t21, t22;  // packed 14-bit thresholds (both lanes): 1-row; 2-row K>=1, K>=2
    uint64_t seed;
    const int64_t *step;
    float *pooled;  // [B, 64]
    float *s_out;   // [B, AW, 64] or null
    float *msum;    // [B, 64] or null
    int32_t *qsched;  // [2] zeroed query-grab / done counters (dynamic scheduling) or null: static striding
    int qsched_reset_by_tail;  // 1: the step's tail kernel zeroes qsched after its wait (no end-of-CTA reset)
    // dynamic scheduling over groups of identical queries (null: one query
    // per unit): [G | start[0..G] | order[0..B)] -- unit u = the queries
    // order[start[u] .. start[u+1]), all with the same anchor tuple, so the
    // unit stages, merges and builds its rows once and runs tiles +
    // reduction per member (each with its own dropout stream and outputs)
    const int32_t *groups;
    int64_t n_units;  // G with groups, else n_batch
    int64_t b_offset;  // index of query 0 in the global batch (dropout key; batch-sharded data parallel)
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}


// byte permute with the sign-replicate mode (selector nibble bit 3)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

__device__ __forceinline__ uint32_t hadd2_u32(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// Output word k of the row [x | 1 | 0...] (16 fp16 columns), where column
// c < A*W is count f = c % W of anchor block j = c / W, taken from the fp16
// table row r[j] (W <= 8 halves in 4 words), column A*W is 1.0.  All
// selectors are compile-time constants after unrolling: one PRMT per word.
template <int A, int W>
__device__ __forceinline__ uint32_t half_src(const uint32_t (&r)[A][4], int c, int &sel_hi) {
    constexpr int AW = A * W;
    if (c < AW) {
        const int j = c / W, f = c % W;
        sel_hi = f & 1;
        return r[j][f >> 1];
    }
    sel_hi = 0;
    return c == AW ? 0x3C003C00u : 0u;
}

template <int A, int W>
__device__ __forceinline__ void splice_row(const uint32_t (&r)[A][4], uint32_t (&out)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        int h0, h1;
        const uint32_t x = half_src<A, W>(r, 2 * k, h0);
        const uint32_t y = half_src<A, W>(r, 2 * k + 1, h1);
        out[k] = __byte_perm(x, y, (h0 ? 0x32u : 0x10u) | ((h1 ? 0x76u : 0x54u) << 8));
    }
}

// row l's two 16-B halves are XOR-swizzled by bit 2 of l, so the 8 rows of
// an ldmatrix phase are bank-conflict-free when they are consecutive
__device__ __forceinline__ uint32_t row_addr(uint32_t base, uint32_t l, uint32_t half) {
    return base + l * kRowB + (((half ^ (l >> 2)) & 1u) << 4);
}

// Cross RPE ids by merging the anchors' sorted lists (merge path): for every
// anchor pair (a, j) thread tid of nthr takes an equal slice of the merged
// order (one diagonal binary search, then a linear merge); equal ids are
// emitted list-a first, so an element of list j finds its partner at list a's
// previous position.  scr[a][jj][l] = RPE id of landing l of anchor a relative
// to the jj-th other anchor (0 if absent).
template <int A>
__device__ __forceinline__ void merge_cross(int tid, int nthr, int mu, const int32_t *sx, const int32_t *sid,
                                            const int (&U)[A], int32_t *scr) {
#pragma unroll
    for (int a = 0; a < A; ++a)
#pragma unroll
        for (int j = a + 1; j < A; ++j) {
            const int n0 = U[a], n1 = U[j], tot = n0 + n1;
            const int32_t *X0 = sx + a * mu, *X1 = sx + j * mu, *I0 = sid + a * mu, *I1 = sid + j * mu;
            int32_t *o0 = scr + (a * (A - 1) + (j - 1)) * mu;  // list a relative to j (jj = j - 1: j > a)
            int32_t *o1 = scr + (j * (A - 1) + a) * mu;        // list j relative to a (jj = a: a < j)
            const int d0 = (tid * tot) / nthr, d1 = ((tid + 1) * tot) / nthr;
            int lo = max(0, d0 - n1), hi = min(d0, n0);
            while (lo < hi) {  // merge-path split of diagonal d0 (ties: list a first)
                const int mid = (lo + hi) >> 1;
                if (X0[mid] <= X1[d0 - mid - 1])
                    lo = mid + 1;
                else
                    hi = mid;
            }
            int i0 = lo, i1 = d0 - lo;
            int32_t x0 = i0 < n0 ? X0[i0] : INT32_MAX, x1 = i1 < n1 ? X1[i1] : INT32_MAX;
            for (int d = d0; d < d1; ++d) {
                if (x0 <= x1 && i0 < n0) {
                    o0[i0] = x0 == x1 ? I1[i1] : 0;
                    ++i0;
                    x0 = i0 < n0 ? X0[i0] : INT32_MAX;
                } else {
                    o1[i1] = (i0 > 0 && X0[i0 - 1] == x1) ? I0[i0 - 1] : 0;
                    ++i1;
                    x1 = i1 < n1 ? X1[i1] : INT32_MAX;
                }
            }
        }
}

// Row build from precomputed cross ids (wj_join_cross): no searches, the
// fp16 table rows of kRowU landings are loaded together.
template <int A, int W, bool INF>
__device__ __forceinline__ void build_rows_x(const EncMmaArgs &g, int tid, int nthr, const int32_t *scr,
                                             const int32_t *sid, const int (&pu)[A + 1], unsigned char *xr,
                                             uint16_t *vl, uint16_t *nl) {
    const int mu = g.mu;
    const int LT = pu[A];
    for (int e0 = tid; e0 < LT; e0 += kRowU * nthr) {
        uint4 t4[kRowU][A];
        int rowi[kRowU];
#pragma unroll
        for (int u = 0; u < kRowU; ++u) {
            const int e = e0 + u * nthr;
            const bool ok = e < LT;
            int a = 0;
#pragma unroll
            for (int t = 1; t < A; ++t) a += e >= pu[t];
            int base_a = 0;
#pragma unroll
            for (int t = 1; t < A; ++t)
                if (a == t) base_a = pu[t];
            const int l = ok ? e - base_a : 0;
            rowi[u] = ok ? a * mu + l : -1;
#pragma unroll
            for (int j = 0; j < A; ++j) {
                const int jj = j < a ? j : j - 1;
                const int id = !ok ? 0 : (j == a ? sid[a * mu + l] : scr[(a * (A - 1) + jj) * mu + l]);
                t4[u][j] = __ldg(g.trow + id);
            }
        }
#pragma unroll
        for (int u = 0; u < kRowU; ++u) {
            if (rowi[u] < 0) continue;
            uint32_t r[A][4];
#pragma unroll
            for (int j = 0; j < A; ++j) {
                r[j][0] = t4[u][j].x;
                r[j][1] = t4[u][j].y;
                r[j][2] = t4[u][j].z;
                r[j][3] = t4[u][j].w;
            }
            uint32_t w[8];
            splice_row<A, W>(r, w);
            const uint32_t row = (uint32_t)rowi[u];
            if (INF) {  // list position e -> row; 2 n_l = twice the own block's row sum (fp16)
                const int a = (int)(row / (uint32_t)g.mu);
                __half2 acc = __floats2half2_rn(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < A; ++j)
                    if (j == a)
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc = __hadd2(acc, *reinterpret_cast<const __half2 *>(&r[j][k]));
                const __half n = __hadd(__low2half(acc), __high2half(acc));  // W <= 8 halves; padding is 0
                const int e = e0 + u * nthr;
                vl[e] = (uint16_t)row;
                nl[e] = __half_as_ushort(__hadd(n, n));
            }
            const uint32_t sw = (row >> 2) & 1u;
            *reinterpret_cast<uint4 *>(xr + row * kRowB + (sw << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4 *>(xr + row * kRowB + ((sw ^ 1u) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
        }
    }
}

using EncMmaKernel = void (*)(EncMmaArgs);

// tcgen05 variant (encode_tc.cu): kernel for (arity, L+1, keep == 1, warps)
// or nullptr outside its envelope, and its dynamic shared memory
EncMmaKernel pick_tc(int A, int W, bool infer, int nw);
size_t tc_smem(int A, int mu, int lcap, int xr_bytes);

}  // namespace wj
