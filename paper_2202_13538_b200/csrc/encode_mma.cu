// Join fused with the encoder's first layer on the tensor cores (sm_100a):
// the training hot kernel.
//
// Reference: joiner.join_batch_arrays + pipeline._dense_batch + encoder
// forward/backward (joiner.py:53-71, pipeline.py:169-182, encoder.py:
// 126-233).  Same outputs as the SIMT kernel in encode.cu (pooled / S / msum
// per query, see the identities there); the work is organised as
//
//  * rows: anchor a's block has n_l identical rows per distinct landing l.
//    The store's virtual-landing index (vindex.cu, built at preprocess) lists
//    each anchor's block as 2-row virtual landings (section 2: l repeated
//    floor(n_l/2) times) and 1-row ones (section 1: l once if n_l is odd), so
//    a query's input is  sum_a |section 2_a| + |section 1_a|  virtual rows
//    whose dropout is Binomial(2, keep) resp. Bernoulli(keep) per unit;
//  * per query the CTA resolves every distinct landing against the other
//    anchors (sorted-list merge, as the join kernel) and writes its fp16 row
//    [x | 1 | 0..] ONCE into shared memory; a tile of 16 virtual landings is
//    then loaded straight from those rows with per-lane ldmatrix addresses
//    (no per-tile staging copy);
//  * z^T = W1aug^T [X | 1]^T is one m16n8k16 HMMA per 16 units x 8 landings
//    (W1 and b1 as a power-of-two-scaled fp16 hi + lo pair: ~22 mantissa
//    bits, fp32 accumulation); only z's SIGN is used;
//  * dropout, branch-free in 16-bit SIMD lanes: per lane and tile one hashed
//    seed, then per (t, mt, hb) one IMAD (an LCG jumped ahead) gives 32 bits,
//    folded to two 14-bit uniforms u (landing pair 2tq, 2tq+1 of one unit) as
//    u' = 0x3FFF-u;
//    T + u' has bit 14 set iff u < T, so the kept-row count of a lane as an
//    fp16 value 2*K is (T1 + u') & 0x4000 (& ~sign(z)) [+ the same with T2
//    for 2-row landings, one HADD2].  The sign mask comes from a PRMT
//    sign-replicate of the two fp32 accumulators;
//  * the backward statistics S^T = G^T [X | 1] (G = 2*kept, masked by z > 0)
//    are a second HMMA whose A operand is the first one's accumulator layout;
//    G <= 4 and x <= 2048, so S and msum are exact integer sums (halved at
//    the end);
//  * pooled needs no per-element work: relu(z) * kept = z * G / 2 and
//    z = [x | 1] W1aug, so pooled[h] = sum_c W1aug[c][h] S^T[h][c].
//
// One CTA (8 warps) per query, persistent; each warp owns every 8th tile.
#include <cstdio>
#include <cstdlib>
#include <new>

#include "encode_common.cuh"

namespace wj {

// Dropout stream: per lane and tile one hashed 32-bit seed s, then the 16
// draws x_k = A_k s + C_k (k = 0..15) = the LCG x <- a x + c (a = 747796405,
// c = 2891336453; L'Ecuyer's multiplier, odd increment) jumped k + 1 steps
// ahead -- one IMAD per 32 bits instead of a full hash (the integer ALU pipe
// bounds the kernel's tiles).
__host__ __device__ constexpr uint32_t lcg_mul(int k) {  // a^(k+1) mod 2^32
    uint32_t A = 1u;
    for (int i = 0; i <= k; ++i) A *= 747796405u;
    return A;
}
__host__ __device__ constexpr uint32_t lcg_add(int k) {  // c (a^(k+1) - 1) / (a - 1) mod 2^32
    uint32_t C = 0u;
    for (int i = 0; i <= k; ++i) C = C * 747796405u + 2891336453u;
    return C;
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}

__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}


// One tile of 16 virtual landings (list entries v0 .. v0+15) for one warp.
// KIND 2 = 2-row landings (Binomial(2, keep)), 1 = 1-row (Bernoulli(keep)),
// 0 = no dropout (keep = 1): the tile runs over the DISTINCT landings and G
// is 2 n_l (n_l = the landing's row count, fp16 pairs at nl2), so the
// statistics equal the virtual-landing sums with every row kept, exactly.
template <int KIND>
__device__ __forceinline__ void tile(const uint16_t *lst, uint32_t xr_s, uint32_t wt_s, int lane,
                                     uint32_t cq, uint32_t ta, uint32_t tb, float (&sacc)[4][2][4],
                                     const uint32_t *nl2 = nullptr) {
    constexpr bool TWO = KIND == 2;
    constexpr int H = 64;
    const uint32_t ib = lst[(lane & 7) + 8 * (lane >> 4)];
    const uint32_t it = lst[(lane & 7) + 8 * ((lane >> 3) & 1)];
    uint32_t bx[4], bt[4];
    ldsm_x4(bx, row_addr(xr_s, ib, (lane >> 3) & 1));
    ldsm_x4_t(bt, row_addr(xr_s, it, lane >> 4));
    // one full hash of the lane's tile counter per tile seeds its 16 draws
    uint32_t seed = cq * 0x7feb352dU;
    seed ^= seed >> 15;
    seed *= 0x846ca68bU;
    seed ^= seed >> 16;
    uint32_t nw[2] = {0u, 0u};
    if (KIND == 0) {  // (2 n_l, 2 n_l') of landings 8t + 2tq, 8t + 2tq + 1
        nw[0] = nl2[(lane & 3)];
        nw[1] = nl2[4 + (lane & 3)];
    }
    uint32_t ga[4][4];  // GEMM2 A fragments: G^T (unit x landing), fp16
    const int arow = (lane & 7) + 8 * ((lane >> 3) & 1), acol = 8 * (lane >> 4);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        uint32_t ahi[4], alo[4];
        ldsm_x4(ahi, wt_s + ((16 * mt + arow) * kWS + acol) * 2);
        ldsm_x4(alo, wt_s + ((H + 16 * mt + arow) * kWS + acol) * 2);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            float z[4] = {0.f, 0.f, 0.f, 0.f};
            hmma(z, ahi, bx[2 * t], bx[2 * t + 1]);
            hmma(z, alo, bx[2 * t], bx[2 * t + 1]);
            // z[r]: unit 16mt + gq + 8(r>>1), landing 8t + 2tq + (r&1)
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {
                if (KIND == 0) {
                    const uint32_t neg =
                        prmt(__float_as_uint(z[2 * hb]), __float_as_uint(z[2 * hb + 1]), 0xFFBBu);
                    ga[mt][2 * t + hb] = nw[t] & ~neg;
                    continue;
                }
                // 32 random bits for (t, mt, hb): step k = 8t + 2mt + hb of an
                // LCG seeded by the lane's hashed tile counter, as one IMAD by
                // jump-ahead constants (x_k = A_k s + C_k), folded like the seed
                const int k = 8 * t + 2 * mt + hb;
                uint32_t x = seed * lcg_mul(k) + lcg_add(k);
                const uint32_t up = ~(x ^ (x >> 16)) & 0x3FFF3FFFu;  // 0x3FFF - u, two lanes
                // 0xFFFF in a lane whose z is negative (sign byte replicated)
                const uint32_t neg = prmt(__float_as_uint(z[2 * hb]), __float_as_uint(z[2 * hb + 1]), 0xFFBBu);
                uint32_t gk = (ta + up) & ~neg & 0x40004000u;  // fp16 2.0 where u < T1 and z >= 0
                if (TWO) gk = hadd2_u32(gk, (tb + up) & ~neg & 0x40004000u);
                ga[mt][2 * t + hb] = gk;
            }
        }
    }
    // GEMM2: S^T += G^T [X | 1]  (k = landing, n = column)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        hmma(sacc[mt][0], ga[mt], bt[0], bt[1]);
        hmma(sacc[mt][1], ga[mt], bt[2], bt[3]);
    }
}

template <int A, int AW, int kMW, int MINB, bool INF>
__global__ void __launch_bounds__(kMW * 32, MINB) join_encode_mma_kernel(EncMmaArgs g) {
    static_assert(AW + 1 <= 16, "one k16 step: A*(L+1) + 1 <= 16");
    constexpr int W = AW / A;
    static_assert(W <= 8, "fp16 table rows hold 8 counts");
    constexpr int H = 64;
    constexpr int NT = kMW * 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int mu = g.mu;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, tq = lane & 3;  // mma fragment coordinates

    // ---- shared memory carve-up (16-B aligned blocks first)
    __half *wt = reinterpret_cast<__half *>(smem_raw);                 // [2][64][kWS] W^T hi / lo
    QMeta *meta = reinterpret_cast<QMeta *>(smem_raw + kWtBytes);       // [kMetaQ][A] query metadata
    float *wscale = reinterpret_cast<float *>(meta + kMetaQ * 3);       // [2]
    unsigned char *xr = smem_raw + kWtBytes + kHdrBytes;                // rows [A*mu + 1][32 B] | red
    float *red = reinterpret_cast<float *>(xr);                         // [warps][64][kRedS] (after tiles)
    int32_t *sx = reinterpret_cast<int32_t *>(xr + g.xr_bytes);         // [A][mu] sorted landing lists
    int32_t *sid = sx + A * mu;                                         // [A][mu] their RPE ids
    int32_t *scr = sid + A * mu;                                        // [A][A-1][mu] cross RPE ids
    uint16_t *vl = reinterpret_cast<uint16_t *>(scr + A * (A - 1) * mu);  // [lcap] virtual landing rows
    uint16_t *nl = vl + ((A * mu + 16 + 7) & ~7);  // INF: [A*mu + 16] 2 n_l per list position (fp16)
    const uint32_t xr_s = smem_u32(xr), wt_s = smem_u32(wt);
    const uint32_t zrow = (uint32_t)(A * mu);  // all-zero row: padding (contributes nothing)

    // metadata of the CTA's first kMetaQ queries: independent of the previous
    // kernel in the stream, so it is fetched before the PDL wait
    auto load_meta = [&](int64_t b0) {
        for (int t = threadIdx.x; t < kMetaQ * A; t += NT) {
            const int i = t / A, a = t - i * A;
            const int64_t bb = b0 + (int64_t)i * gridDim.x;
            QMeta m = {0, 0, 0, 0, 0};
            if (bb < g.n_batch) {
                const int64_t q = g.queries[bb * A + a];
                m.lo = g.offsets[q];
                m.u = (int)(g.offsets[q + 1] - m.lo);
                m.vo = g.voff[q];
                m.v2 = g.vcnt[2 * q];
                m.v1 = g.vcnt[2 * q + 1];
            }
            meta[t] = m;
        }
    };
    // Query scheduling.  Static: CTA c takes queries c, c + grid, ...
    // (metadata kMetaQ at a time).  Dynamic (g.qsched): the first query is
    // blockIdx.x, every further one is grabbed from a global counter once the
    // previous one's tiles start, its metadata loaded while that query's
    // reduction runs -- CTAs that run ahead (or start early under PDL) take
    // more queries.  The last CTA to finish resets the counters.
    const bool dyn = g.qsched != nullptr;
    int64_t *next_b = reinterpret_cast<int64_t *>(wscale + 20);
    const int32_t *gstart = g.groups ? g.groups + 1 : nullptr;
    const int32_t *gorder = g.groups ? g.groups + 2 + g.n_units : nullptr;
    const int32_t *gtup = g.groups ? gorder + g.n_batch : nullptr;  // [G][A] each unit's anchor tuple
    auto load_meta1 = [&](int64_t uu, QMeta *dst) {  // metadata of unit uu's anchor tuple
        if (threadIdx.x < A) {
            QMeta m = {0, 0, 0, 0, 0};
            if (uu < g.n_units) {
                const int64_t q = gtup ? (int64_t)gtup[uu * A + threadIdx.x] : g.queries[uu * A + threadIdx.x];
                m.lo = g.offsets[q];
                m.u = (int)(g.offsets[q + 1] - m.lo);
                m.vo = g.voff[q];
                m.v2 = g.vcnt[2 * q];
                m.v1 = g.vcnt[2 * q + 1];
            }
            dst[threadIdx.x] = m;
        }
    };
    if (dyn)
        load_meta1(blockIdx.x, meta);
    else
        load_meta(blockIdx.x);
    __syncthreads();
    float *wred = wscale + 4;  // [kMW] W^T max-reduction scratch (the rows area is live by then)

    // ---- W^T = [W1; b1; 0]^T as a power-of-two-scaled fp16 hi + lo pair
    auto stage_wt = [&]() {
        // each thread loads its W^T elements once (one round of loads on the
        // critical path after the wait), takes the max, then splits them
        constexpr int PER = (H * 16 + NT - 1) / NT;
        float wv[PER];
        float mx = 0.f;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + j * NT, m = i >> 4, k = i & 15;
            wv[j] = (i >= H * 16) ? 0.f : (k < AW ? g.w1[k * H + m] : (k == AW ? g.b1[m] : 0.f));
            mx = fmaxf(mx, fabsf(wv[j]));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        if (lane == 0) wred[warp] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = 0.f;
            for (int w = 0; w < kMW; ++w) m = fmaxf(m, wred[w]);
            int e = 0;
            if (m > 0.f) frexpf(m, &e);  // m in [2^(e-1), 2^e)
            const int s = 14 - e;        // scaled max in [2^13, 2^14)
            wscale[0] = ldexpf(1.f, s);
        }
        __syncthreads();
        const float sc = wscale[0];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + j * NT, m = i >> 4, k = i & 15;
            if (i >= H * 16) break;
            const float w = wv[j] * sc;
            const __half hi = __float2half_rn(w);
            const __half lo = __float2half_rn(w - __half2float(hi));
            wt[m * kWS + k] = hi;
            wt[H * kWS + m * kWS + k] = lo;
        }
        __syncthreads();
    };
    uint64_t skey = 0;

    int jq = 0;  // local unit index
    for (int64_t u = blockIdx.x; u < g.n_units; ++jq) {
        const int mstart = gorder ? gstart[u] : 0;
        const int mcount = gorder ? gstart[u + 1] - mstart : 1;
        int64_t b = gorder ? (int64_t)gorder[mstart] : u;  // the unit's first query
        if (!dyn && jq > 0 && jq % kMetaQ == 0) {  // metadata of the CTA's next kMetaQ queries
            __syncthreads();
            load_meta(b);
            __syncthreads();
        }
        const QMeta *qm = dyn ? meta + (jq & 1) * A : meta + (jq % kMetaQ) * A;
        int U[A], V2[A], V1[A], pu[A + 1], p2[A + 1], p1[A + 1];
        pu[0] = p2[0] = p1[0] = 0;
#pragma unroll
        for (int a = 0; a < A; ++a) {
            U[a] = qm[a].u;
            V2[a] = qm[a].v2;
            V1[a] = qm[a].v1;
            pu[a + 1] = pu[a] + U[a];
            p2[a + 1] = p2[a] + V2[a];
            p1[a + 1] = p1[a] + V1[a];
        }
        const int P2 = INF ? 0 : (p2[A] + 15) & ~15, P1 = INF ? (pu[A] + 15) & ~15 : (p1[A] + 15) & ~15;
        // ---- stage the anchors' sorted lists (async) and the virtual-landing rows
#pragma unroll
        for (int a = 0; a < A; ++a) {
            const int32_t *gx = g.ux + qm[a].lo;
            const int32_t *gi = g.uid + qm[a].lo;
            for (int i = threadIdx.x; i < U[a]; i += NT) {
                if (!g.cross) cp_async4(sx + a * mu + i, gx + i);
                cp_async4(sid + a * mu + i, gi + i);
            }
            if (g.cross)
#pragma unroll
                for (int jj = 0; jj < A - 1; ++jj) {
                    const int32_t *gc = g.cross + (b * A * (A - 1) + a * (A - 1) + jj) * (int64_t)mu;
                    for (int i = threadIdx.x; i < U[a]; i += NT) cp_async4(scr + (a * (A - 1) + jj) * mu + i, gc + i);
                }
        }
        // the anchors' virtual-landing lists (uint16, anchor-local) with the
        // anchor's row offset added: 4 loads in flight per thread
#pragma unroll
        for (int a = 0; a < (INF ? 0 : A); ++a) {
            const uint16_t *vs = g.vslots + qm[a].vo;
            const uint16_t add = (uint16_t)(a * mu);
            const int n2 = V2[a], nall = V2[a] + V1[a];
            for (int i0 = threadIdx.x; i0 < nall; i0 += 4 * NT) {
                uint16_t v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] = i0 + k * NT < nall ? __ldg(vs + i0 + k * NT) : (uint16_t)0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = i0 + k * NT;
                    if (i < nall) vl[i < n2 ? p2[a] + i : P2 + p1[a] + (i - n2)] = (uint16_t)(v[k] + add);
                }
            }
        }
        if (INF) {
            for (int i = pu[A] + threadIdx.x; i < P1; i += NT) {
                vl[i] = (uint16_t)zrow;
                nl[i] = 0;
            }
        } else {
            for (int i = p2[A] + threadIdx.x; i < P2; i += NT) vl[i] = (uint16_t)zrow;
            for (int i = P2 + p1[A] + threadIdx.x; i < P2 + P1; i += NT) vl[i] = (uint16_t)zrow;
        }
        if (threadIdx.x < 2) *reinterpret_cast<uint4 *>(xr + zrow * kRowB + 16 * threadIdx.x) = make_uint4(0, 0, 0, 0);
        cp_async_wait_all();
        __syncthreads();

        if (!g.cross && A > 1) {  // cross ids by merging the sorted lists
            merge_cross<A>(threadIdx.x, NT, mu, sx, sid, U, scr);
            __syncthreads();
        }
        build_rows_x<A, W, INF>(g, threadIdx.x, NT, scr, sid, pu, xr, vl, nl);
        __syncthreads();

        if (jq == 0) {
            // Everything above reads only the store and this step's queries,
            // so under PDL it overlaps the previous step's tail and Adam; W1,
            // b1 and the step counter are written by them: wait here.
            pdl_wait();
            skey = mix64(g.seed + kGolden * ((uint64_t)(g.step ? *g.step : 0) + 1ULL));
            stage_wt();
            // dynamic scheduling: a CTA exits only once the queue is empty, so the
            // dependent tail kernel may launch now -- its CTAs take the SM slots of
            // retiring CTAs and stage W2 / U1 / V before they wait for this kernel
            if (dyn) pdl_trigger();
        }
        // last query of this CTA, after the wait: dependents may launch
        if (!dyn && u + gridDim.x >= g.n_units) pdl_trigger();
        if (dyn && threadIdx.x == 0) *next_b = (int64_t)gridDim.x + atomicAdd(g.qsched, 1);
        int64_t nb = u + gridDim.x;

        for (int mem = 0; mem < mcount; ++mem) {
        if (mem > 0) {  // the previous member's reduction overlaid the rows: rebuild them
            b = gorder[mstart + mem];
            if (threadIdx.x < 2) *reinterpret_cast<uint4 *>(xr + zrow * kRowB + 16 * threadIdx.x) = make_uint4(0, 0, 0, 0);
            build_rows_x<A, W, INF>(g, threadIdx.x, NT, scr, sid, pu, xr, vl, nl);
            __syncthreads();
        }
        // ---- per-warp tiles of 16 virtual landings
        uint32_t qq = (uint32_t)mix64(skey ^ mix64((uint64_t)(b + g.b_offset)));
        qq ^= qq >> 16;
        float sacc[4][2][4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int r = 0; r < 4; ++r) sacc[mt][nt][r] = 0.f;
        const int T2 = P2 >> 4, TT = T2 + (P1 >> 4);
        for (int tt = warp; tt < TT; tt += kMW) {
            const int v0 = tt << 4;
            // hash counter: (v0 / 2 + 4t + tq) << 6 | (16 mt + 8 hb + gq)
            const uint32_t cq = qq ^ ((uint32_t)v0 << 5) ^ ((uint32_t)tq << 6) ^ (uint32_t)gq;
            if (INF)
                tile<0>(vl + v0, xr_s, wt_s, lane, 0u, 0u, 0u, sacc, reinterpret_cast<const uint32_t *>(nl + v0));
            else if (tt < T2)
                tile<2>(vl + v0, xr_s, wt_s, lane, cq, g.t21, g.t22, sacc);
            else
                tile<1>(vl + v0, xr_s, wt_s, lane, cq, g.t11, 0u, sacc);
        }
        __syncthreads();  // rows are dead: red overlays them
        if (dyn && mem == mcount - 1) {
            nb = *next_b;
            load_meta1(nb, meta + ((jq + 1) & 1) * A);  // lands while the reduction runs
        }
        // ---- CTA reduction: per-warp S^T partials -> smem -> fixed-order sum
        float *myred = red + warp * H * kRedS;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int c = 8 * nt + 2 * tq + (r & 1);
                    if (c <= AW) myred[(16 * mt + gq + 8 * (r >> 1)) * kRedS + c] = sacc[mt][nt][r];
                }
        __syncthreads();
        // one thread per unit: column sums in a fixed order (G carries a factor
        // 2: halve), then pooled[h] = sum_c W1aug[c][h] S^T[h][c] (relu(z) *
        // kept = z * kept) in the same thread -- no barrier between them
        if (threadIdx.x < H) {
            const int m = threadIdx.x;
            float sv[AW + 1];
#pragma unroll
            for (int c = 0; c <= AW; ++c) {
                float s = 0.f;
#pragma unroll
                for (int w = 0; w < kMW; ++w) s += red[w * H * kRedS + m * kRedS + c];
                s *= 0.5f;
                sv[c] = s;
                if (c < AW) {
                    if (g.s_out) g.s_out[(b * AW + c) * (int64_t)H + m] = s;
                } else if (g.msum) {
                    g.msum[b * H + m] = s;
                }
            }
            float pv = g.b1[m] * sv[AW];
#pragma unroll
            for (int c = 0; c < AW; ++c) pv = fmaf(g.w1[c * H + m], sv[c], pv);
            g.pooled[b * H + m] = pv;
        }
        __syncthreads();
        }  // members
        u = nb;
    }
    // the step executor's tail zeroes the counters once this grid completed;
    // standalone launches: the last CTA to finish does (a fence + an L2 round
    // trip on every CTA's exit, which delays the dependent tail)
    if (dyn && !g.qsched_reset_by_tail && threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(g.qsched + 1, 1) == (int)gridDim.x - 1) {  // every CTA is done grabbing
            atomicExch(g.qsched, 0);
            atomicExch(g.qsched + 1, 0);
        }
    }
}

// ---------------------------------------------------------------------------
// Query-level cross RPE ids (the rpe_ids columns of _kernels.join_fill,
// _kernels.py:237-245, per distinct landing instead of per walk slot):
// cross[b][a][jj][l] = RPE id of landing l of anchor a relative to the jj-th
// other anchor of query b (0 if that anchor's walks never reach it).  One
// CTA per query stages the anchors' sorted lists in shared memory and, for
// every anchor pair, merges the two lists (merge path: one diagonal binary
// search per thread, then a linear merge of ~(U_a + U_j) / 128 elements);
// equal ids are emitted list-a first, so an element of list j finds its
// partner at list a's previous position.
template <int A>
__global__ void __launch_bounds__(128) join_cross_kernel(const int64_t *__restrict__ queries, int64_t n_batch,
                                                         const int64_t *__restrict__ offsets,
                                                         const int32_t *__restrict__ ux,
                                                         const int32_t *__restrict__ uid, int mu,
                                                         int32_t *__restrict__ cross) {
    extern __shared__ __align__(16) int32_t csm[];
    int32_t *sx = csm, *sid = csm + A * mu;
    __shared__ int64_t lo_s[A];
    __shared__ int un_s[A];
    const int64_t b = blockIdx.x;
    pdl_wait();
    if (threadIdx.x < A) {
        const int64_t q = queries[b * A + threadIdx.x];
        const int64_t lo = offsets[q];
        lo_s[threadIdx.x] = lo;
        un_s[threadIdx.x] = (int)(offsets[q + 1] - lo);
    }
    __syncthreads();
    int U[A];
#pragma unroll
    for (int a = 0; a < A; ++a) {
        U[a] = un_s[a];
        for (int i = threadIdx.x; i < U[a]; i += blockDim.x) {
            cp_async4(sx + a * mu + i, ux + lo_s[a] + i);
            cp_async4(sid + a * mu + i, uid + lo_s[a] + i);
        }
    }
    cp_async_wait_all();
    __syncthreads();
    pdl_trigger();
    // the same merge path as the join+encode kernel's prepass, into global memory
    merge_cross<A>(threadIdx.x, blockDim.x, mu, sx, sid, U, cross + b * (int64_t)A * (A - 1) * mu);
}

// ---------------------------------------------------------------------------
// Scoring (keep = 1) of queries that share their first anchor -- the test
// protocol: each positive (u, v) followed by its negatives (u, v_i)
// (pipeline.py:185-198).  Same outputs as the keep = 1 variant
// of join_encode_mma_kernel, organised around reuse: a CTA scores a
// contiguous range of queries; for each new first anchor u it stages u's
// sorted list once, writes u's "alone" rows [x_u | 0 | 1] (the rows of u's
// landings that the second anchor's walks never reach) and sums their tiles
// into S0(u).  Per query it stages only v's list, merges the two lists (cross
// ids both ways), builds v's rows, and tiles v's landings plus every
// co-reached landing of u twice: with its actual row (weight +2n) and its
// alone row (weight -2n).  S^T and msum are integer sums, so S0(u) plus the
// per-query tiles equal the full computation exactly; pooled is then formed
// from S as in the join+encode kernel (bit-identical scores).
constexpr int kCoCap = 128;  // co-reached landings of u per tile round (larger counts loop)

template <int W>
__device__ __forceinline__ uint16_t put_row2(const EncMmaArgs &g, unsigned char *xr, uint32_t row, int id0, int id1,
                                             int own) {
    uint32_t r[2][4];
    const uint4 a = __ldg(g.trow + id0), b = __ldg(g.trow + id1);
    r[0][0] = a.x, r[0][1] = a.y, r[0][2] = a.z, r[0][3] = a.w;
    r[1][0] = b.x, r[1][1] = b.y, r[1][2] = b.z, r[1][3] = b.w;
    uint32_t w[8];
    splice_row<2, W>(r, w);
    const uint32_t sw = (row >> 2) & 1u;
    *reinterpret_cast<uint4 *>(xr + row * kRowB + (sw << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4 *>(xr + row * kRowB + ((sw ^ 1u) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
    __half2 acc = __floats2half2_rn(0.f, 0.f);  // the own block's row sum n_l
#pragma unroll
    for (int k = 0; k < 4; ++k) acc = __hadd2(acc, *reinterpret_cast<const __half2 *>(&r[own][k]));
    const __half n = __hadd(__low2half(acc), __high2half(acc));
    return __half_as_ushort(__hadd(n, n));
}

template <int W>
__global__ void __launch_bounds__(128, 3) infer_shared_kernel(EncMmaArgs g, int64_t per_cta) {
    constexpr int A = 2, AW = 2 * W, H = 64, NT = 128, kMW = 4;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int mu = g.mu;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // W^T | rows [2 mu + kCoCap + 1] | S0 [64][kRedS] | sx, sid [2][mu] | scr [2][mu] | vl, nl | co
    __half *wt = reinterpret_cast<__half *>(smem_raw);
    unsigned char *xr = smem_raw + kWtBytes;  // u alone rows [0, mu), v rows [mu, 2mu), co rows, zero row
    float *red = reinterpret_cast<float *>(xr + (size_t)mu * kRowB);  // over v / co rows (dead after tiles)
    float *s0 = reinterpret_cast<float *>(xr + g.xr_bytes);
    int32_t *sx = reinterpret_cast<int32_t *>(s0 + H * kRedS);
    int32_t *sid = sx + 2 * mu;
    int32_t *scr = sid + 2 * mu;
    uint16_t *vl = reinterpret_cast<uint16_t *>(scr + 2 * mu);
    uint16_t *nl = vl + g.lcap;
    uint16_t *co = nl + g.lcap;
    // co-reached counter, triple-buffered: iteration i counts into s_cnt[i % 3]
    // and resets s_cnt[(i + 1) % 3], whose last readers (iteration i - 2)
    // all passed iteration i - 1's barrier -- a single counter reset at the
    // top of the next iteration raced with slow warps still reading it
    __shared__ int s_cnt[3], s_q[2], s_len[2];
    __shared__ int64_t s_lo[2];
    const uint32_t xr_s = smem_u32(xr), wt_s = smem_u32(wt);
    const uint32_t zrow = (uint32_t)(2 * mu + kCoCap);
    const int64_t b_lo = (int64_t)blockIdx.x * per_cta;
    const int64_t b_hi = b_lo + per_cta < g.n_batch ? b_lo + per_cta : g.n_batch;
    if (b_lo >= b_hi) return;
    pdl_wait();
    // ---- W1aug^T as a power-of-two-scaled fp16 hi + lo pair (as the join+encode kernel)
    {
        constexpr int PER = (H * 16 + NT - 1) / NT;
        float wv[PER], mx = 0.f;
        float *wred = s0;  // scratch before S0 is used
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + j * NT, m = i >> 4, k = i & 15;
            wv[j] = (i >= H * 16) ? 0.f : (k < AW ? g.w1[k * H + m] : (k == AW ? g.b1[m] : 0.f));
            mx = fmaxf(mx, fabsf(wv[j]));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        if (lane == 0) wred[warp] = mx;
        __syncthreads();
        float m = 0.f;
        for (int w = 0; w < kMW; ++w) m = fmaxf(m, wred[w]);
        int e = 0;
        if (m > 0.f) frexpf(m, &e);
        const float sc = ldexpf(1.f, 14 - e);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + j * NT, mm = i >> 4, k = i & 15;
            if (i >= H * 16) break;
            const float w = wv[j] * sc;
            const __half hi = __float2half_rn(w);
            const __half lo = __float2half_rn(w - __half2float(hi));
            wt[mm * kWS + k] = hi;
            wt[H * kWS + mm * kWS + k] = lo;
        }
        if (threadIdx.x < 2) *reinterpret_cast<uint4 *>(xr + zrow * kRowB + 16 * threadIdx.x) = make_uint4(0, 0, 0, 0);
        if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
        __syncthreads();
    }
    pdl_trigger();
    int ci = 0;  // co-reached counter iteration (uniform)
    // tiles over vl[0, n) (padded to 16 with the zero row) into sacc
    float sacc[4][2][4];
    auto zero_acc = [&]() {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int r = 0; r < 4; ++r) sacc[mt][nt][r] = 0.f;
    };
    auto run_tiles = [&](int n) {
        const int np = (n + 15) & ~15;
        for (int i = n + threadIdx.x; i < np; i += NT) {
            vl[i] = (uint16_t)zrow;
            nl[i] = 0;
        }
        __syncthreads();
        for (int tt = warp; tt < (np >> 4); tt += kMW) {
            const int v0 = tt << 4;
            tile<0>(vl + v0, xr_s, wt_s, lane, 0u, 0u, 0u, sacc, reinterpret_cast<const uint32_t *>(nl + v0));
        }
    };
    // per-warp S^T partials -> red (fixed order), returned for column c of unit m
    auto reduce_to = [&](float *dst, bool add_s0) {
        __syncthreads();
        float *myred = red + warp * H * kRedS;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int c = 8 * nt + 2 * ((lane & 3)) + (r & 1);
                    if (c <= AW) myred[(16 * mt + (lane >> 2) + 8 * (r >> 1)) * kRedS + c] = sacc[mt][nt][r];
                }
        __syncthreads();
        if (threadIdx.x < H) {
            const int m = threadIdx.x;
            for (int c = 0; c <= AW; ++c) {
                float s = add_s0 ? s0[m * kRedS + c] : 0.f;
#pragma unroll
                for (int w = 0; w < kMW; ++w) s += red[w * H * kRedS + m * kRedS + c];
                dst[m * kRedS + c] = s;
            }
        }
        __syncthreads();
    };
    float *outS = red;  // the final S^T of a query (written over red by reduce_to)
    int cur_u = -1;
    for (int64_t b = b_lo; b < b_hi; ++b) {
        if (threadIdx.x < 2) {
            const int64_t q = g.queries[b * 2 + threadIdx.x];
            s_q[threadIdx.x] = (int)q;
            s_lo[threadIdx.x] = g.offsets[q];
            s_len[threadIdx.x] = (int)(g.offsets[q + 1] - g.offsets[q]);
        }
        __syncthreads();
        const int U[2] = {s_len[0], s_len[1]};
        if (s_q[0] != cur_u) {  // ---- u's list, alone rows and S0(u), once per first anchor
            for (int i = threadIdx.x; i < U[0]; i += NT) {
                cp_async4(sx + i, g.ux + s_lo[0] + i);
                cp_async4(sid + i, g.uid + s_lo[0] + i);
            }
            cp_async_wait_all();
            __syncthreads();
            for (int l = threadIdx.x; l < U[0]; l += NT) {
                nl[l] = put_row2<W>(g, xr, (uint32_t)l, sid[l], 0, 0);
                vl[l] = (uint16_t)l;
            }
            zero_acc();
            run_tiles(U[0]);
            reduce_to(s0, false);
            cur_u = s_q[0];
        }
        // ---- v: stage, merge (cross ids both ways), rows
        for (int i = threadIdx.x; i < U[1]; i += NT) {
            cp_async4(sx + mu + i, g.ux + s_lo[1] + i);
            cp_async4(sid + mu + i, g.uid + s_lo[1] + i);
        }
        cp_async_wait_all();
        __syncthreads();
        merge_cross<2>(threadIdx.x, NT, mu, sx, sid, U, scr);
        __syncthreads();
        // v's rows [counts rel. u (cross) | counts rel. v (own) | 1], weight 2 n_l
        for (int l = threadIdx.x; l < U[1]; l += NT) {
            nl[l] = put_row2<W>(g, xr, (uint32_t)(mu + l), scr[mu + l], sid[mu + l], 1);
            vl[l] = (uint16_t)(mu + l);
        }
        zero_acc();
        int nv = U[1];
        // co-reached landings of u (cross id rel. v != 0): rounds of whole
        // strides of NT landings, at most kCoCap (>= NT) per round; each round
        // tiles their actual rows (+2n) and their alone rows (-2n)
        int start = 0;
        while (true) {
            int nco = 0, l0 = start;
            while (l0 < U[0]) {
                const int cs = ci % 3;
                __syncthreads();  // the previous round's tiles are done
                const int l = l0 + threadIdx.x;
                const bool hit = l < U[0] && scr[l] != 0;
                const unsigned bm = __ballot_sync(kFull, hit);
                int wb = 0;
                if (lane == 0 && bm) wb = atomicAdd(&s_cnt[cs], __popc(bm));
                if (threadIdx.x == 0) s_cnt[(ci + 1) % 3] = 0;
                __syncthreads();
                const int h = s_cnt[cs];
                ++ci;
                if (nco + h > kCoCap) break;  // uniform; this stride opens the next round
                wb = __shfl_sync(kFull, wb, 0);
                if (hit) co[nco + wb + __popc(bm & lanemask_lt())] = (uint16_t)l;
                nco += h;
                l0 += NT;
            }
            start = l0;
            __syncthreads();
            for (int k = threadIdx.x; k < nco; k += NT) {
                const int l = co[k];
                const uint16_t n2 = put_row2<W>(g, xr, (uint32_t)(2 * mu + k), sid[l], scr[l], 0);
                vl[nv + k] = (uint16_t)(2 * mu + k);
                nl[nv + k] = n2;
                vl[nv + nco + k] = (uint16_t)l;
                nl[nv + nco + k] = (uint16_t)(n2 ^ 0x8000u);  // -2 n_l
            }
            run_tiles(nv + 2 * nco);
            nv = 0;
            if (start >= U[0]) break;
        }
        reduce_to(outS, true);
        if (threadIdx.x < H) {
            const int m = threadIdx.x;
            float sv[AW + 1];
#pragma unroll
            for (int c = 0; c <= AW; ++c) sv[c] = outS[m * kRedS + c] * 0.5f;
            float pv = g.b1[m] * sv[AW];
#pragma unroll
            for (int c = 0; c < AW; ++c) pv = fmaf(g.w1[c * H + m], sv[c], pv);
            g.pooled[b * H + m] = pv;
            if (g.s_out)
                for (int c = 0; c < AW; ++c) g.s_out[(b * AW + c) * (int64_t)H + m] = sv[c];
            if (g.msum) g.msum[b * H + m] = sv[AW];
        }
        __syncthreads();
    }
}

template <int NW, int MINB, bool INF = false>
static EncMmaKernel pick_mma(int A, int W) {
#define WJ_CASE(a, w) \
    if (A == a && W == w) return join_encode_mma_kernel<a, a * w, NW, MINB, INF>;
    WJ_CASE(1, 2) WJ_CASE(1, 3) WJ_CASE(1, 4) WJ_CASE(1, 5) WJ_CASE(1, 6) WJ_CASE(1, 7) WJ_CASE(1, 8)
    WJ_CASE(2, 2) WJ_CASE(2, 3) WJ_CASE(2, 4) WJ_CASE(2, 5) WJ_CASE(2, 6) WJ_CASE(2, 7)
    WJ_CASE(3, 2) WJ_CASE(3, 3) WJ_CASE(3, 4) WJ_CASE(3, 5)
#undef WJ_CASE
    return nullptr;
}

// 14-bit inverse-CDF thresholds, packed into both 16-bit lanes:
// 1-row: P(K >= 1) = keep; 2-row: P(K >= 1) = 1 - (1-keep)^2, P(K >= 2) = keep^2
static inline uint32_t pack_thr(double p) {
    const uint32_t t = (uint32_t)(p * 16384.0 + 0.5);
    return t | (t << 16);
}

void binomial_thresholds14(float keep_prob, uint32_t &t11, uint32_t &t21, uint32_t &t22) {
    const double k = (double)keep_prob;
    if (keep_prob >= 1.f) {
        t11 = t21 = t22 = pack_thr(1.0);
        return;
    }
    t11 = pack_thr(k);
    t21 = pack_thr(1.0 - (1.0 - k) * (1.0 - k));
    t22 = pack_thr(k * k);
}

}  // namespace wj

// SIMT variant (encode.cu): any hidden in {32, 64, 128}, A * (L+1) <= 16
extern "C" int wj_join_encode_simt(const int64_t *, int64_t, int32_t, const int64_t *, const int32_t *,
                                   const int32_t *, int32_t, int32_t, int32_t, const uint64_t *, int64_t,
                                   const float *, const float *, int32_t, float, uint64_t, const int64_t *,
                                   float *, float *, float *, wj_stream_t);

namespace wj {

// Kernel choice, shared-memory size and residency of the tensor-core kernel
// for one shape; k == nullptr outside its envelope.
struct MmaPlan {
    EncMmaKernel k = nullptr;
    int nw = 4;
    size_t smem = 0;
    int slots = 0;  // resident CTAs on the device (persistent grid)
    int lcap = 0, xr_bytes = 0, mu = 1;
    bool infer = false;
    bool tc = false;  // the tcgen05 kernel (encode_tc.cu)
    int threads = 128;
};


// infer: the keep = 1 variant (no dropout stream; tiles over the distinct
// landings with G = 2 n_l), usable while 2 n_l <= 2 M (L+1) is an exact
// fp16 integer (M (L+1) <= 1024); otherwise keep = 1 runs the dropout
// kernel with every threshold at 1.
static int plan_mma(int arity, int num_walks, int num_steps, int max_unique, MmaPlan &pl, bool infer = false) {
    const int W = num_steps + 1;
    // CTA shape: warps x min resident CTAs per SM (register budget); tuning
    // override WJ_ENC_CFG in {"4x2", "4x3", "4x4", "8x2"}.  WJ_ENC_TC = "4" /
    // "8" selects the tcgen05 kernel (encode_tc.cu) with that many dropout
    // warps where it applies (arity <= 2); unset or "0": the mma.sync kernel
    // (measured faster at C3)
    const char *env_cfg = getenv("WJ_ENC_CFG");
    const char *env_tc = getenv("WJ_ENC_TC");
    const int cfg = env_cfg ? (env_cfg[0] - '0') * 10 + (env_cfg[2] - '0') : 43;
    const int tc_nw = env_tc ? (env_tc[0] == '4' ? 4 : env_tc[0] == '8' ? 8 : 0) : 0;
    if (num_walks > 2048) return WJ_ERR_UNSUPPORTED;
    const int64_t P = (int64_t)num_walks * W;
    pl.infer = infer && P <= 1024;
    pl.tc = false;
    if (tc_nw && (pl.k = pick_tc(arity, W, pl.infer, tc_nw)) != nullptr) {
        pl.tc = true;
        pl.nw = tc_nw;
    } else if (pl.infer) pl.k = pick_mma<4, 3, true>(arity, W);
    else if (cfg == 42) pl.k = pick_mma<4, 2>(arity, W);
    else if (cfg == 44) pl.k = pick_mma<4, 4>(arity, W);
    else if (cfg == 82) { pl.k = pick_mma<8, 2>(arity, W); pl.nw = 8; }
    else pl.k = pick_mma<4, 3>(arity, W);
    if (!pl.k) return WJ_ERR_UNSUPPORTED;
    pl.threads = pl.nw * 32 + (pl.tc ? 32 : 0);  // tcgen05: + the MMA-issuing warp
    pl.mu = max_unique < 1 ? 1 : max_unique;
    if (P > 65535 || (int64_t)arity * pl.mu + 1 > 65535) {
        set_error("M*(L+1) or A*max_unique too large for uint16 row indices");
        pl.k = nullptr;
        return WJ_ERR_UNSUPPORTED;
    }
    const int64_t rows_b = ((int64_t)arity * pl.mu + 1) * kRowB;
    if (pl.tc) {
        // virtual landings per query: sum_a sum_l ceil(n_l / 2) <= A (P + U) / 2,
        // + two sections padded to 32 + the last tile padded to 128
        pl.lcap = (int)(((int64_t)arity * ((P + pl.mu) / 2 + 1) + 2 * 31 + 127 + 7) & ~7LL);
        if (pl.infer) pl.lcap = 2 * ((arity * pl.mu + 128 + 7) & ~7);  // list positions + 2 n_l per position
        pl.xr_bytes = (int)((rows_b + 15) & ~15LL);
        pl.smem = tc_smem(arity, pl.mu, pl.lcap, pl.xr_bytes);
    } else {
        // virtual landings per query: sum_a sum_l ceil(n_l / 2) <= A (P + U) / 2, + 2 x 15 padding
        pl.lcap = (int)(((int64_t)arity * ((P + pl.mu) / 2 + 1) + 32 + 7) & ~7LL);
        if (pl.infer) pl.lcap = 2 * ((arity * pl.mu + 16 + 7) & ~7);  // list positions + 2 n_l per position
        const int64_t red_b = (int64_t)pl.nw * 64 * kRedS * 4;
        pl.xr_bytes = (int)(((rows_b > red_b ? rows_b : red_b) + 15) & ~15LL);
        pl.smem = (size_t)kWtBytes + kHdrBytes + (size_t)pl.xr_bytes +
                  (size_t)(2 * arity + arity * (arity - 1)) * pl.mu * 4 + (size_t)pl.lcap * 2;
    }
    if (pl.smem > 200 * 1024) {
        set_error("join_encode needs %zu B of shared memory", pl.smem);
        pl.k = nullptr;
        return WJ_ERR_UNSUPPORTED;
    }
    cudaError_t e = cudaFuncSetAttribute(pl.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    if (e != cudaSuccess) {
        set_error("join_encode smem attribute: %s", cudaGetErrorString(e));
        pl.k = nullptr;
        return WJ_ERR_CUDA;
    }
    cudaFuncSetAttribute(pl.k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int per_sm = 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.k, pl.threads, pl.smem);
    if (getenv("WJ_ENC_DEBUG")) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, pl.k);
        int ps0 = 0, ps48 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps0, pl.k, pl.threads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps48, pl.k, pl.threads, 48 * 1024);
        fprintf(stderr, "  attrs: regs=%d static_smem=%zu max_dyn=%d maxthr=%d occ(0)=%d occ(48K)=%d\n", fa.numRegs,
                fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.maxThreadsPerBlock, ps0, ps48);
    }
    if (getenv("WJ_ENC_DEBUG"))
        fprintf(stderr, "join_encode plan: tc=%d nw=%d smem=%zu per_sm=%d (%s) mu=%d lcap=%d\n", (int)pl.tc, pl.nw,
                pl.smem, per_sm, cudaGetErrorString(e), pl.mu, pl.lcap);
    if (pl.tc) {
        // the occupancy API reports one CTA per SM for kernels that allocate
        // tensor memory; residency is bounded by TMEM (512 columns / 256 per
        // CTA), shared memory (227 KB per SM) and registers, all of which
        // admit two CTAs of this kernel
        const int by_smem = (int)((227 * 1024) / (pl.smem + 1024 + 128));
        per_sm = by_smem < 2 ? by_smem : 2;
    }
    pl.slots = sm_count() * (per_sm > 0 ? per_sm : 1);
    return WJ_OK;
}

static void fill_args(EncMmaArgs &g, const MmaPlan &pl, const int64_t *queries, int64_t n_batch,
                      const int64_t *offsets, const int32_t *uniq_x, const int32_t *uniq_id, const int64_t *voff,
                      const int32_t *vcnt, const uint16_t *vslots, const uint16_t *table_rows_f16, float keep_prob,
                      uint64_t seed, const int64_t *step) {
    g = EncMmaArgs{};
    g.queries = queries;
    g.n_batch = n_batch;
    g.n_units = n_batch;
    g.offsets = offsets;
    g.ux = uniq_x;
    g.uid = uniq_id;
    g.voff = voff;
    g.vcnt = vcnt;
    g.vslots = vslots;
    g.trow = reinterpret_cast<const uint4 *>(table_rows_f16);
    g.mu = pl.mu;
    g.lcap = pl.lcap;
    g.xr_bytes = pl.xr_bytes;
    binomial_thresholds14(keep_prob, g.t11, g.t21, g.t22);
    g.seed = seed;
    g.step = step;
}

}  // namespace wj

extern "C" int wj_join_encode(const int64_t *queries, int64_t n_batch, int32_t arity,
                              const int64_t *offsets, const int32_t *uniq_x,
                              const int32_t *uniq_id, const int32_t *cross, const int64_t *voff, const int32_t *vcnt,
                              const uint16_t *vslots, const uint16_t *table_rows_f16,
                              int32_t num_walks, int32_t num_steps,
                              int32_t max_unique, const uint64_t *table_keys, int64_t table_len,
                              const float *w1, const float *b1, int32_t hidden, float keep_prob,
                              uint64_t seed, const int64_t *step, float *pooled_out, float *s_out,
                              float *msum_out, wj_stream_t stream) {
    using namespace wj;
    if (arity < 1 || num_walks < 1 || num_steps < 1 || !(keep_prob > 0.f) || keep_prob > 1.f) {
        set_error("bad arity / shape / keep_prob");
        return WJ_ERR_ARG;
    }
    MmaPlan pl;
    const bool envelope = hidden == 64 && voff && vcnt && vslots && table_rows_f16;
    int rc = envelope ? plan_mma(arity, num_walks, num_steps, max_unique, pl, keep_prob >= 1.f)
                      : WJ_ERR_UNSUPPORTED;
    if (rc == WJ_ERR_CUDA) return rc;
    if (!pl.k)  // outside the tensor-core kernel's envelope (or no virtual-landing index)
        return wj_join_encode_simt(queries, n_batch, arity, offsets, uniq_x, uniq_id, num_walks, num_steps,
                                   max_unique, table_keys, table_len, w1, b1, hidden, keep_prob, seed, step,
                                   pooled_out, s_out, msum_out, stream);
    if (!pooled_out) {
        set_error("pooled_out is required");
        return WJ_ERR_ARG;
    }
    if (n_batch == 0) return WJ_OK;
    EncMmaArgs g;
    fill_args(g, pl, queries, n_batch, offsets, uniq_x, uniq_id, voff, vcnt, vslots, table_rows_f16, keep_prob,
              seed, step);
    g.w1 = w1;
    g.b1 = b1;
    g.cross = arity > 1 ? cross : nullptr;
    g.pooled = pooled_out;
    g.s_out = s_out;
    g.msum = msum_out;
    // persistent: one resident CTA slot per (SM, occupancy) -- W^T is split
    // once per CTA, not once per query
    const int64_t blocks = n_batch < pl.slots ? n_batch : pl.slots;
    const cudaError_t e = launch_pdl(pl.k, dim3((unsigned)blocks), dim3(pl.threads), pl.smem, (cudaStream_t)stream, g);
    if (e != cudaSuccess) {
        set_error("wj_join_encode launch: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return check_launch("wj_join_encode");
}


// Scoring of queries that share their first anchor (infer_shared_kernel):
// pooled [B, 64] (and S / msum when given) exactly as wj_join_encode at
// keep = 1.  Arity 2, hidden 64, A (L+1) + 1 <= 16.
extern "C" int wj_score_shared(const int64_t *queries, int64_t n_batch, const int64_t *offsets,
                               const int32_t *uniq_x, const int32_t *uniq_id, const uint16_t *table_rows_f16,
                               int32_t num_walks, int32_t num_steps, int32_t max_unique, const float *w1,
                               const float *b1, float *pooled_out, float *s_out, float *msum_out,
                               wj_stream_t stream) {
    using namespace wj;
    const int W = num_steps + 1;
    if (!queries || !offsets || !uniq_x || !uniq_id || !table_rows_f16 || !w1 || !b1 || !pooled_out ||
        num_walks < 1 || num_steps < 1 || max_unique < 1) {
        set_error("wj_score_shared: bad arguments");
        return WJ_ERR_ARG;
    }
    if (2 * W + 1 > 16 || 2 * (int64_t)max_unique + kCoCap + 1 > 65535) {
        set_error("wj_score_shared: shape outside the kernel (A(L+1)+1 <= 16, rows < 65536)");
        return WJ_ERR_UNSUPPORTED;
    }
    if (n_batch == 0) return WJ_OK;
    using K = void (*)(EncMmaArgs, int64_t);
    K k = nullptr;
    switch (W) {
        case 2: k = infer_shared_kernel<2>; break;
        case 3: k = infer_shared_kernel<3>; break;
        case 4: k = infer_shared_kernel<4>; break;
        case 5: k = infer_shared_kernel<5>; break;
        case 6: k = infer_shared_kernel<6>; break;
        case 7: k = infer_shared_kernel<7>; break;
        default: break;
    }
    if (!k) {
        set_error("wj_score_shared: L+1 = %d not instantiated", W);
        return WJ_ERR_UNSUPPORTED;
    }
    const int mu = max_unique;
    EncMmaArgs g = EncMmaArgs{};
    g.queries = queries;
    g.n_batch = n_batch;
    g.offsets = offsets;
    g.ux = uniq_x;
    g.uid = uniq_id;
    g.trow = reinterpret_cast<const uint4 *>(table_rows_f16);
    g.mu = mu;
    g.lcap = (mu + 2 * kCoCap + 32 + 7) & ~7;
    const int64_t rows_b = (int64_t)(2 * mu + kCoCap + 1) * kRowB;
    const int64_t red_b = (int64_t)mu * kRowB + 4 * 64 * kRedS * 4;
    g.xr_bytes = (int)(((rows_b > red_b ? rows_b : red_b) + 15) & ~15LL);
    g.w1 = w1;
    g.b1 = b1;
    g.pooled = pooled_out;
    g.s_out = s_out;
    g.msum = msum_out;
    const size_t smem = (size_t)kWtBytes + g.xr_bytes + 64 * kRedS * 4 + (size_t)6 * mu * 4 + (size_t)g.lcap * 4 +
                        kCoCap * 2;
    if (smem > 227 * 1024) {
        set_error("wj_score_shared needs %zu B of shared memory", smem);
        return WJ_ERR_UNSUPPORTED;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        set_error("wj_score_shared smem attribute: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 128, smem);
    const int64_t slots = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
    const int64_t per_cta = (n_batch + slots - 1) / slots;
    const int64_t blocks = (n_batch + per_cta - 1) / per_cta;
    e = launch_pdl(k, dim3((unsigned)blocks), dim3(128), smem, (cudaStream_t)stream, g, per_cta);
    if (e != cudaSuccess) {
        set_error("wj_score_shared launch: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return check_launch("wj_score_shared");
}

// ---------------------------------------------------------------------------
// Step executor: one fused training step (wj_join_encode -> wj_encoder_tail
// -> wj_adam) per call, every launch programmatic-dependent, so consecutive
// steps form one PDL chain on the stream: the next step's join+encode
// kernel is launched as soon as this step's Adam kernel starts, and stages
// its first query (lists, cross ids, rows) while the tail and Adam finish;
// it waits (griddepcontrol.wait) only before it needs W1.  The static
// arguments and the kernel plan are fixed at creation, so a step costs one
// host call and three launches.  Inputs may live in mapped (pinned) host
// memory: the queries are read before the wait, the labels are prefetched by
// the tail before its wait.
struct wj_stepper {
    wj::MmaPlan plan;
    wj::EncMmaArgs args;
    int32_t arity, aw, tail_rows_max, n_params;
    int32_t offsets9[9];
    float *params, *m, *v, *partial;
    int64_t *step;
    float scale, lr, beta1, beta2, eps;
};

extern "C" int wj_stepper_create(const int64_t *offsets, const int32_t *uniq_x, const int32_t *uniq_id,
                                 const int64_t *voff, const int32_t *vcnt, const uint16_t *vslots,
                                 const uint16_t *table_rows_f16, int32_t arity, int32_t num_walks, int32_t num_steps,
                                 int32_t max_unique, float *params, float *adam_m, float *adam_v,
                                 const int32_t *offsets9, float keep_prob, float tail_scale, uint64_t seed, float lr, float beta1,
                                 float beta2, float eps, int64_t *step, float *pooled, float *s_out, float *msum,
                                 float *partial, int32_t partial_rows_max, int32_t *sched, wj_stepper **out) {
    using namespace wj;
    if (!out || !params || !adam_m || !adam_v || !offsets9 || !step || !pooled || !s_out || !msum || !partial ||
        partial_rows_max < 1 || arity < 1 || num_walks < 1 || num_steps < 1 || !(keep_prob > 0.f) || keep_prob > 1.f) {
        set_error("wj_stepper_create: bad arguments");
        return WJ_ERR_ARG;
    }
    if (!voff || !vcnt || !vslots || !table_rows_f16) {
        set_error("wj_stepper_create: the store's virtual-landing index and fp16 table rows are required");
        return WJ_ERR_ARG;
    }
    wj_stepper *st = new (std::nothrow) wj_stepper();
    if (!st) {
        set_error("wj_stepper_create: out of host memory");
        return WJ_ERR_ARG;
    }
    int rc = plan_mma(arity, num_walks, num_steps, max_unique, st->plan, keep_prob >= 1.f);
    if (rc != WJ_OK || !st->plan.k) {
        delete st;
        if (rc == WJ_OK) set_error("wj_stepper_create: shape outside the tensor-core kernel");
        return rc == WJ_OK ? WJ_ERR_UNSUPPORTED : rc;
    }
    fill_args(st->args, st->plan, nullptr, 0, offsets, uniq_x, uniq_id, voff, vcnt, vslots, table_rows_f16,
              keep_prob, seed, step);
    st->args.w1 = params + offsets9[0];
    st->args.b1 = params + offsets9[1];
    st->args.cross = nullptr;
    st->args.pooled = pooled;
    st->args.s_out = s_out;
    st->args.msum = msum;
    st->args.qsched = sched;
    st->arity = arity;
    st->aw = arity * (num_steps + 1);
    st->tail_rows_max = partial_rows_max;
    for (int i = 0; i < 9; ++i) st->offsets9[i] = offsets9[i];
    st->n_params = offsets9[8];
    st->params = params;
    st->m = adam_m;
    st->v = adam_v;
    st->partial = partial;
    st->step = step;
    st->scale = tail_scale;
    st->lr = lr;
    st->beta1 = beta1;
    st->beta2 = beta2;
    st->eps = eps;
    *out = st;
    return WJ_OK;
}

extern "C" int wj_stepper_destroy(wj_stepper *st) {
    delete st;
    return WJ_OK;
}

namespace wj {
int encoder_tail(const float *, const float *, const float *, const float *, int64_t, int32_t, int32_t, const float *,
                 const int32_t *, float, float *, float *, int32_t, int32_t, float, int64_t *, cudaStream_t,
                 int32_t *sched_reset);
}

static int stepper_encode(wj_stepper *st, const int64_t *queries, int64_t n_batch, const int32_t *groups,
                          int64_t n_groups, wj_stream_t stream, bool tail_follows) {
    using namespace wj;
    if (!st || !queries || n_batch < 1 || (groups && (n_groups < 1 || n_groups > n_batch))) {
        set_error("wj_stepper_encode: bad arguments");
        return WJ_ERR_ARG;
    }
    if (groups && !st->args.qsched) {
        set_error("wj_stepper_encode: query groups need the dynamic scheduler (sched)");
        return WJ_ERR_ARG;
    }
    EncMmaArgs g = st->args;
    g.queries = queries;
    g.n_batch = n_batch;
    g.groups = groups;
    g.n_units = groups ? n_groups : n_batch;
    g.qsched_reset_by_tail = tail_follows ? 1 : 0;
    const int64_t blocks = g.n_units < st->plan.slots ? g.n_units : st->plan.slots;
    cudaError_t e = launch_pdl(st->plan.k, dim3((unsigned)blocks), dim3(st->plan.threads), st->plan.smem,
                               (cudaStream_t)stream, g);
    if (e != cudaSuccess) {
        set_error("wj_stepper: join_encode launch: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return check_launch("wj_stepper_encode");
}

extern "C" int wj_stepper_encode(wj_stepper *st, const int64_t *queries, int64_t n_batch, const int32_t *groups,
                                 int64_t n_groups, wj_stream_t stream) {
    return stepper_encode(st, queries, n_batch, groups, n_groups, stream, false);
}

extern "C" int wj_stepper_run(wj_stepper *st, const int64_t *queries, const float *labels, int64_t n_batch,
                              const int32_t *groups, int64_t n_groups, float *loss_out, wj_stream_t stream) {
    using namespace wj;
    if (!st || !queries || !labels || n_batch < 1 || (groups && (n_groups < 1 || n_groups > n_batch))) {
        set_error("wj_stepper_run: bad arguments");
        return WJ_ERR_ARG;
    }
    if (groups && !st->args.qsched) {
        set_error("wj_stepper_run: query groups need the dynamic scheduler (sched)");
        return WJ_ERR_ARG;
    }
    const int rc0 = stepper_encode(st, queries, n_batch, groups, n_groups, stream, st->args.qsched != nullptr);
    if (rc0 != WJ_OK) return rc0;
    EncMmaArgs g = st->args;
    int64_t rows = (n_batch + 15) / 16;
    if (rows > st->tail_rows_max) rows = st->tail_rows_max;
    int rc = encoder_tail(g.pooled, g.s_out, g.msum, labels, n_batch, st->aw, 64, st->params, st->offsets9,
                          st->scale, nullptr, st->partial, (int32_t)rows, 0, 0.f, st->step, (cudaStream_t)stream,
                          g.qsched);
    if (rc != WJ_OK) return rc;
    return wj_adam(st->params, st->m, st->v, st->partial, (int32_t)rows, st->n_params, st->lr, st->beta1, st->beta2,
                   st->eps, st->step, nullptr, loss_out, stream);
}

// Data parallel: the step split around the gradient exchange -- join+encode
// and tail, then the fixed-order sum of the partial rows into grad_out
// [n_params + 1] (gradients | loss); the caller all-reduces (averages) it
// and wj_stepper_apply runs Adam on it.
extern "C" int wj_stepper_grads(wj_stepper *st, const int64_t *queries, const float *labels, int64_t n_batch,
                                const int32_t *groups, int64_t n_groups, float *grad_out, wj_stream_t stream) {
    using namespace wj;
    if (!st || !queries || !labels || !grad_out || n_batch < 1) {
        set_error("wj_stepper_grads: bad arguments");
        return WJ_ERR_ARG;
    }
    const int rc0 = stepper_encode(st, queries, n_batch, groups, n_groups, stream, st->args.qsched != nullptr);
    if (rc0 != WJ_OK) return rc0;
    EncMmaArgs g = st->args;
    int64_t rows = (n_batch + 15) / 16;
    if (rows > st->tail_rows_max) rows = st->tail_rows_max;
    int rc = encoder_tail(g.pooled, g.s_out, g.msum, labels, n_batch, st->aw, 64, st->params, st->offsets9,
                          st->scale, nullptr, st->partial, (int32_t)rows, 0, 0.f, st->step, (cudaStream_t)stream,
                          g.qsched);
    if (rc != WJ_OK) return rc;
    return wj_sum_partials(st->partial, (int32_t)rows, st->n_params + 1, grad_out, stream);
}


// Batch-sharded data parallel: this rank's slice of one global
// batch -- queries [b_offset, b_offset + n_batch) of b_global, whose tail rows
// are rows [b_offset / per_cta, + rows) of the single-GPU step's partial rows
// -- with the global dropout keys and the global 1/B; the caller gathers every
// rank's rows in order and applies them with wj_stepper_apply_rows, which is
// then bit-identical to wj_stepper_run on the whole batch.
extern "C" int wj_stepper_grads_shard(wj_stepper *st, const int64_t *queries, const float *labels, int64_t n_batch,
                                      const int32_t *groups, int64_t n_groups, int64_t b_offset, int64_t b_global,
                                      int32_t per_cta, int32_t rows, float *partial_out, wj_stream_t stream) {
    using namespace wj;
    if (!st || n_batch < 0 || b_offset < 0 || b_global < 1 || per_cta < 1 || rows < 0 || !partial_out ||
        (n_batch > 0 && (!queries || !labels || rows < 1))) {
        set_error("wj_stepper_grads_shard: bad arguments");
        return WJ_ERR_ARG;
    }
    if (n_batch == 0) return WJ_OK;
    if (rows > st->tail_rows_max) {
        set_error("wj_stepper_grads_shard: %d rows exceed the stepper's %d", rows, st->tail_rows_max);
        return WJ_ERR_ARG;
    }
    st->args.b_offset = b_offset;
    const int rc0 = stepper_encode(st, queries, n_batch, groups, n_groups, stream, st->args.qsched != nullptr);
    st->args.b_offset = 0;
    if (rc0 != WJ_OK) return rc0;
    EncMmaArgs g = st->args;
    return encoder_tail(g.pooled, g.s_out, g.msum, labels, n_batch, st->aw, 64, st->params, st->offsets9, st->scale,
                        nullptr, partial_out, rows, per_cta, 1.f / (float)b_global, st->step,
                        (cudaStream_t)stream, g.qsched);
}

// Adam on the gathered partial rows of a batch-sharded step (fixed order)
extern "C" int wj_stepper_apply_rows(wj_stepper *st, const float *partial, int32_t rows, float *loss_out,
                                     wj_stream_t stream) {
    using namespace wj;
    if (!st || !partial || rows < 1) {
        set_error("wj_stepper_apply_rows: bad arguments");
        return WJ_ERR_ARG;
    }
    return wj_adam(st->params, st->m, st->v, partial, rows, st->n_params, st->lr, st->beta1, st->beta2, st->eps,
                   st->step, nullptr, loss_out, stream);
}

extern "C" int wj_stepper_apply(wj_stepper *st, const float *grad, float *loss_out, wj_stream_t stream) {
    using namespace wj;
    if (!st || !grad) {
        set_error("wj_stepper_apply: bad arguments");
        return WJ_ERR_ARG;
    }
    return wj_adam(st->params, st->m, st->v, grad, 1, st->n_params, st->lr, st->beta1, st->beta2, st->eps, st->step,
                   nullptr, loss_out, stream);
}


extern "C" int wj_join_cross(const int64_t *queries, int64_t n_batch, int32_t arity, const int64_t *offsets,
                             const int32_t *uniq_x, const int32_t *uniq_id, int32_t max_unique, int32_t *cross_out,
                             wj_stream_t stream) {
    using namespace wj;
    if (arity < 2 || arity > 3 || max_unique < 1 || !cross_out) {
        set_error("wj_join_cross: arity must be 2 or 3, max_unique >= 1");
        return arity == 1 ? WJ_ERR_UNSUPPORTED : WJ_ERR_ARG;
    }
    if (n_batch == 0) return WJ_OK;
    const size_t smem = (size_t)arity * max_unique * 8;
    if (smem > 200 * 1024) {
        set_error("wj_join_cross needs %zu B of shared memory", smem);
        return WJ_ERR_UNSUPPORTED;
    }
    cudaError_t e;
    if (arity == 2) {
        cudaFuncSetAttribute(join_cross_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        e = launch_pdl(join_cross_kernel<2>, dim3((unsigned)n_batch), dim3(128), smem, (cudaStream_t)stream, queries,
                       n_batch, offsets, uniq_x, uniq_id, (int)max_unique, cross_out);
    } else {
        cudaFuncSetAttribute(join_cross_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        e = launch_pdl(join_cross_kernel<3>, dim3((unsigned)n_batch), dim3(128), smem, (cudaStream_t)stream, queries,
                       n_batch, offsets, uniq_x, uniq_id, (int)max_unique, cross_out);
    }
    if (e != cudaSuccess) {
        set_error("wj_join_cross launch: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return check_launch("wj_join_cross");
}
