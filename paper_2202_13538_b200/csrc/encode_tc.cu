// Join fused with the encoder's first layer on the 5th-generation tensor
// cores (tcgen05 + TMEM): the training hot kernel for arity <= 2.
//
// Reference: joiner.join_batch_arrays + pipeline._dense_batch + encoder
// forward/backward (joiner.py:53-71, pipeline.py:169-182, encoder.py:
// 126-233).  Same outputs and identities as encode_mma.cu (pooled / S / msum
// per query); what changes is who does the per-tile work:
//
//  * a tile is 128 virtual landings.  Its rows [x | 1 | 0..] (fp16, 32 B)
//    are gathered from the unit's distinct-landing rows into a K-major
//    operand Xv [128 x 16] in shared memory (no-swizzle core matrices);
//  * z = Xv W1aug^T [128 x 64] is ONE tcgen05.mma pair (W1aug as a
//    power-of-two-scaled fp16 hi + lo pair, fp32 accumulation) issued by one
//    thread into TMEM; TMEM lane l = landing l of the tile;
//  * thread (landing l, hidden half) reads its 32 z values with one
//    tcgen05.ld and draws the dropout of its (landing, unit) pairs: one
//    32-bit hash per unit pair gives two 14-bit uniforms, the kept-row count
//    as fp16 2K is (T1 + u') & 0x4000 & ~sign(z) [+ the T2 term for 2-row
//    landings] -- exactly the encode_mma.cu arithmetic, with the counter
//    (landing v of the query, unit pair k);
//  * G [128 landings x 64 units] goes to shared memory as the MN-major A
//    operand of S^T += G^T Xv (M = 64 units, N = 16 columns, K = 128
//    landings: 8 tcgen05.mma k-steps), accumulated in TMEM across the
//    unit's tiles -- no per-warp partials, no cross-warp reduction;
//  * the next tile's Xv gather and z MMA overlap this tile's dropout work
//    (four Xv buffers, two z accumulators, two G buffers, mbarrier
//    completion tracking; one CTA barrier per tile).
//
// Descriptors (pinned on B200 by profiles/tc05_probe.cu): no-swizzle smem
// descriptor, LBO = byte stride between core matrices along K, SBO = along
// M/N, for both K-major and MN-major operands; an M = 64 accumulator row m
// sits in TMEM lane (m / 16) * 32 + m % 16.
#include "encode_common.cuh"

namespace wj {

namespace tc {

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // sm100 version, no swizzle
}

// kind::f16 instruction descriptor: fp16 A/B, fp32 D, M x N, A/B major
constexpr uint32_t idesc_f16(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        smem_u32(bar)));
}

__device__ __forceinline__ void bar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void bar_init_n(uint64_t *bar, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(n));
}

__device__ __forceinline__ void bar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

constexpr int kTile = 128;                // virtual landings per tile (= MMA M, = TMEM lanes)
constexpr int kXvBytes = kTile * 32;      // [128 x 16] fp16 K-major operand
constexpr int kGBytes = kTile * 64 * 2;   // [128 landings x 64 units] fp16 (MN-major A of S^T)
constexpr int kWBytes = 2 * 64 * 16 * 2;  // W1aug^T hi | lo, [64 x 16] fp16 K-major each
constexpr uint32_t kTmemCols = 256;       // z: two buffers, columns [0, 128); S^T: [128, 144)
constexpr uint32_t kSCol = 128;
constexpr uint32_t kIdZ = idesc_f16(128, 64, 0, 0);  // z = Xv W^T: K-major A and B
constexpr uint32_t kIdS = idesc_f16(64, 16, 1, 1);   // S^T = G^T Xv: MN-major A and B

// byte offset of element (r, k) of a [rows x 16] fp16 K-major operand: 8 x 16 B
// core matrices, K-adjacent ones 128 B apart (LBO), row-adjacent 256 B (SBO)
__host__ __device__ constexpr uint32_t kmaj16(uint32_t r, uint32_t k) {
    return (r >> 3) * 256 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

}  // namespace tc

// Kernel: A anchors, AW = A (L+1) columns, NW warps (4: a thread covers all
// 64 units of its landing; 8: two threads per landing, 32 units each).
template <int A, int AW, int NW, int MINB, bool INF>
__global__ void __launch_bounds__(NW * 32 + 32, MINB) join_encode_tc_kernel(EncMmaArgs g) {
    using namespace tc;
    static_assert(AW + 1 <= 16, "one k16 step: A*(L+1) + 1 <= 16");
    static_assert(NW == 4 || NW == 8, "4 or 8 warps");
    constexpr int W = AW / A;
    static_assert(W <= 8, "fp16 table rows hold 8 counts");
    constexpr int H = 64;
    constexpr int NT = NW * 32 + 32;  // NW dropout warps + one MMA-issuing warp
    constexpr int NH = NW * 32;       // dropout threads
    constexpr int HPT = H * 4 / NW;   // units per thread (64 or 32)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // z MMA of TMEM buffer 0 / 1 done; S MMA of G buffer 0 / 1 done; G buffer
    // 0 / 1 written by every warp (NW arrivals)
    __shared__ uint64_t bars[6];
    __shared__ uint32_t tmem_base;
    const int mu = g.mu;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int lt = tid & (kTile - 1);       // landing of the tile = TMEM lane
    const int ch = tid >> 7;                // unit half (NW = 8)
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;

    // ---- shared memory: W^T | header | Xv[2] | rows | lists / G | vl (| nl)
    unsigned char *wt = smem_raw;
    QMeta *meta = reinterpret_cast<QMeta *>(smem_raw + kWBytes);
    float *wscale = reinterpret_cast<float *>(meta + kMetaQ * 3);
    int64_t *next_b = reinterpret_cast<int64_t *>(wscale + 20);
    unsigned char *xv = smem_raw + kWBytes + kHdrBytes;
    unsigned char *xr = xv + 4 * kXvBytes;
    unsigned char *lg = xr + g.xr_bytes;  // lists (staging, merge, rows) overlaid by G (tiles)
    int32_t *sx = reinterpret_cast<int32_t *>(lg);
    int32_t *sid = sx + A * mu;
    int32_t *scr = sid + A * mu;
    const int lg_bytes = (((2 * A + A * (A - 1)) * mu * 4 > 2 * kGBytes ? (2 * A + A * (A - 1)) * mu * 4 : 2 * kGBytes) + 15) & ~15;
    uint16_t *vl = reinterpret_cast<uint16_t *>(lg + lg_bytes);
    uint16_t *nl = vl + ((g.lcap / (INF ? 2 : 1) + 7) & ~7);  // INF: 2 n_l per list position (fp16)
    const uint32_t wt_s = smem_u32(wt), xv_s = smem_u32(xv), g_s = smem_u32(lg);
    const uint32_t zrow = (uint32_t)(A * mu);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) bar_init(&bars[i]);
        bar_init_n(&bars[4], NW);  // one arrival per dropout warp
        bar_init_n(&bars[5], NW);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }

    auto load_meta = [&](int64_t b0) {
        for (int t = tid; t < kMetaQ * A; t += NT) {
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
    const bool dyn = g.qsched != nullptr;
    const int32_t *gstart = g.groups ? g.groups + 1 : nullptr;
    const int32_t *gorder = g.groups ? g.groups + 2 + g.n_units : nullptr;
    const int32_t *gtup = g.groups ? gorder + g.n_batch : nullptr;
    auto load_meta1 = [&](int64_t uu, QMeta *dst) {
        if (tid < A) {
            QMeta m = {0, 0, 0, 0, 0};
            if (uu < g.n_units) {
                const int64_t q = gtup ? (int64_t)gtup[uu * A + tid] : g.queries[uu * A + tid];
                m.lo = g.offsets[q];
                m.u = (int)(g.offsets[q + 1] - m.lo);
                m.vo = g.voff[q];
                m.v2 = g.vcnt[2 * q];
                m.v1 = g.vcnt[2 * q + 1];
            }
            dst[tid] = m;
        }
    };
    if (dyn)
        load_meta1(blockIdx.x, meta);
    else
        load_meta(blockIdx.x);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tmem_base;
    float *wred = wscale + 4;

    // W1aug^T = [W1; b1; 0]^T (64 x 16) as a power-of-two-scaled fp16 hi + lo
    // pair in the K-major B layout
    auto stage_wt = [&]() {
        constexpr int PER = (H * 16 + NT - 1) / NT;
        float wv[PER];
        float mx = 0.f;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = tid + j * NT, m = i >> 4, k = i & 15;
            wv[j] = (i >= H * 16) ? 0.f : (k < AW ? g.w1[k * H + m] : (k == AW ? g.b1[m] : 0.f));
            mx = fmaxf(mx, fabsf(wv[j]));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        if (lane == 0) wred[warp] = mx;
        __syncthreads();
        if (tid == 0) {
            float m = 0.f;
            for (int w = 0; w < NW; ++w) m = fmaxf(m, wred[w]);
            int e = 0;
            if (m > 0.f) frexpf(m, &e);
            wscale[0] = ldexpf(1.f, 14 - e);
        }
        __syncthreads();
        const float sc = wscale[0];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = tid + j * NT, m = i >> 4, k = i & 15;
            if (i >= H * 16) break;
            const float w = wv[j] * sc;
            const __half hi = __float2half_rn(w);
            const __half lo = __float2half_rn(w - __half2float(hi));
            *reinterpret_cast<__half *>(wt + kmaj16(m, k)) = hi;
            *reinterpret_cast<__half *>(wt + 2048 + kmaj16(m, k)) = lo;
        }
        fence_async_smem();
        __syncthreads();
    };

    uint64_t skey = 0;
    uint32_t ph = 0;  // mbarrier phase bits: z buffers 0, 1; S of G buffers 0, 1; G ready 0, 1 (tid 0)
    int jq = 0;
    for (int64_t u = blockIdx.x; u < g.n_units; ++jq) {
        const int mstart = gorder ? gstart[u] : 0;
        const int mcount = gorder ? gstart[u + 1] - mstart : 1;
        int64_t b = gorder ? (int64_t)gorder[mstart] : u;
        if (!dyn && jq > 0 && jq % kMetaQ == 0) {
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
        // sections padded to 32 (one warp's landings share a kind), total to a tile
        const int P2 = INF ? 0 : (p2[A] + 31) & ~31;
        const int P1 = INF ? pu[A] : p1[A];
        const int PT = (P2 + P1 + kTile - 1) & ~(kTile - 1);
        // ---- stage the anchors' sorted lists (async) and the virtual-landing list
#pragma unroll
        for (int a = 0; a < A; ++a) {
            const int32_t *gx = g.ux + qm[a].lo;
            const int32_t *gi = g.uid + qm[a].lo;
            for (int i = tid; i < U[a]; i += NT) {
                if (!g.cross) cp_async4(sx + a * mu + i, gx + i);
                cp_async4(sid + a * mu + i, gi + i);
            }
            if (g.cross)
#pragma unroll
                for (int jj = 0; jj < A - 1; ++jj) {
                    const int32_t *gc = g.cross + (b * A * (A - 1) + a * (A - 1) + jj) * (int64_t)mu;
                    for (int i = tid; i < U[a]; i += NT) cp_async4(scr + (a * (A - 1) + jj) * mu + i, gc + i);
                }
        }
#pragma unroll
        for (int a = 0; a < (INF ? 0 : A); ++a) {
            const uint16_t *vs = g.vslots + qm[a].vo;
            const uint16_t add = (uint16_t)(a * mu);
            const int n2 = V2[a], nall = V2[a] + V1[a];
            for (int i0 = tid; i0 < nall; i0 += 4 * NT) {
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
            for (int i = pu[A] + tid; i < PT; i += NT) {
                vl[i] = (uint16_t)zrow;
                nl[i] = 0;
            }
        } else {
            for (int i = p2[A] + tid; i < P2; i += NT) vl[i] = (uint16_t)zrow;
            for (int i = P2 + p1[A] + tid; i < PT; i += NT) vl[i] = (uint16_t)zrow;
        }
        if (tid < 2) *reinterpret_cast<uint4 *>(xr + zrow * kRowB + 16 * tid) = make_uint4(0, 0, 0, 0);
        cp_async_wait_all();
        __syncthreads();
        if (!g.cross && A > 1) {
            merge_cross<A>(tid, NT, mu, sx, sid, U, scr);
            __syncthreads();
        }
        build_rows_x<A, W, INF>(g, tid, NT, scr, sid, pu, xr, vl, nl);
        __syncthreads();  // the lists are dead from here: G overlays them

        if (jq == 0) {
            pdl_wait();
            skey = mix64(g.seed + kGolden * ((uint64_t)(g.step ? *g.step : 0) + 1ULL));
            stage_wt();
            if (dyn) pdl_trigger();
        }
        if (!dyn && u + gridDim.x >= g.n_units) pdl_trigger();
        if (dyn && tid == 0) *next_b = (int64_t)gridDim.x + atomicAdd(g.qsched, 1);
        int64_t nb = u + gridDim.x;
        const int TT = PT / kTile;

        // Xv of tile i into buffer i & 3: row of landing lt, K-half hh
        auto gather = [&](int i) {
            unsigned char *dst = xv + (i & 3) * kXvBytes;
#pragma unroll
            for (int hh = (NW == 8 ? ch : 0); hh < 2; hh += (NW == 8 ? 2 : 1)) {
                const uint32_t r = vl[i * kTile + lt];
                const uint4 v = *reinterpret_cast<const uint4 *>(xr + r * kRowB + (((hh ^ (r >> 2)) & 1u) << 4));
                *reinterpret_cast<uint4 *>(dst + kmaj16(lt, 8 * hh)) = v;
            }
        };
        // z of tile i into TMEM buffer i & 1 (the MMA warp)
        auto issue_z = [&](int i) {
            const uint64_t ad = sdesc(xv_s + (i & 3) * kXvBytes, 128, 256);
            const uint32_t d = tb + (uint32_t)((i & 1) * 64);
            mma(d, ad, sdesc(wt_s, 128, 256), kIdZ, 0u);
            mma(d, ad, sdesc(wt_s + 2048, 128, 256), kIdZ, 1u);
            commit(&bars[i & 1]);
        };

        for (int mem = 0; mem < mcount; ++mem) {
            if (mem > 0) b = gorder[mstart + mem];
            uint32_t qq = (uint32_t)mix64(skey ^ mix64((uint64_t)(b + g.b_offset)));
            qq ^= qq >> 16;
            // pipeline: tile i's z was issued two tiles earlier (two TMEM
            // buffers), its G goes to G buffer i & 1 once S(i - 2) has read it,
            // and the barrier after it releases S(i) and z(i + 2) at once
            if (tid < NH) {
                gather(0);
                if (TT > 1) gather(1);
            }
            fence_async_smem();
            __syncthreads();
            if (warp == NW) {
                // the MMA warp: z of the first two tiles, then per tile, once
                // every dropout warp has written its G rows: S(i) and z(i + 2)
                if (lane == 0) {
                    fence_after();
                    issue_z(0);
                    if (TT > 1) issue_z(1);
                    for (int i = 0; i < TT; ++i) {
                        const int zb = i & 1;
                        bar_wait(&bars[4 + zb], (ph >> (4 + zb)) & 1u);
                        ph ^= 1u << (4 + zb);
                        fence_after();
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks) {  // S^T += G^T Xv (8 k16 steps)
                            const uint64_t ad = sdesc(g_s + zb * kGBytes + ks * 2048, 1024, 128);
                            const uint64_t bd = sdesc(xv_s + (i & 3) * kXvBytes + ks * 512, 256, 128);
                            mma(tb + kSCol, ad, bd, kIdS, (i > 0 || ks > 0) ? 1u : 0u);
                        }
                        commit(&bars[2 + zb]);
                        if (i + 2 < TT) issue_z(i + 2);
                    }
                }
                __syncwarp();
            } else for (int i = 0; i < TT; ++i) {
                const int v = i * kTile + lt;
                const int zb = i & 1;
                // this tile's z (my landing, my units) into registers
                bar_wait(&bars[zb], (ph >> zb) & 1u);
                ph ^= 1u << zb;
                fence_after();
                uint32_t zr[HPT];
                const uint32_t zcol = tb + lane_off + (uint32_t)(zb * 64 + ch * HPT);
                ld32(zcol, *reinterpret_cast<uint32_t(*)[32]>(zr));
                if constexpr (HPT == 64) ld32(zcol + 32u, *reinterpret_cast<uint32_t(*)[32]>(zr + 32));
                ld_wait();
                // ---- dropout: kept count (fp16 2K) per (landing, unit), masked by z > 0
                const bool two = !INF && (i * kTile + 32 * (warp & 3)) < P2;  // warp-uniform
                const uint32_t ta = two ? g.t21 : g.t11, tbb = two ? g.t22 : 0u;
                uint32_t gw[HPT / 2];
                if (INF) {
                    const uint32_t n2 = nl[v];
                    const uint32_t nw = n2 | (n2 << 16);
#pragma unroll
                    for (int j = 0; j < HPT / 2; ++j) gw[j] = nw & ~prmt(zr[2 * j], zr[2 * j + 1], 0xFFBBu);
                } else {
                    // counter (v, unit pair k): x = (qq + (v << 5) + k) * C1, then
                    // one xorshift-multiply-xorshift round; two 14-bit lanes
                    const uint32_t base = (qq + ((uint32_t)v << 5) + (uint32_t)(ch * (HPT / 2))) * 0x7feb352dU;
                    if (two) {
#pragma unroll
                        for (int j = 0; j < HPT / 2; ++j) {
                            uint32_t x = base + (uint32_t)j * 0x7feb352dU;
                            x ^= x >> 15;
                            x *= 0x846ca68bU;
                            const uint32_t up = ~(x ^ (x >> 16)) & 0x3FFF3FFFu;
                            const uint32_t neg = prmt(zr[2 * j], zr[2 * j + 1], 0xFFBBu);
                            const uint32_t g1 = (ta + up) & ~neg & 0x40004000u;
                            gw[j] = hadd2_u32(g1, (tbb + up) & ~neg & 0x40004000u);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < HPT / 2; ++j) {
                            uint32_t x = base + (uint32_t)j * 0x7feb352dU;
                            x ^= x >> 15;
                            x *= 0x846ca68bU;
                            const uint32_t up = ~(x ^ (x >> 16)) & 0x3FFF3FFFu;
                            const uint32_t neg = prmt(zr[2 * j], zr[2 * j + 1], 0xFFBBu);
                            gw[j] = (ta + up) & ~neg & 0x40004000u;
                        }
                    }
                }
                // S(i - 2) read G buffer zb and Xv buffer (i + 2) & 3
                if (i >= 2) {
                    bar_wait(&bars[2 + zb], (ph >> (2 + zb)) & 1u);
                    ph ^= 1u << (2 + zb);
                }
                // G row of my landing: units ch*HPT .. +HPT, 8 per core-matrix row
                unsigned char *gbuf = lg + zb * kGBytes;
#pragma unroll
                for (int c = 0; c < HPT / 8; ++c) {
                    const uint32_t mb = (uint32_t)(ch * (HPT / 8) + c);
                    *reinterpret_cast<uint4 *>(gbuf + (lt >> 3) * 1024 + mb * 128 + (lt & 7) * 16) =
                        make_uint4(gw[4 * c], gw[4 * c + 1], gw[4 * c + 2], gw[4 * c + 3]);
                }
                if (i + 2 < TT) gather(i + 2);
                // this warp's G rows (and Xv rows of tile i + 2) are written and
                // its z reads are done: one arrival per warp for the MMA warp
                fence_async_smem();
                fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&bars[4 + zb]);
            }
            // the unit's last two S MMAs (the dropout threads track those phases)
            if (tid < NH)
                for (int i = (TT > 2 ? TT - 2 : 0); i < TT; ++i) {
                    bar_wait(&bars[2 + (i & 1)], (ph >> (2 + (i & 1))) & 1u);
                    ph ^= 1u << (2 + (i & 1));
                }
            __syncthreads();
            fence_after();
            if (dyn && mem == mcount - 1) {
                nb = *next_b;
                load_meta1(nb, meta + ((jq + 1) & 1) * A);
            }
            // ---- S^T row h = unit 16w + l (lanes < 16 of warps 0-3): outputs
            if (warp < 4) {
                uint32_t sr[16];
                ld16(tb + lane_off + kSCol, sr);
                ld_wait();
                if (lane < 16) {
                    const int m = 16 * warp + lane;
                    float sv[AW + 1];
#pragma unroll
                    for (int c = 0; c <= AW; ++c) {
                        const float s = __uint_as_float(sr[c]) * 0.5f;  // G carries a factor 2
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
            }
            fence_before();
            __syncthreads();
        }  // members
        u = nb;
    }
    if (dyn && tid == 0) {
        __threadfence();
        if (atomicAdd(g.qsched + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(g.qsched, 0);
            atomicExch(g.qsched + 1, 0);
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tb), "n"(kTmemCols));
    }
}

// Kernel choice for (arity, L+1); nullptr outside the envelope (arity <= 2,
// A (L+1) + 1 <= 16).  Shared memory: see tc_smem.
EncMmaKernel pick_tc(int A, int W, bool infer, int nw) {
#define WJ_TC(a, w)                                                                                         \
    if (A == a && W == w)                                                                                   \
        return nw == 8 ? (infer ? join_encode_tc_kernel<a, a * w, 8, 2, true> : join_encode_tc_kernel<a, a * w, 8, 2, false>) \
                       : (infer ? join_encode_tc_kernel<a, a * w, 4, 2, true> : join_encode_tc_kernel<a, a * w, 4, 2, false>);
    WJ_TC(1, 2) WJ_TC(1, 3) WJ_TC(1, 4) WJ_TC(1, 5) WJ_TC(1, 6) WJ_TC(1, 7) WJ_TC(1, 8)
    WJ_TC(2, 2) WJ_TC(2, 3) WJ_TC(2, 4) WJ_TC(2, 5) WJ_TC(2, 6) WJ_TC(2, 7)
#undef WJ_TC
    return nullptr;
}

size_t tc_smem(int A, int mu, int lcap, int xr_bytes) {
    const int lists = (2 * A + A * (A - 1)) * mu * 4;
    const int lg = ((lists > 2 * tc::kGBytes ? lists : 2 * tc::kGBytes) + 15) & ~15;
    return (size_t)tc::kWBytes + kHdrBytes + 4 * tc::kXvBytes + (size_t)xr_bytes + (size_t)lg +
           (size_t)lcap * 2 + 16;
}

}  // namespace wj
