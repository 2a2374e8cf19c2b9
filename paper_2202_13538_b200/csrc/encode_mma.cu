// Join fused with the encoder's first layer on the tensor cores (sm_100a):
// the training hot kernel.
//
// Reference: joiner.join_batch_arrays + pipeline._dense_batch + encoder
// forward/backward (joiner.py:53-71, pipeline.py:169-182, encoder.py:
// 126-233).  Same outputs as the SIMT kernel in encode.cu (pooled / S / msum
// per query, see the identities there); what changes is how the per-landing
// work is organised:
//
//  * the distinct landings of the query's anchor blocks are cut into
//    "virtual landings" of at most 2 rows each (a landing that occurs n times
//    in its block has ceil(n/2) of them), so every element of the layer-1
//    activation matrix is (virtual landing v, hidden unit h) with a row count
//    cnt_v in {1, 2};
//  * z = [x_v | 1] [W1; b1] is one m16n8k16 HMMA per 8 landings x 16 units
//    (x_v = the query-level RPE row: small integer counts, exact in fp16; W1
//    and b1 enter as a power-of-two-scaled fp16 hi + lo pair, so z carries
//    ~22 mantissa bits, with fp32 accumulation);
//  * dropout: the number of kept rows of (v, h) is Binomial(cnt_v, keep),
//    drawn by inverse CDF from one 16-bit uniform (two thresholds), the
//    uniforms coming from a counter hash of (step, query, v, h);
//  * the backward statistics S^T = G^T [X | 1] (G = kept rows masked by
//    z > 0) are a second HMMA whose A operand is the first one's accumulator
//    fragment re-packed to fp16 (G <= 2 and x <= 2048: exact), so S and msum
//    are exact integer-weighted sums;
//  * pooled needs no per-element work at all: relu(z) * kept = z * G and
//    z = [x | 1] W1aug, so pooled[h] = sum_c W1aug[c][h] * S^T[h][c] -- one
//    AW+1 term dot product per unit and query, from the exact S.  z itself
//    is only needed for its sign.
//
// One CTA (8 warps) per query; each warp owns every 8th tile of 16 virtual
// landings.  Nothing of size [rows, 64] touches memory.
#include <cuda_fp16.h>

#include "common.cuh"

namespace wj {

constexpr int kMW = 8;          // warps per CTA
constexpr int kXS = 24;         // halves per staged row (48 B: conflict-free ldmatrix)
constexpr int kRedS = 17;       // floats per unit in the reduction buffer (16 S^T cols + pad)
constexpr int kBigCap = 512;    // heavy landings expanded cooperatively per query

struct EncMmaArgs {
    const int64_t *queries;
    int64_t n_batch;
    const int64_t *offsets;
    const int32_t *ux;
    const int32_t *uid;
    int P, max_u, vcap;
    const uint64_t *tkeys;
    int64_t tlen;
    int stage_table;
    int cb;
    const float *w1;  // [AW, 64]
    const float *b1;  // [64]
    uint32_t thr[3][2];  // inverse-CDF thresholds of Binomial(cnt, keep), cnt = 0, 1, 2
    uint64_t seed;
    const int64_t *step;
    float *pooled;  // [B, 64]
    float *s_out;   // [B, AW, 64] or null
    float *msum;    // [B, 64] or null
};

// 32-bit integer hash (lowbias32): the dropout uniforms
__host__ __device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
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

// clamp(a - b, 0, 1) in one FADD.SAT
__device__ __forceinline__ float sub_sat(float a, float b) {
    float r;
    asm("sub.ftz.sat.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&h);
}

__device__ __forceinline__ int lb_i32(const int32_t *a, int n, int32_t x) {
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

// Output word k of the staged row [x | 1 | 0...] (16 fp16 columns), where
// column c < A*W is count f = c % W of anchor block j = c / W, taken from
// the fp16 table row r[j] (W <= 8 halves in 4 words), column A*W is 1.0.
// All selectors are compile-time constants after unrolling: one PRMT per word.
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

template <int A, int AW>
__global__ void __launch_bounds__(kMW * 32, 2) join_encode_mma_kernel(EncMmaArgs g) {
    static_assert(AW + 1 <= 16, "one k16 step: A*(L+1) + 1 <= 16");
    constexpr int W = AW / A;
    constexpr int H = 64;
    constexpr int NT = kMW * 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int mu = g.max_u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, tq = lane & 3;  // mma fragment coordinates

    // ---- shared memory carve-up (16-B aligned blocks first)
    __half *wt = reinterpret_cast<__half *>(smem_raw);              // [2][64][kXS] W^T hi / lo
    __half *xt = wt + 2 * H * kXS;                                  // [warps][16][kXS]
    float *red = reinterpret_cast<float *>(xt + kMW * 16 * kXS);    // [warps][64][kRedS]
    int64_t *qa = reinterpret_cast<int64_t *>(red + kMW * H * kRedS);  // [4]
    int *un = reinterpret_cast<int *>(qa + 4);                       // U_a [4], prefix [4], heavy count, pad
    unsigned long long *wsum = reinterpret_cast<unsigned long long *>(un + 10);  // [warps + 2]
    float *wscale = reinterpret_cast<float *>(wsum + kMW + 2);       // [2]
    uint64_t *tks = reinterpret_cast<uint64_t *>(wscale + 2);       // [tlen] (staged table keys)
    uint4 *th = reinterpret_cast<uint4 *>(                          // [tlen] fp16 count rows
        (reinterpret_cast<uintptr_t>(tks + ((g.stage_table & 1) ? g.tlen : 0)) + 15) & ~uintptr_t(15));
    int32_t *sx = reinterpret_cast<int32_t *>(th + ((g.stage_table & 2) ? g.tlen : 0));  // [A][mu]
    int32_t *sid = sx + A * mu;                                      // [A][mu]
    int32_t *cross = sid + A * mu;                                   // [A][A-1][mu]
    uint32_t *vmap = reinterpret_cast<uint32_t *>(cross + A * (A - 1) * mu);  // [vcap]

    const uint64_t cmask = (1ULL << g.cb) - 1;
    const uint64_t skey = mix64(g.seed + kGolden * ((uint64_t)(g.step ? *g.step : 0) + 1ULL));

    // ---- W^T = [W1; b1; 0]^T as a power-of-two-scaled fp16 hi + lo pair
    {
        float mx = 0.f;
        for (int i = threadIdx.x; i < (AW + 1) * H; i += NT) {
            const float w = i < AW * H ? g.w1[i] : g.b1[i - AW * H];
            mx = fmaxf(mx, fabsf(w));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        if (lane == 0) red[warp] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = 0.f;
            for (int w = 0; w < kMW; ++w) m = fmaxf(m, red[w]);
            int e = 0;
            if (m > 0.f) frexpf(m, &e);  // m in [2^(e-1), 2^e)
            const int s = 14 - e;        // scaled max in [2^13, 2^14)
            wscale[0] = ldexpf(1.f, s);
            wscale[1] = ldexpf(1.f, -s);
        }
        __syncthreads();
        const float sc = wscale[0];
        for (int i = threadIdx.x; i < H * 16; i += NT) {
            const int m = i >> 4, k = i & 15;
            const float w = (k < AW ? g.w1[k * H + m] : (k == AW ? g.b1[m] : 0.f)) * sc;
            const __half hi = __float2half_rn(w);
            const __half lo = __float2half_rn(w - __half2float(hi));
            wt[m * kXS + k] = hi;
            wt[H * kXS + m * kXS + k] = lo;
        }
        if (g.stage_table & 1) {
            for (int64_t i = threadIdx.x; i < g.tlen; i += NT) cp_async8(tks + i, g.tkeys + i);
            cp_async_wait_all();
            __syncthreads();
        }
        if (g.stage_table & 2)  // each RPE vector as W fp16 counts (exact: counts <= 2048), zero padded
            for (int64_t i = threadIdx.x; i < g.tlen; i += NT) {
                const uint64_t key = tks[i];
                float f[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) f[c] = c < W ? (float)(uint32_t)((key >> (g.cb * c)) & cmask) : 0.f;
                th[i] = make_uint4(pack_h2(f[0], f[1]), pack_h2(f[2], f[3]), pack_h2(f[4], f[5]), pack_h2(f[6], f[7]));
            }
        __syncthreads();
    }
        const uint64_t *tkp = (g.stage_table & 1) ? tks : g.tkeys;
    __half *myx = xt + warp * 16 * kXS;
    float *myred = red + warp * H * kRedS;

    for (int64_t b = blockIdx.x; b < g.n_batch; b += gridDim.x) {
        if (threadIdx.x < A) {
            const int64_t q = g.queries[b * A + threadIdx.x];
            qa[threadIdx.x] = q;
            un[threadIdx.x] = (int)(g.offsets[q + 1] - g.offsets[q]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0;
#pragma unroll
            for (int a = 0; a < A; ++a) {
                un[4 + a] = run;
                run += un[a];
            }
            un[4 + A] = run;
            un[8] = 0;  // heavy-landing list length
        }
#pragma unroll
        for (int a = 0; a < A; ++a) {
            const int64_t lo = g.offsets[qa[a]];
            for (int i = threadIdx.x; i < un[a]; i += NT) {
                cp_async4(sx + a * mu + i, g.ux + lo + i);
                cp_async4(sid + a * mu + i, g.uid + lo + i);
            }
        }
        cp_async_wait_all();
        __syncthreads();
        // RPE id of every landing of anchor a relative to every other anchor
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
                    const int pos = lb_i32(xj, nj, x);
                    dst[k] = (pos < nj && xj[pos] == x) ? sid[j * mu + pos] : 0;
                }
            }
        }
        // ---- virtual landings: thread t owns landings [t*per, (t+1)*per) of the
        // concatenated blocks; chunks = ceil(rows / 2); CTA exclusive scan
        const int LT = un[4 + A];
        const int per = (LT + NT - 1) / NT;
        const int l0 = min((int)threadIdx.x * per, LT), l1 = min(l0 + per, LT);
        int mine = 0;
        for (int lam = l0; lam < l1; ++lam) {
            int a = 0;
#pragma unroll
            for (int t = 1; t < A; ++t) a += lam >= un[4 + t];
            const uint64_t key = tkp[sid[a * mu + lam - un[4 + a]]];
            int rows = 0;
#pragma unroll
            for (int c = 0; c < W; ++c) rows += (int)((key >> (g.cb * c)) & cmask);
            mine += (rows + 1) >> 1;
        }
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[warp] = (unsigned long long)incl;
        __syncthreads();  // also: cross ready
        if (threadIdx.x == 0) {
            unsigned long long run = 0;
            for (int w = 0; w < kMW; ++w) {
                const unsigned long long t = wsum[w];
                wsum[w] = run;
                run += t;
            }
            wsum[kMW] = run;
        }
        __syncthreads();
        // vmap entries: a thread writes at most 4 chunks of a landing; the rest
        // of a heavy landing (the anchor itself: >= M rows) goes to a short
        // list that the warps expand 32 chunks at a time, so no thread walks
        // a 100-chunk loop while the CTA waits at the barrier
        int *big = reinterpret_cast<int *>(red);  // [kBigCap][3]; red is free until the tiles end
        {
            int v = (int)wsum[warp] + incl - mine;
            for (int lam = l0; lam < l1; ++lam) {
                int a = 0;
#pragma unroll
                for (int t = 1; t < A; ++t) a += lam >= un[4 + t];
                const uint64_t key = tkp[sid[a * mu + lam - un[4 + a]]];
                int rows = 0;
#pragma unroll
                for (int c = 0; c < W; ++c) rows += (int)((key >> (g.cb * c)) & cmask);
                for (int k = 0; k < 4 && rows > 0; ++k, rows -= 2) vmap[v++] = ((uint32_t)lam << 2) | (uint32_t)min(rows, 2);
                if (rows > 0) {
                    const int slot = atomicAdd(&un[8], 1);
                    if (slot < kBigCap) {
                        big[3 * slot] = lam;
                        big[3 * slot + 1] = v;
                        big[3 * slot + 2] = rows;
                        v += (rows + 1) >> 1;
                    } else {
                        for (; rows > 0; rows -= 2) vmap[v++] = ((uint32_t)lam << 2) | (uint32_t)min(rows, 2);
                    }
                }
            }
        }
        const int V = (int)wsum[kMW];
        __syncthreads();
        {
            const int nbig = min(un[8], kBigCap);
            for (int e = warp; e < nbig; e += kMW) {
                const uint32_t lam = (uint32_t)big[3 * e];
                const int v0 = big[3 * e + 1], rows = big[3 * e + 2];
                for (int c = lane; 2 * c < rows; c += 32) vmap[v0 + c] = (lam << 2) | (uint32_t)min(rows - 2 * c, 2);
            }
        }
        __syncthreads();

        // ---- per-warp tiles of 16 virtual landings
        const uint64_t qkey = mix64(skey ^ mix64((uint64_t)b));
        const uint32_t qlo = (uint32_t)qkey;
        float sacc[4][2][4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int r = 0; r < 4; ++r) sacc[mt][nt][r] = 0.f;
        }
        for (int v0 = warp * 16; v0 < V; v0 += kMW * 16) {
            // stage [x_v | 1 | 0] rows: lane i < 16 builds row i (and its
            // Binomial(cnt, keep) thresholds)
            // thresholds as floats 2^23 + t (exact): the kept-row count is then
            // sat(T1 - uf) + sat(T2 - uf) with uf = 2^23 + u -- FMA-pipe ops
            float my_t1 = 8388608.f, my_t2 = 8388608.f;
            if (lane < 16) {
                const int v = v0 + lane;
                uint32_t wrow[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                if (v < V) {
                    const uint32_t e = vmap[v];
                    const int cnt = (int)(e & 3u);
                    my_t1 = 8388608.f + (float)(cnt == 1 ? g.thr[1][0] : g.thr[2][0]);
                    my_t2 = 8388608.f + (float)(cnt == 1 ? 0u : g.thr[2][1]);
                    const int lam = (int)(e >> 2);
                    int a = 0;
#pragma unroll
                    for (int t = 1; t < A; ++t) a += lam >= un[4 + t];
                    const int l = lam - un[4 + a];
                    int ids[A];
#pragma unroll
                    for (int j = 0; j < A; ++j) {
                        if (j == a) {
                            ids[j] = sid[a * mu + l];
                        } else {
                            const int jj = j < a ? j : j - 1;
                            ids[j] = cross[(a * (A - 1) + jj) * mu + l];
                        }
                    }
                    if (W <= 8 && (g.stage_table & 2)) {
                        // fp16 rows from the staged table, spliced with byte permutes
                        uint32_t r[A][4];
#pragma unroll
                        for (int j = 0; j < A; ++j) {
                            const uint4 q4 = th[ids[j]];
                            r[j][0] = q4.x;
                            r[j][1] = q4.y;
                            r[j][2] = q4.z;
                            r[j][3] = q4.w;
                        }
                        splice_row<A, W>(r, wrow);
                    } else {
                        float x[16];
#pragma unroll
                        for (int c = 0; c < 16; ++c) x[c] = 0.f;
#pragma unroll
                        for (int j = 0; j < A; ++j) {
                            const uint64_t key = tkp[ids[j]];
#pragma unroll
                            for (int c = 0; c < W; ++c) x[j * W + c] = (float)(uint32_t)((key >> (g.cb * c)) & cmask);
                        }
                        x[AW] = 1.f;
#pragma unroll
                        for (int k = 0; k < 8; ++k) wrow[k] = pack_h2(x[2 * k], x[2 * k + 1]);
                    }
                }
                *reinterpret_cast<uint4 *>(myx + lane * kXS) = make_uint4(wrow[0], wrow[1], wrow[2], wrow[3]);
                *reinterpret_cast<uint4 *>(myx + lane * kXS + 8) = make_uint4(wrow[4], wrow[5], wrow[6], wrow[7]);
            }
            __syncwarp();
            // this thread's 4 landings: n = 8t + 2tq + s -> thresholds, hash bases
            float t1[2][2], t2[2][2];
            uint32_t hb0[2][2];
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int n = 8 * t + 2 * tq + s;
                    t1[t][s] = __shfl_sync(kFull, my_t1, n);
                    t2[t][s] = __shfl_sync(kFull, my_t2, n);
                    hb0[t][s] = qlo ^ (((uint32_t)(v0 + n) << 5) | ((uint32_t)gq << 2));
                }
            // GEMM1 operands: X^T tiles (k = column, n = landing)
            uint32_t bx[4];
            ldsm_x4(bx, smem_u32(myx + ((lane & 7) + 8 * (lane >> 4)) * kXS + 8 * ((lane >> 3) & 1)));
            uint32_t ga[4][4];  // GEMM2 A fragments: G^T (unit x landing), fp16
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                uint32_t ahi[4], alo[4];
                const int arow = 16 * mt + (lane & 7) + 8 * ((lane >> 3) & 1);
                const int acol = 8 * (lane >> 4);
                ldsm_x4(ahi, smem_u32(wt + arow * kXS + acol));
                ldsm_x4(alo, smem_u32(wt + H * kXS + arow * kXS + acol));
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    float z[4] = {0.f, 0.f, 0.f, 0.f};
                    hmma(z, ahi, bx[2 * t], bx[2 * t + 1]);
                    hmma(z, alo, bx[2 * t], bx[2 * t + 1]);
                    // z[r]: unit 16mt + gq + 8(r>>1), landing 8t + 2tq + (r&1);
                    // G = kept rows if z > 0 else 0 (only z's sign is needed)
                    float gv[4];
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        const uint32_t w = hash32(hb0[t][s] ^ (uint32_t)mt);
#pragma unroll
                        for (int hb = 0; hb < 2; ++hb) {
                            // uf = 2^23 + (16-bit uniform): one PRMT
                            const float uf = __int_as_float(__byte_perm(w, 0x4B000000u, hb ? 0x7632u : 0x7610u));
                            const float kept = sub_sat(t1[t][s], uf) + sub_sat(t2[t][s], uf);
                            // 1[z > 0] exactly: positive z is >= 2^-24 here (fp16 lattice)
                            const float pos = __saturatef(z[2 * hb + s] * 0x1p64f);
                            gv[2 * hb + s] = kept * pos;
                        }
                    }
                    ga[mt][2 * t] = pack_h2(gv[0], gv[1]);
                    ga[mt][2 * t + 1] = pack_h2(gv[2], gv[3]);
                }
            }
            // GEMM2: S^T += G^T [X | 1]  (k = landing, n = column)
            uint32_t bt[4];
            ldsm_x4_t(bt, smem_u32(myx + ((lane & 7) + 8 * ((lane >> 3) & 1)) * kXS + 8 * (lane >> 4)));
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const uint32_t a[4] = {ga[mt][0], ga[mt][1], ga[mt][2], ga[mt][3]};
                hmma(sacc[mt][0], a, bt[0], bt[1]);
                hmma(sacc[mt][1], a, bt[2], bt[3]);
            }
            __syncwarp();
        }
        // ---- CTA reduction: per-warp S^T partials -> smem -> fixed-order sum
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    myred[(16 * mt + gq + 8 * (r >> 1)) * kRedS + 8 * nt + 2 * tq + (r & 1)] = sacc[mt][nt][r];
        __syncthreads();
        // column sums in a fixed order; S^T[h][c] for c <= AW stays in red[0]
        for (int i = threadIdx.x; i < (AW + 1) * H; i += NT) {
            const int c = i / H, m = i - c * H;
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < kMW; ++w) s += red[w * H * kRedS + m * kRedS + c];
            if (c < AW) {
                if (g.s_out) g.s_out[(b * AW + c) * (int64_t)H + m] = s;
            } else if (g.msum) {
                g.msum[b * H + m] = s;
            }
            red[m * kRedS + c] = s;  // warp 0's slot: only this thread read it
        }
        __syncthreads();
        // pooled[h] = sum_c W1aug[c][h] S^T[h][c]  (relu(z) * kept = z * G)
        if (threadIdx.x < H) {
            const int m = threadIdx.x;
            float s = g.b1[m] * red[m * kRedS + AW];
#pragma unroll
            for (int c = 0; c < AW; ++c) s = fmaf(g.w1[c * H + m], red[m * kRedS + c], s);
            g.pooled[b * H + m] = s;
        }
        __syncthreads();
    }
}

using EncMmaKernel = void (*)(EncMmaArgs);

static EncMmaKernel pick_mma(int A, int W) {
#define WJ_CASE(a, w) \
    if (A == a && W == w) return join_encode_mma_kernel<a, a * w>;
    WJ_CASE(1, 2) WJ_CASE(1, 3) WJ_CASE(1, 4) WJ_CASE(1, 5) WJ_CASE(1, 6) WJ_CASE(1, 7) WJ_CASE(1, 8)
    WJ_CASE(2, 2) WJ_CASE(2, 3) WJ_CASE(2, 4) WJ_CASE(2, 5) WJ_CASE(2, 6) WJ_CASE(2, 7)
    WJ_CASE(3, 2) WJ_CASE(3, 3) WJ_CASE(3, 4) WJ_CASE(3, 5)
#undef WJ_CASE
    return nullptr;
}

// inverse-CDF thresholds (16-bit) of Binomial(cnt, keep) for cnt = 1, 2
void binomial_thresholds(float keep_prob, uint32_t thr[3][2]) {
    const double k = (double)keep_prob;
    thr[0][0] = thr[0][1] = 0;
    if (keep_prob >= 1.f) {
        thr[1][0] = thr[2][0] = thr[2][1] = 65536u;
        thr[1][1] = 0;
        return;
    }
    thr[1][0] = (uint32_t)(k * 65536.0 + 0.5);
    thr[1][1] = 0;
    thr[2][0] = (uint32_t)((1.0 - (1.0 - k) * (1.0 - k)) * 65536.0 + 0.5);
    thr[2][1] = (uint32_t)(k * k * 65536.0 + 0.5);
}

}  // namespace wj

// SIMT variant (encode.cu): any hidden in {32, 64, 128}, A * (L+1) <= 16
extern "C" int wj_join_encode_simt(const int64_t *, int64_t, int32_t, const int64_t *, const int32_t *,
                                   const int32_t *, int32_t, int32_t, int32_t, const uint64_t *, int64_t,
                                   const float *, const float *, int32_t, float, uint64_t, const int64_t *,
                                   float *, float *, float *, wj_stream_t);

extern "C" int wj_join_encode(const int64_t *queries, int64_t n_batch, int32_t arity,
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
    EncMmaKernel k = (hidden == 64 && num_walks <= 2048) ? pick_mma(arity, W) : nullptr;
    if (!k)  // outside the tensor-core kernel's envelope
        return wj_join_encode_simt(queries, n_batch, arity, offsets, uniq_x, uniq_id, num_walks, num_steps,
                                   max_unique, table_keys, table_len, w1, b1, hidden, keep_prob, seed, step,
                                   pooled_out, s_out, msum_out, stream);
    if ((int64_t)num_walks * W > 65535) {
        set_error("M*(L+1) too large");
        return WJ_ERR_UNSUPPORTED;
    }
    if (n_batch == 0) return WJ_OK;
    EncMmaArgs g;
    g.queries = queries;
    g.n_batch = n_batch;
    g.offsets = offsets;
    g.ux = uniq_x;
    g.uid = uniq_id;
    g.P = num_walks * W;
    g.max_u = max_unique < 1 ? 1 : max_unique;
    // virtual landings per query: sum_a sum_l ceil(n_l / 2) <= A (P + U) / 2
    g.vcap = arity * ((g.P + g.max_u) / 2 + 1) + 16;
    g.tkeys = table_keys;
    g.tlen = table_len;
    g.cb = bits_for((uint64_t)num_walks);
    g.w1 = w1;
    g.b1 = b1;
    binomial_thresholds(keep_prob, g.thr);
    g.seed = seed;
    g.step = step;
    g.pooled = pooled_out;
    g.s_out = s_out;
    g.msum = msum_out;
    const int H = 64;
    size_t base = (size_t)2 * H * kXS * 2 + (size_t)kMW * 16 * kXS * 2 + (size_t)kMW * H * kRedS * 4 + 32 + 48 +
                  8 * (kMW + 2) + 8 + (size_t)arity * g.max_u * 8 + (size_t)arity * (arity - 1) * g.max_u * 4 +
                  (size_t)g.vcap * 4 + 16;
    const size_t limit = 200 * 1024;
    // stage the packed keys (bit 0) and, when they fit too, the fp16 count rows (bit 1)
    const size_t budget = 110 * 1024;
    g.stage_table = (base + (size_t)table_len * 8 <= budget && table_len <= 8192) ? 1 : 0;
    if (g.stage_table && W <= 8 && base + (size_t)table_len * 24 + 16 <= budget) g.stage_table |= 2;
    const size_t smem = base + ((g.stage_table & 1) ? (size_t)table_len * 8 : 0) +
                        ((g.stage_table & 2) ? (size_t)table_len * 16 + 16 : 0);
    if (smem > limit) {
        set_error("join_encode needs %zu B of shared memory", smem);
        return WJ_ERR_UNSUPPORTED;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        set_error("join_encode smem attribute: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kMW * 32, smem);
    // persistent: one resident CTA slot per (SM, occupancy) -- the W^T split
    // and the staged table are set up once per CTA, not once per query
    int64_t blocks = n_batch;
    const int64_t cap = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
    if (blocks > cap) blocks = cap;
    k<<<(unsigned)blocks, kMW * 32, smem, (cudaStream_t)stream>>>(g);
    return check_launch("wj_join_encode");
}
