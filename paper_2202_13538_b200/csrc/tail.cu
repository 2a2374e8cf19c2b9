// Encoder tail + Adam for sm_100a: everything after the fused layer-1 kernel
// in two launches instead of ~100 small PyTorch kernels.
//
// Reference: encoder.py:159-249 (W2 layer on the pooled walk encodings,
// 2-layer classifier, BCE, hand-written backward, Adam).  Input per query b
// is what wj_join_encode produced: pooled_b (sum of relu(z)*d over rows),
// S_b and msum_b.  With pm = pooled * scale (scale = 1 / (keep * rows), the
// reference row mean of the inverted-dropout activations):
//   hq = pm W2 + b2,  z2 = hq U1 + c1,  a2 = relu(z2),  logit = a2 . u2 + c2
//   loss = mean_b [max(z,0) - z y + log1p(exp(-|z|))]
//   dlogit = (sigmoid(z) - y) / B,  dz2 = dlogit u2 * 1[z2 > 0]
//   dhq = dz2 U1^T,  g = (dhq W2^T) * scale
//   dW2 += pm^T dhq, dU1 += hq^T dz2, dW1 += S_b * g, db1 += msum_b * g
// tail_tc_kernel: one CTA per chunk of 16 queries runs every [16 x 64] x
// [64 x 64] product above (and the rank-16 gradient updates) on the tensor
// cores in 3-pass TF32 (fp32-level accuracy) and writes its partial
// gradients to its own row of a [grid, n_params + 1] buffer; the Adam kernel
// reduces those rows in a fixed order (deterministic) and applies the
// bias-corrected update (encoder.py:236-249).
#include "common.cuh"

namespace wj {

constexpr int kH = 64;

struct ParamOffsets {
    int w1, b1, w2, b2, u1, c1, u2, c2, total;
};

struct TailArgs {
    const float *pooled;  // [B, H]
    const float *s;       // [B, AW, H] (nullable: inference)
    const float *msum;    // [B, H]
    const float *labels;  // [B] (nullable: inference)
    int64_t B;
    const float *params;
    ParamOffsets off;
    float scale;          // 1 / (keep * rows)
    float inv_b;          // 1 / B (mean BCE)
    int64_t *step_inc;    // incremented once the tail is done (nullable)
    float *logits;        // [B] nullable
    float *partial;       // [grid, total + 1] (last column: loss partial)
    float *work;          // [B, kVecStride] per-query vectors (training)
    int per_cta;          // queries per gradient CTA
    int32_t *sched_reset; // [2] join+encode queue counters, zeroed after the wait (nullable)
};

// Sum the per-CTA partial gradients in a fixed order and apply Adam
// (encoder.py:236-249) with bias corrections from the device step counter.
// A CTA owns 32 consecutive parameters; its 8 warps each sum every 8th
// partial row (coalesced 128-B rows), then warp 0 adds the 8 sums in order:
// deterministic, and 8x the memory parallelism of one thread per column.
// (4 or 16 groups measured slower: 0.0893 / 0.0909 ms per C3 step vs 0.0876)
constexpr int kAdamCols = 32, kAdamGroups = 8;
constexpr int kAdamUnroll = 128 / kAdamGroups;  // loads per thread in flight (rows <= 128)

// bias-corrected Adam on one parameter (encoder.py:236-249); explicit
// roundings so every kernel that applies it produces the same bits
__device__ __forceinline__ void adam_update(float *p, float *m, float *v, float g, float lr, float beta1,
                                            float beta2, float eps, float bc1, float bc2) {
    const float mi = __fadd_rn(__fmul_rn(beta1, *m), __fmul_rn(1.f - beta1, g));
    const float vi = __fadd_rn(__fmul_rn(beta2, *v), __fmul_rn(__fmul_rn(1.f - beta2, g), g));
    *m = mi;
    *v = vi;
    *p = __fsub_rn(*p, __fdiv_rn(__fmul_rn(lr, __fdiv_rn(mi, bc1)), __fadd_rn(__fsqrt_rn(__fdiv_rn(vi, bc2)), eps)));
}

// sum of p[r * ld] over rows r = grp, grp + 8, ... < rows: four independent
// chains (four loads in flight), combined in a fixed order
__device__ __forceinline__ float strided_sum(const float *p, int64_t ld, int grp, int rows) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    if (rows <= kAdamUnroll * kAdamGroups) {
        // every load of the thread in flight at once (one L2 round trip, not
        // one per four rows), then the same additions in the same order
        float v[kAdamUnroll];
#pragma unroll
        for (int i = 0; i < kAdamUnroll; ++i) {
            const int r = grp + kAdamGroups * i;
            v[i] = r < rows ? p[(int64_t)r * ld] : 0.f;
        }
#pragma unroll
        for (int k = 0; k < kAdamUnroll / 4; ++k) {
            const int r = grp + 4 * kAdamGroups * k;
            if (r + 3 * kAdamGroups < rows) {  // a full group of four: one per chain
                s0 += v[4 * k];
                s1 += v[4 * k + 1];
                s2 += v[4 * k + 2];
                s3 += v[4 * k + 3];
            } else {  // the remainder rows, all into chain 0
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (r + kAdamGroups * j < rows) s0 += v[4 * k + j];
            }
        }
        return (s0 + s1) + (s2 + s3);
    }
    int r = grp;
    for (; r + 3 * kAdamGroups < rows; r += 4 * kAdamGroups) {
        s0 += p[(int64_t)r * ld];
        s1 += p[(int64_t)(r + kAdamGroups) * ld];
        s2 += p[(int64_t)(r + 2 * kAdamGroups) * ld];
        s3 += p[(int64_t)(r + 3 * kAdamGroups) * ld];
    }
    for (; r < rows; r += kAdamGroups) s0 += p[(int64_t)r * ld];
    return (s0 + s1) + (s2 + s3);
}

__global__ void __launch_bounds__(kAdamCols *kAdamGroups) adam_kernel(
    float *params, float *m, float *v, const float *partial, int rows, int n, float lr, float beta1,
    float beta2, float eps, const int64_t *step, float *grad_out, float *loss_out) {
    __shared__ float part[kAdamGroups][kAdamCols];
    const int c = threadIdx.x & (kAdamCols - 1), grp = threadIdx.x / kAdamCols;
    const int i = blockIdx.x * kAdamCols + c;
    // the next step's join+encode kernel may launch now: before its own wait
    // it only reads the store and its queries, which this kernel never writes
    pdl_trigger();
    // this parameter's p / m / v: written only by the previous step's Adam
    // (complete before the tail started), so fetched before the wait -- the
    // update then needs no load after the reduction
    float pi = 0.f, mi = 0.f, vi = 0.f;
    if (grp == 0 && i < n) {
        pi = params[i];
        mi = m[i];
        vi = v[i];
    }
    pdl_wait();  // the partial rows of the tail kernel
    // the step counter (advanced by the tail): its load and the bias
    // corrections overlap the reduction's loads
    const int64_t t = *step;
    float gsum = 0.f;
    if (i <= n) gsum = strided_sum(partial + i, (int64_t)(n + 1), grp, rows);
    const float bc1 = 1.f - powf(beta1, (float)t);
    const float bc2 = 1.f - powf(beta2, (float)t);
    part[grp][c] = gsum;
    __syncthreads();
    if (grp != 0 || i > n) return;
    gsum = 0.f;
#pragma unroll
    for (int k = 0; k < kAdamGroups; ++k) gsum += part[k][c];
    if (i == n) {
        if (loss_out) *loss_out = gsum;
        return;
    }
    if (grad_out) grad_out[i] = gsum;
    adam_update(&pi, &mi, &vi, gsum, lr, beta1, beta2, eps, bc1, bc2);
    params[i] = pi;
    m[i] = mi;
    v[i] = vi;
}

// Fixed-order column sums of the partial rows (the data-parallel path:
// reduce locally, all-reduce the [n+1] vector over ranks, then Adam on it).
__global__ void __launch_bounds__(kAdamCols *kAdamGroups) sum_rows_kernel(const float *partial, int rows,
                                                                        int cols, float *out) {
    __shared__ float part[kAdamGroups][kAdamCols];
    const int c = threadIdx.x & (kAdamCols - 1), grp = threadIdx.x / kAdamCols;
    const int i = blockIdx.x * kAdamCols + c;
    float gsum = 0.f;
    if (i < cols) gsum = strided_sum(partial + i, (int64_t)cols, grp, rows);
    part[grp][c] = gsum;
    __syncthreads();
    if (grp != 0 || i >= cols) return;
    gsum = 0.f;
#pragma unroll
    for (int k = 0; k < kAdamGroups; ++k) gsum += part[k][c];
    out[i] = gsum;
}

// ---------------------------------------------------------------------------
// Tensor-core tail: one CTA (4 warps) per chunk of 16 queries.  The five
// [16 x 64] x [64 x 64] products of the tail (hq, z2, dhq, g) and the rank-16
// gradient updates (dW2 += pm^T dhq, dU1 += hq^T dz2) run as m16n8k8 TF32
// MMAs in the 3-pass split (a_hi b_hi + a_hi b_lo + a_lo b_hi: fp32-level
// accuracy); W2 / U1 are staged once per CTA in shared memory.
constexpr int kTQ = 16;   // queries per chunk (the MMA M dimension)
constexpr int kTP = 68;   // shared-memory row pitch (floats)

__device__ __forceinline__ void tf32_split(float x, uint32_t &hi, uint32_t &lo) {
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
    const float r = x - __uint_as_float(hi);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// acc[nt] += A[16 x 8KS] B[8KS x 8NT] for one warp, via mo / no row / column
// offsets; la(m, k) = A[m][k], lb(k, n) = B[k][n].  Even and odd k-steps
// accumulate into separate fragments (two independent MMA chains), added at
// the end.
template <int NT, int KS, class LA, class LB>
__device__ __forceinline__ void warp_mma3(float (&acc)[NT][4], int lane, LA la, LB lb) {
    const int gq = lane >> 2, tq = lane & 3;
    float acc2[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc2[nt][r] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
        uint32_t ah[4], al[4];
        tf32_split(la(gq, 8 * ks + tq), ah[0], al[0]);
        tf32_split(la(gq + 8, 8 * ks + tq), ah[1], al[1]);
        tf32_split(la(gq, 8 * ks + tq + 4), ah[2], al[2]);
        tf32_split(la(gq + 8, 8 * ks + tq + 4), ah[3], al[3]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            uint32_t bh0, bl0, bh1, bl1;
            tf32_split(lb(8 * ks + tq, 8 * nt + gq), bh0, bl0);
            tf32_split(lb(8 * ks + tq + 4, 8 * nt + gq), bh1, bl1);
            float(&d)[4] = (ks & 1) ? acc2[nt] : acc[nt];
            mma_tf32(d, al, bh0, bh1);
            mma_tf32(d, ah, bl0, bl1);
            mma_tf32(d, ah, bh0, bh1);
        }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[nt][r] += acc2[nt][r];
}

// Two products sharing the A operand: acc1 += A B1, acc2 += A B2 (16 x 8
// each, K = 8 * KS), 3-pass TF32 like warp_mma3; the two chains interleave.
template <int KS, class LA, class LB1, class LB2>
__device__ __forceinline__ void warp_mma3_dual(float (&acc1)[4], float (&acc2)[4], int lane, LA la, LB1 lb1,
                                               LB2 lb2) {
    const int gq = lane >> 2, tq = lane & 3;
    float x1[4] = {0.f, 0.f, 0.f, 0.f}, x2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
        uint32_t ah[4], al[4];
        tf32_split(la(gq, 8 * ks + tq), ah[0], al[0]);
        tf32_split(la(gq + 8, 8 * ks + tq), ah[1], al[1]);
        tf32_split(la(gq, 8 * ks + tq + 4), ah[2], al[2]);
        tf32_split(la(gq + 8, 8 * ks + tq + 4), ah[3], al[3]);
        uint32_t bh0, bl0, bh1, bl1, ch0, cl0, ch1, cl1;
        tf32_split(lb1(8 * ks + tq, gq), bh0, bl0);
        tf32_split(lb1(8 * ks + tq + 4, gq), bh1, bl1);
        tf32_split(lb2(8 * ks + tq, gq), ch0, cl0);
        tf32_split(lb2(8 * ks + tq + 4, gq), ch1, cl1);
        float(&d1)[4] = (ks & 1) ? x1 : acc1;
        float(&d2)[4] = (ks & 1) ? x2 : acc2;
        mma_tf32(d1, al, bh0, bh1);
        mma_tf32(d2, al, ch0, ch1);
        mma_tf32(d1, ah, bl0, bl1);
        mma_tf32(d2, ah, cl0, cl1);
        mma_tf32(d1, ah, bh0, bh1);
        mma_tf32(d2, ah, ch0, ch1);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        acc1[r] += x1[r];
        acc2[r] += x2[r];
    }
}

constexpr int kTW = 8;  // warps per tail CTA
constexpr int kTailLabels = 64;  // labels per CTA prefetched into shared memory

template <int AW>
__global__ void __launch_bounds__(kTW * 32) tail_tc_kernel(TailArgs g) {
    constexpr int NT = kTW * 32;
    extern __shared__ __align__(16) float tsm[];
    float *W2s = tsm, *U1s = W2s + 64 * kTP;               // [64][kTP] row-major W2, U1
    float *PM = U1s + 64 * kTP, *HQ = PM + kTQ * kTP, *Z2 = HQ + kTQ * kTP;
    float *DZ2 = Z2 + kTQ * kTP, *DHQ = DZ2 + kTQ * kTP, *G = DHQ + kTQ * kTP;  // [kTQ][kTP] each
    float *vsm = G + kTQ * kTP;                             // [kTW][64] du2 partials | dc2 | loss
    float *SS = vsm + kTW * 64 + 2 * kTW;                   // [kTQ][(AW+1)*64] S | msum of the chunk
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const float *P = g.params;
    for (int i = tid; i < 64 * 16; i += NT) {
        const int r = i >> 4, c = (i & 15) * 4;
        cp_async16(W2s + r * kTP + c, P + g.off.w2 + r * 64 + c);
        cp_async16(U1s + r * kTP + c, P + g.off.u1 + r * 64 + c);
    }
    const float u2a = P[g.off.u2 + lane], u2b = P[g.off.u2 + lane + 32], c2 = P[g.off.c2];
    const bool train = g.labels != nullptr;
    const int64_t q_lo = (int64_t)blockIdx.x * g.per_cta;
    const int64_t q_hi = min(g.B, q_lo + g.per_cta);
    // this CTA's labels (inputs, possibly in mapped host memory): fetched
    // before the wait so their latency overlaps the join+encode kernel
    float *LB = SS + kTQ * (AW + 1) * 64;  // [kTailLabels]
    float *VS = LB + kTailLabels;           // [64][kTP] V = W2 U1
    float *C1P = VS + 64 * kTP;             // [64] c1' = b2 U1 + c1
    if (train)
        for (int64_t i = tid; i < min((int64_t)kTailLabels, q_hi - q_lo); i += NT) LB[i] = g.labels[q_lo + i];
    // V = W2 U1 and c1' = b2 U1 + c1 (parameters only, so before the wait):
    // z2 = scale pooled V + c1' and g = scale dz2 V^T take one product each
    // on the critical path instead of two (hq and dhq, needed only for
    // dU1 / dW2, ride along in the same passes)
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    {
        const int vm = warp & 3, vn = (warp >> 2) * 32;
        float va[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int r = 0; r < 4; ++r) va[i][r] = 0.f;
        warp_mma3<4, 8>(va, lane, [&](int m, int k) { return W2s[(16 * vm + m) * kTP + k]; },
                        [&](int k, int n) { return U1s[k * kTP + vn + n]; });
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r0 = 16 * vm + gq, c = vn + 8 * j + 2 * tq;
            VS[r0 * kTP + c] = va[j][0];
            VS[r0 * kTP + c + 1] = va[j][1];
            VS[(r0 + 8) * kTP + c] = va[j][2];
            VS[(r0 + 8) * kTP + c + 1] = va[j][3];
        }
        if (tid < 64) {
            float c1p = P[g.off.c1 + tid];
            for (int k = 0; k < 64; ++k) c1p = fmaf(P[g.off.b2 + k], U1s[k * kTP + tid], c1p);
            C1P[tid] = c1p;
        }
    }
    pdl_wait();     // pooled / S / msum of the join+encode kernel
    pdl_trigger();  // the Adam kernel may get scheduled
    // the join+encode grid has completed: zero its queue counters for the
    // next step (its CTAs skip the end-of-CTA reset under the step executor)
    if (g.sched_reset && blockIdx.x == 0 && tid < 2) g.sched_reset[tid] = 0;
    constexpr int NW1 = ((AW + 1) * 64 + NT - 1) / NT;
    // dW2 / dU1 tiles of this warp: m-tile (warp & 3), n-tiles 4 (warp >> 2) .. +3
    const int fm = warp & 3, fn = (warp >> 2) * 4;
    float aw2[4][4], au1[4][4], aw1[NW1], vacc = 0.f, du2a = 0.f, du2b = 0.f, dc2 = 0.f, lsum = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int r = 0; r < 4; ++r) aw2[i][r] = au1[i][r] = 0.f;
#pragma unroll
    for (int i = 0; i < NW1; ++i) aw1[i] = 0.f;
    for (int64_t q0 = q_lo; q0 < q_hi; q0 += kTQ) {
        const int nq = (int)min((int64_t)kTQ, q_hi - q0);
        // the chunk's pooled rows (unscaled: the scale is applied to hq and dW2)
        for (int i = tid; i < kTQ * 16; i += NT) {
            const int q = i >> 4, c = (i & 15) * 4;
            if (q < nq)
                cp_async16(PM + q * kTP + c, g.pooled + (q0 + q) * 64 + c);
            else
                *reinterpret_cast<float4 *>(PM + q * kTP + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        cp_async_commit();  // group: pooled rows (+ W2 / U1 on the first chunk)
        if (train) {  // S and msum, in flight while the products run
            for (int i = tid; i < nq * AW * 16; i += NT) {
                const int q = i / (AW * 16), c = i - q * AW * 16;
                cp_async16(SS + q * (AW + 1) * 64 + c * 4, g.s + (q0 + q) * AW * 64 + c * 4);
            }
            for (int i = tid; i < nq * 16; i += NT)
                cp_async16(SS + (i >> 4) * (AW + 1) * 64 + AW * 64 + (i & 15) * 4, g.msum + (q0 + (i >> 4)) * 64 + (i & 15) * 4);
            cp_async_commit();
        }
        // wait for W2 / U1 (first chunk) and the pooled rows; S may still be in flight
        if (train) cp_async_wait_group1(); else cp_async_wait_all();
        __syncthreads();
        // hq = scale pooled W2 + b2 and z2 = scale pooled V + c1' in one pass
        // (warp w: output columns 8w .. 8w+7)
        {
            float ah[4] = {0.f, 0.f, 0.f, 0.f}, az[4] = {0.f, 0.f, 0.f, 0.f};
            warp_mma3_dual<8>(ah, az, lane, [&](int m, int k) { return PM[m * kTP + k]; },
                              [&](int k, int n) { return W2s[k * kTP + 8 * warp + n]; },
                              [&](int k, int n) { return VS[k * kTP + 8 * warp + n]; });
            const int c = 8 * warp + 2 * tq;
            const float *b2 = P + g.off.b2;
            HQ[gq * kTP + c] = fmaf(ah[0], g.scale, b2[c]);
            HQ[gq * kTP + c + 1] = fmaf(ah[1], g.scale, b2[c + 1]);
            HQ[(gq + 8) * kTP + c] = fmaf(ah[2], g.scale, b2[c]);
            HQ[(gq + 8) * kTP + c + 1] = fmaf(ah[3], g.scale, b2[c + 1]);
            Z2[gq * kTP + c] = fmaf(az[0], g.scale, C1P[c]);
            Z2[gq * kTP + c + 1] = fmaf(az[1], g.scale, C1P[c + 1]);
            Z2[(gq + 8) * kTP + c] = fmaf(az[2], g.scale, C1P[c]);
            Z2[(gq + 8) * kTP + c + 1] = fmaf(az[3], g.scale, C1P[c + 1]);
            __syncthreads();
        }
        // logits, BCE and dz2 (warp w: queries w, w + 8; unrolled, so the two
        // shuffle / exp chains interleave; accumulation order unchanged)
#pragma unroll
        for (int qi = 0; qi < kTQ / kTW; ++qi) {
            const int q = warp + qi * kTW;
            const float za = Z2[q * kTP + lane], zb = Z2[q * kTP + lane + 32];
            float part = fmaxf(za, 0.f) * u2a + fmaxf(zb, 0.f) * u2b;
#pragma unroll
            for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
            const float z = part + c2;
            float dl = 0.f;
            if (q < nq) {
                if (g.logits && lane == 0) g.logits[q0 + q] = z;
                if (train) {
                    const int64_t li = q0 + q - q_lo;
                    const float y = li < kTailLabels ? LB[li] : g.labels[q0 + q];
                    const float sig = z >= 0.f ? 1.f / (1.f + expf(-z)) : expf(z) / (1.f + expf(z));
                    dl = (sig - y) * g.inv_b;
                    if (lane == 0) {
                        dc2 += dl;
                        lsum += fmaxf(z, 0.f) - z * y + log1pf(expf(-fabsf(z)));
                    }
                    du2a = fmaf(fmaxf(za, 0.f), dl, du2a);
                    du2b = fmaf(fmaxf(zb, 0.f), dl, du2b);
                }
            }
            DZ2[q * kTP + lane] = za > 0.f ? dl * u2a : 0.f;
            DZ2[q * kTP + lane + 32] = zb > 0.f ? dl * u2b : 0.f;
        }
        __syncthreads();
        if (!train) continue;
        // dhq[q][k] = sum_h dz2[q][h] U1[k][h] and g[q][k] = scale sum_h dz2[q][h] V[k][h]
        // (= scale sum_h dhq[q][h] W2[k][h]) in one pass
        {
            float ad[4] = {0.f, 0.f, 0.f, 0.f}, ag[4] = {0.f, 0.f, 0.f, 0.f};
            warp_mma3_dual<8>(ad, ag, lane, [&](int m, int k) { return DZ2[m * kTP + k]; },
                              [&](int k, int n) { return U1s[(8 * warp + n) * kTP + k]; },
                              [&](int k, int n) { return VS[(8 * warp + n) * kTP + k]; });
            const int c = 8 * warp + 2 * tq;
            DHQ[gq * kTP + c] = ad[0];
            DHQ[gq * kTP + c + 1] = ad[1];
            DHQ[(gq + 8) * kTP + c] = ad[2];
            DHQ[(gq + 8) * kTP + c + 1] = ad[3];
            G[gq * kTP + c] = ag[0] * g.scale;
            G[gq * kTP + c + 1] = ag[1] * g.scale;
            G[(gq + 8) * kTP + c] = ag[2] * g.scale;
            G[(gq + 8) * kTP + c + 1] = ag[3] * g.scale;
            // S / msum were issued before the first product (long landed):
            // this barrier publishes them too, so the dW2 / dU1 products and
            // the dW1 FMAs below share one barrier interval
            cp_async_wait_all();
            __syncthreads();
        }
        // dW2 += pooled^T dhq (scaled at the end), dU1 += hq^T dz2
        warp_mma3<4, 2>(aw2, lane, [&](int m, int k) { return PM[k * kTP + 16 * fm + m]; },
                        [&](int k, int n) { return DHQ[k * kTP + 8 * fn + n]; });
        warp_mma3<4, 2>(au1, lane, [&](int m, int k) { return HQ[k * kTP + 16 * fm + m]; },
                        [&](int k, int n) { return DZ2[k * kTP + 8 * fn + n]; });
        // dW1[c][h] += S_q[c][h] g_q[h], db1[h] += msum_q[h] g_q[h]; db2 = sum dhq, dc1 = sum dz2
#pragma unroll
        for (int i = 0; i < NW1; ++i) {
            const int e = tid + NT * i;
            if (e < (AW + 1) * 64) {
                float a = aw1[i];
                for (int q = 0; q < nq; ++q) a = fmaf(SS[q * (AW + 1) * 64 + e], G[q * kTP + (e & 63)], a);
                aw1[i] = a;
            }
        }
        if (tid < 128) {
            const float *V = tid < 64 ? DHQ : DZ2;
            for (int q = 0; q < nq; ++q) vacc += V[q * kTP + (tid & 63)];
        }
        // the next chunk overwrites the chunk buffers (the epilogue below only
        // uses registers and vsm: no barrier after the last chunk)
        if (q0 + kTQ < q_hi) __syncthreads();
    }
    if (g.step_inc && blockIdx.x == 0 && tid == 0) *g.step_inc += 1;
    if (!train) return;
    // ---- partial row of this CTA: [grads | loss], 8-B stores straight from
    // the accumulator pairs (full 32-B sectors per quad of lanes)
    float *row = g.partial + (int64_t)blockIdx.x * (g.off.total + 1);
    vsm[warp * 64 + lane] = du2a;
    vsm[warp * 64 + lane + 32] = du2b;
    if (lane == 0) {
        vsm[kTW * 64 + warp] = dc2;
        vsm[kTW * 64 + kTW + warp] = lsum;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int r0 = 16 * fm + gq, c = 8 * (fn + j) + 2 * tq;
        *reinterpret_cast<float2 *>(row + g.off.w2 + r0 * 64 + c) = make_float2(aw2[j][0] * g.scale, aw2[j][1] * g.scale);
        *reinterpret_cast<float2 *>(row + g.off.w2 + (r0 + 8) * 64 + c) = make_float2(aw2[j][2] * g.scale, aw2[j][3] * g.scale);
        *reinterpret_cast<float2 *>(row + g.off.u1 + r0 * 64 + c) = make_float2(au1[j][0], au1[j][1]);
        *reinterpret_cast<float2 *>(row + g.off.u1 + (r0 + 8) * 64 + c) = make_float2(au1[j][2], au1[j][3]);
    }
#pragma unroll
    for (int i = 0; i < NW1; ++i) {
        const int e = tid + NT * i;
        if (e < AW * 64)
            row[g.off.w1 + e] = aw1[i];
        else if (e < (AW + 1) * 64)
            row[g.off.b1 + e - AW * 64] = aw1[i];
    }
    if (tid < 128) row[(tid < 64 ? g.off.b2 : g.off.c1) + (tid & 63)] = vacc;
    __syncthreads();
    if (tid < 64) {
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < kTW; ++w) v += vsm[w * 64 + tid];
        row[g.off.u2 + tid] = v;
    } else if (tid == 64 || tid == 65) {
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < kTW; ++w) v += vsm[kTW * 64 + (tid - 64) * kTW + w];
        if (tid == 64)
            row[g.off.c2] = v;
        else
            row[g.off.total] = v * g.inv_b;
    }
}

template <int AW>
constexpr size_t tail_smem() {
    return (size_t)(2 * 64 * kTP + 6 * kTQ * kTP + kTW * 64 + 2 * kTW + kTQ * (AW + 1) * 64 + kTailLabels + 64 * kTP +
                    64) * 4;
}

using TailKernel = void (*)(TailArgs);

static TailKernel pick_tail(int aw, size_t &smem) {
    switch (aw) {
#define WJ_T(x) \
    case x: smem = tail_smem<x>(); return tail_tc_kernel<x>;
        WJ_T(2) WJ_T(3) WJ_T(4) WJ_T(5) WJ_T(6) WJ_T(7) WJ_T(8) WJ_T(9) WJ_T(10) WJ_T(12) WJ_T(14) WJ_T(15)
        WJ_T(16)
#undef WJ_T
        default: return nullptr;
    }
}

}  // namespace wj

namespace wj {

// training: exactly partial_rows CTAs, CTA i owns queries [i*q, (i+1)*q) with
// q = per_cta (0: ceil(B / partial_rows)), rows past the last query are zeros;
// inference: one CTA per 16 queries.  inv_b: the mean's 1 / B (0: 1 / n_batch).
int encoder_tail(const float *pooled, const float *s, const float *msum, const float *labels, int64_t n_batch,
                 int32_t aw, int32_t hidden, const float *params, const int32_t *offsets9, float scale,
                 float *logits_out, float *partial, int32_t partial_rows, int32_t per_cta, float inv_b,
                 int64_t *step_inc, cudaStream_t stream, int32_t *sched_reset) {
    if (hidden != kH) {
        set_error("encoder tail kernel supports hidden=64 (got %d)", hidden);
        return WJ_ERR_UNSUPPORTED;
    }
    size_t smem = 0;
    TailKernel k = pick_tail(aw, smem);
    if (!k) {
        set_error("encoder tail not instantiated for A*(L+1)=%d", aw);
        return WJ_ERR_UNSUPPORTED;
    }
    if (labels && (!s || !msum || !partial || partial_rows < 1)) {
        set_error("training tail needs S, msum and a partial buffer");
        return WJ_ERR_ARG;
    }
    // the partial rows are written with 8-B stores: [rows, total + 1] with
    // total + 1 even (every parameter block is a multiple of 64 but c2)
    if (labels && ((reinterpret_cast<uintptr_t>(partial) & 7u) || ((offsets9[8] + 1) & 1) ||
                   ((offsets9[2] | offsets9[4]) & 1))) {
        set_error("training tail: partial must be 8-byte aligned (and W2 / U1 offsets even)");
        return WJ_ERR_ARG;
    }
    if (n_batch == 0 && !labels) return WJ_OK;
    TailArgs g;
    g.pooled = pooled;
    g.s = s;
    g.msum = msum;
    g.labels = labels;
    g.B = n_batch;
    g.params = params;
    g.off = {offsets9[0], offsets9[1], offsets9[2], offsets9[3], offsets9[4],
             offsets9[5], offsets9[6], offsets9[7], offsets9[8]};
    g.scale = scale;
    g.inv_b = inv_b > 0.f ? inv_b : (n_batch > 0 ? 1.f / (float)n_batch : 0.f);
    g.logits = logits_out;
    g.partial = partial;
    g.work = nullptr;
    g.step_inc = step_inc;
    g.sched_reset = sched_reset;
    const int64_t rows = labels ? partial_rows : (n_batch + kTQ - 1) / kTQ;
    g.per_cta = per_cta > 0 ? per_cta : (int)((n_batch + rows - 1) / rows);
    // the smem attribute is per (device, kernel): set once (a repeat is harmless)
    static bool attr_done[64][17] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaSuccess;
    if (dev < 0 || dev >= 64 || !attr_done[dev][aw]) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            set_error("tail smem attribute: %s", cudaGetErrorString(e));
            return WJ_ERR_CUDA;
        }
        if (dev >= 0 && dev < 64) attr_done[dev][aw] = true;
    }
    e = launch_pdl(k, dim3((unsigned)rows), dim3(kTW * 32), smem, stream, g);
    if (e != cudaSuccess) {
        set_error("wj_encoder_tail launch: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return check_launch("wj_encoder_tail");
}

}  // namespace wj

extern "C" int wj_encoder_tail(const float *pooled, const float *s, const float *msum,
                               const float *labels, int64_t n_batch, int32_t aw, int32_t hidden,
                               const float *params, const int32_t *offsets9, float scale,
                               float *logits_out, float *partial, int32_t partial_rows, float *work,
                               int64_t *step_inc, wj_stream_t stream) {
    (void)work;  // not needed by the tensor-core tail (kept for ABI stability)
    return wj::encoder_tail(pooled, s, msum, labels, n_batch, aw, hidden, params, offsets9, scale, logits_out,
                            partial, partial_rows, 0, 0.f, step_inc, (cudaStream_t)stream, nullptr);
}

extern "C" int wj_adam(float *params, float *m, float *v, const float *partial,
                       int32_t partial_rows, int32_t n_params, float lr, float beta1, float beta2,
                       float eps, const int64_t *step, float *grad_out, float *loss_out,
                       wj_stream_t stream) {
    using namespace wj;
    if (n_params < 1 || partial_rows < 1) {
        set_error("bad adam sizes");
        return WJ_ERR_ARG;
    }
    const int blocks = (n_params + 1 + kAdamCols - 1) / kAdamCols;
    const cudaError_t e = launch_pdl(adam_kernel, dim3(blocks), dim3(kAdamCols * kAdamGroups), 0, (cudaStream_t)stream,
                                     params, m, v, partial, partial_rows, n_params, lr, beta1, beta2, eps, step,
                                     grad_out, loss_out);
    if (e != cudaSuccess) {
        set_error("wj_adam launch: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return check_launch("wj_adam");
}

extern "C" int wj_sum_partials(const float *partial, int32_t partial_rows, int32_t n_cols, float *out,
                               wj_stream_t stream) {
    using namespace wj;
    if (n_cols < 1 || partial_rows < 1) {
        set_error("bad partial sizes");
        return WJ_ERR_ARG;
    }
    const int blocks = (n_cols + kAdamCols - 1) / kAdamCols;
    sum_rows_kernel<<<blocks, kAdamCols * kAdamGroups, 0, (cudaStream_t)stream>>>(partial, partial_rows, n_cols,
                                                                                 out);
    return check_launch("wj_sum_partials");
}
