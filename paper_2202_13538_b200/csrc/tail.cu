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
// One warp per query (lane owns hidden units lane and lane+32: conflict-free
// shared-memory access to both W and W^T with a 65-float row pitch); the
// rank-1 updates of the 64x64 gradients are split by rows across the CTA's 8
// warps.  Each CTA writes its partial gradients to its own row of a
// [grid, n_params] buffer; the Adam kernel reduces those rows in a fixed
// order (deterministic) and applies the bias-corrected update
// (encoder.py:236-249).
#include "common.cuh"

namespace wj {

constexpr int kTailWarps = 8;
constexpr int kH = 64;
constexpr int kPitch = 65;

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
    float *logits;        // [B] nullable
    float *partial;       // [grid, total + 1] (last column: loss partial)
    float *work;          // [B, kVecStride] per-query vectors (training)
    int per_cta;          // queries per gradient CTA
};

// per-query vectors in the work buffer: pm, hq, dz2, dhq, g, a2*dl | dl, loss
constexpr int kVecStride = 6 * kH + 8;
enum { kPM = 0, kHQ = kH, kDZ2 = 2 * kH, kDHQ = 3 * kH, kG = 4 * kH, kA2DL = 5 * kH, kDL = 6 * kH, kLOSS };

// out[c] = sum_k in[k] M[k][c] for the lane's columns c = lane, lane + 32
// (in: the warp's 64-vector, lane holds k = lane, lane + 32).  Four
// independent accumulator chains per output instead of one 64-long chain.
__device__ __forceinline__ void matvec(const float (&in)[2], const float *Ms, int lane, float (&out)[2]) {
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int k = 0; k < kH; ++k) {
        const float x = __shfl_sync(kFull, in[k >> 5], k & 31);
        acc[0][k & 3] = fmaf(x, Ms[k * kPitch + lane], acc[0][k & 3]);
        acc[1][k & 3] = fmaf(x, Ms[k * kPitch + lane + 32], acc[1][k & 3]);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) out[j] = (acc[j][0] + acc[j][1]) + (acc[j][2] + acc[j][3]);
}

// out[r] = sum_h in[h] M[r][h] for the lane's rows r = lane, lane + 32
__device__ __forceinline__ void matvec_t(const float (&in)[2], const float *Ms, int lane, float (&out)[2]) {
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int h = 0; h < kH; ++h) {
        const float x = __shfl_sync(kFull, in[h >> 5], h & 31);
        acc[0][h & 3] = fmaf(x, Ms[lane * kPitch + h], acc[0][h & 3]);
        acc[1][h & 3] = fmaf(x, Ms[(lane + 32) * kPitch + h], acc[1][h & 3]);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) out[j] = (acc[j][0] + acc[j][1]) + (acc[j][2] + acc[j][3]);
}

// Phase 1: one warp per query -- forward (logits) and, for training, the
// per-query backward vectors into the work buffer.  No cross-query state.
__global__ void __launch_bounds__(kTailWarps * 32) tail_vec_kernel(TailArgs g) {
    __shared__ float wts[2 * kH * kPitch];
    float *w2s = wts;
    float *u1s = wts + kH * kPitch;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float *P = g.params;
    for (int i = threadIdx.x; i < kH * kH; i += blockDim.x) {
        const int r = i / kH, c = i % kH;
        cp_async4(w2s + r * kPitch + c, P + g.off.w2 + i);
        cp_async4(u1s + r * kPitch + c, P + g.off.u1 + i);
    }
    float b2v[2], c1v[2], u2v[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        b2v[j] = P[g.off.b2 + lane + 32 * j];
        c1v[j] = P[g.off.c1 + lane + 32 * j];
        u2v[j] = P[g.off.u2 + lane + 32 * j];
    }
    const float c2 = P[g.off.c2];
    cp_async_wait_all();
    __syncthreads();
    const float invB = 1.f / (float)g.B;
    for (int64_t b = (int64_t)blockIdx.x * kTailWarps + warp; b < g.B; b += (int64_t)gridDim.x * kTailWarps) {
        float pm[2], hq[2], z2[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) pm[j] = g.pooled[b * kH + lane + 32 * j] * g.scale;
        matvec(pm, w2s, lane, hq);  // hq = pm W2 + b2
        hq[0] += b2v[0];
        hq[1] += b2v[1];
        matvec(hq, u1s, lane, z2);  // z2 = hq U1 + c1
        z2[0] += c1v[0];
        z2[1] += c1v[1];
        const float a2[2] = {fmaxf(z2[0], 0.f), fmaxf(z2[1], 0.f)};
        float part = a2[0] * u2v[0] + a2[1] * u2v[1];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
        const float z = part + c2;
        if (g.logits && lane == 0) g.logits[b] = z;
        if (!g.labels) continue;
        const float y = g.labels[b];
        const float loss = fmaxf(z, 0.f) - z * y + log1pf(expf(-fabsf(z)));
        const float sig = z >= 0.f ? 1.f / (1.f + expf(-z)) : expf(z) / (1.f + expf(z));
        const float dl = (sig - y) * invB;
        float dz2[2], dhq[2], gk[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) dz2[j] = z2[j] > 0.f ? dl * u2v[j] : 0.f;
        matvec_t(dz2, u1s, lane, dhq);  // dhq[k] = sum_h dz2[h] U1[k][h]
        matvec_t(dhq, w2s, lane, gk);   // g[k] = sum_h dhq[h] W2[k][h] * scale
        float *wk = g.work + b * kVecStride;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int h = lane + 32 * j;
            wk[kPM + h] = pm[j];
            wk[kHQ + h] = hq[j];
            wk[kDZ2 + h] = dz2[j];
            wk[kDHQ + h] = dhq[j];
            wk[kG + h] = gk[j] * g.scale;
            wk[kA2DL + h] = a2[j] * dl;
        }
        if (lane == 0) {
            wk[kDL] = dl;
            wk[kLOSS] = loss;
        }
    }
}

// Phase 2: CTA r reduces queries [r*per, (r+1)*per) in a fixed order into
// partial row r.  Thread t owns column h = t % 64 of rows k = t/64 + 4i of
// dW2 / dU1 / dW1 and one of the bias vectors; the chunk's vectors are staged
// in shared memory, so the inner loop is pure FMA (no dependent chains).
template <int AW>
__global__ void __launch_bounds__(256) tail_grad_kernel(TailArgs g) {
    constexpr int CH = 8;                   // queries per staged chunk
    constexpr int NK = (AW + 3) / 4;        // dW1 rows per thread
    __shared__ float wv[CH][kVecStride];
    __shared__ float sv[CH][AW * kH + kH];  // S rows then msum
    const int t = threadIdx.x, h = t & (kH - 1), kq = t >> 6;
    float dW2[16], dU1[16], dW1[NK], vec = 0.f, dc2 = 0.f, loss = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) dW2[i] = dU1[i] = 0.f;
#pragma unroll
    for (int i = 0; i < NK; ++i) dW1[i] = 0.f;
    const int64_t b0 = (int64_t)blockIdx.x * g.per_cta;
    const int64_t b1 = min((int64_t)g.B, b0 + g.per_cta);
    for (int64_t cb = b0; cb < b1; cb += CH) {
        const int nq = (int)min((int64_t)CH, b1 - cb);
        __syncthreads();
        for (int i = t; i < nq * kVecStride; i += blockDim.x)
            cp_async4(&wv[i / kVecStride][i % kVecStride], g.work + cb * kVecStride + i);
        for (int i = t; i < nq * AW * kH; i += blockDim.x)
            cp_async4(&sv[i / (AW * kH)][i % (AW * kH)], g.s + cb * AW * kH + i);
        for (int i = t; i < nq * kH; i += blockDim.x) cp_async4(&sv[i / kH][AW * kH + i % kH], g.msum + cb * kH + i);
        cp_async_wait_all();
        __syncthreads();
        for (int q = 0; q < nq; ++q) {
            const float *w = wv[q];
            const float dhq = w[kDHQ + h], dz2 = w[kDZ2 + h], gg = w[kG + h];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                dW2[i] = fmaf(w[kPM + kq + 4 * i], dhq, dW2[i]);
                dU1[i] = fmaf(w[kHQ + kq + 4 * i], dz2, dU1[i]);
            }
#pragma unroll
            for (int i = 0; i < NK; ++i)
                if (kq + 4 * i < AW) dW1[i] = fmaf(sv[q][(kq + 4 * i) * kH + h], gg, dW1[i]);
            if (kq == 0)
                vec = fmaf(sv[q][AW * kH + h], gg, vec);  // db1
            else if (kq == 1)
                vec += dhq;                               // db2
            else if (kq == 2)
                vec += dz2;                               // dc1
            else
                vec += w[kA2DL + h];                      // du2
            if (t == 0) {
                dc2 += w[kDL];
                loss += w[kLOSS];
            }
        }
    }
    float *row = g.partial + (int64_t)blockIdx.x * (g.off.total + 1);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        row[g.off.w2 + (kq + 4 * i) * kH + h] = dW2[i];
        row[g.off.u1 + (kq + 4 * i) * kH + h] = dU1[i];
    }
#pragma unroll
    for (int i = 0; i < NK; ++i)
        if (kq + 4 * i < AW) row[g.off.w1 + (kq + 4 * i) * kH + h] = dW1[i];
    const int vo = kq == 0 ? g.off.b1 : (kq == 1 ? g.off.b2 : (kq == 2 ? g.off.c1 : g.off.u2));
    row[vo + h] = vec;
    if (t == 0) {
        row[g.off.c2] = dc2;
        row[g.off.total] = loss / (float)g.B;
    }
}

// Sum the per-CTA partial gradients in a fixed order and apply Adam
// (encoder.py:236-249) with bias corrections from the device step counter.
// A CTA owns 32 consecutive parameters; its 8 warps each sum every 8th
// partial row (coalesced 128-B rows), then warp 0 adds the 8 sums in order:
// deterministic, and 8x the memory parallelism of one thread per column.
constexpr int kAdamCols = 32, kAdamGroups = 8;

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
    float gsum = 0.f;
    if (i <= n) gsum = strided_sum(partial + i, (int64_t)(n + 1), grp, rows);
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
    const int64_t t = *step;
    const float bc1 = 1.f - powf(beta1, (float)t);
    const float bc2 = 1.f - powf(beta2, (float)t);
    if (grad_out) grad_out[i] = gsum;
    adam_update(params + i, m + i, v + i, gsum, lr, beta1, beta2, eps, bc1, bc2);
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

using TailKernel = void (*)(TailArgs);

static TailKernel pick_tail(int aw) {
    switch (aw) {
#define WJ_T(x) \
    case x: return tail_grad_kernel<x>;
        WJ_T(2) WJ_T(3) WJ_T(4) WJ_T(5) WJ_T(6) WJ_T(8) WJ_T(9) WJ_T(10) WJ_T(12) WJ_T(14) WJ_T(15)
        WJ_T(16)
#undef WJ_T
        default: return nullptr;
    }
}

}  // namespace wj

extern "C" int wj_encoder_tail(const float *pooled, const float *s, const float *msum,
                               const float *labels, int64_t n_batch, int32_t aw, int32_t hidden,
                               const float *params, const int32_t *offsets9, float scale,
                               float *logits_out, float *partial, int32_t partial_rows, float *work,
                               wj_stream_t stream) {
    using namespace wj;
    if (hidden != kH) {
        set_error("encoder tail kernel supports hidden=64 (got %d)", hidden);
        return WJ_ERR_UNSUPPORTED;
    }
    TailKernel k = pick_tail(aw);
    if (!k) {
        set_error("encoder tail not instantiated for A*(L+1)=%d", aw);
        return WJ_ERR_UNSUPPORTED;
    }
    if (labels && (!s || !msum || !partial || !work || partial_rows < 1)) {
        set_error("training tail needs S, msum, a partial buffer and a work buffer");
        return WJ_ERR_ARG;
    }
    if (n_batch == 0) return WJ_OK;
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
    g.logits = logits_out;
    g.partial = partial;
    g.work = work;
    g.per_cta = (int)((n_batch + partial_rows - 1) / partial_rows);
    const int64_t groups = (n_batch + kTailWarps - 1) / kTailWarps;
    const int64_t grid = groups < 4096 ? groups : 4096;
    tail_vec_kernel<<<(unsigned)grid, kTailWarps * 32, 0, (cudaStream_t)stream>>>(g);
    if (!labels) return check_launch("wj_encoder_tail");
    // exactly partial_rows CTAs: rows past the last query write zeros
    k<<<(unsigned)partial_rows, 256, 0, (cudaStream_t)stream>>>(g);
    return check_launch("wj_encoder_tail");
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
    adam_kernel<<<blocks, kAdamCols * kAdamGroups, 0, (cudaStream_t)stream>>>(
        params, m, v, partial, partial_rows, n_params, lr, beta1, beta2, eps, step, grad_out, loss_out);
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
