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
};

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

template <int AW>
__global__ void __launch_bounds__(kTailWarps * 32) encoder_tail_kernel(TailArgs g) {
    __shared__ float wts[2 * kH * kPitch];
    float *w2s = wts;
    float *u1s = wts + kH * kPitch;
    __shared__ float vec[kTailWarps][4][kH];  // pm, hq, dz2, dhq of the group's queries
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float *P = g.params;
    for (int i = threadIdx.x; i < kH * kH; i += blockDim.x) {
        const int r = i / kH, c = i % kH;
        w2s[r * kPitch + c] = P[g.off.w2 + i];
        u1s[r * kPitch + c] = P[g.off.u1 + i];
    }
    float b2v[2], c1v[2], u2v[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        b2v[j] = P[g.off.b2 + lane + 32 * j];
        c1v[j] = P[g.off.c1 + lane + 32 * j];
        u2v[j] = P[g.off.u2 + lane + 32 * j];
    }
    const float c2 = P[g.off.c2];
    const bool train = g.labels != nullptr;
    // register accumulators
    float dW1[AW][2], db1[2] = {0.f, 0.f}, du2[2] = {0.f, 0.f}, dc1[2] = {0.f, 0.f},
                      db2[2] = {0.f, 0.f}, dc2 = 0.f, loss = 0.f;
    float dU1[8][2], dW2[8][2];  // rows k = 8*warp + i, cols lane, lane+32
#pragma unroll
    for (int c = 0; c < AW; ++c) dW1[c][0] = dW1[c][1] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) dU1[i][0] = dU1[i][1] = dW2[i][0] = dW2[i][1] = 0.f;
    __syncthreads();
    const float invB = 1.f / (float)g.B;
    const int64_t groups = (g.B + kTailWarps - 1) / kTailWarps;
    for (int64_t grp = blockIdx.x; grp < groups; grp += gridDim.x) {
        const int64_t b = grp * kTailWarps + warp;
        const bool active = b < g.B;
        float pm[2] = {0.f, 0.f}, hq[2], dz2[2] = {0.f, 0.f}, dhq[2] = {0.f, 0.f};
        if (active) {
#pragma unroll
            for (int j = 0; j < 2; ++j) pm[j] = g.pooled[b * kH + lane + 32 * j] * g.scale;
            matvec(pm, w2s, lane, hq);  // hq = pm W2 + b2
            hq[0] += b2v[0];
            hq[1] += b2v[1];
            float z2[2];
            matvec(hq, u1s, lane, z2);  // z2 = hq U1 + c1
            z2[0] += c1v[0];
            z2[1] += c1v[1];
            const float a2[2] = {fmaxf(z2[0], 0.f), fmaxf(z2[1], 0.f)};
            float part = a2[0] * u2v[0] + a2[1] * u2v[1];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
            const float z = part + c2;
            if (g.logits && lane == 0) g.logits[b] = z;
            if (train) {
                const float y = g.labels[b];
                loss += fmaxf(z, 0.f) - z * y + log1pf(expf(-fabsf(z)));
                const float sig = z >= 0.f ? 1.f / (1.f + expf(-z)) : expf(z) / (1.f + expf(z));
                const float dl = (sig - y) * invB;
                dc2 += dl;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    du2[j] = fmaf(a2[j], dl, du2[j]);
                    dz2[j] = z2[j] > 0.f ? dl * u2v[j] : 0.f;
                    dc1[j] += dz2[j];
                }
                // dhq[k] = sum_h dz2[h] U1[k][h], k = lane, lane + 32
                matvec_t(dz2, u1s, lane, dhq);
                db2[0] += dhq[0];
                db2[1] += dhq[1];
                // gk[k] = sum_h dhq[h] W2[k][h] * scale, k = lane, lane + 32
                float gk[2];
                matvec_t(dhq, w2s, lane, gk);
                gk[0] *= g.scale;
                gk[1] *= g.scale;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    db1[j] = fmaf(g.msum[b * kH + lane + 32 * j], gk[j], db1[j]);
#pragma unroll
                    for (int c = 0; c < AW; ++c)
                        dW1[c][j] = fmaf(g.s[(b * AW + c) * kH + lane + 32 * j], gk[j], dW1[c][j]);
                }
            }
        }
        if (!train) continue;
        // rank-1 updates of dU1 = hq^T dz2 and dW2 = pm^T dhq, split by rows over warps
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            vec[warp][0][lane + 32 * j] = pm[j];
            vec[warp][1][lane + 32 * j] = active ? hq[j] : 0.f;
            vec[warp][2][lane + 32 * j] = dz2[j];
            vec[warp][3][lane + 32 * j] = dhq[j];
        }
        __syncthreads();
        for (int q = 0; q < kTailWarps; ++q) {
            const float dzl[2] = {vec[q][2][lane], vec[q][2][lane + 32]};
            const float dhl[2] = {vec[q][3][lane], vec[q][3][lane + 32]};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int k = warp * 8 + i;
                const float hk = vec[q][1][k], pk = vec[q][0][k];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    dU1[i][j] = fmaf(hk, dzl[j], dU1[i][j]);
                    dW2[i][j] = fmaf(pk, dhl[j], dW2[i][j]);
                }
            }
        }
        __syncthreads();
    }
    if (!train) return;
    // this CTA's partial gradients -> its row of the partial buffer
    float *row = g.partial + (int64_t)blockIdx.x * (g.off.total + 1);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int k = warp * 8 + i;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            row[g.off.u1 + k * kH + lane + 32 * j] = dU1[i][j];
            row[g.off.w2 + k * kH + lane + 32 * j] = dW2[i][j];
        }
    }
    // per-warp vectors: reduce over warps through shared memory (reusing the
    // weight tiles, which are dead after the query loop), 8 vectors at a time
    constexpr int NVEC = AW + 4;  // dW1 rows, db1, db2, dc1, du2
    constexpr int CH = 8;
    static_assert(kTailWarps * CH * kH <= 2 * kH * kPitch, "reduction tile too large");
    float(*red)[CH][kH] = reinterpret_cast<float(*)[CH][kH]>(wts);
    __shared__ float sred[kTailWarps][2];
    float vals[NVEC][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int c = 0; c < AW; ++c) vals[c][j] = dW1[c][j];
        vals[AW + 0][j] = db1[j];
        vals[AW + 1][j] = db2[j];
        vals[AW + 2][j] = dc1[j];
        vals[AW + 3][j] = du2[j];
    }
    if (lane == 0) {
        sred[warp][0] = dc2;   // dc2 and the loss are warp-uniform: take lane 0
        sred[warp][1] = loss;
    }
#pragma unroll
    for (int v0 = 0; v0 < NVEC; v0 += CH) {
        __syncthreads();
#pragma unroll
        for (int vv = 0; vv < CH; ++vv) {
            if (v0 + vv < NVEC) {
                red[warp][vv][lane] = vals[v0 + vv][0];
                red[warp][vv][lane + 32] = vals[v0 + vv][1];
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < CH * kH; i += blockDim.x) {
            const int v = v0 + i / kH, h = i % kH;
            if (v >= NVEC) continue;
            float sum = 0.f;
#pragma unroll
            for (int w = 0; w < kTailWarps; ++w) sum += red[w][i / kH][h];
            int dst;
            if (v < AW)
                dst = g.off.w1 + v * kH + h;
            else if (v == AW)
                dst = g.off.b1 + h;
            else if (v == AW + 1)
                dst = g.off.b2 + h;
            else if (v == AW + 2)
                dst = g.off.c1 + h;
            else
                dst = g.off.u2 + h;
            row[dst] = sum;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.f, l = 0.f;
        for (int w = 0; w < kTailWarps; ++w) {
            s += sred[w][0];
            l += sred[w][1];
        }
        row[g.off.c2] = s;
        row[g.off.total] = l * invB;
    }
}

// Sum the per-CTA partial gradients in a fixed order and apply Adam
// (encoder.py:236-249) with bias corrections from the device step counter.
// A CTA owns 32 consecutive parameters; its 8 warps each sum every 8th
// partial row (coalesced 128-B rows), then warp 0 adds the 8 sums in order:
// deterministic, and 8x the memory parallelism of one thread per column.
constexpr int kAdamCols = 32, kAdamGroups = 8;

__global__ void __launch_bounds__(kAdamCols *kAdamGroups) adam_kernel(
    float *params, float *m, float *v, const float *partial, int rows, int n, float lr, float beta1,
    float beta2, float eps, const int64_t *step, float *grad_out, float *loss_out) {
    __shared__ float part[kAdamGroups][kAdamCols];
    const int c = threadIdx.x & (kAdamCols - 1), grp = threadIdx.x / kAdamCols;
    const int i = blockIdx.x * kAdamCols + c;
    float gsum = 0.f;
    if (i <= n)
        for (int r = grp; r < rows; r += kAdamGroups) gsum += partial[(int64_t)r * (n + 1) + i];
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
    const float mi = beta1 * m[i] + (1.f - beta1) * gsum;
    const float vi = beta2 * v[i] + (1.f - beta2) * gsum * gsum;
    m[i] = mi;
    v[i] = vi;
    params[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
}

// Fixed-order column sums of the partial rows (the data-parallel path:
// reduce locally, all-reduce the [n+1] vector over ranks, then Adam on it).
__global__ void __launch_bounds__(kAdamCols *kAdamGroups) sum_rows_kernel(const float *partial, int rows,
                                                                        int cols, float *out) {
    __shared__ float part[kAdamGroups][kAdamCols];
    const int c = threadIdx.x & (kAdamCols - 1), grp = threadIdx.x / kAdamCols;
    const int i = blockIdx.x * kAdamCols + c;
    float gsum = 0.f;
    if (i < cols)
        for (int r = grp; r < rows; r += kAdamGroups) gsum += partial[(int64_t)r * cols + i];
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
    case x: return encoder_tail_kernel<x>;
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
                               float *logits_out, float *partial, int32_t partial_rows,
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
    if (labels && (!s || !msum || !partial || partial_rows < 1)) {
        set_error("training tail needs S, msum and a partial buffer");
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
    const int64_t groups = (n_batch + kTailWarps - 1) / kTailWarps;
    int64_t grid = labels ? partial_rows : (groups < 1024 ? groups : 1024);
    if (grid > groups && !labels) grid = groups;
    k<<<(unsigned)grid, kTailWarps * 32, 0, (cudaStream_t)stream>>>(g);
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
