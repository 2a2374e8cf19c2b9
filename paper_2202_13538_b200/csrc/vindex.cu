// Virtual-landing index of the store: the per-anchor input layout of the
// tensor-core join+encode kernel (encode_mma.cu), built once after interning.
//
// Anchor u's block of the joined input has one row per walk slot; the rows
// of a landing l (one distinct node x of u's walks) are identical and there
// are n_l = (row sum of l's count vector) of them.  The encoder kernel draws
// the dropout of a landing's rows in "virtual landings" of at most 2 rows
// (Binomial(2, keep) or Bernoulli(keep) per unit), so anchor u's block is
// described once, at preprocess time, by
//
//   section 2: landing l repeated floor(n_l / 2) times  (2-row virtual landings)
//   section 1: every landing with odd n_l, once          (1-row virtual landings)
//
// stored as uint16 landing indices at vslots[voff[u], voff[u+1]) with
// vcnt[u] = {|section 2|, |section 1|}.  Sum over sections = sum ceil(n_l/2).
// The reference has no such structure: it is the device layout of the rows
// that pipeline._dense_batch (pipeline.py:169-182) materialises densely.
#include <cuda_fp16.h>

#include "common.cuh"

namespace wj {

__device__ __forceinline__ int row_sum(uint64_t key, int cb, int W) {
    const uint64_t m = (1ULL << cb) - 1;
    int s = 0;
    for (int c = 0; c < W; ++c) s += (int)((key >> (cb * c)) & m);
    return s;
}

// one warp per anchor: {sum floor(n/2), sum (n & 1)}
__global__ void vindex_count_kernel(const int64_t *__restrict__ off, const int32_t *__restrict__ uid,
                                    int64_t n, const uint64_t *__restrict__ tk, int cb, int W,
                                    int32_t *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (u >= n) return;
    const int64_t lo = off[u], hi = off[u + 1];
    int c2 = 0, c1 = 0;
    for (int64_t e0 = lo + lane; e0 < hi; e0 += 4 * 32) {  // four ids per lane in flight
        int32_t id[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) id[j] = e0 + 32 * j < hi ? __ldg(uid + e0 + 32 * j) : -1;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (id[j] < 0) continue;
            const int r = row_sum(__ldg(tk + id[j]), cb, W);
            c2 += r >> 1;
            c1 += r & 1;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        c2 += __shfl_xor_sync(kFull, c2, o);
        c1 += __shfl_xor_sync(kFull, c1, o);
    }
    if (lane == 0) {
        cnt[2 * u] = c2;
        cnt[2 * u + 1] = c1;
    }
}

// one warp per anchor, 32 landings at a time; the 2-row section of a chunk
// is expanded cooperatively (heavy landings -- the anchor itself has >= M
// rows -- would otherwise serialise on one lane)
__global__ void vindex_fill_kernel(const int64_t *__restrict__ off, const int32_t *__restrict__ uid,
                                   int64_t n, const uint64_t *__restrict__ tk, int cb, int W,
                                   const int64_t *__restrict__ voff, const int32_t *__restrict__ cnt,
                                   uint16_t *__restrict__ vs) {
    __shared__ int incl_s[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (u >= n) return;
    const int64_t lo = off[u], hi = off[u + 1];
    uint16_t *out2 = vs + voff[u];
    uint16_t *out1 = out2 + cnt[2 * u];
    int run2 = 0, run1 = 0;
    for (int64_t base = lo; base < hi; base += 32) {
        const int64_t e = base + lane;
        int r = 0;
        if (e < hi) r = row_sum(__ldg(tk + __ldg(uid + e)), cb, W);
        const int k2 = r >> 1, k1 = r & 1;
        int i2 = k2;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(kFull, i2, o);
            if (lane >= o) i2 += t;
        }
        const unsigned b1 = __ballot_sync(kFull, k1);
        const int l = (int)(e - lo);
        if (k1) out1[run1 + __popc(b1 & lanemask_lt())] = (uint16_t)l;
        incl_s[wib][lane] = i2;
        __syncwarp();
        const int tot2 = __shfl_sync(kFull, i2, 31);
        for (int p = lane; p < tot2; p += 32) {
            int a = 0, b = 31;  // first lane with incl > p
            while (a < b) {
                const int m = (a + b) >> 1;
                if (incl_s[wib][m] > p)
                    b = m;
                else
                    a = m + 1;
            }
            out2[run2 + p] = (uint16_t)(base - lo + a);
        }
        __syncwarp();
        run2 += tot2;
        run1 += __popc(b1);
    }
}

// fp16 count rows of the RPE table (8 halves per id, zero padded; W <= 8):
// the X operand rows of the tensor-core kernel
__global__ void table_rows_kernel(const uint64_t *__restrict__ tk, int64_t tlen, int cb, int W,
                                  uint4 *__restrict__ rows) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= tlen) return;
    const uint64_t key = tk[i], m = (1ULL << cb) - 1;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float lo = 2 * k < W ? (float)(uint32_t)((key >> (cb * 2 * k)) & m) : 0.f;
        const float hi = 2 * k + 1 < W ? (float)(uint32_t)((key >> (cb * (2 * k + 1))) & m) : 0.f;
        const __half2 h = __floats2half2_rn(lo, hi);
        w[k] = *reinterpret_cast<const uint32_t *>(&h);
    }
    rows[i] = make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace wj

extern "C" int wj_vindex_count(const int64_t *offsets, const int32_t *uniq_id, int64_t n_anchors,
                               const uint64_t *table_keys, int32_t num_walks, int32_t num_steps,
                               int32_t *vcnt_out, wj_stream_t stream) {
    using namespace wj;
    if (n_anchors < 0 || num_walks < 1 || num_steps < 1 || num_steps + 1 > 64) {
        set_error("bad shape");
        return WJ_ERR_ARG;
    }
    if (n_anchors == 0) return WJ_OK;
    const int cb = bits_for((uint64_t)num_walks);
    const int64_t blocks = (n_anchors * 32 + 255) / 256;
    vindex_count_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(offsets, uniq_id, n_anchors, table_keys,
                                                                            cb, num_steps + 1, vcnt_out);
    return check_launch("wj_vindex_count");
}

extern "C" int wj_vindex_fill(const int64_t *offsets, const int32_t *uniq_id, int64_t n_anchors,
                              const uint64_t *table_keys, int32_t num_walks, int32_t num_steps,
                              const int64_t *voff, const int32_t *vcnt, uint16_t *vslots_out,
                              wj_stream_t stream) {
    using namespace wj;
    if (n_anchors < 0 || num_walks < 1 || num_steps < 1 || num_steps + 1 > 64) {
        set_error("bad shape");
        return WJ_ERR_ARG;
    }
    if ((int64_t)num_walks * (num_steps + 1) > 65535) {
        set_error("M*(L+1) > 65535: landing index does not fit uint16");
        return WJ_ERR_UNSUPPORTED;
    }
    if (n_anchors == 0) return WJ_OK;
    const int cb = bits_for((uint64_t)num_walks);
    const int64_t blocks = (n_anchors * 32 + 255) / 256;
    vindex_fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(offsets, uniq_id, n_anchors, table_keys, cb,
                                                                           num_steps + 1, voff, vcnt, vslots_out);
    return check_launch("wj_vindex_fill");
}

extern "C" int wj_table_rows_f16(const uint64_t *table_keys, int64_t table_len, int32_t num_walks,
                                 int32_t num_steps, uint16_t *rows_out, wj_stream_t stream) {
    using namespace wj;
    if (table_len < 0 || num_walks < 1 || num_steps < 1 || num_walks > 2048) {
        set_error("bad shape (fp16 rows need M <= 2048)");
        return WJ_ERR_ARG;
    }
    if (num_steps + 1 > 8) {
        set_error("fp16 table rows need L+1 <= 8");
        return WJ_ERR_UNSUPPORTED;
    }
    if (table_len == 0) return WJ_OK;
    const int cb = bits_for((uint64_t)num_walks);
    table_rows_kernel<<<(unsigned)((table_len + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        table_keys, table_len, cb, num_steps + 1, reinterpret_cast<uint4 *>(rows_out));
    return check_launch("wj_table_rows_f16");
}
