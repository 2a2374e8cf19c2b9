// Query-level join fused with densify, plus the small store kernels
// (gather_rpe, reference dict export, point lookup) for sm_100a.
//
// Reference: _kernels.py:209-245 (join_fill) probes anchor j's hash dict for
// every landing of every query anchor a -- A^2*M*(L+1) random probes per
// query -- and pipeline.py:178 then densifies table[rpe_ids] to float64 in a
// separate numpy pass.  Here one CTA owns one query: it stages the A anchors'
// sorted unique-id lists in shared memory, resolves each DISTINCT landing of
// anchor a against anchor j once (binary search in shared memory over the
// sorted list, A*(A-1)*U searches instead of A^2*M*(L+1) probes), and then
// expands to the M*(L+1) walk slots through the per-slot unique index,
// writing the RPE ids and/or the dense count rows straight into the
// encoder's input buffer.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace wj {

template <typename T>
__device__ __forceinline__ T to_out(uint32_t v);
template <>
__device__ __forceinline__ float to_out<float>(uint32_t v) { return (float)v; }
template <>
__device__ __forceinline__ double to_out<double>(uint32_t v) { return (double)v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(uint32_t v) {
    return __float2bfloat16_rn((float)v);
}
template <>
__device__ __forceinline__ __half to_out<__half>(uint32_t v) { return __float2half_rn((float)v); }

struct JoinArgs {
    const int64_t *queries;
    int64_t n_batch;
    int A;
    const int32_t *walks;
    const int64_t *offsets;
    const int32_t *ux;
    const int32_t *uid;
    const uint16_t *slot_idx;
    int M, W, P, max_u;
    const uint64_t *tkeys;
    int64_t tlen;
    int stage_table;
    int cb;
    int32_t *walk_nodes;
    int32_t *rpe_ids;
    void *dense;
    int64_t row_stride;
};

__device__ __forceinline__ int lower_bound_s(const int32_t *a, int n, int32_t x) {
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

template <typename OutT>
__global__ void __launch_bounds__(256) join_kernel(JoinArgs g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int A = g.A, P = g.P, W = g.W, mu = g.max_u;
    int64_t *qa = reinterpret_cast<int64_t *>(smem_raw);            // [A]
    int *un = reinterpret_cast<int *>(qa + 4);                         // [A]
    int32_t *sx = reinterpret_cast<int32_t *>(un + 4);                 // [A][mu]
    int32_t *sid = sx + (size_t)A * mu;                                // [A][mu]
    int32_t *cross = sid + (size_t)A * mu;                             // [A][A-1][mu]
    uint16_t *sl = reinterpret_cast<uint16_t *>(cross + (size_t)A * (A - 1) * mu);  // [P]
    uint64_t *tks = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(sl + P) + 15) & ~uintptr_t(15));  // [tlen] if staged
    const uint64_t cmask = (1ULL << g.cb) - 1;

    if (g.stage_table) {
        for (int64_t i = threadIdx.x; i < g.tlen; i += blockDim.x) tks[i] = g.tkeys[i];
    }
    for (int64_t b = blockIdx.x; b < g.n_batch; b += gridDim.x) {
        if (threadIdx.x < A) {
            const int64_t q = g.queries[b * A + threadIdx.x];
            qa[threadIdx.x] = q;
            un[threadIdx.x] = (int)(g.offsets[q + 1] - g.offsets[q]);
        }
        __syncthreads();
        for (int a = 0; a < A; ++a) {
            const int64_t lo = g.offsets[qa[a]];
            const int n = un[a];
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                sx[a * mu + i] = __ldg(g.ux + lo + i);
                sid[a * mu + i] = __ldg(g.uid + lo + i);
            }
        }
        __syncthreads();
        if (g.rpe_ids || g.dense) {
            // resolve each distinct landing of anchor a against anchor j != a
            for (int a = 0; a < A; ++a) {
                for (int jj = 0; jj < A - 1; ++jj) {
                    const int j = jj < a ? jj : jj + 1;
                    const int nj = un[j];
                    const int32_t *xj = sx + j * mu;
                    int32_t *dst = cross + (a * (A - 1) + jj) * mu;
                    for (int k = threadIdx.x; k < un[a]; k += blockDim.x) {
                        const int32_t x = sx[a * mu + k];
                        const int pos = lower_bound_s(xj, nj, x);
                        dst[k] = (pos < nj && xj[pos] == x) ? sid[j * mu + pos] : 0;
                    }
                }
            }
        }
        __syncthreads();
        for (int a = 0; a < A; ++a) {
            const int64_t q = qa[a];
            if (g.walk_nodes) {
                const int32_t *src = g.walks + q * (int64_t)P;
                int32_t *dst = g.walk_nodes + (b * A + a) * (int64_t)P;
                for (int i = threadIdx.x; i < P; i += blockDim.x) dst[i] = __ldg(src + i);
            }
            if (!(g.rpe_ids || g.dense)) continue;
            const uint16_t *slq = g.slot_idx + q * (int64_t)P;
            for (int i = threadIdx.x; i < P; i += blockDim.x) sl[i] = __ldg(slq + i);
            __syncthreads();
            for (int p = threadIdx.x; p < P; p += blockDim.x) {
                const int local = sl[p];
                const int64_t row = b * (int64_t)A * P + (int64_t)a * P + p;
                int32_t ids[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j < A) {
                        const int jj = j < a ? j : j - 1;
                        ids[j] = (j == a) ? sid[a * mu + local]
                                          : cross[(a * (A - 1) + jj) * mu + local];
                    }
                }
                if (g.rpe_ids) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (j < A) g.rpe_ids[row * A + j] = ids[j];
                }
                if (g.dense) {
                    OutT *out = reinterpret_cast<OutT *>(g.dense) + row * g.row_stride;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (j < A) {
                            const uint64_t key =
                                g.stage_table ? tks[ids[j]] : __ldg(g.tkeys + ids[j]);
                            for (int c = 0; c < W; ++c)
                                out[j * W + c] = to_out<OutT>((uint32_t)((key >> (g.cb * c)) & cmask));
                        }
                    }
                }
            }
            __syncthreads();
        }
        __syncthreads();
    }
}

__global__ void gather_rpe_kernel(const int32_t *__restrict__ ids, int64_t n,
                                  const int32_t *__restrict__ table, int64_t tlen, int width,
                                  void *out, int dtype, int32_t *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t id = ids[i];
        if (id < 0 || id >= tlen) {
            *bad = 1;
            id = 0;
        }
        for (int c = 0; c < width; ++c) {
            const uint32_t v = (uint32_t)table[(int64_t)id * width + c];
            const int64_t o = i * width + c;
            switch (dtype) {
                case WJ_F32: reinterpret_cast<float *>(out)[o] = (float)v; break;
                case WJ_F64: reinterpret_cast<double *>(out)[o] = (double)v; break;
                case WJ_BF16: reinterpret_cast<__nv_bfloat16 *>(out)[o] = __float2bfloat16_rn((float)v); break;
                default: reinterpret_cast<__half *>(out)[o] = __float2half_rn((float)v); break;
            }
        }
    }
}

// Reference dict layout (_kernels.py:174-188): insertion in first-appearance
// order, hash mix64(x) & mask, linear probing.  Walking the slots in order and
// inserting a node when its first appearance is reached reproduces the
// insertion order without a sort.
__global__ void export_dicts_kernel(const int64_t *__restrict__ offsets,
                                    const int32_t *__restrict__ ux, const int32_t *__restrict__ uid,
                                    const uint16_t *__restrict__ ufirst,
                                    const uint16_t *__restrict__ slot_idx, int64_t n_anchors, int P,
                                    const int64_t *__restrict__ cap_offsets, int32_t *keys,
                                    int32_t *vals) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_anchors;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = cap_offsets[k];
        const uint64_t mask = (uint64_t)(cap_offsets[k + 1] - base - 1);
        const int64_t lo = offsets[k];
        const uint16_t *sl = slot_idx + k * (int64_t)P;
        for (int p = 0; p < P; ++p) {
            const int r = sl[p];
            if (ufirst[lo + r] != p) continue;
            const int32_t x = ux[lo + r];
            uint64_t h = mix64((uint64_t)(int64_t)x) & mask;
            while (keys[base + h] != -1) h = (h + 1) & mask;
            keys[base + h] = x;
            vals[base + h] = uid[lo + r];
        }
    }
}

__global__ void lookup_kernel(const int64_t *__restrict__ u, const int64_t *__restrict__ x,
                              int64_t n, const int64_t *__restrict__ offsets,
                              const int32_t *__restrict__ ux, const int32_t *__restrict__ uid,
                              int32_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = offsets[u[i]], hi = offsets[u[i] + 1];
        const int64_t xv = x[i];
        int64_t a = lo, b = hi;
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if ((int64_t)ux[mid] < xv)
                a = mid + 1;
            else
                b = mid;
        }
        out[i] = (a < hi && (int64_t)ux[a] == xv) ? uid[a] : 0;
    }
}

}  // namespace wj

extern "C" int wj_join(const int64_t *queries, int64_t n_batch, int32_t arity,
                       const int32_t *walks, const int64_t *offsets, const int32_t *uniq_x,
                       const int32_t *uniq_id, const uint16_t *slot_idx, int32_t num_walks,
                       int32_t num_steps, int32_t max_unique, const uint64_t *table_keys,
                       int64_t table_len, int32_t *walk_nodes_out, int32_t *rpe_ids_out,
                       void *dense_out, int32_t dense_dtype, int64_t row_stride,
                       wj_stream_t stream) {
    using namespace wj;
    if (arity < 1 || arity > 4) {
        set_error("query arity %d outside the supported 1..4", arity);
        return arity < 1 ? WJ_ERR_ARG : WJ_ERR_UNSUPPORTED;
    }
    if (num_walks < 1 || num_steps < 1 || max_unique < 0) {
        set_error("bad store shape");
        return WJ_ERR_ARG;
    }
    if (n_batch == 0) return WJ_OK;
    JoinArgs g;
    g.queries = queries;
    g.n_batch = n_batch;
    g.A = arity;
    g.walks = walks;
    g.offsets = offsets;
    g.ux = uniq_x;
    g.uid = uniq_id;
    g.slot_idx = slot_idx;
    g.M = num_walks;
    g.W = num_steps + 1;
    g.P = num_walks * g.W;
    g.max_u = max_unique < 1 ? 1 : max_unique;
    g.tkeys = table_keys;
    g.tlen = table_len;
    g.cb = bits_for((uint64_t)num_walks);
    g.walk_nodes = walk_nodes_out;
    g.rpe_ids = rpe_ids_out;
    g.dense = dense_out;
    g.row_stride = row_stride;
    if (dense_out && row_stride < (int64_t)arity * g.W) {
        set_error("row_stride %lld < arity*(L+1)", (long long)row_stride);
        return WJ_ERR_ARG;
    }
    size_t base = 64 + (size_t)arity * g.max_u * 8 + (size_t)arity * (arity - 1) * g.max_u * 4 +
                  (size_t)g.P * 2 + 16;
    const size_t limit = 200 * 1024;
    g.stage_table = (dense_out && base + (size_t)table_len * 8 <= limit && table_len <= 8192) ? 1 : 0;
    const size_t smem = base + (g.stage_table ? (size_t)table_len * 8 : 0);
    if (smem > limit) {
        set_error("join needs %zu B of shared memory (arity %d, max_unique %d)", smem, arity,
                  max_unique);
        return WJ_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    int64_t blocks = n_batch;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    cudaError_t e = cudaSuccess;
#define WJ_LAUNCH_JOIN(T)                                                                     \
    do {                                                                                      \
        e = cudaFuncSetAttribute(join_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)smem);                                                  \
        if (e == cudaSuccess) join_kernel<T><<<(unsigned)blocks, 256, smem, s>>>(g);          \
    } while (0)
    switch (dense_dtype) {
        case WJ_F32: WJ_LAUNCH_JOIN(float); break;
        case WJ_F64: WJ_LAUNCH_JOIN(double); break;
        case WJ_BF16: WJ_LAUNCH_JOIN(__nv_bfloat16); break;
        case WJ_F16: WJ_LAUNCH_JOIN(__half); break;
        default:
            set_error("unknown dense dtype %d", dense_dtype);
            return WJ_ERR_ARG;
    }
#undef WJ_LAUNCH_JOIN
    if (e != cudaSuccess) {
        set_error("wj_join smem attribute: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return check_launch("wj_join");
}

extern "C" int wj_gather_rpe(const int32_t *rpe_ids, int64_t n_ids, const int32_t *table,
                             int64_t table_len, int32_t width, void *out, int32_t dtype,
                             int32_t *bad_flag, wj_stream_t stream) {
    using namespace wj;
    if (dtype < WJ_F32 || dtype > WJ_F16 || width < 1) {
        set_error("bad dtype/width");
        return WJ_ERR_ARG;
    }
    if (n_ids == 0) return WJ_OK;
    int64_t blocks = (n_ids + 255) / 256;
    if (blocks > sm_count() * 32) blocks = sm_count() * 32;
    gather_rpe_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        rpe_ids, n_ids, table, table_len, width, out, dtype, bad_flag);
    return check_launch("wj_gather_rpe");
}

extern "C" int wj_export_dicts(const int64_t *offsets, const int32_t *uniq_x,
                               const int32_t *uniq_id, const uint16_t *uniq_first,
                               const uint16_t *slot_idx, int64_t n_anchors, int32_t num_walks,
                               int32_t num_steps, const int64_t *cap_offsets, int32_t *dict_keys,
                               int32_t *dict_vals, wj_stream_t stream) {
    using namespace wj;
    if (n_anchors == 0) return WJ_OK;
    int64_t blocks = (n_anchors + 127) / 128;
    if (blocks > sm_count() * 32) blocks = sm_count() * 32;
    export_dicts_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(
        offsets, uniq_x, uniq_id, uniq_first, slot_idx, n_anchors, num_walks * (num_steps + 1),
        cap_offsets, dict_keys, dict_vals);
    return check_launch("wj_export_dicts");
}

extern "C" int wj_lookup(const int64_t *u, const int64_t *x, int64_t count,
                         const int64_t *offsets, const int32_t *uniq_x, const int32_t *uniq_id,
                         int32_t *out, wj_stream_t stream) {
    using namespace wj;
    if (count == 0) return WJ_OK;
    int64_t blocks = (count + 255) / 256;
    if (blocks > sm_count() * 32) blocks = sm_count() * 32;
    lookup_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(u, x, count, offsets, uniq_x,
                                                                      uniq_id, out);
    return check_launch("wj_lookup");
}
