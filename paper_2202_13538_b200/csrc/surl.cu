// Reference store-file (SURL v1) records on the device.
//
// store._write_store (store.py:167-193) writes, after the header and table,
// one record per node: capacity (u32), walks[u] (M*(L+1) int32), then the
// node's dict_keys and dict_vals (capacity int32 each).  These kernels build
// (pack) or read (unpack) that record region as 4-byte words, one warp per
// node, with rec_off[u] = word offset of node u's record; the host adds the
// header, table and id map.
#include "common.cuh"

namespace wj {

__global__ void surl_pack_kernel(const int32_t *__restrict__ walks, int64_t n, int mw,
                                 const int64_t *__restrict__ doff, const int32_t *__restrict__ dk,
                                 const int32_t *__restrict__ dv, const int64_t *__restrict__ rec_off,
                                 int32_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (u >= n) return;
    const int64_t lo = doff[u];
    const int cap = (int)(doff[u + 1] - lo);
    int32_t *r = out + rec_off[u];
    if (lane == 0) r[0] = cap;
    const int32_t *w = walks + u * (int64_t)mw;
    for (int i = lane; i < mw; i += 32) r[1 + i] = w[i];
    for (int i = lane; i < cap; i += 32) {
        r[1 + mw + i] = dk[lo + i];
        r[1 + mw + cap + i] = dv[lo + i];
    }
}

__global__ void surl_unpack_kernel(const int32_t *__restrict__ in, int64_t n, int mw,
                                   const int64_t *__restrict__ rec_off, const int64_t *__restrict__ doff,
                                   int32_t *__restrict__ walks, int32_t *__restrict__ dk, int32_t *__restrict__ dv) {
    const int lane = threadIdx.x & 31;
    const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (u >= n) return;
    const int32_t *r = in + rec_off[u];
    const int64_t lo = doff[u];
    const int cap = (int)(doff[u + 1] - lo);
    int32_t *w = walks + u * (int64_t)mw;
    for (int i = lane; i < mw; i += 32) w[i] = r[1 + i];
    if (dk)
        for (int i = lane; i < cap; i += 32) {
            dk[lo + i] = r[1 + mw + i];
            dv[lo + i] = r[1 + mw + cap + i];
        }
}

}  // namespace wj

extern "C" int wj_surl_pack(const int32_t *walks, int64_t n_nodes, int32_t walk_words,
                            const int64_t *dict_offsets, const int32_t *dict_keys, const int32_t *dict_vals,
                            const int64_t *rec_off, int32_t *out, wj_stream_t stream) {
    using namespace wj;
    if (n_nodes < 0 || walk_words < 1) {
        set_error("bad shape");
        return WJ_ERR_ARG;
    }
    if (n_nodes == 0) return WJ_OK;
    surl_pack_kernel<<<(unsigned)((n_nodes * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        walks, n_nodes, walk_words, dict_offsets, dict_keys, dict_vals, rec_off, out);
    return check_launch("wj_surl_pack");
}

extern "C" int wj_surl_unpack(const int32_t *records, int64_t n_nodes, int32_t walk_words, const int64_t *rec_off,
                              const int64_t *dict_offsets, int32_t *walks_out, int32_t *dict_keys_out,
                              int32_t *dict_vals_out, wj_stream_t stream) {
    using namespace wj;
    if (n_nodes < 0 || walk_words < 1 || (dict_keys_out && !dict_vals_out)) {
        set_error("bad shape");
        return WJ_ERR_ARG;
    }
    if (n_nodes == 0) return WJ_OK;
    surl_unpack_kernel<<<(unsigned)((n_nodes * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        records, n_nodes, walk_words, rec_off, dict_offsets, walks_out, dict_keys_out, dict_vals_out);
    return check_launch("wj_surl_unpack");
}
