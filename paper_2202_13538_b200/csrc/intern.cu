// Global interning of positional count vectors for sm_100a.
//
// Reference: _kernels.py:137-171 (intern_rows) scans every (anchor, node) row
// sequentially in (anchor ascending, first appearance) order and gives each
// new vector the next id -- 64% of the reference preprocess, all on one core.
// The ids equal 1 + rank of each distinct vector's FIRST occurrence in that
// order, which is an order-independent fact: phase 1 here inserts every entry
// into an open-addressing table keyed by the packed vector, keeping the
// minimum scan order (anchor << 16 | first position) with atomicMin; a CTA
// first folds its entries into a shared-memory table so the hot vectors (a
// handful of shapes cover most rows) cost one global atomic per CTA, not one
// per row.  Phase 2 (sort the few distinct vectors by that minimum) is host
// plumbing; phase 3 maps every entry to its id.
#include "common.cuh"

namespace wj {

constexpr int kSmemSlots = 2048;  // 32 KB of (key, order) per CTA
constexpr int kInternThreads = 512;
constexpr uint64_t kEmpty = 0ULL;  // a packed vector always has a nonzero count

__device__ __forceinline__ bool global_insert(uint64_t *keys, uint64_t *order, uint64_t mask,
                                              uint64_t key, uint64_t ord) {
    uint64_t h = mix64(key) & mask;
    for (uint64_t probes = 0; probes <= mask; ++probes) {
        unsigned long long prev = atomicCAS((unsigned long long *)&keys[h], kEmpty, key);
        if (prev == kEmpty || prev == key) {
            atomicMin((unsigned long long *)&order[h], (unsigned long long)ord);
            return true;
        }
        h = (h + 1) & mask;
    }
    return false;
}

__global__ void __launch_bounds__(kInternThreads) intern_insert_kernel(
    const uint64_t *__restrict__ ukey, const uint16_t *__restrict__ ufirst,
    const int64_t *__restrict__ offsets, int64_t n_anchors, int64_t anchor_base, uint64_t *gkeys,
    uint64_t *gorder, uint64_t gmask, int32_t *overflow) {
    __shared__ unsigned long long skeys[kSmemSlots];
    __shared__ unsigned long long sorder[kSmemSlots];
    for (int i = threadIdx.x; i < kSmemSlots; i += blockDim.x) {
        skeys[i] = kEmpty;
        sorder[i] = ~0ULL;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    for (int64_t k = (int64_t)blockIdx.x * nwarps + warp; k < n_anchors;
         k += (int64_t)gridDim.x * nwarps) {
        const int64_t lo = offsets[k], hi = offsets[k + 1];
        const uint64_t ahi = (uint64_t)(anchor_base + k) << 16;
        // four entries per lane in flight (the loads, not the table, bound
        // this pass), then inserted in entry order
        for (int64_t e0 = lo + lane; e0 < hi; e0 += 4 * 32) {
            uint64_t kv[4];
            uint16_t fv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t e = e0 + 32 * j;
                kv[j] = e < hi ? __ldg(ukey + e) : kEmpty;
                fv[j] = e < hi ? __ldg(ufirst + e) : (uint16_t)0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t key = kv[j];
                if (key == kEmpty) continue;
                const uint64_t ord = ahi | fv[j];
                uint32_t h = (uint32_t)(mix64(key) & (kSmemSlots - 1));
                bool done = false;
                for (int probes = 0; probes < 64; ++probes) {
                    // a slot only ever goes empty -> key, so a plain read that
                    // sees the key needs no atomic; the scan order only needs
                    // an atomic when it would lower it
                    unsigned long long prev = *reinterpret_cast<volatile unsigned long long *>(&skeys[h]);
                    if (prev == kEmpty) prev = atomicCAS(&skeys[h], kEmpty, key);
                    if (prev == kEmpty || prev == key) {
                        if ((unsigned long long)ord < *reinterpret_cast<volatile unsigned long long *>(&sorder[h]))
                            atomicMin(&sorder[h], (unsigned long long)ord);
                        done = true;
                        break;
                    }
                    h = (h + 1) & (kSmemSlots - 1);
                }
                if (!done && !global_insert(gkeys, gorder, gmask, key, ord)) *overflow = 1;
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSmemSlots; i += blockDim.x) {
        const uint64_t key = skeys[i];
        if (key != kEmpty && !global_insert(gkeys, gorder, gmask, key, sorder[i])) *overflow = 1;
    }
}

__global__ void intern_assign_kernel(const uint64_t *__restrict__ ukey, int64_t n,
                                     const uint64_t *__restrict__ gkeys,
                                     const int32_t *__restrict__ gids, uint64_t gmask,
                                     int32_t *__restrict__ uid) {
    // four entries per thread in flight (grid-strided, coalesced)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < n; e0 += 4 * stride) {
        uint64_t kv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t e = e0 + j * stride;
            kv[j] = e < n ? __ldg(ukey + e) : kEmpty;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t e = e0 + j * stride;
            if (e >= n) break;
            const uint64_t key = kv[j];
            uint64_t h = mix64(key) & gmask;
            int32_t id = 0;
            for (uint64_t probes = 0; probes <= gmask; ++probes) {
                const uint64_t k = __ldg(gkeys + h);
                if (k == key) {
                    id = __ldg(gids + h);
                    break;
                }
                if (k == kEmpty) break;
                h = (h + 1) & gmask;
            }
            uid[e] = id;
        }
    }
}

}  // namespace wj

extern "C" int wj_intern_insert(const uint64_t *uniq_key, const uint16_t *uniq_first,
                                const int64_t *offsets, int64_t n_anchors, int64_t anchor_base,
                                uint64_t *table_keys, uint64_t *table_order, int64_t table_cap,
                                int32_t *overflow_flag, wj_stream_t stream) {
    using namespace wj;
    if (table_cap < 2 || (table_cap & (table_cap - 1))) {
        set_error("table_cap must be a power of two >= 2");
        return WJ_ERR_ARG;
    }
    if (n_anchors == 0) return WJ_OK;
    const int nw = kInternThreads / 32;
    int64_t blocks = (n_anchors + nw - 1) / nw;
    const int64_t cap = (int64_t)sm_count() * 2;  // persistent: one smem table per CTA
    if (blocks > cap) blocks = cap;
    intern_insert_kernel<<<(unsigned)blocks, kInternThreads, 0, (cudaStream_t)stream>>>(
        uniq_key, uniq_first, offsets, n_anchors, anchor_base, table_keys, table_order,
        (uint64_t)(table_cap - 1), overflow_flag);
    return check_launch("wj_intern_insert");
}

extern "C" int wj_intern_assign(const uint64_t *uniq_key, int64_t n_entries,
                                const uint64_t *table_keys, const int32_t *table_ids,
                                int64_t table_cap, int32_t *uniq_id, wj_stream_t stream) {
    using namespace wj;
    if (table_cap < 2 || (table_cap & (table_cap - 1))) {
        set_error("table_cap must be a power of two >= 2");
        return WJ_ERR_ARG;
    }
    if (n_entries == 0) return WJ_OK;
    int64_t blocks = (n_entries + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 32;
    if (blocks > cap) blocks = cap;
    intern_assign_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        uniq_key, n_entries, table_keys, table_ids, (uint64_t)(table_cap - 1), uniq_id);
    return check_launch("wj_intern_assign");
}
