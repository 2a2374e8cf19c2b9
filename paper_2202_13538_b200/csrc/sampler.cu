// Walk sampler for sm_100a.
//
// Reference: _kernels.py:53-74 (sample_node_walks / sample_all_walks).  The
// reference draws sequentially from one splitmix64 stream per node; because a
// walk only consumes a draw at a node with degree > 0 and the CSR is always
// symmetric (graph.py:92-97), draw k of node u is mix64(S0(u) + (k+1)*G) with
// k = j*L + (i-1) for walk j, step i.  That makes every (node, walk) an
// independent unit: one thread per walk, 32 consecutive walks per warp (a
// warp covers one anchor's walks, as in the north-star design) and no shared
// state.  A mid-walk dead end (only possible for a hand-built non-symmetric
// CSR) breaks the counter identity; such anchors are flagged and re-sampled
// by one sequential device thread each, which is exactly the reference loop.
#include "common.cuh"

namespace wj {

template <typename IdxT>
__global__ void __launch_bounds__(256) sample_walks_kernel(
    const IdxT *__restrict__ idxptr, const int32_t *__restrict__ indices, int64_t lo,
    int64_t n_walks_total, int32_t M, int32_t L, uint64_t seed, int32_t *__restrict__ walks,
    uint8_t *__restrict__ fix_flags) {
    const int W = L + 1;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_walks_total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / M;  // anchor offset within [lo, hi)
        const int32_t j = (int32_t)(t - k * M);
        const int64_t u = lo + k;
        int32_t *out = walks + t * W;
        int64_t cur = u;
        out[0] = (int32_t)u;
        const IdxT b0 = __ldg(idxptr + u), e0 = __ldg(idxptr + u + 1);
        if (e0 == b0) {  // isolated anchor: repeat, no draws (_kernels.py:61-65)
            for (int i = 1; i <= L; ++i) out[i] = (int32_t)u;
            continue;
        }
        uint64_t state = node_stream_state(seed, u) + (uint64_t)j * (uint64_t)L * kGolden;
        IdxT beg = b0, deg = e0 - b0;
        bool dead = false;
#pragma unroll 4
        for (int i = 1; i <= L; ++i) {
            if (deg > 0) {
                state += kGolden;
                const uint64_t z = mix64(state);
                cur = __ldg(indices + beg + bounded(z, (uint32_t)deg));
                if (i < L) {
                    beg = __ldg(idxptr + cur);
                    deg = __ldg(idxptr + cur + 1) - beg;
                }
            } else {
                dead = true;  // reached a node without out-edges
            }
            out[i] = (int32_t)cur;
        }
        if (dead) fix_flags[k] = 1;
    }
}

// Sequential re-sample of flagged anchors: the literal reference loop.
template <typename IdxT>
__device__ uint64_t sample_node_sequential(const IdxT *__restrict__ idxptr,
                                           const int32_t *__restrict__ indices, int64_t u,
                                           int32_t M, int32_t L, uint64_t state, int32_t *out) {
    const int W = L + 1;
    for (int j = 0; j < M; ++j) {
        int64_t cur = u;
        out[j * W] = (int32_t)cur;
        for (int i = 1; i <= L; ++i) {
            const IdxT b = idxptr[cur];
            const IdxT deg = idxptr[cur + 1] - b;
            if (deg > 0) {
                state += kGolden;
                cur = indices[b + bounded(mix64(state), (uint32_t)deg)];
            }
            out[j * W + i] = (int32_t)cur;
        }
    }
    return state;
}

template <typename IdxT>
__global__ void fix_walks_kernel(const IdxT *__restrict__ idxptr,
                                 const int32_t *__restrict__ indices, int64_t lo,
                                 int64_t n_anchors, int32_t M, int32_t L, uint64_t seed,
                                 int32_t *__restrict__ walks, const uint8_t *__restrict__ fix_flags) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_anchors;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (!fix_flags[k]) continue;
        const int64_t u = lo + k;
        sample_node_sequential(idxptr, indices, u, M, L, node_stream_state(seed, u),
                               walks + k * (int64_t)M * (L + 1));
    }
}

// Single anchor with an explicit state (sampler.sample_walks): one warp,
// lanes run walks under the counter identity, lane 0 redoes the anchor
// sequentially if any lane met a dead end, and publishes the end state.
template <typename IdxT>
__global__ void sample_node_kernel(const IdxT *__restrict__ idxptr,
                                   const int32_t *__restrict__ indices, int64_t u, int32_t M,
                                   int32_t L, uint64_t state0, int32_t *__restrict__ out,
                                   uint64_t *__restrict__ end_state) {
    const int lane = threadIdx.x;
    const int W = L + 1;
    const IdxT b0 = idxptr[u], e0 = idxptr[u + 1];
    bool dead_any = false;
    if (e0 > b0) {
        for (int j = lane; j < M; j += 32) {
            uint64_t state = state0 + (uint64_t)j * (uint64_t)L * kGolden;
            int64_t cur = u;
            out[j * W] = (int32_t)u;
            for (int i = 1; i <= L; ++i) {
                const IdxT b = idxptr[cur];
                const IdxT deg = idxptr[cur + 1] - b;
                if (deg > 0) {
                    state += kGolden;
                    cur = indices[b + bounded(mix64(state), (uint32_t)deg)];
                } else {
                    dead_any = true;
                }
                out[j * W + i] = (int32_t)cur;
            }
        }
    } else {
        for (int j = lane; j < M; j += 32)
            for (int i = 0; i <= L; ++i) out[j * W + i] = (int32_t)u;
    }
    const bool redo = __any_sync(kFull, dead_any);
    __syncwarp();
    if (lane == 0) {
        if (redo) {
            *end_state = sample_node_sequential(idxptr, indices, u, M, L, state0, out);
        } else {
            *end_state = state0 + (e0 > b0 ? (uint64_t)M * (uint64_t)L * kGolden : 0ULL);
        }
    }
}

template <typename IdxT>
static int launch_sample(const IdxT *idxptr, const int32_t *indices, int64_t lo, int64_t hi,
                         int32_t M, int32_t L, uint64_t seed, int32_t *walks, uint8_t *flags,
                         cudaStream_t s) {
    const int64_t n_anchors = hi - lo;
    const int64_t total = n_anchors * (int64_t)M;
    if (total == 0) return WJ_OK;
    const int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    const int64_t cap = (int64_t)sm_count() * 8 * 64;  // grid-stride beyond 64 waves
    if (blocks > cap) blocks = cap;
    sample_walks_kernel<IdxT><<<(unsigned)blocks, threads, 0, s>>>(idxptr, indices, lo, total, M,
                                                                     L, seed, walks, flags);
    int rc = check_launch("wj_sample_walks");
    if (rc) return rc;
    int64_t fblocks = (n_anchors + 255) / 256;
    if (fblocks > sm_count() * 16) fblocks = sm_count() * 16;
    fix_walks_kernel<IdxT><<<(unsigned)fblocks, 256, 0, s>>>(idxptr, indices, lo, n_anchors, M, L,
                                                             seed, walks, flags);
    return check_launch("wj_sample_walks(fixup)");
}

}  // namespace wj

extern "C" int wj_sample_walks(const void *idxptr, int idxptr_bytes, const int32_t *indices,
                               int64_t n_nodes, int64_t lo, int64_t hi, int32_t num_walks,
                               int32_t num_steps, uint64_t seed, int32_t *walks_out,
                               uint8_t *fix_flags, wj_stream_t stream) {
    using namespace wj;
    if (num_walks < 1 || num_steps < 1) {
        set_error("num_walks and num_steps must be >= 1");
        return WJ_ERR_ARG;
    }
    if (lo < 0 || hi < lo || hi > n_nodes || n_nodes >= (1LL << 31)) {
        set_error("bad node range [%lld, %lld) for %lld nodes", (long long)lo, (long long)hi,
                  (long long)n_nodes);
        return WJ_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (idxptr_bytes == 4)
        return launch_sample((const int32_t *)idxptr, indices, lo, hi, num_walks, num_steps, seed,
                             walks_out, fix_flags, s);
    if (idxptr_bytes == 8)
        return launch_sample((const int64_t *)idxptr, indices, lo, hi, num_walks, num_steps, seed,
                             walks_out, fix_flags, s);
    set_error("idxptr_bytes must be 4 or 8");
    return WJ_ERR_ARG;
}

extern "C" int wj_sample_node_walks(const void *idxptr, int idxptr_bytes, const int32_t *indices,
                                    int64_t u, int32_t num_walks, int32_t num_steps,
                                    uint64_t state, int32_t *out, uint64_t *end_state_out,
                                    wj_stream_t stream) {
    using namespace wj;
    if (num_walks < 1 || num_steps < 1) {
        set_error("num_walks and num_steps must be >= 1");
        return WJ_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (idxptr_bytes == 4)
        sample_node_kernel<int32_t><<<1, 32, 0, s>>>((const int32_t *)idxptr, indices, u, num_walks,
                                                     num_steps, state, out, end_state_out);
    else if (idxptr_bytes == 8)
        sample_node_kernel<int64_t><<<1, 32, 0, s>>>((const int64_t *)idxptr, indices, u, num_walks,
                                                     num_steps, state, out, end_state_out);
    else {
        set_error("idxptr_bytes must be 4 or 8");
        return WJ_ERR_ARG;
    }
    return check_launch("wj_sample_node_walks");
}

namespace wj {

// ---------------------------------------------------------------------------
// Typed / metapath walks.  The reference has no typed sampler
// (SPEC.md:121-124 leaves "how edge types enter the walk sampler" open), so
// this is our definition, chosen so that its homogeneous special case IS the
// reference sampler: step i of walk j from anchor u must follow an edge of
// type metapath[(i-1) mod P] (a negative entry = any edge), chosen uniformly
// among the current node's edges of that type in CSR order with draw
// mix64(S0(u) + (j*L + i)*G) -- the reference's counter -- and a walk with no
// edge of the required type stays where it is for that step.  With metapath
// [-1] (or one type on every edge) and the reference's symmetric CSR this is
// bit-identical to wj_sample_walks.
//
// Layout: typed_indices holds each node's neighbours grouped by edge type
// (stable: CSR order inside a type), type_off[c*T + t] is the start of node
// c's type-t group, type_off[n*T] = 2E.  wj_typed_csr builds both.
struct Metapath {
    int8_t t[32];
    int32_t len;
};

template <typename IdxT>
__global__ void __launch_bounds__(256) sample_typed_kernel(
    const IdxT *__restrict__ idxptr, const int32_t *__restrict__ indices, const int64_t *__restrict__ type_off,
    const int32_t *__restrict__ typed_indices, int32_t T, Metapath mp, int64_t lo, int64_t n_walks_total,
    int32_t M, int32_t L, uint64_t seed, int32_t *__restrict__ walks) {
    const int W = L + 1;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_walks_total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / M;
        const int32_t j = (int32_t)(t - k * M);
        const int64_t u = lo + k;
        int32_t *out = walks + t * W;
        int64_t cur = u;
        out[0] = (int32_t)u;
        uint64_t state = node_stream_state(seed, u) + (uint64_t)j * (uint64_t)L * kGolden;
        for (int i = 1; i <= L; ++i) {
            state += kGolden;
            const int ty = mp.t[(i - 1) % mp.len];
            int64_t beg, deg;
            const int32_t *src;
            if (ty < 0) {
                beg = (int64_t)__ldg(idxptr + cur);
                deg = (int64_t)__ldg(idxptr + cur + 1) - beg;
                src = indices;
            } else {
                beg = __ldg(type_off + cur * T + ty);
                deg = __ldg(type_off + cur * T + ty + 1) - beg;
                src = typed_indices;
            }
            if (deg > 0) cur = __ldg(src + beg + bounded(mix64(state), (uint32_t)deg));
            out[i] = (int32_t)cur;
        }
    }
}

// One warp per node: per type, a ballot compaction over the node's edges in
// CSR order (stable grouping); lane 0 writes the node's T group starts.
template <typename IdxT>
__global__ void typed_csr_kernel(const IdxT *__restrict__ idxptr, const int32_t *__restrict__ indices,
                                 const uint8_t *__restrict__ etype, int64_t n, int32_t T,
                                 int64_t *__restrict__ type_off, int32_t *__restrict__ typed_indices) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < n; c += warps) {
        const int64_t b = (int64_t)idxptr[c], e = (int64_t)idxptr[c + 1];
        int64_t w = b;
        for (int ty = 0; ty < T; ++ty) {
            if (lane == 0) type_off[c * T + ty] = w;
            for (int64_t p = b; p < e; p += 32) {
                const int64_t q = p + lane;
                const bool hit = q < e && (int)__ldg(etype + q) == ty;
                const uint32_t m = __ballot_sync(kFull, hit);
                if (hit) typed_indices[w + __popc(m & ((1u << lane) - 1u))] = __ldg(indices + q);
                w += __popc(m);
            }
        }
        if (c == n - 1 && lane == 0) type_off[n * T] = e;
    }
}

template <typename IdxT>
static int launch_typed(const IdxT *idxptr, const int32_t *indices, const int64_t *type_off,
                        const int32_t *typed_indices, int32_t T, const Metapath &mp, int64_t lo, int64_t hi,
                        int32_t M, int32_t L, uint64_t seed, int32_t *walks, cudaStream_t s) {
    const int64_t total = (hi - lo) * (int64_t)M;
    if (total == 0) return WJ_OK;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8 * 64;
    if (blocks > cap) blocks = cap;
    sample_typed_kernel<IdxT><<<(unsigned)blocks, 256, 0, s>>>(idxptr, indices, type_off, typed_indices, T, mp,
                                                               lo, total, M, L, seed, walks);
    return check_launch("wj_sample_walks_typed");
}

template <typename IdxT>
static int launch_typed_csr(const IdxT *idxptr, const int32_t *indices, const uint8_t *etype, int64_t n,
                            int32_t T, int64_t *type_off, int32_t *typed_indices, cudaStream_t s) {
    if (n == 0) return WJ_OK;
    int64_t blocks = (n + 7) / 8;  // 8 warps per CTA, one node per warp
    if (blocks > (int64_t)sm_count() * 64) blocks = (int64_t)sm_count() * 64;
    typed_csr_kernel<IdxT><<<(unsigned)blocks, 256, 0, s>>>(idxptr, indices, etype, n, T, type_off, typed_indices);
    return check_launch("wj_typed_csr");
}

}  // namespace wj

extern "C" int wj_typed_csr(const void *idxptr, int idxptr_bytes, const int32_t *indices, const uint8_t *edge_types,
                            int64_t n_nodes, int32_t num_types, int64_t *type_off_out, int32_t *typed_indices_out,
                            wj_stream_t stream) {
    using namespace wj;
    if (num_types < 1 || num_types > 64 || n_nodes < 0 || n_nodes >= (1LL << 31)) {
        set_error("num_types must be in [1, 64] (got %d) and n_nodes < 2^31", num_types);
        return WJ_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (idxptr_bytes == 4)
        return launch_typed_csr((const int32_t *)idxptr, indices, edge_types, n_nodes, num_types, type_off_out,
                                typed_indices_out, s);
    if (idxptr_bytes == 8)
        return launch_typed_csr((const int64_t *)idxptr, indices, edge_types, n_nodes, num_types, type_off_out,
                                typed_indices_out, s);
    set_error("idxptr_bytes must be 4 or 8");
    return WJ_ERR_ARG;
}

extern "C" int wj_sample_walks_typed(const void *idxptr, int idxptr_bytes, const int32_t *indices,
                                     const int64_t *type_off, const int32_t *typed_indices, int32_t num_types,
                                     const int8_t *metapath, int32_t metapath_len, int64_t n_nodes, int64_t lo,
                                     int64_t hi, int32_t num_walks, int32_t num_steps, uint64_t seed,
                                     int32_t *walks_out, wj_stream_t stream) {
    using namespace wj;
    if (num_walks < 1 || num_steps < 1) {
        set_error("num_walks and num_steps must be >= 1");
        return WJ_ERR_ARG;
    }
    if (lo < 0 || hi < lo || hi > n_nodes || n_nodes >= (1LL << 31)) {
        set_error("bad node range [%lld, %lld) for %lld nodes", (long long)lo, (long long)hi, (long long)n_nodes);
        return WJ_ERR_ARG;
    }
    if (!metapath || metapath_len < 1 || metapath_len > 32) {
        set_error("metapath length must be in [1, 32] (got %d)", metapath_len);
        return WJ_ERR_ARG;
    }
    Metapath mp;
    mp.len = metapath_len;
    bool typed = false;
    for (int i = 0; i < 32; ++i) mp.t[i] = i < metapath_len ? metapath[i] : (int8_t)-1;
    for (int i = 0; i < metapath_len; ++i) {
        if (metapath[i] >= num_types) {
            set_error("metapath entry %d = %d is not an edge type (num_types %d)", i, (int)metapath[i], num_types);
            return WJ_ERR_ARG;
        }
        typed |= metapath[i] >= 0;
    }
    if (typed && (!type_off || num_types < 1)) {
        set_error("a typed metapath needs type_off / typed_indices (wj_typed_csr)");
        return WJ_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (idxptr_bytes == 4)
        return launch_typed((const int32_t *)idxptr, indices, type_off, typed_indices, num_types, mp, lo, hi,
                            num_walks, num_steps, seed, walks_out, s);
    if (idxptr_bytes == 8)
        return launch_typed((const int64_t *)idxptr, indices, type_off, typed_indices, num_types, mp, lo, hi,
                            num_walks, num_steps, seed, walks_out, s);
    set_error("idxptr_bytes must be 4 or 8");
    return WJ_ERR_ARG;
}
