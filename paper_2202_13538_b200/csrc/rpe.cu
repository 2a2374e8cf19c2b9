// Per-anchor RPE index for sm_100a: sort + unique of each anchor's M*(L+1)
// walk landings in shared memory, one warp per anchor.
//
// Reference: _kernels.py:77-126 (count_distinct_all / fill_distinct_all) build
// a per-anchor hash table and list the distinct landings in first-appearance
// order with their positional count vectors.  Here each landing becomes the
// key (x << pbits) | p (p = flat slot, so the input is already in p order) and
// a stable warp-level LSD radix sort on the x bits (8-bit digits, ranks from
// __match_any_sync + popc) orders the slots by node id while keeping slot
// order inside equal ids.  A ballot/popc pass then marks segment heads: the
// head's p is the first appearance, a segmented 64-bit warp scan of
// 1 << (cb * (p % W)) yields the packed count vector, and every slot learns
// the index of its node in the sorted unique list (slot_idx).
#include "common.cuh"

namespace wj {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kRpeWarps = 8;

// Stable LSD radix sort of n keys (bits [lo_bit, lo_bit+nbits)) by one warp.
// Returns the buffer holding the result.  R: rounds of 32 keys (n <= 32 * R):
// each round's peer mask (__match_any_sync, on the ADU pipe that bounds this
// kernel) is computed once per pass, kept in a register, and reused by the
// histogram and the scatter.
template <typename K, int R>
__device__ __forceinline__ K *warp_radix_sort(K *a, K *b, int n, int lo_bit, int nbits,
                                              uint32_t *hist, int lane) {
    const unsigned lt = lanemask_lt();
    for (int shift = lo_bit; shift < lo_bit + nbits; shift += kRadixBits) {
        for (int i = lane; i < kBins; i += 32) hist[i] = 0;
        __syncwarp();
        unsigned peers[R];
        // histogram: one smem update per distinct digit per round
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r * 32 < n) {
                const int i = r * 32 + lane;
                const uint32_t d = i < n ? (uint32_t)((a[i] >> shift) & (kBins - 1)) : 0xFFFFu;
                peers[r] = __match_any_sync(kFull, d);
                if (i < n && (peers[r] & lt) == 0) hist[d] += __popc(peers[r]);
                __syncwarp();
            }
        }
        // exclusive scan over the bins, 8 per lane
        uint32_t v[kBins / 32];
        uint32_t s = 0;
#pragma unroll
        for (int q = 0; q < kBins / 32; ++q) {
            v[q] = hist[lane * (kBins / 32) + q];
            s += v[q];
        }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += t;
        }
        uint32_t run = incl - s;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kBins / 32; ++q) {
            hist[lane * (kBins / 32) + q] = run;
            run += v[q];
        }
        __syncwarp();
        // stable scatter: rank inside the round = peers before me
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r * 32 < n) {
                const int i = r * 32 + lane;
                const K key = i < n ? a[i] : (K)0;
                const uint32_t d = (uint32_t)((key >> shift) & (kBins - 1));
                uint32_t pos = 0;
                if (i < n) pos = hist[d] + __popc(peers[r] & lt);
                __syncwarp();
                if (i < n) {
                    b[pos] = key;
                    if ((peers[r] & lt) == 0) hist[d] += __popc(peers[r]);
                }
                __syncwarp();
            }
        }
        K *t = a;
        a = b;
        b = t;
    }
    return a;
}

struct RpeShape {
    int P;          // landings per anchor = M * W
    int W;          // L + 1
    int pbits;      // bits for p in [0, P)
    int xbits;      // bits for node ids in [0, n)
    int cb;         // bits per packed count (counts <= M)
    uint32_t wmag;  // magic for p / W
    uint32_t lmag;  // magic for t / L (L = W - 1)
    int pcap;       // P rounded up to a multiple of 32
};

template <typename K, bool FILL, int R>
__global__ void __launch_bounds__(kRpeWarps * 32, 3) rpe_kernel(
    const int32_t *__restrict__ walks, int64_t n_anchors, RpeShape sh,
    int32_t *__restrict__ counts_out, const int64_t *__restrict__ offsets,
    int32_t *__restrict__ uniq_x, uint64_t *__restrict__ uniq_key,
    uint16_t *__restrict__ uniq_first, uint16_t *__restrict__ slot_idx) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t per_warp = 2 * (size_t)sh.pcap * sizeof(K) + kBins * sizeof(uint32_t);
    unsigned char *mine = smem_raw + warp * per_warp;
    K *bufa = reinterpret_cast<K *>(mine);
    K *bufb = bufa + sh.pcap;
    uint32_t *hist = reinterpret_cast<uint32_t *>(bufb + sh.pcap);
    const int P = sh.P;
    const int M = sh.P / sh.W;
    const K pmask = ((K)1 << sh.pbits) - 1;
    const unsigned le = lanemask_le();

    for (int64_t k = (int64_t)blockIdx.x * kRpeWarps + warp; k < n_anchors;
         k += (int64_t)gridDim.x * kRpeWarps) {
        const int32_t *src = walks + k * (int64_t)P;
        // Every walk starts at the anchor: its M step-0 landings become ONE
        // key (x0, p = 0) of weight M, so the sort sees M*L + 1 keys, not
        // M*(L+1) (checked per anchor: walks given by a caller may differ)
        const int32_t x0 = __ldg(src);
        bool col0 = true;
        for (int j = lane; j < M; j += 32) col0 &= __ldg(src + (int64_t)j * sh.W) == x0;
        col0 = __all_sync(kFull, col0);
        const int n = col0 ? M * (sh.W - 1) + 1 : P;
        if (col0) {
            for (int t = lane; t < n; t += 32) {
                uint32_t p = 0;
                if (t > 0) {
                    const uint32_t tt = (uint32_t)t - 1, j = sh.W == 2 ? tt : fast_div16(tt, sh.lmag);
                    p = j * sh.W + 1 + (tt - j * (sh.W - 1));
                }
                bufa[t] = ((K)(uint32_t)__ldg(src + p) << sh.pbits) | (K)p;
            }
        } else {
            for (int i = lane; i < P; i += 32) bufa[i] = ((K)(uint32_t)__ldg(src + i) << sh.pbits) | (K)i;
        }
        __syncwarp();
        K *s = warp_radix_sort<K, R>(bufa, bufb, n, sh.pbits, sh.xbits, hist, lane);
        uint16_t *slot = reinterpret_cast<uint16_t *>(s == bufa ? bufb : bufa);

        int carry = 0;               // heads so far
        uint64_t scarry = 0;         // running inclusive sum of count increments
        uint64_t seg_base_carry = 0; // exclusive prefix at the open segment's head
        const int64_t off = FILL ? offsets[k] : 0;
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            const bool valid = i < n;
            const K key = valid ? s[i] : (K)0;
            const K x = key >> sh.pbits;
            const bool head = valid && (i == 0 || (s[i - 1] >> sh.pbits) != x);
            const unsigned hb = __ballot_sync(kFull, head);
            const int r = carry + __popc(hb & le) - 1;
            carry += __popc(hb);
            if (FILL) {
                const uint32_t p = (uint32_t)(key & pmask);
                const bool tail = valid && (i == n - 1 || (s[i + 1] >> sh.pbits) != x);
                const uint32_t step = p - fast_div16(p, sh.wmag) * sh.W;
                uint64_t v = valid ? (1ULL << (sh.cb * step)) : 0ULL;
                if (col0 && valid && p == 0) v = (uint64_t)M;  // the anchor's M step-0 landings
                // inclusive warp scan of v
                uint64_t incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t t = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += t;
                }
                incl += scarry;
                const uint64_t excl = incl - v;
                const unsigned hm = hb & le;
                const int hl = hm ? 31 - __clz(hm) : 0;
                const uint64_t hb_excl = __shfl_sync(kFull, excl, hl);
                const uint64_t seg_base = hm ? hb_excl : seg_base_carry;
                if (head) {
                    uniq_x[off + r] = (int32_t)x;
                    uniq_first[off + r] = (uint16_t)p;
                }
                if (tail) uniq_key[off + r] = incl - seg_base;
                if (valid) slot[p] = (uint16_t)r;
                const int last = hb ? 31 - __clz(hb) : 0;
                const uint64_t lb = __shfl_sync(kFull, excl, last);
                if (hb) seg_base_carry = lb;
                scarry = __shfl_sync(kFull, incl, 31);
            }
        }
        if (FILL) {
            __syncwarp();
            if (col0) {  // every step-0 slot holds the anchor: its unique index
                const uint16_t ru = slot[0];
                for (int j = lane + 1; j < M; j += 32) slot[j * sh.W] = ru;
                __syncwarp();
            }
            uint16_t *dst = slot_idx + k * (int64_t)P;
            for (int i = lane; i < P; i += 32) dst[i] = slot[i];
        } else if (lane == 0) {
            counts_out[k] = carry;
        }
        __syncwarp();
    }
}

// Count-only pass: the number of distinct landings of each anchor, which
// only sizes the fill pass, needs no sort -- each warp inserts its anchor's
// P landings into an open-addressing set in shared memory (atomicCAS, load
// <= 1/2) and counts the successful inserts.  Same result as the sort's
// segment-head count.
constexpr int kCountWarps = 8;

__global__ void __launch_bounds__(kCountWarps * 32) rpe_count_hash_kernel(
    const int32_t *__restrict__ walks, int64_t n_anchors, int P, int tbits, int32_t *__restrict__ counts_out) {
    extern __shared__ __align__(16) uint32_t tabs[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = 1 << tbits;
    uint32_t *tab = tabs + (size_t)warp * T;
    for (int64_t k = (int64_t)blockIdx.x * kCountWarps + warp; k < n_anchors;
         k += (int64_t)gridDim.x * kCountWarps) {
        for (int i = lane * 4; i < T; i += 128) *reinterpret_cast<uint4 *>(tab + i) = make_uint4(~0u, ~0u, ~0u, ~0u);
        __syncwarp();
        const int32_t *src = walks + k * (int64_t)P;
        // landings equal to the anchor (every walk's step 0, and returns) are
        // not inserted -- one same-address CAS per such slot serialised the
        // warp -- the anchor counts once (it is present: it is slot 0); the
        // next round's keys are loaded before this round's probes
        int count = 0;
        bool has_u = false;
        int32_t xn = lane < P ? __ldg(src + lane) : 0;
        const int32_t u = __shfl_sync(kFull, xn, 0);  // walk 0's step 0: the anchor (any value is exact)
        for (int base = 0; base < P; base += 32) {
            const int i = base + lane;
            const int32_t xs = xn;
            xn = i + 32 < P ? __ldg(src + i + 32) : 0;
            bool fresh = false;
            if (i < P) {
                if (xs == u) {
                    has_u = true;
                } else {
                    const uint32_t x = (uint32_t)xs;
                    uint32_t h = (x * 0x9E3779B1u) >> (32 - tbits);
                    while (true) {
                        const uint32_t old = atomicCAS(tab + h, ~0u, x);
                        if (old == ~0u) {
                            fresh = true;
                            break;
                        }
                        if (old == x) break;
                        h = (h + 1) & (T - 1);
                    }
                }
            }
            count += __popc(__ballot_sync(kFull, fresh));
        }
        count += __any_sync(kFull, has_u) ? 1 : 0;
        if (lane == 0) counts_out[k] = count;
        __syncwarp();
    }
}

static int make_shape(int32_t M, int32_t L, int64_t n_nodes, RpeShape &sh, bool &wide) {
    if (M < 1 || L < 1) {
        set_error("num_walks and num_steps must be >= 1");
        return WJ_ERR_ARG;
    }
    sh.W = L + 1;
    const int64_t P = (int64_t)M * sh.W;
    if (P > 4096) {
        set_error("M*(L+1) = %lld exceeds the 4096-landing envelope of the RPE kernel",
                  (long long)P);
        return WJ_ERR_UNSUPPORTED;
    }
    sh.P = (int)P;
    sh.pbits = bits_for((uint64_t)(P - 1));
    sh.xbits = bits_for((uint64_t)(n_nodes > 0 ? n_nodes - 1 : 0));
    sh.cb = bits_for((uint64_t)M);
    if (sh.cb * sh.W > 64) {
        set_error("(L+1)*bits(M) = %d exceeds the 64-bit packed count vector", sh.cb * sh.W);
        return WJ_ERR_UNSUPPORTED;
    }
    sh.wmag = div_magic((uint32_t)sh.W);
    sh.lmag = div_magic((uint32_t)L);
    sh.pcap = (sh.P + 31) / 32 * 32;
    wide = sh.pbits + sh.xbits > 32;
    return WJ_OK;
}

template <typename K, bool FILL, int R>
static int launch_rpe_r(const int32_t *walks, int64_t n_anchors, const RpeShape &sh,
                      int32_t *counts, const int64_t *offsets, int32_t *ux, uint64_t *ukey,
                      uint16_t *ufirst, uint16_t *slot, cudaStream_t s) {
    if (n_anchors == 0) return WJ_OK;
    const size_t per_warp = 2 * (size_t)sh.pcap * sizeof(K) + kBins * sizeof(uint32_t);
    const size_t smem = per_warp * kRpeWarps;
    auto kern = rpe_kernel<K, FILL, R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        set_error("rpe smem attribute (%zu B): %s", smem, cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRpeWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (n_anchors + kRpeWarps - 1) / kRpeWarps;
    const int64_t cap = (int64_t)sm_count() * per_sm * 16;
    if (blocks > cap) blocks = cap;
    kern<<<(unsigned)blocks, kRpeWarps * 32, smem, s>>>(walks, n_anchors, sh, counts, offsets, ux,
                                                         ukey, ufirst, slot);
    return check_launch(FILL ? "wj_rpe_fill" : "wj_rpe_count");
}

// rounds of 32 landings held in registers by the sort: 8, 16, 32, 64 or 128
template <typename K, bool FILL>
static int launch_rpe(const int32_t *walks, int64_t n_anchors, const RpeShape &sh, int32_t *counts,
                      const int64_t *offsets, int32_t *ux, uint64_t *ukey, uint16_t *ufirst, uint16_t *slot,
                      cudaStream_t s) {
    const int rounds = sh.pcap / 32;
    if (rounds <= 8) return launch_rpe_r<K, FILL, 8>(walks, n_anchors, sh, counts, offsets, ux, ukey, ufirst, slot, s);
    if (rounds <= 16) return launch_rpe_r<K, FILL, 16>(walks, n_anchors, sh, counts, offsets, ux, ukey, ufirst, slot, s);
    if (rounds <= 32) return launch_rpe_r<K, FILL, 32>(walks, n_anchors, sh, counts, offsets, ux, ukey, ufirst, slot, s);
    if (rounds <= 64) return launch_rpe_r<K, FILL, 64>(walks, n_anchors, sh, counts, offsets, ux, ukey, ufirst, slot, s);
    return launch_rpe_r<K, FILL, 128>(walks, n_anchors, sh, counts, offsets, ux, ukey, ufirst, slot, s);
}

}  // namespace wj

extern "C" int wj_rpe_count(const int32_t *walks, int64_t n_anchors, int32_t num_walks,
                            int32_t num_steps, int64_t n_nodes, int32_t *counts_out,
                            wj_stream_t stream) {
    using namespace wj;
    RpeShape sh;
    bool wide;
    int rc = make_shape(num_walks, num_steps, n_nodes, sh, wide);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (sh.P <= 2048) {  // hash-set count (table <= 16 KB per warp)
        if (n_anchors == 0) return WJ_OK;
        const int tbits = bits_for((uint64_t)(2 * sh.P - 1)) < 5 ? 5 : bits_for((uint64_t)(2 * sh.P - 1));
        const size_t smem = ((size_t)1 << tbits) * 4 * kCountWarps;
        cudaError_t e = cudaFuncSetAttribute(rpe_count_hash_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) {
            set_error("rpe count smem attribute: %s", cudaGetErrorString(e));
            return WJ_ERR_CUDA;
        }
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rpe_count_hash_kernel, kCountWarps * 32, smem);
        int64_t blocks = (n_anchors + kCountWarps - 1) / kCountWarps;
        const int64_t cap = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1) * 16;
        if (blocks > cap) blocks = cap;
        rpe_count_hash_kernel<<<(unsigned)blocks, kCountWarps * 32, smem, s>>>(walks, n_anchors, sh.P, tbits,
                                                                               counts_out);
        return check_launch("wj_rpe_count");
    }
    if (wide)
        return launch_rpe<uint64_t, false>(walks, n_anchors, sh, counts_out, nullptr, nullptr,
                                           nullptr, nullptr, nullptr, s);
    return launch_rpe<uint32_t, false>(walks, n_anchors, sh, counts_out, nullptr, nullptr, nullptr,
                                       nullptr, nullptr, s);
}

extern "C" int wj_rpe_fill(const int32_t *walks, int64_t n_anchors, int32_t num_walks,
                           int32_t num_steps, int64_t n_nodes, const int64_t *offsets,
                           int32_t *uniq_x, uint64_t *uniq_key, uint16_t *uniq_first,
                           uint16_t *slot_idx, wj_stream_t stream) {
    using namespace wj;
    RpeShape sh;
    bool wide;
    int rc = make_shape(num_walks, num_steps, n_nodes, sh, wide);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (wide)
        return launch_rpe<uint64_t, true>(walks, n_anchors, sh, nullptr, offsets, uniq_x, uniq_key,
                                          uniq_first, slot_idx, s);
    return launch_rpe<uint32_t, true>(walks, n_anchors, sh, nullptr, offsets, uniq_x, uniq_key,
                                      uniq_first, slot_idx, s);
}
