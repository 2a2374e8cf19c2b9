// Host-side training mini-batch planner: the reference's BFS batch growth
// and in-seed negative sampling (pipeline.py:77-166, driven per batch by
// train() at pipeline.py:292-304) restated in C++ on numpy's own PCG64
// stream, so that for the same Generator state it returns the reference's
// batches exactly -- seeds, BFS order, positives, negatives, labels -- and
// leaves the generator in the same state.
//
// numpy pieces restated (numpy 2.x, pinned by tests against numpy itself):
//  * PCG64 (128-bit LCG, XSL-RR output) with the buffered 32-bit half-word
//    (pcg64_next32: low half first, high half kept in uinteger/has_uint32);
//  * bounded draws: random_bounded_uint64 -> buffered_bounded_lemire_uint32
//    for ranges < 2^32 (Generator.integers with int64 output uses the same);
//  * Generator.choice(a, k, replace=False) for k <= 16: Floyd's algorithm
//    followed by a Fisher-Yates shuffle of the k picks.
//
// The reference spends ~7 ms of Python per batch here at the citation2 shape
// (SURVEY 8(f) f1), ~60x the device training step; this runs in tens of us.
// The planner is a caller-owned handle holding host memory (the node ->
// query index and the positive-tuple hash set); it touches no device state.
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <exception>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include <sys/mman.h>

#include "walkjoin_b200.h"

namespace wj {
void set_error(const char *fmt, ...);
}

namespace {

typedef unsigned __int128 u128;

// ------------------------------------------------------------- numpy PCG64
struct Pcg64 {
    u128 state, inc;
    int has_uint32;
    uint32_t uinteger;

    uint64_t next64() {
        const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
        state = state * mult + inc;
        uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
        unsigned r = (unsigned)(state >> 122);
        return (x >> r) | (x << ((64 - r) & 63));
    }
    uint32_t next32() {
        if (has_uint32) {
            has_uint32 = 0;
            return uinteger;
        }
        uint64_t v = next64();
        has_uint32 = 1;
        uinteger = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    // uniform in [0, rng] (inclusive), rng < 2^32 - 1: Lemire with rejection
    uint32_t lemire32(uint32_t rng) {
        const uint32_t excl = rng + 1;
        uint64_t m = (uint64_t)next32() * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t thresh = (UINT32_MAX - rng) % excl;
            while (left < thresh) {
                m = (uint64_t)next32() * excl;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
    // random_bounded_uint64(off=0, rng, use_masked=false), rng < 2^32
    uint64_t bounded(uint64_t rng) {
        if (rng == 0) return 0;
        if (rng == 0xFFFFFFFFULL) return next32();
        return lemire32((uint32_t)rng);
    }
};

inline uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Run fn(lo, hi) over [0, n) split across up to 16 host threads (small n:
// the calling thread alone).
template <typename F>
void parallel_for(int64_t n, F fn, unsigned reserve = 0) {
    // ``reserve``: host threads left to concurrent work of the caller
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    unsigned nt = std::max(1u, std::min(hc > reserve ? hc - reserve : 1u, 16u));
    if (n < (1 << 20)) nt = 1;
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(fn, n * t / nt, n * (t + 1) / nt);
    fn(0, n / nt);
    for (auto &x : th) x.join();
}

// Host array on transparent huge pages: the filter table and the per-node
// arrays are hundreds of MB at the citation2 shape and read at random, so
// 4 KB pages would add a TLB miss to every probe.
template <typename T>
struct HugeArray {
    T *ptr = nullptr;
    size_t n = 0;
    HugeArray() = default;
    HugeArray(const HugeArray &) = delete;
    HugeArray &operator=(const HugeArray &) = delete;
    ~HugeArray() { std::free(ptr); }
    void allocate(size_t count) {
        std::free(ptr);
        const size_t align = size_t(1) << 21;
        size_t bytes = ((count * sizeof(T) + align - 1) / align) * align;
        ptr = static_cast<T *>(std::aligned_alloc(align, bytes ? bytes : align));
        if (!ptr) throw std::bad_alloc();
        static const bool thp = !getenv("WJ_PLANNER_THP") || getenv("WJ_PLANNER_THP")[0] != '0';
        if (thp) madvise(ptr, bytes, MADV_HUGEPAGE);
        n = count;
    }
    void fill(const T &v) { std::fill(ptr, ptr + n, v); }
    T &operator[](size_t i) { return ptr[i]; }
    const T &operator[](size_t i) const { return ptr[i]; }
    T *data() { return ptr; }
    size_t size() const { return n; }
};

// ----------------------------------------------- canonical-tuple hash set
// Keys are the sorted tuple's node ids (< 2^31), 32 bits each: one 64-bit
// word for arity <= 2, two for arity 3-4.  Open addressing, power-of-two
// capacity, load <= 0.5; an all-ones word is the empty slot (no id has it).
struct Key2 {
    uint64_t a, b;
    bool operator==(const Key2 &o) const { return a == o.a && b == o.b; }
};

inline void sort_small(uint32_t *s, int n) {
    for (int i = 1; i < n; ++i) {
        uint32_t v = s[i];
        int j = i - 1;
        while (j >= 0 && s[j] > v) {
            s[j + 1] = s[j];
            --j;
        }
        s[j + 1] = v;
    }
}

template <int A>
inline uint64_t pack1(const int64_t *t) {
    if (A == 1) return (uint64_t)t[0];
    uint32_t x = (uint32_t)t[0], y = (uint32_t)t[1];
    return x < y ? ((uint64_t)x << 32) | y : ((uint64_t)y << 32) | x;
}

inline Key2 pack2(const int64_t *t, int arity) {
    uint32_t s[4] = {0, 0, 0, 0};
    for (int i = 0; i < arity; ++i) s[i] = (uint32_t)t[i];
    sort_small(s, arity);
    return Key2{((uint64_t)s[0] << 32) | s[1], ((uint64_t)s[2] << 32) | s[3]};
}

// multiplicative (Fibonacci) hashing: the table index is the top bits
inline uint64_t hash_of(uint64_t k) { return (k ^ (k >> 29)) * 0x9E3779B97F4A7C15ULL; }
inline uint64_t hash_of(const Key2 &k) { return (k.a * 0x9E3779B97F4A7C15ULL) ^ ((k.b ^ (k.b >> 31)) * 0xC2B2AE3D27D4EB4FULL); }
inline bool is_empty(uint64_t k) { return k == ~0ULL; }
inline bool is_empty(const Key2 &k) { return k.a == ~0ULL; }
inline void set_empty(uint64_t &k) { k = ~0ULL; }
inline void set_empty(Key2 &k) { k.a = k.b = ~0ULL; }

template <typename K>
struct TupleSet {
    HugeArray<K> slots;
    uint64_t mask = 0;
    int shift = 60;

    void reserve(int64_t n) {
        uint64_t cap = 16;
        shift = 60;
        while (cap < (uint64_t)(2 * n)) cap <<= 1, --shift;
        slots.allocate(cap);
        // all-ones bytes are the empty key; first touch in parallel
        char *base = reinterpret_cast<char *>(slots.data());
        parallel_for((int64_t)(cap * sizeof(K)),
                     [&](int64_t lo, int64_t hi) { std::memset(base + lo, 0xFF, (size_t)(hi - lo)); });
        mask = cap - 1;
    }
    uint64_t slot_of(const K &k) const { return hash_of(k) >> shift; }
    void insert(const K &k) {
        uint64_t h = slot_of(k);
        while (!is_empty(slots[h])) {
            if (slots[h] == k) return;
            h = (h + 1) & mask;
        }
        slots[h] = k;
    }
    // concurrent insert of 64-bit keys
    void insert_atomic(uint64_t k) {
        uint64_t h = slot_of(k);
        while (true) {
            uint64_t expected = ~0ULL;
            if (__atomic_compare_exchange_n(&slots[h], &expected, k, false, __ATOMIC_RELAXED, __ATOMIC_RELAXED) ||
                expected == k)
                return;
            h = (h + 1) & mask;
        }
    }
    bool contains(const K &k, uint64_t h) const {
        while (true) {
            const K &s = slots[h];
            if (s == k) return true;
            if (is_empty(s)) return false;
            h = (h + 1) & mask;
        }
    }
    void prefetch(uint64_t h) const { __builtin_prefetch(&slots[h]); }
};

}  // namespace

struct wj_planner {
    int32_t arity;
    int64_t n_pos, num_nodes;
    int32_t capacity, batch_size, k_neg;
    HugeArray<int64_t> pos;          // [n_pos, arity]
    HugeArray<int64_t> node_off;     // [num_nodes + 1] node -> range of qids
    HugeArray<int64_t> node_qids;    // qids per node, ascending
    std::vector<int64_t> nodes;      // sorted distinct nodes of the positives
    std::vector<int64_t> pool;       // optional fixed negative pool [n_pool, arity]
    TupleSet<uint64_t> filter1;  // arity <= 2
    TupleSet<Key2> filter2;      // arity 3-4
    // grouping of a batch's identical pairs by seed-local ids (the producer
    // thread): every node of a batch is in its seed set
    std::vector<int64_t> sset;
    std::vector<int32_t> sidx, pair_unit, gcnt, gfirst, gmem, gorder;
    Pcg64 rng;
    // per-batch scratch: generation stamps instead of clearing sets
    HugeArray<uint32_t> seed_stamp, batch_stamp;
    uint32_t gen = 0;
    std::vector<int64_t> seed_list, queue, batch, draws;
    std::vector<uint64_t> hashes, keys1;
    std::vector<Key2> keys2;
    // epoch producer (wj_planner_start_epoch): two threads fill a caller-owned
    // ring of batch slots in order -- the planner thread plans a batch into a
    // slot (slot_ready 0 -> 1, its seed set copied to slot_seeds), the
    // grouping thread groups it (1 -> 2: ready), so grouping batch b overlaps
    // planning batch b + 1; the consumer acquires a ready slot and releases
    // it (-> 0)
    struct Slot {
        int64_t n_queries, n_pos;  // n_queries -1: end of epoch; -2: error
    };
    std::thread worker, grouper;
    std::vector<std::vector<int64_t>> slot_seeds;
    std::atomic<int> stop{0};
    bool running = false;
    int64_t *ring_q = nullptr;
    float *ring_y = nullptr;
    int32_t *ring_g = nullptr;
    int32_t group_max = 4;  // unit size of wj_group_queries on the producer thread
    int32_t n_slots = 0;
    int64_t ring_cap = 0, consumed_batches = 0;
    std::unique_ptr<std::atomic<int>[]> slot_ready;
    std::vector<Slot> slot_meta;
    char worker_err[256] = "";

    ~wj_planner() {
        stop.store(1);
        if (worker.joinable()) worker.join();
        if (grouper.joinable()) grouper.join();
    }
};

extern "C" int wj_planner_create(const int64_t *positives, int64_t n_pos, int32_t arity,
                                 const int64_t *filter_tuples, int64_t n_filter, int64_t num_nodes,
                                 int32_t batch_capacity, int32_t batch_size, int32_t k_neg,
                                 const int64_t *neg_pool, int64_t n_pool, wj_planner **out) {
    if (!out || !positives || n_pos < 1 || arity < 1 || arity > 4 || num_nodes < 1 ||
        num_nodes > 0x7FFFFFFFLL || batch_capacity < 1 || batch_size < 1 || k_neg < 1 ||
        (n_filter > 0 && !filter_tuples) || (n_pool > 0 && !neg_pool)) {
        wj::set_error("wj_planner_create: bad arguments (n_pos=%lld arity=%d num_nodes=%lld)",
                      (long long)n_pos, arity, (long long)num_nodes);
        return arity > 4 ? WJ_ERR_UNSUPPORTED : WJ_ERR_ARG;
    }
    for (int64_t i = 0; i < n_pos * arity; ++i)
        if (positives[i] < 0 || positives[i] >= num_nodes) {
            wj::set_error("wj_planner_create: positive node id %lld out of range [0, %lld)",
                          (long long)positives[i], (long long)num_nodes);
            return WJ_ERR_ARG;
        }
    std::atomic<int64_t> bad{-1};
    parallel_for(n_filter * arity, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i)
            if (filter_tuples[i] < 0 || filter_tuples[i] >= num_nodes) bad.store(i);
    });
    if (bad.load() >= 0) {
        wj::set_error("wj_planner_create: filter node id %lld out of range", (long long)filter_tuples[bad.load()]);
        return WJ_ERR_ARG;
    }
    // WJ_PLANNER_TIMING=1: phase times of the build on stderr (profiling aid)
    static const bool timing = getenv("WJ_PLANNER_TIMING") != nullptr;
    auto t_start = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
        if (!timing) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "wj_planner_create %s: %.1f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t_start).count());
    };
    wj_planner *p = new (std::nothrow) wj_planner();
    if (!p) {
        wj::set_error("wj_planner_create: out of host memory");
        return WJ_ERR_ARG;
    }
    try {
        p->arity = arity;
        p->n_pos = n_pos;
        p->num_nodes = num_nodes;
        p->capacity = batch_capacity;
        p->batch_size = batch_size;
        p->k_neg = k_neg;
        p->pos.allocate(n_pos * arity);
        std::memcpy(p->pos.data(), positives, sizeof(int64_t) * n_pos * arity);
        if (n_pool > 0) p->pool.assign(neg_pool, neg_pool + n_pool * arity);
        // node -> qids (QueryOverlapIndex, pipeline.py:54-69): counting sort in
        // qid order keeps each node's list ascending, repeats included.  It
        // runs on its own thread while the filter set is built in parallel.
        std::exception_ptr index_err;
        std::thread index_thread([&]() {
            try {
                p->node_off.allocate(num_nodes + 1);
                p->node_off.fill(0);
                for (int64_t i = 0; i < n_pos * arity; ++i) p->node_off[positives[i] + 1]++;
                for (int64_t u = 0; u < num_nodes; ++u) {
                    if (p->node_off[u + 1] > 0) p->nodes.push_back(u);
                    p->node_off[u + 1] += p->node_off[u];
                }
                p->node_qids.allocate(n_pos * arity);
                std::vector<int64_t> fillp(p->node_off.data(), p->node_off.data() + num_nodes);
                for (int64_t q = 0; q < n_pos; ++q)
                    for (int a = 0; a < arity; ++a) p->node_qids[fillp[positives[q * arity + a]]++] = q;
            } catch (...) {
                index_err = std::current_exception();
            }
        });
        struct Joiner {
            std::thread &t;
            ~Joiner() {
                if (t.joinable()) t.join();
            }
        } joiner{index_thread};
        if (arity <= 2) {
            p->filter1.reserve(n_filter);
            lap("filter table allocate + clear");
            // lock-free parallel build (CAS on the 64-bit slots): the set holds
            // every positive of the split, ~30 M tuples at the citation2 shape
            // (each insert is a random DRAM access: the bucket of the tuple
            // 16 ahead is prefetched, for write)
            parallel_for(n_filter, [&](int64_t lo, int64_t hi) {
                auto key = [&](int64_t i) {
                    return arity == 1 ? pack1<1>(filter_tuples + i) : pack1<2>(filter_tuples + 2 * i);
                };
                constexpr int64_t D = 16;
                for (int64_t i = lo; i < hi; ++i) {
                    if (i + D < hi) __builtin_prefetch(&p->filter1.slots[p->filter1.slot_of(key(i + D))], 1);
                    p->filter1.insert_atomic(key(i));
                }
            }, 3);  // cores left to the query-index thread and the caller (device preprocess)
        } else {
            p->filter2.reserve(n_filter);
            for (int64_t i = 0; i < n_filter; ++i) p->filter2.insert(pack2(filter_tuples + i * arity, arity));
        }
        index_thread.join();
        if (index_err) std::rethrow_exception(index_err);
        lap("filter insert + query index");
        p->seed_stamp.allocate(num_nodes);
        p->seed_stamp.fill(0);
        p->batch_stamp.allocate(n_pos);
        p->batch_stamp.fill(0);
        p->rng = Pcg64{0, 1, 0, 0};
    } catch (...) {
        delete p;
        wj::set_error("wj_planner_create: out of host memory");
        return WJ_ERR_ARG;
    }
    *out = p;
    return WJ_OK;
}

extern "C" int wj_planner_destroy(wj_planner *p) {
    delete p;
    return WJ_OK;
}

extern "C" int wj_planner_set_rng(wj_planner *p, const uint64_t *words) {
    if (!p || !words) {
        wj::set_error("wj_planner_set_rng: null argument");
        return WJ_ERR_ARG;
    }
    if (p->running) {
        wj::set_error("wj_planner_set_rng: an epoch producer is running on this planner");
        return WJ_ERR_ARG;
    }
    p->rng.state = ((u128)words[0] << 64) | words[1];
    p->rng.inc = ((u128)words[2] << 64) | words[3];
    p->rng.has_uint32 = words[4] ? 1 : 0;
    p->rng.uinteger = (uint32_t)words[5];
    return WJ_OK;
}

extern "C" int wj_planner_get_rng(const wj_planner *p, uint64_t *words) {
    if (!p || !words) {
        wj::set_error("wj_planner_get_rng: null argument");
        return WJ_ERR_ARG;
    }
    if (p->running) {
        wj::set_error("wj_planner_get_rng: an epoch producer is running on this planner");
        return WJ_ERR_ARG;
    }
    words[0] = (uint64_t)(p->rng.state >> 64);
    words[1] = (uint64_t)p->rng.state;
    words[2] = (uint64_t)(p->rng.inc >> 64);
    words[3] = (uint64_t)p->rng.inc;
    words[4] = (uint64_t)p->rng.has_uint32;
    words[5] = (uint64_t)p->rng.uinteger;
    return WJ_OK;
}

namespace {

// sample_minibatch (pipeline.py:77-129): Floyd seeds, BFS over query-sharing
// neighbours until batch_size queries or batch_capacity seed nodes.
void grow_batch(wj_planner *p) {
    Pcg64 &rng = p->rng;
    if (++p->gen == 0) {  // stamp wrap: clear once every 2^32 batches
        p->seed_stamp.fill(0);
        p->batch_stamp.fill(0);
        p->gen = 1;
    }
    const uint32_t gen = p->gen;
    const int64_t pop = (int64_t)p->nodes.size();
    const int64_t k = std::min<int64_t>(std::min<int64_t>(16, p->capacity), pop);
    // Generator.choice(nodes, k, replace=False): Floyd + shuffle
    int64_t idx[16];
    for (int64_t j = pop - k; j < pop; ++j) {
        int64_t val = (int64_t)rng.bounded((uint64_t)j);
        bool seen = false;
        for (int64_t t = 0; t < j - (pop - k); ++t) seen |= (idx[t] == val);
        idx[j - pop + k] = seen ? j : val;
    }
    for (int64_t i = k - 1; i >= 1; --i) {
        int64_t j = (int64_t)rng.bounded((uint64_t)i);
        std::swap(idx[i], idx[j]);
    }
    p->seed_list.clear();
    p->queue.clear();
    p->batch.clear();
    for (int64_t i = 0; i < k; ++i) {
        int64_t s = p->nodes[idx[i]];
        if (p->seed_stamp[s] != gen) {
            p->seed_stamp[s] = gen;
            p->seed_list.push_back(s);
            p->queue.push_back(s);
        }
    }
    bool full = false;
    size_t head = 0;
    while (head < p->queue.size() && !full) {
        int64_t u = p->queue[head++];
        for (int64_t e = p->node_off[u]; e < p->node_off[u + 1]; ++e) {
            int64_t qid = p->node_qids[e];
            if (p->batch_stamp[qid] == gen) continue;
            if ((int64_t)p->batch.size() >= p->batch_size) {
                full = true;
                break;
            }
            p->batch_stamp[qid] = gen;
            p->batch.push_back(qid);
            for (int a = 0; a < p->arity; ++a) {
                int64_t w = p->pos[qid * p->arity + a];
                if (p->seed_stamp[w] != gen) {
                    if ((int64_t)p->seed_list.size() >= p->capacity) {
                        full = true;
                        break;
                    }
                    p->seed_stamp[w] = gen;
                    p->seed_list.push_back(w);
                    p->queue.push_back(w);
                }
            }
            if (full) break;
        }
    }
}

// sample_negatives (pipeline.py:132-166): chunks of uniform in-seed tuples,
// rows with a repeated node or in the positive set rejected, accepted rows
// kept in draw order.  Returns the number written, -1 on budget exhaustion.
// The generator is held in a local for the draw loop; each chunk's rows are
// hashed first with their buckets prefetched, then probed in draw order.
template <int A, typename K>
int64_t negatives_t(wj_planner *p, const TupleSet<K> &filter, std::vector<K> &keys, int64_t count,
                    int64_t *out) {
    Pcg64 rng = p->rng;
    const int64_t *seeds = p->seed_list.data();
    const uint32_t hi = (uint32_t)(p->seed_list.size() - 1);
    int64_t have = 0, budget = 1000 * count;
    while (have < count) {
        int64_t chunk = std::min<int64_t>(std::max<int64_t>(2 * (count - have), 64), budget);
        if (chunk <= 0) break;
        p->draws.resize(chunk * A);
        int64_t *d = p->draws.data();
        if (hi == 0) {
            for (int64_t i = 0; i < chunk * A; ++i) d[i] = seeds[0];
        } else {
            for (int64_t i = 0; i < chunk * A; ++i) d[i] = seeds[rng.lemire32(hi)];
        }
        budget -= chunk;
        keys.resize(chunk);
        p->hashes.resize(chunk);
        K *kk = keys.data();
        uint64_t *hh = p->hashes.data();
        // software pipeline: row r is hashed and its bucket prefetched D rows
        // before it is probed (the filter table is DRAM-resident at scale)
        constexpr int64_t D = 24;
        for (int64_t r = 0; r < chunk + D && have < count; ++r) {
            if (r < chunk) {
                const int64_t *row = d + r * A;
                bool distinct = true;
                for (int a = 0; a < A; ++a)
                    for (int b = a + 1; b < A; ++b) distinct &= row[a] != row[b];
                if (!distinct) {
                    hh[r] = ~0ULL;
                } else {
                    if constexpr (A <= 2) kk[r] = pack1<A>(row);
                    else kk[r] = pack2(row, A);
                    hh[r] = filter.slot_of(kk[r]);
                    filter.prefetch(hh[r]);
                }
            }
            const int64_t j = r - D;
            if (j < 0 || hh[j] == ~0ULL || filter.contains(kk[j], hh[j])) continue;
            for (int a = 0; a < A; ++a) out[have * A + a] = d[j * A + a];
            ++have;
        }
        if (budget <= 0 && have < count) {
            p->rng = rng;
            return -1;
        }
    }
    p->rng = rng;
    return have;
}

int64_t negatives(wj_planner *p, int64_t count, int64_t *out) {
    switch (p->arity) {
        case 1: return negatives_t<1>(p, p->filter1, p->keys1, count, out);
        case 2: return negatives_t<2>(p, p->filter1, p->keys1, count, out);
        case 3: return negatives_t<3>(p, p->filter2, p->keys2, count, out);
        default: return negatives_t<4>(p, p->filter2, p->keys2, count, out);
    }
}

}  // namespace

namespace {
// Per-thread scratch of wj_group_queries, reused across calls (a call is a
// few microseconds; allocating and clearing a table each time was 40 us).
struct GroupScratch {
    std::vector<Key2> keys;
    std::vector<uint32_t> stamp;
    std::vector<int32_t> gid, of, cnt, tstart, members, ustart, usize, ufirst, bucket;
    uint32_t gen = 0;
};

void emit_units(GroupScratch &sc, const int64_t *queries, int32_t arity, int64_t n, int32_t max_group,
                int32_t *groups_out) {
    // each tuple's queries in batch order, cut into units of <= max_group
    // members (the join+encode kernel runs a unit's members one after the
    // other in one CTA: a long unit would straggle), larger units first
    // (counting sort on the unit size, stable)
    const int32_t T = (int32_t)sc.cnt.size();
    sc.tstart.assign(T + 1, 0);
    for (int32_t t = 0; t < T; ++t) sc.tstart[t + 1] = sc.tstart[t] + sc.cnt[t];
    sc.members.resize(n);
    sc.cnt.assign(sc.tstart.begin(), sc.tstart.end() - 1);  // reuse as fill pointers
    for (int64_t i = 0; i < n; ++i) sc.members[sc.cnt[sc.of[i]]++] = (int32_t)i;
    const int32_t cap_m = max_group > 0 ? max_group : (int32_t)(n > 0 ? n : 1);
    sc.ufirst.clear();
    sc.usize.clear();
    int32_t big = 1;
    for (int32_t t = 0; t < T; ++t)
        for (int32_t a = sc.tstart[t]; a < sc.tstart[t + 1]; a += cap_m) {
            const int32_t sz = std::min(cap_m, sc.tstart[t + 1] - a);
            sc.ufirst.push_back(a);
            sc.usize.push_back(sz);
            big = std::max(big, sz);
        }
    const int32_t G = (int32_t)sc.usize.size();
    sc.bucket.assign(big + 2, 0);  // units per size, then start positions (largest first)
    for (int32_t g = 0; g < G; ++g) sc.bucket[big - sc.usize[g] + 1]++;
    for (int32_t b = 1; b <= big + 1; ++b) sc.bucket[b] += sc.bucket[b - 1];
    sc.ustart.resize(G);
    for (int32_t g = 0; g < G; ++g) sc.ustart[sc.bucket[big - sc.usize[g]]++] = g;
    int32_t *start = groups_out + 1, *order = groups_out + 2 + G;
    groups_out[0] = G;
    start[0] = 0;
    for (int32_t r = 0; r < G; ++r) {
        const int32_t g = sc.ustart[r];
        start[r + 1] = start[r] + sc.usize[g];
        for (int32_t k = 0; k < sc.usize[g]; ++k) order[start[r] + k] = sc.members[sc.ufirst[g] + k];
    }
    int32_t *tup = order + n;  // each unit's anchor tuple (one load for the kernel's unit metadata)
    for (int32_t r = 0; r < G; ++r)
        for (int a = 0; a < arity; ++a) tup[r * arity + a] = (int32_t)queries[(int64_t)order[start[r]] * arity + a];
}

}  // namespace

extern "C" int wj_group_queries(const int64_t *queries, int64_t n, int32_t arity, int32_t max_group,
                                int32_t *groups_out, int64_t *n_groups_out) {
    if (!queries || !groups_out || n < 0 || arity < 1 || arity > 4 || n > 0x3FFFFFFF || max_group < 0) {
        wj::set_error("wj_group_queries: bad arguments");
        return arity > 4 ? WJ_ERR_UNSUPPORTED : WJ_ERR_ARG;
    }
    static thread_local GroupScratch sc;
    // ordered tuple -> tuple id (first occurrence order): open addressing
    // with generation stamps instead of clearing the table
    uint64_t cap = 16;
    int cbits = 4;
    while (cap < (uint64_t)(2 * n)) cap <<= 1, ++cbits;
    if (sc.keys.size() < cap) {
        sc.keys.assign(cap, Key2{0, 0});
        sc.stamp.assign(cap, 0);
        sc.gid.assign(cap, 0);
        sc.gen = 0;
    }
    if (++sc.gen == 0) {
        std::fill(sc.stamp.begin(), sc.stamp.end(), 0);
        sc.gen = 1;
    }
    const uint32_t gen = sc.gen;
    const uint64_t mask = cap - 1;
    sc.of.resize(n);
    sc.cnt.clear();
    for (int64_t i = 0; i < n; ++i) {
        const int64_t *t = queries + i * arity;
        uint32_t v[4] = {0, 0, 0, 0};
        for (int a = 0; a < arity; ++a) v[a] = (uint32_t)t[a];
        const Key2 k{((uint64_t)v[0] << 32) | v[1], ((uint64_t)v[2] << 32) | v[3]};
        uint64_t h = hash_of(k) >> (64 - cbits);  // top bits: they mix every id
        while (sc.stamp[h] == gen && !(sc.keys[h] == k)) h = (h + 1) & mask;
        if (sc.stamp[h] != gen) {
            sc.stamp[h] = gen;
            sc.keys[h] = k;
            sc.gid[h] = (int32_t)sc.cnt.size();
            sc.cnt.push_back(0);
        }
        sc.of[i] = sc.gid[h];
        sc.cnt[sc.gid[h]]++;
    }
    emit_units(sc, queries, arity, n, max_group, groups_out);
    if (n_groups_out) *n_groups_out = groups_out[0];
    return WJ_OK;
}


namespace {

// One batch of train() (pipeline.py:292-304) into queries_out / labels_out;
// on error returns a WJ_ERR_* code with the message in err.
int plan_one(wj_planner *p, int64_t *queries_out, float *labels_out, int64_t cap, int64_t *n_queries_out,
             int64_t *n_pos_out, int64_t *n_seeds_out, char *err, size_t err_len) {
    grow_batch(p);
    const int A = p->arity;
    const int64_t nb = (int64_t)p->batch.size();
    if (n_seeds_out) *n_seeds_out = (int64_t)p->seed_list.size();
    *n_pos_out = nb;
    *n_queries_out = 0;
    if (nb == 0) return WJ_OK;  // train() stops the epoch on an empty batch
    const int64_t n_neg = (int64_t)p->k_neg * nb;
    if (nb + n_neg > cap) {
        snprintf(err, err_len, "wj_planner: output capacity %lld < %lld queries", (long long)cap,
                 (long long)(nb + n_neg));
        return WJ_ERR_ARG;
    }
    for (int64_t i = 0; i < nb; ++i)
        std::memcpy(queries_out + i * A, &p->pos[p->batch[i] * A], sizeof(int64_t) * A);
    int64_t got;
    if (!p->pool.empty()) {  // fixed negative pool (pipeline.py:298-300)
        const int64_t np_ = (int64_t)p->pool.size() / A;
        for (int64_t i = 0; i < n_neg; ++i) {
            int64_t pick = (int64_t)p->rng.bounded((uint64_t)(np_ - 1));
            std::memcpy(queries_out + (nb + i) * A, &p->pool[pick * A], sizeof(int64_t) * A);
        }
        got = n_neg;
    } else {
        if ((int64_t)p->seed_list.size() < A) {
            snprintf(err, err_len, "seed set of %lld nodes cannot host arity-%d negatives",
                     (long long)p->seed_list.size(), A);
            return WJ_ERR_ARG;
        }
        got = negatives(p, n_neg, queries_out + nb * A);
        if (got < 0) {
            snprintf(err, err_len, "negative sampling budget exhausted for %lld queries", (long long)n_neg);
            return WJ_ERR_ARG;
        }
    }
    if (labels_out)
        for (int64_t i = 0; i < nb + got; ++i) labels_out[i] = i < nb ? 1.0f : 0.0f;
    *n_queries_out = nb + got;
    return WJ_OK;
}

// Units of identical queries of a just-planned batch, on the producer
// thread.  Every node of the batch is in its seed set, so for pairs over a
// small seed set the tuple id comes from a dense (local a, local b) table
// instead of hashing the tuples; otherwise wj_group_queries.
void group_planned(wj_planner *p, const std::vector<int64_t> &seed_list, const int64_t *q, int64_t n, int32_t *out) {
    const int64_t ns = (int64_t)seed_list.size();
    if (p->arity != 2 || ns > 128 || !p->pool.empty()) {
        wj_group_queries(q, n, p->arity, p->group_max, out, nullptr);
        return;
    }
    static thread_local GroupScratch sc;
    int sbits = 4;
    while ((1ll << sbits) < 2 * ns + 2) ++sbits;
    const uint64_t smask = ((uint64_t)1 << sbits) - 1;
    p->sset.assign((size_t)1 << sbits, -1);
    p->sidx.assign((size_t)1 << sbits, 0);
    for (int64_t i = 0; i < ns; ++i) {
        const int64_t a = seed_list[i];
        uint64_t h = hash_of((uint64_t)a) >> (64 - sbits);
        while (p->sset[h] >= 0) h = (h + 1) & smask;
        p->sset[h] = a;
        p->sidx[h] = (int32_t)i;
    }
    auto local = [&](int64_t x) -> int32_t {
        uint64_t h = hash_of((uint64_t)x) >> (64 - sbits);
        while (p->sset[h] >= 0) {
            if (p->sset[h] == x) return p->sidx[h];
            h = (h + 1) & smask;
        }
        return -1;
    };
    p->pair_unit.assign((size_t)(ns * ns), -1);
    sc.of.resize(n);
    sc.cnt.clear();
    for (int64_t i = 0; i < n; ++i) {
        const int32_t la = local(q[2 * i]), lb = local(q[2 * i + 1]);
        if (la < 0 || lb < 0) {  // a positive cut off by the seed-capacity limit
            wj_group_queries(q, n, p->arity, p->group_max, out, nullptr);
            return;
        }
        int32_t &t = p->pair_unit[(size_t)la * ns + lb];
        if (t < 0) {
            t = (int32_t)sc.cnt.size();
            sc.cnt.push_back(0);
        }
        sc.of[i] = t;
        sc.cnt[t]++;
    }
    emit_units(sc, q, 2, n, p->group_max, out);
}

// The epoch loop of train() (pipeline.py:287-305): batches until the
// positives consumed reach len(positives) or a batch comes back empty.
void epoch_worker(wj_planner *p) {
    int64_t consumed = 0;
    for (int64_t b = 0;; ++b) {
        const int32_t s = (int32_t)(b % p->n_slots);
        while (p->slot_ready[s].load(std::memory_order_acquire) != 0) {
            if (p->stop.load(std::memory_order_relaxed)) return;
            std::this_thread::yield();
        }
        if (p->stop.load(std::memory_order_relaxed)) return;
        auto &m = p->slot_meta[s];
        if (consumed >= p->n_pos) {
            m.n_queries = -1;
            m.n_pos = 0;
        } else {
            int64_t nq = 0, npos = 0;
            int rc = plan_one(p, p->ring_q + (int64_t)s * p->ring_cap * p->arity, p->ring_y + (int64_t)s * p->ring_cap,
                              p->ring_cap, &nq, &npos, nullptr, p->worker_err, sizeof(p->worker_err));
            m.n_queries = rc != WJ_OK ? -2 : (npos == 0 ? -1 : nq);
            m.n_pos = npos;
            consumed += npos;
            if (m.n_queries > 0 && p->ring_g) p->slot_seeds[s] = p->seed_list;  // the grouper's copy
        }
        const bool last = m.n_queries < 0;
        p->slot_ready[s].store(1, std::memory_order_release);
        if (last) return;
    }
}

// the grouping stage of the epoch producer (see wj_planner)
void group_worker(wj_planner *p) {
    for (int64_t b = 0;; ++b) {
        const int32_t s = (int32_t)(b % p->n_slots);
        while (p->slot_ready[s].load(std::memory_order_acquire) != 1) {
            if (p->stop.load(std::memory_order_relaxed)) return;
            std::this_thread::yield();
        }
        const auto m = p->slot_meta[s];
        if (m.n_queries > 0 && p->ring_g)
            group_planned(p, p->slot_seeds[s], p->ring_q + (int64_t)s * p->ring_cap * p->arity, m.n_queries,
                          p->ring_g + (int64_t)s * ((2 + p->arity) * p->ring_cap + 2));
        p->slot_ready[s].store(2, std::memory_order_release);
        if (m.n_queries < 0) return;
    }
}

}  // namespace

extern "C" int wj_planner_next(wj_planner *p, int64_t *queries_out, float *labels_out, int64_t cap,
                               int64_t *n_queries_out, int64_t *n_pos_out, int64_t *n_seeds_out) {
    if (!p || !queries_out || !n_queries_out || !n_pos_out) {
        wj::set_error("wj_planner_next: null argument");
        return WJ_ERR_ARG;
    }
    if (p->running) {
        wj::set_error("wj_planner_next: an epoch producer is running on this planner");
        return WJ_ERR_ARG;
    }
    char err[256];
    int rc = plan_one(p, queries_out, labels_out, cap, n_queries_out, n_pos_out, n_seeds_out, err, sizeof(err));
    if (rc != WJ_OK) wj::set_error("%s", err);
    return rc;
}

extern "C" int wj_planner_start_epoch(wj_planner *p, int64_t *ring_queries, float *ring_labels, int32_t *ring_groups,
                                      int32_t n_slots, int64_t cap) {
    if (!p || !ring_queries || !ring_labels || n_slots < 1 || cap < 1) {
        wj::set_error("wj_planner_start_epoch: bad arguments");
        return WJ_ERR_ARG;
    }
    if (p->running) {
        wj::set_error("wj_planner_start_epoch: an epoch is already running");
        return WJ_ERR_ARG;
    }
    p->ring_q = ring_queries;
    p->ring_y = ring_labels;
    p->ring_g = ring_groups;
    p->n_slots = n_slots;
    p->ring_cap = cap;
    p->consumed_batches = 0;
    p->slot_ready.reset(new std::atomic<int>[n_slots]);
    for (int32_t i = 0; i < n_slots; ++i) p->slot_ready[i].store(0);
    p->slot_meta.assign(n_slots, {0, 0});
    p->slot_seeds.assign(n_slots, {});
    p->worker_err[0] = 0;
    p->stop.store(0);
    p->running = true;
    p->worker = std::thread(epoch_worker, p);
    p->grouper = std::thread(group_worker, p);
    return WJ_OK;
}

extern "C" int wj_planner_acquire(wj_planner *p, int32_t *slot_out, int64_t *n_queries_out, int64_t *n_pos_out) {
    if (!p || !slot_out || !n_queries_out || !n_pos_out || !p->running) {
        wj::set_error("wj_planner_acquire: no epoch running");
        return WJ_ERR_ARG;
    }
    const int32_t s = (int32_t)(p->consumed_batches % p->n_slots);
    while (p->slot_ready[s].load(std::memory_order_acquire) != 2) {
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    const auto m = p->slot_meta[s];
    if (m.n_queries < 0) {  // end of epoch or error: both producer threads have returned
        p->worker.join();
        p->grouper.join();
        p->running = false;
        *slot_out = -1;
        *n_queries_out = 0;
        *n_pos_out = 0;
        if (m.n_queries == -2) {
            wj::set_error("%s", p->worker_err);
            return WJ_ERR_ARG;
        }
        return WJ_OK;
    }
    ++p->consumed_batches;
    *slot_out = s;
    *n_queries_out = m.n_queries;
    *n_pos_out = m.n_pos;
    return WJ_OK;
}

extern "C" int wj_planner_release(wj_planner *p, int32_t slot) {
    if (!p || slot < 0 || slot >= p->n_slots) {
        wj::set_error("wj_planner_release: bad slot");
        return WJ_ERR_ARG;
    }
    p->slot_ready[slot].store(0, std::memory_order_release);
    return WJ_OK;
}

extern "C" int wj_planner_stop(wj_planner *p) {
    if (!p) return WJ_OK;
    p->stop.store(1);
    if (p->worker.joinable()) p->worker.join();
    if (p->grouper.joinable()) p->grouper.join();
    p->running = false;
    return WJ_OK;
}
