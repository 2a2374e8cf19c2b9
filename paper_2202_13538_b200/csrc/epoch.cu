// Native training-epoch loop: planner slots (pinned host ring, filled by the
// planner's producer thread) -> H2D on a copy stream one batch ahead -> the
// step executor (join+encode -> tail -> Adam, PDL-chained) -> the loss into
// the caller's buffer, for every batch of the epoch, with no Python between
// steps.  Replaces train()'s batch loop body (pipeline.py:287-310) when the
// planner and the step executor are both native; same batches, same
// kernels, same results as the per-step Python path (DeviceFeeder +
// TrainStep chain calls), which stays the reference for the tests.
//
// Ordering: a device slot is refilled only after the step that read it
// (its "done" event, waited on the copy stream); a planner slot is handed
// back once its copy has completed; before a step is launched the host
// checks its batch's copy event, so the training stream carries no copy or
// cross-stream wait and its PDL chain stays unbroken.
#include <cuda_runtime.h>

#include <cstdint>
#include <deque>
#include <vector>

#include "common.cuh"
#include "walkjoin_b200.h"

extern "C" int wj_train_epoch(wj_stepper *st, wj_planner *pl, const int64_t *ring_q, const int32_t *ring_g,
                              int32_t n_slots, int64_t cap, int32_t arity, int64_t *dev_q, int32_t *dev_g,
                              int32_t dev_depth, const float *dev_labels, float *loss_out, int64_t max_steps,
                              wj_stream_t stream, wj_stream_t copy_stream, int64_t *steps_done,
                              int64_t *h2d_bytes) {
    if (!st || !pl || !ring_q || !ring_g || n_slots < 2 || cap < 1 || arity < 1 || !dev_q || !dev_g ||
        dev_depth < 2 || !dev_labels || !loss_out || !steps_done) {
        wj::set_error("wj_train_epoch: bad arguments");
        return WJ_ERR_ARG;
    }
    *steps_done = 0;
    int64_t bytes = 0;
    const cudaStream_t s_main = (cudaStream_t)stream, s_copy = (cudaStream_t)copy_stream;
    const int64_t gstride = (2 + (int64_t)arity) * cap + 2;
    std::vector<cudaEvent_t> copied(dev_depth), done(dev_depth);
    std::vector<bool> used(dev_depth, false);
    for (int i = 0; i < dev_depth; ++i) {
        cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
    }
    struct Batch {
        int32_t slot, dslot;
        int64_t B, n_pos, G;
    };
    std::deque<Batch> unreleased;  // planner slots whose copies may still be in flight
    int rc = WJ_OK;
    int64_t k_issue = 0;

    auto release_done = [&](bool force_one) {
        while (!unreleased.empty()) {
            const Batch &b = unreleased.front();
            const cudaError_t q = force_one ? cudaEventSynchronize(copied[b.dslot]) : cudaEventQuery(copied[b.dslot]);
            if (q == cudaErrorNotReady) break;
            wj_planner_release(pl, b.slot);
            unreleased.pop_front();
            force_one = false;
        }
    };
    // next planner batch -> its device slot (copy stream); false at the end of the epoch
    auto issue = [&](Batch &out) -> bool {
        if (max_steps >= 0 && k_issue >= max_steps) return false;
        // keep at most n_slots - 1 planner slots outstanding so the producer can advance
        while ((int64_t)unreleased.size() >= n_slots - 1) release_done(true);
        int32_t s = -1;
        int64_t B = 0, n_pos = 0;
        if (wj_planner_acquire(pl, &s, &B, &n_pos) != WJ_OK) {
            rc = WJ_ERR_ARG;
            return false;
        }
        if (s < 0) return false;
        if (B > cap) {
            wj::set_error("wj_train_epoch: batch of %lld queries exceeds the ring capacity %lld", (long long)B,
                          (long long)cap);
            rc = WJ_ERR_ARG;
            return false;
        }
        const int32_t d = (int32_t)(k_issue % dev_depth);
        ++k_issue;
        if (used[d]) cudaStreamWaitEvent(s_copy, done[d], 0);  // the step that last read this slot
        const int32_t *g = ring_g + (int64_t)s * gstride;
        const int64_t G = g[0];
        cudaMemcpyAsync(dev_q + (int64_t)d * cap * arity, ring_q + (int64_t)s * cap * arity,
                        (size_t)B * arity * sizeof(int64_t), cudaMemcpyHostToDevice, s_copy);
        cudaMemcpyAsync(dev_g + (int64_t)d * gstride, g, (size_t)(G + 2 + B + G * arity) * sizeof(int32_t),
                        cudaMemcpyHostToDevice, s_copy);
        cudaEventRecord(copied[d], s_copy);
        bytes += (int64_t)B * arity * (int64_t)sizeof(int64_t) + (G + 2 + B + G * arity) * (int64_t)sizeof(int32_t);
        out = Batch{s, d, B, n_pos, G};
        unreleased.push_back(out);
        return true;
    };

    Batch cur{}, nxt{};
    bool have = issue(cur);
    int64_t k = 0;
    while (have && rc == WJ_OK) {
        const bool more = issue(nxt);  // the next batch's copy goes out before this step
        if (rc != WJ_OK) break;
        cudaEventSynchronize(copied[cur.dslot]);  // long complete: issued a step ago
        const int64_t d = cur.dslot;
        const int r = wj_stepper_run(st, dev_q + d * cap * arity, dev_labels + (cap - cur.n_pos), cur.B,
                                     dev_g + d * gstride, cur.G, loss_out + k, stream);
        if (r != WJ_OK) {
            rc = r;
            break;
        }
        cudaEventRecord(done[d], s_main);
        used[d] = true;
        ++k;
        release_done(false);
        cur = nxt;
        have = more;
    }
    // hand every planner slot back once its copy is done
    while (!unreleased.empty()) release_done(true);
    *steps_done = k;
    if (h2d_bytes) *h2d_bytes = bytes;
    for (int i = 0; i < dev_depth; ++i) {
        cudaEventDestroy(copied[i]);
        cudaEventDestroy(done[i]);
    }
    if (rc != WJ_OK) return rc;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        wj::set_error("wj_train_epoch: %s", cudaGetErrorString(e));
        return WJ_ERR_CUDA;
    }
    return WJ_OK;
}
