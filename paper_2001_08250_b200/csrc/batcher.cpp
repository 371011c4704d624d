// Read batcher: concurrent single-request callers of
// the read path — server::answer_share (server.cpp:115-135), called per client
// read from the session and link threads of node.cpp:263-266 / 528-530 — are
// coalesced into one device batch ("Read requests are batched and forwarded to
// the GPU").
//
// Host-side only; it calls the public scan entry point xpir_answer_batch.
// Two pinned staging batches alternate: while one is being scanned on the GPU,
// callers join the other. A caller copies its own query (and mask seed) into
// the forming batch's pinned rows and, when the batch is done, copies its own
// answer out, so packing and unpacking run on the callers' threads in parallel;
// the worker thread only seals a batch (full, or max_wait_us after its first
// request) and runs the scan. Requests with and without a mask seed go to
// separate batches (pir::answer vs pir::mask_answer(pir::answer(..)), pir.cpp:29-39, 65-69).
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include "../../include/xpir.h"

namespace xpir {
int set_error(int code, const std::string& msg);  // capi.cu: the thread's xpir_last_error()
}

namespace {

enum class BState { Idle, Forming, Sealed, Running, Done };

struct BBuf {
    uint8_t* rows = nullptr;
    uint8_t* seeds = nullptr;
    uint8_t* out = nullptr;
    BState state = BState::Idle;
    bool masked = false;
    uint32_t count = 0, filled = 0;
    uint64_t gen = 0;
    // completion without the mutex: the worker publishes rc/err, then stores the
    // batch generation (release) and notifies; callers wait on it (futex) and
    // count themselves out with `readers`
    std::atomic<uint64_t> done_gen{0};
    std::atomic<uint32_t> readers{0};
    std::chrono::steady_clock::time_point first;
    int rc = 0;
    std::string err;
};

}  // namespace

struct xpir_batcher {
    xpir_store* st = nullptr;
    uint32_t N = 0, S = 0, nb = 0, max_batch = 0, max_wait_us = 0;
    std::mutex mu;
    // Separate wake-up channels so a state change wakes only the threads that wait
    // for it (hundreds of callers may be blocked at once):
    std::condition_variable cv_work;     // worker: a batch started / filled / packed
    std::condition_variable cv_free;     // callers: a staging batch became idle
    BBuf buf[2];
    bool stop = false;
    std::thread worker;
    uint64_t n_requests = 0, n_batches = 0, max_seen = 0;

    void run() {
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
            BBuf* b = nullptr;
            cv_work.wait(lk, [&] {
                for (auto& x : buf)
                    if (x.state == BState::Forming) return true;
                return stop;
            });
            for (auto& x : buf)  // the older forming batch first
                if (x.state == BState::Forming && (!b || x.gen < b->gen)) b = &x;
            if (!b) return;  // stop, nothing pending
            const auto deadline = b->first + std::chrono::microseconds(max_wait_us);
            cv_work.wait_until(lk, deadline, [&] { return stop || b->count >= max_batch; });
            b->state = BState::Sealed;  // no more joins
            cv_work.wait(lk, [&] { return b->filled == b->count; });
            b->state = BState::Running;
            const uint32_t B = b->count;
            const bool masked = b->masked;
            lk.unlock();
            const int rc = xpir_answer_batch(st, b->rows, nb, N, B, masked ? b->seeds : nullptr, b->out);
            const std::string err = rc ? std::string(xpir_last_error()) : std::string();
            lk.lock();
            b->rc = rc;
            b->err = err;
            b->readers.store(B, std::memory_order_relaxed);
            b->state = BState::Done;
            n_batches += 1;
            if (B > max_seen) max_seen = B;
            b->done_gen.store(b->gen, std::memory_order_release);
            b->done_gen.notify_all();
        }
    }
};

namespace {
int bfail(int code, const std::string& m) { return xpir::set_error(code, m); }
}  // namespace

extern "C" {

int xpir_batcher_create(xpir_store* st, uint32_t max_batch, uint32_t max_wait_us, xpir_batcher** out) {
    if (!st || !out) return bfail(XPIR_EINVAL, "batcher_create: null argument");
    if (max_batch == 0) return bfail(XPIR_EINVAL, "batcher_create: max_batch must be positive");
    uint32_t N, S, lo, hi;
    uint64_t epoch;
    int rc = xpir_store_info(st, &N, &S, &lo, &hi, &epoch, nullptr);
    if (rc) return rc;
    auto* b = new xpir_batcher;
    b->st = st;
    b->N = N;
    b->S = S;
    b->nb = (N + 7) / 8;
    b->max_batch = max_batch;
    b->max_wait_us = max_wait_us;
    for (auto& x : b->buf) {
        cudaError_t e = cudaHostAlloc(&x.rows, size_t(max_batch) * b->nb + 16, cudaHostAllocPortable);
        if (e == cudaSuccess) e = cudaHostAlloc(&x.seeds, size_t(max_batch) * 32, cudaHostAllocPortable);
        if (e == cudaSuccess) e = cudaHostAlloc(&x.out, size_t(max_batch) * S + 16, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            for (auto& y : b->buf)
                for (uint8_t* p : {y.rows, y.seeds, y.out})
                    if (p) cudaFreeHost(p);
            delete b;
            return bfail(e == cudaErrorMemoryAllocation ? XPIR_ENOMEM : XPIR_ECUDA,
                         std::string("batcher_create: ") + cudaGetErrorString(e));
        }
    }
    b->worker = std::thread([b] { b->run(); });
    *out = b;
    return XPIR_OK;
}

int xpir_batcher_destroy(xpir_batcher* b) {
    if (!b) return XPIR_OK;
    {
        std::lock_guard<std::mutex> lk(b->mu);
        b->stop = true;
    }
    b->cv_work.notify_all();
    b->cv_free.notify_all();
    b->worker.join();
    for (auto& x : b->buf)
        for (uint8_t* p : {x.rows, x.seeds, x.out})
            if (p) cudaFreeHost(p);
    delete b;
    return XPIR_OK;
}

int xpir_batcher_answer(xpir_batcher* b, const uint8_t* q, uint32_t q_bits, const uint8_t* mask_seed,
                        uint8_t* out) {
    if (!b || !q || !out) return bfail(XPIR_EINVAL, "batcher_answer: null argument");
    if (q_bits != b->N) return bfail(XPIR_EINVAL, "answer: query length mismatch");  // pir.cpp:30-31
    const bool masked = mask_seed != nullptr;
    std::unique_lock<std::mutex> lk(b->mu);
    BBuf* buf = nullptr;
    for (;;) {
        if (b->stop) return bfail(XPIR_ESTATE, "batcher_answer: batcher is shutting down");
        for (auto& x : b->buf)
            if (x.state == BState::Forming && x.masked == masked && x.count < b->max_batch) buf = &x;
        if (!buf)
            for (auto& x : b->buf)
                if (x.state == BState::Idle) {
                    buf = &x;
                    uint64_t g = 0;
                    for (auto& y : b->buf) g = y.gen > g ? y.gen : g;
                    x.state = BState::Forming;
                    x.masked = masked;
                    x.count = x.filled = 0;
                    x.gen = g + 1;
                    x.first = std::chrono::steady_clock::now();
                    break;
                }
        if (buf) break;
        b->cv_free.wait(lk);
    }
    const uint32_t k = buf->count++;
    const uint64_t gen = buf->gen;
    b->n_requests += 1;
    if (k == 0 || buf->count == b->max_batch) b->cv_work.notify_one();
    lk.unlock();
    std::memcpy(buf->rows + size_t(k) * b->nb, q, b->nb);
    if (masked) std::memcpy(buf->seeds + size_t(k) * 32, mask_seed, 32);
    lk.lock();
    buf->filled += 1;
    if (buf->filled == buf->count && buf->state == BState::Sealed) b->cv_work.notify_one();
    lk.unlock();
    for (uint64_t d = buf->done_gen.load(std::memory_order_acquire); d != gen;
         d = buf->done_gen.load(std::memory_order_acquire))
        buf->done_gen.wait(d, std::memory_order_acquire);
    const int rc = buf->rc;
    const std::string err = rc ? buf->err : std::string();
    if (!rc) std::memcpy(out, buf->out + size_t(k) * b->S, b->S);
    if (buf->readers.fetch_sub(1, std::memory_order_acq_rel) == 1) {
        lk.lock();
        buf->state = BState::Idle;
        lk.unlock();
        b->cv_free.notify_all();
    }
    if (rc) return bfail(rc, err);
    return XPIR_OK;
}

int xpir_batcher_stats(xpir_batcher* b, uint64_t* requests, uint64_t* batches, uint64_t* max_batch_seen) {
    if (!b) return bfail(XPIR_EINVAL, "batcher_stats: null batcher");
    std::lock_guard<std::mutex> lk(b->mu);
    if (requests) *requests = b->n_requests;
    if (batches) *batches = b->n_batches;
    if (max_batch_seen) *max_batch_seen = b->max_seen;
    return XPIR_OK;
}

}  // extern "C"
