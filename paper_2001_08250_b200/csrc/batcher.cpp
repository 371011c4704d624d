// Read batcher: concurrent single-request callers of
// the read path — server::answer_share (server.cpp:115-135), called per client
// read from the session and link threads of node.cpp:263-266 / 528-530 — are
// coalesced into one device batch ("Read requests are batched and forwarded to
// the GPU").
//
// Host-side only; it calls the public device-pointer scan entry point
// xpir_answer_batch_dev. Three pinned staging batches rotate through
//   Idle -> Forming (callers join) -> Sealed (callers finish packing)
//        -> InFlight (H2D, scan, D2H queued on the batch's own stream)
//        -> Done (answers in pinned memory) -> Idle (last caller unpacked).
// The worker thread only seals batches (full, or max_wait_us after their first
// request) and queues them without waiting for the GPU; a completer thread waits
// on each batch's event in order and publishes it. So one batch can be scanned
// while the next one's transfers run and a third one forms. Callers copy their
// own query (and mask seed) in and their own answer out, in parallel on their
// threads; completion is a futex wait on the batch generation. Requests with and
// without a mask seed go to separate batches (pir::answer vs
// pir::mask_answer(pir::answer(..)), pir.cpp:29-39, 65-69).
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>

#include "../../include/xpir.h"

namespace xpir {
int set_error(int code, const std::string& msg);  // capi.cu: the thread's xpir_last_error()
void store_release_stream_scratch(xpir_store* st, cudaStream_t s);  // capi.cu
}

namespace {

enum class BState { Idle, Forming, Sealed, InFlight, Done };
constexpr int NBUF = 3;

// Batches in flight before a forming one waits (adaptive sealing). 1 (default):
// closed-loop 381k requests/s at 512 callers; 2 (XPIR_BATCHER_INFLIGHT=2): lower
// open-loop latency (250k/s offered: p50 290 vs 469 us) for 6% less peak (359k).
static size_t inflight_cap() {
    static const size_t cap = getenv("XPIR_BATCHER_INFLIGHT") ? size_t(atoi(getenv("XPIR_BATCHER_INFLIGHT"))) : 1;
    return cap;
}

struct BBuf {
    uint8_t* rows = nullptr;   // pinned
    uint8_t* seeds = nullptr;  // pinned
    uint8_t* out = nullptr;    // pinned
    uint8_t *d_rows = nullptr, *d_seeds = nullptr, *d_out = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done_ev = nullptr;
    BState state = BState::Idle;
    xpir_store* st = nullptr;  // the store this batch scans (fixed when it starts forming)
    bool masked = false;
    uint32_t count = 0;
    std::atomic<uint32_t> filled{0};  // callers done packing (no lock: the worker polls it after sealing)
    uint64_t gen = 0;
    std::chrono::steady_clock::time_point first;
    int rc = 0;
    std::string err;
    std::atomic<uint64_t> done_gen{0};
    std::atomic<uint32_t> readers{0};
};

}  // namespace

struct xpir_batcher {
    xpir_store* st = nullptr;
    int device = 0;
    uint32_t N = 0, S = 0, nb = 0, max_batch = 0, max_wait_us = 0;
    std::mutex mu;
    std::condition_variable cv_work;  // worker: a batch started / filled / packed, a slot freed
    std::condition_variable cv_done;  // completer: a batch went in flight
    std::condition_variable cv_free;  // callers: a staging batch became idle
    BBuf buf[NBUF];
    std::deque<BBuf*> inflight;  // in submission order
    std::atomic<bool> stop{false};
    bool completer_stop = false;
    std::atomic<uint32_t> active{0};  // callers inside xpir_batcher_answer (destroy waits for them)
    std::thread worker, completer;
    uint64_t n_requests = 0, n_batches = 0, max_seen = 0;

    void publish(BBuf* b, int rc, const std::string& err) {  // under mu
        b->rc = rc;
        b->err = err;
        b->readers.store(b->count, std::memory_order_relaxed);
        b->state = BState::Done;
        n_batches += 1;
        if (b->count > max_seen) max_seen = b->count;
        b->done_gen.store(b->gen, std::memory_order_release);
        b->done_gen.notify_all();
    }

    void run() {
        cudaSetDevice(device);
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
            BBuf* b = nullptr;
            cv_work.wait(lk, [&] {
                for (auto& x : buf)
                    if (x.state == BState::Forming) return true;
                return stop.load();
            });
            for (auto& x : buf)  // the oldest forming batch first
                if (x.state == BState::Forming && (!b || x.gen < b->gen)) b = &x;
            if (!b) break;  // stop, nothing pending
            // Adaptive sealing: while the device is idle a batch is sealed at once (a lone
            // caller pays no batching delay); while a batch is in flight it keeps forming
            // until it is full, max_wait_us have passed, or the device goes idle.
            const auto deadline = b->first + std::chrono::microseconds(max_wait_us);
            cv_work.wait_until(lk, deadline,
                               [&] { return stop.load() || b->count >= max_batch || inflight.size() < inflight_cap(); });
            b->state = BState::Sealed;  // no more joins
            const uint32_t B = b->count;
            const bool masked = b->masked;
            xpir_store* const bst = b->st;
            lk.unlock();
            // the joined callers are copying their rows in (a few microseconds)
            while (b->filled.load(std::memory_order_acquire) != B) std::this_thread::yield();
            lk.lock();
            b->state = BState::InFlight;
            lk.unlock();
            // queue H2D, scan, D2H on the batch's stream; do not wait
            int rc = XPIR_OK;
            std::string err;
            cudaError_t e = cudaMemcpyAsync(b->d_rows, b->rows, size_t(B) * nb, cudaMemcpyHostToDevice, b->stream);
            if (e == cudaSuccess && masked)
                e = cudaMemcpyAsync(b->d_seeds, b->seeds, size_t(B) * 32, cudaMemcpyHostToDevice, b->stream);
            if (e != cudaSuccess) {
                rc = XPIR_ECUDA;
                err = std::string("batcher H2D: ") + cudaGetErrorString(e);
            }
            if (!rc) {
                rc = xpir_answer_batch_dev(bst, b->d_rows, nb, N, B, masked ? b->d_seeds : nullptr, b->d_out,
                                           b->stream);
                if (rc) err = xpir_last_error();
            }
            if (!rc) {
                e = cudaMemcpyAsync(b->out, b->d_out, size_t(B) * S, cudaMemcpyDeviceToHost, b->stream);
                if (e == cudaSuccess) e = cudaEventRecord(b->done_ev, b->stream);
                if (e != cudaSuccess) {
                    rc = XPIR_ECUDA;
                    err = std::string("batcher D2H: ") + cudaGetErrorString(e);
                }
            }
            lk.lock();
            if (rc) {
                // earlier in-flight batches complete first; this one fails now
                publish(b, rc, err);
            } else {
                inflight.push_back(b);
                cv_done.notify_one();
            }
        }
        // drain: the completer publishes what is still in flight, then exits
        completer_stop = true;
        cv_done.notify_one();
    }

    void complete() {
        cudaSetDevice(device);
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
            cv_done.wait(lk, [&] { return !inflight.empty() || completer_stop; });
            if (inflight.empty()) break;
            BBuf* b = inflight.front();
            lk.unlock();
            const cudaError_t e = cudaEventSynchronize(b->done_ev);
            lk.lock();
            inflight.pop_front();
            publish(b, e == cudaSuccess ? XPIR_OK : XPIR_ECUDA,
                    e == cudaSuccess ? std::string() : std::string("batcher: ") + cudaGetErrorString(e));
            if (inflight.size() < inflight_cap()) cv_work.notify_one();  // a forming batch may go now
        }
    }
};

namespace {
int bfail(int code, const std::string& m) { return xpir::set_error(code, m); }

void free_bufs(xpir_batcher* b) {
    for (auto& x : b->buf) {
        if (x.stream) {
            cudaStreamSynchronize(x.stream);
            if (b->st) xpir::store_release_stream_scratch(b->st, x.stream);
        }
        for (uint8_t* p : {x.rows, x.seeds, x.out})
            if (p) cudaFreeHost(p);
        for (uint8_t* p : {x.d_rows, x.d_seeds, x.d_out})
            if (p) cudaFree(p);
        if (x.done_ev) cudaEventDestroy(x.done_ev);
        if (x.stream) cudaStreamDestroy(x.stream);
    }
}
}  // namespace

extern "C" {

static int batcher_create(xpir_store* st, int dev, uint32_t N, uint32_t S, uint32_t max_batch,
                          uint32_t max_wait_us, xpir_batcher** out) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    auto* b = new xpir_batcher;
    b->st = st;
    b->device = dev;
    b->N = N;
    b->S = S;
    b->nb = (N + 7) / 8;
    b->max_batch = max_batch;
    b->max_wait_us = max_wait_us;
    cudaError_t e = cudaSuccess;
    for (auto& x : b->buf) {
        auto H = [&](uint8_t** p, size_t n) {
            if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(p), n, cudaHostAllocPortable);
        };
        auto D = [&](uint8_t** p, size_t n) {
            if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(p), n);
        };
        H(&x.rows, size_t(max_batch) * b->nb + 16);
        H(&x.seeds, size_t(max_batch) * 32);
        H(&x.out, size_t(max_batch) * S + 16);
        D(&x.d_rows, size_t(max_batch) * b->nb + 16);
        D(&x.d_seeds, size_t(max_batch) * 32);
        D(&x.d_out, size_t(max_batch) * S + 16);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&x.stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x.done_ev, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        free_bufs(b);
        delete b;
        return bfail(e == cudaErrorMemoryAllocation ? XPIR_ENOMEM : XPIR_ECUDA,
                     std::string("batcher_create: ") + cudaGetErrorString(e));
    }
    b->worker = std::thread([b] { b->run(); });
    b->completer = std::thread([b] { b->complete(); });
    *out = b;
    return XPIR_OK;
}

int xpir_batcher_create(xpir_store* st, uint32_t max_batch, uint32_t max_wait_us, xpir_batcher** out) {
    if (!st || !out) return bfail(XPIR_EINVAL, "batcher_create: null argument");
    if (max_batch == 0) return bfail(XPIR_EINVAL, "batcher_create: max_batch must be positive");
    uint32_t N, S, lo, hi;
    uint64_t epoch;
    void* data = nullptr;
    int rc = xpir_store_info(st, &N, &S, &lo, &hi, &epoch, &data);
    if (rc) return rc;
    int dev = 0;
    cudaPointerAttributes pa{};
    if (data && cudaPointerGetAttributes(&pa, data) == cudaSuccess) dev = pa.device;
    return batcher_create(st, dev, N, S, max_batch, max_wait_us, out);
}

int xpir_batcher_create_geometry(int device, uint32_t N, uint32_t S, uint32_t max_batch, uint32_t max_wait_us,
                                 xpir_batcher** out) {
    if (!out) return bfail(XPIR_EINVAL, "batcher_create: null argument");
    if (max_batch == 0) return bfail(XPIR_EINVAL, "batcher_create: max_batch must be positive");
    if (N == 0 || S == 0) return bfail(XPIR_EINVAL, "batcher_create: empty geometry");
    return batcher_create(nullptr, device, N, S, max_batch, max_wait_us, out);
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
    b->completer.join();
    {
        // callers of the last batches may still be copying their answers out
        std::unique_lock<std::mutex> lk(b->mu);
        b->cv_free.wait(lk, [&] { return b->active.load() == 0; });
    }
    free_bufs(b);
    delete b;
    return XPIR_OK;
}

int xpir_batcher_answer(xpir_batcher* b, const uint8_t* q, uint32_t q_bits, const uint8_t* mask_seed,
                        uint8_t* out) {
    if (!b) return bfail(XPIR_EINVAL, "batcher_answer: null argument");
    if (!b->st) return bfail(XPIR_EINVAL, "batcher_answer: batcher created by geometry: use xpir_batcher_answer_on");
    return xpir_batcher_answer_on(b, b->st, q, q_bits, mask_seed, out);
}

int xpir_batcher_answer_on(xpir_batcher* b, xpir_store* st, const uint8_t* q, uint32_t q_bits,
                           const uint8_t* mask_seed, uint8_t* out) {
    if (!b || !st || !q || !out) return bfail(XPIR_EINVAL, "batcher_answer: null argument");
    if (q_bits != b->N) return bfail(XPIR_EINVAL, "answer: query length mismatch");  // pir.cpp:30-31
    if (st != b->st) {  // another snapshot of the same geometry (e.g. another sealed epoch)
        uint32_t N = 0, S = 0, lo = 0, hi = 0;
        int rc = xpir_store_info(st, &N, &S, &lo, &hi, nullptr, nullptr);
        if (rc) return rc;
        if (N != b->N || S != b->S || lo != 0 || hi != N)
            return bfail(XPIR_EINVAL, "batcher_answer: store geometry differs from the batcher's");
    }
    const bool masked = mask_seed != nullptr;
    std::unique_lock<std::mutex> lk(b->mu);
    if (b->stop) return bfail(XPIR_ESTATE, "batcher_answer: batcher is shutting down");
    b->active.fetch_add(1);
    struct Leave {  // the last one out lets a pending destroy proceed
        xpir_batcher* b;
        ~Leave() {
            // The decrement happens under mu: destroy evaluates its "active == 0"
            // predicate under mu too, so it cannot free `b` until this caller has
            // released the lock — the caller's last touch of `b`.
            std::lock_guard<std::mutex> g(b->mu);
            if (b->active.fetch_sub(1) == 1 && b->stop.load()) b->cv_free.notify_all();
        }
    };
    BBuf* buf = nullptr;
    for (;;) {
        if (b->stop) {
            lk.unlock();
            Leave leave{b};
            return bfail(XPIR_ESTATE, "batcher_answer: batcher is shutting down");
        }
        for (auto& x : b->buf)
            if (x.state == BState::Forming && x.masked == masked && x.st == st && x.count < b->max_batch) buf = &x;
        if (!buf)
            for (auto& x : b->buf)
                if (x.state == BState::Idle) {
                    buf = &x;
                    uint64_t g = 0;
                    for (auto& y : b->buf) g = y.gen > g ? y.gen : g;
                    x.state = BState::Forming;
                    x.st = st;
                    x.masked = masked;
                    x.count = 0;
                    x.filled.store(0, std::memory_order_relaxed);
                    x.gen = g + 1;
                    x.first = std::chrono::steady_clock::now();
                    break;
                }
        if (buf) break;
        b->cv_free.wait(lk);
    }
    Leave leave{b};  // (constructed after the join loop: the lock above is released below)
    const uint32_t k = buf->count++;
    const uint64_t gen = buf->gen;
    b->n_requests += 1;
    if (k == 0 || buf->count == b->max_batch) b->cv_work.notify_one();
    lk.unlock();
    std::memcpy(buf->rows + size_t(k) * b->nb, q, b->nb);
    if (masked) std::memcpy(buf->seeds + size_t(k) * 32, mask_seed, 32);
    buf->filled.fetch_add(1, std::memory_order_release);
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
        b->cv_work.notify_one();
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
