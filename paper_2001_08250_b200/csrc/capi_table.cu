// C-ABI (include/xpir.h): the blocked cuckoo table — cuckoo::Table (cuckoo.hpp:37-84, cuckoo.cpp).
#include "capi_internal.cuh"

// ===========================================================================
// cuckoo table
// ===========================================================================

static const uint32_t DRAW_CAP = 1u << 18;  // DetRng draws staged per refill (2 MiB)

static void table_free_all(xpir_table* t) {
    cudaFree(t->d.used);
    cudaFree(t->d.beta1);
    cudaFree(t->d.beta2);
    cudaFree(t->d.stamp);
    cudaFree(t->d.origin);
    cudaFree(t->d.touched_mark);
    cudaFree(t->d.touched);
    cudaFree(t->d.mod_batch);
    cudaFree(t->d.chain_pre);
    cudaFree(t->d.fifo);
    cudaFree(t->d.draws);
    cudaFree(t->dstate);
    cudaFree(t->data);
    t->in_b1.release();
    t->in_b2.release();
    t->in_payload.release();
    t->in_reports.release();
    t->gather.release();
    t->chk.release();
    t->in_pack.release();
    t->stage.release();
    t->state_h.release();
    if (t->g1) cudaGraphExecDestroy(t->g1);
    t->g1 = nullptr;
    t->g1_stage.release();
    t->g1_dev.release();
    t->par.release();
    if (t->stream) cudaStreamDestroy(t->stream);
}

extern "C" {

int xpir_table_create(int device, uint32_t buckets, uint32_t depth, uint64_t capacity,
                      uint64_t item_size, const uint8_t seed[32], xpir_table** out) {
    return xpir_table_create_shard(device, buckets, depth, capacity, item_size, seed, 0, buckets, out);
}

int xpir_table_create_shard(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                            const uint8_t seed[32], uint32_t lo, uint32_t hi, xpir_table** out) {
    if (!out || !seed) return fail(XPIR_EINVAL, "table_create: null argument");
    if (buckets == 0 || depth == 0 || item_size == 0)  // cuckoo.cpp:15-16
        return fail(XPIR_EINVAL, "cuckoo: table dimensions must be positive");
    if (capacity == 0 || capacity > uint64_t(buckets) * depth)  // cuckoo.cpp:17-18
        return fail(XPIR_EINVAL, "cuckoo: capacity must be in [1, buckets*depth]");
    if (uint64_t(buckets) * depth >= (uint64_t(1) << 32))
        return fail(XPIR_EINVAL, "cuckoo: more than 2^32 slots");
    if (lo >= hi || hi > buckets) return fail(XPIR_EINVAL, "table_create: bad shard bucket range");
    int ndev = 0;
    XCK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(XPIR_EINVAL, "table_create: bad device");
    DeviceGuard g(device);
    auto* t = new xpir_table;
    t->device = device;
    std::memcpy(t->seed, seed, 32);
    t->d.buckets = buckets;
    t->d.depth = depth;
    t->d.capacity = capacity;
    t->d.item = item_size;
    const uint64_t slots = t->slots();
    uint64_t fc = 1;
    while (fc < 2 * slots + 1024) fc <<= 1;
    t->d.fifo_cap = fc;
    t->d.draw_cap = DRAW_CAP;
    cudaError_t e = cudaSuccess;
    auto M = [&](void** p, size_t n) {
        if (e == cudaSuccess) e = cudaMalloc(p, std::max<size_t>(n, 16));
        if (e == cudaSuccess) e = cudaMemset(*p, 0, std::max<size_t>(n, 16));
    };
    M(reinterpret_cast<void**>(&t->d.used), slots);
    M(reinterpret_cast<void**>(&t->d.beta1), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.beta2), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.stamp), 8 * slots);
    M(reinterpret_cast<void**>(&t->d.origin), 8 * slots);
    M(reinterpret_cast<void**>(&t->d.touched_mark), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.touched), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.mod_batch), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.chain_pre), 8 * 3 * 512);
    M(reinterpret_cast<void**>(&t->d.fifo), 8 * fc);
    M(reinterpret_cast<void**>(&t->d.draws), 8 * uint64_t(DRAW_CAP));
    M(reinterpret_cast<void**>(&t->dstate), sizeof(CuckooState));
    t->lo = lo;
    t->hi = hi;
    M(reinterpret_cast<void**>(&t->data), uint64_t(hi - lo) * depth * item_size);
    if (e == cudaSuccess) e = cudaMemset(t->d.fifo, 0xff, 8 * fc);  // -1: no entry
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking);
    // the memsets above ran on the legacy stream, which the table's non-blocking
    // stream does not wait for
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        table_free_all(t);
        delete t;
        return fail(e == cudaErrorMemoryAllocation ? XPIR_ENOMEM : XPIR_ECUDA,
                    std::string("table_create: ") + cudaGetErrorString(e));
    }
    t->h = CuckooState{};
    t->h.limit = ~0ull;
    // pinned state mirror allocated now: cudaHostAlloc inside a write can take milliseconds
    if (t->state_h.ensure(sizeof(CuckooState)) != cudaSuccess) {
        table_free_all(t);
        delete t;
        return fail(XPIR_ENOMEM, "table_create: pinned state mirror");
    }
    if (const char* ev = std::getenv("XPIR_CUCKOO_SEQUENTIAL")) t->parallel_prefix = ev[0] != '1';
    *out = t;
    return XPIR_OK;
}

int xpir_table_destroy(xpir_table* t) {
    if (!t) return XPIR_OK;
    DeviceGuard g(t->device);
    cudaStreamSynchronize(t->stream);
    table_free_all(t);
    delete t;
    return XPIR_OK;
}

}  // extern "C"

// Host round trip of the walk state after an asynchronous walk (one sync).
static int sync_state(xpir_table* t, cudaStream_t s) {
    if (!t->state_on_device) return XPIR_OK;
    XCK(t->state_h.ensure(sizeof(CuckooState)));
    XCK(cudaMemcpyAsync(t->state_h.p, t->dstate, sizeof(CuckooState), cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    std::memcpy(&t->h, t->state_h.p, sizeof(CuckooState));
    t->state_on_device = false;  // status 1 (draws) / 2 (FIFO ring full): the caller resumes the walk
    return XPIR_OK;
}

// The FIFO ring (stamp -> slot, replacing the reference's std::map, cuckoo.hpp:79)
// holds the stamps [fifo_head, next_stamp); live items that are never GC'd keep
// fifo_head back while stamps grow (capacity == slots with failing chains), so the
// ring doubles and is refilled from the live slots instead of failing.
static int grow_fifo(xpir_table* t, cudaStream_t s) {
    uint64_t cap = t->d.fifo_cap * 2;
    while (t->h.next_stamp + 4096 - t->h.fifo_head >= cap) cap *= 2;
    int64_t* ring = nullptr;
    XCK(cudaStreamSynchronize(s));
    XCK(cudaMalloc(&ring, cap * 8));
    cudaError_t e = launch_fifo_rebuild(t->d, ring, cap, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        cudaFree(ring);
        XCK(e);
    }
    cudaFree(t->d.fifo);
    t->d.fifo = ring;
    t->d.fifo_cap = cap;
    if (t->g1) {  // the single-write graph holds the old ring in its kernel parameters
        cudaGraphExecDestroy(t->g1);
        t->g1 = nullptr;
    }
    return XPIR_OK;
}

static int refill_draws(xpir_table* t, uint64_t need, cudaStream_t s) {
    if (t->h.rng_block + need > t->h.draw_base + t->h.draw_count) {
        // (re)fill the draw window starting at the next unconsumed nonce (draws are a
        // pure function of the nonce, so a window stays valid across rounds)
        t->h.draw_base = t->h.rng_block;
        t->h.draw_count = DRAW_CAP;
        XCK(launch_draws(t->seed, t->h.draw_base, DRAW_CAP, t->d.draws, s));
        count_launches(1);
    }
    return XPIR_OK;
}

// The host-driven walk loop from insert i: one launch per draw window.
static int walk_loop(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, uint64_t i, uint64_t n,
                     uint32_t* d_reports, cudaStream_t s) {
    while (i < n) {
        int rc = refill_draws(t, 1024, s);
        if (rc) return rc;
        XCK(cudaMemcpyAsync(t->dstate, &t->h, sizeof(CuckooState), cudaMemcpyHostToDevice, s));
        XCK(launch_cuckoo_walk(t->d, t->dstate, d_b1, d_b2, i, n, d_reports, s));
        count_launches(1);
        t->walked = true;
        XCK(cudaMemcpyAsync(&t->h, t->dstate, sizeof(CuckooState), cudaMemcpyDeviceToHost, s));
        XCK(cudaStreamSynchronize(s));
        if (t->h.status == 2) {  // the FIFO ring is full: grow it, resume at the same insert
            if (int rc = grow_fifo(t, s)) return rc;
        } else if (t->h.resume_at <= i && t->h.status != 1) {
            return fail(XPIR_ESTATE, "table_insert: walk made no progress");
        }
        i = t->h.resume_at;
        if (t->h.status == 1) t->h.draw_count = 0;  // force a refill
        t->h.status = 0;
    }
    return XPIR_OK;
}

// cuckoo.cpp:57-58 for device-resident inputs: the index of the first item whose
// beta1 or beta2 is >= buckets (n when all are in range). The walk kernels index
// the metadata and payload arrays with these values directly, so a bad one must
// never reach them.
static int beta_check(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, uint64_t n, cudaStream_t s,
                      uint64_t* n_ok) {
    XCK(t->chk.ensure(8));
    XCK(launch_beta_check(d_b1, d_b2, n, t->d.buckets, t->chk.as<unsigned long long>(), s));
    count_launches(1);
    unsigned long long first_bad = 0;
    XCK(cudaMemcpyAsync(&first_bad, t->chk.p, 8, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    *n_ok = first_bad < n ? first_bad : n;
    return XPIR_OK;
}

// Push the host mirror of the walk state to the device (pinned staging, async).
static int push_state(xpir_table* t, cudaStream_t s) {
    XCK(t->state_h.ensure(sizeof(CuckooState)));
    std::memcpy(t->state_h.p, &t->h, sizeof(CuckooState));
    XCK(cudaMemcpyAsync(t->dstate, t->state_h.p, sizeof(CuckooState), cudaMemcpyHostToDevice, s));
    XCK(t->state_h.release_after(s));
    return XPIR_OK;
}

// The rest of a batch started on device (parallel prefix + walk from its resume
// point, or the small asynchronous walk): one host round trip for the state;
// *n_ok = the first insert with a bucket out of range (n when none); a walk that
// paused for draws is finished on the host-driven path.
static int finish_walk(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, uint64_t n, uint32_t* d_reports,
                       cudaStream_t s, uint64_t* n_ok) {
    int rc = sync_state(t, s);
    if (rc) return rc;
    *n_ok = t->h.limit < n ? t->h.limit : n;
    t->h.limit = ~0ull;
    if (t->h.status == 1 || t->h.status == 2) {  // the walk paused (draws / FIFO ring): resume
        if (t->h.status == 2) {
            if (int rc2 = grow_fifo(t, s)) return rc2;
        } else {
            t->h.draw_count = 0;  // refill, then resume
        }
        t->h.status = 0;
        return walk_loop(t, d_b1, d_b2, t->h.resume_at, *n_ok, d_reports, s);
    }
    return push_state(t, s);  // the device copy stays authoritative
}

// The walk of a batch. checked: beta1/beta2 already validated (host inputs);
// otherwise the range check runs on device — inside the parallel-prefix kernel
// when that runs, else as its own kernel — and *n_ok is the first bad insert
// (n when none): only inserts before it are walked.
//  * n >= 64: the parallel prefix and the walk from its resume point are launched
//    back to back from and into the device state (no host round trip between);
//  * a batch small against the table (one apply_write) is walked with its draws
//    pre-staged and the state pushed asynchronously;
// with allow_async both leave t->state_on_device (the caller finishes the batch
// and calls finish_walk), else the batch is finished here.
static int walk_impl(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, uint64_t n, uint32_t* d_reports,
                     cudaStream_t s, bool allow_async, bool checked, uint64_t* n_ok) {
    int rc = sync_state(t, s);
    if (rc) return rc;
    *n_ok = n;
    t->h.n_touched = 0;
    t->h.walked = 0;
    t->h.limit = ~0ull;
    t->walked = false;
    const uint64_t slots = t->slots();
    if (t->parallel_prefix && n >= 64) {
        // K6a: the eviction-free, GC-free prefix of the round is placed in parallel
        // (exactly what the sequential walk would do); the walk continues on device
        // from the first insert that needs an eviction or a FIFO GC
        if ((rc = refill_draws(t, 1024, s)) || (rc = push_state(t, s))) return rc;
        XCK(cuckoo_parallel_prefix(t->d, t->dstate, d_b1, d_b2, n, d_reports, t->par, s));
        XCK(launch_cuckoo_walk(t->d, t->dstate, d_b1, d_b2, WALK_FROM_STATE, n, d_reports, s));
        count_launches(1);
        t->walked = true;  // the device flag says whether the walk had work
        t->state_on_device = true;
        t->max_touched = uint32_t(slots);
        if (!allow_async) return finish_walk(t, d_b1, d_b2, n, d_reports, s, n_ok);
        return XPIR_OK;
    }
    t->h.batch_id += 1;
    if (!checked) {
        if ((rc = beta_check(t, d_b1, d_b2, n, s, n_ok))) return rc;
        n = *n_ok;
    }
    if (allow_async && n * 256 < slots && n <= 64) {
        // worst case per insert: uniform(2) + 500 hops (cuckoo.cpp:86-120), with slack
        if ((rc = refill_draws(t, n * 1024 + 1024, s)) || (rc = push_state(t, s))) return rc;
        XCK(launch_cuckoo_walk(t->d, t->dstate, d_b1, d_b2, 0, n, d_reports, s));
        count_launches(1);
        t->walked = true;
        t->state_on_device = true;
        // a GC plus a chain of at most 500 moves per insert
        const uint64_t bound = n * 502;
        t->max_touched = uint32_t(bound < slots ? bound : slots);
        return XPIR_OK;
    }
    return walk_loop(t, d_b1, d_b2, 0, n, d_reports, s);
}

int table_walk_impl(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, uint64_t n, uint32_t* d_reports,
                    void* stream) {
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    uint64_t ok = n;
    int rc = walk_impl(t, d_b1, d_b2, n, d_reports, s, false, true, &ok);
    if (rc) return rc;
    if (!stream) XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

// Payload moves of the batch. With the state on device the touched count is read
// there (no host round trip); the staging buffer is NOT grown then — a batch that
// touched more slots than it holds makes the gather flag status 3 and both kernels
// skip, and the caller redoes them with the host count.
static int gather_impl(xpir_table* t, const ShardMap& m, cudaStream_t s) {
    // only eviction chains and FIFO GC (the walk kernels) move pre-existing items;
    // a round placed entirely by the parallel prefix has nothing to stage
    if (!t->walked || (!t->state_on_device && !t->h.walked)) return XPIR_OK;
    uint32_t cap;
    if (t->state_on_device) {
        if (t->max_touched < uint32_t(1) << 16) XCK(t->gather.ensure(uint64_t(t->max_touched) * t->d.item));
        cap = uint32_t(t->gather.cap / t->d.item);
    } else {
        XCK(t->gather.ensure(uint64_t(t->h.n_touched) * t->d.item));
        cap = t->h.n_touched;
    }
    t->d.gather = t->gather.as<uint8_t>();
    XCK(launch_cuckoo_gather_sharded(t->d, &t->h, t->lo, t->hi, t->data, m, s,
                                     t->state_on_device ? t->dstate : nullptr, t->max_touched, cap));
    count_launches(1);
    return XPIR_OK;
}

static int scatter_impl(xpir_table* t, const uint8_t* d_payload, cudaStream_t s) {
    XCK(launch_cuckoo_scatter_sharded(t->d, &t->h, t->lo, t->hi, t->data, d_payload, s,
                                      t->state_on_device ? t->dstate : nullptr, t->max_touched));
    count_launches(1);
    return XPIR_OK;
}

// Walk + payload gather/scatter of a whole (unsharded) table, one host round
// trip when the batch ran on device (the optional D2H of its reports into
// rep_host is queued before it). If the walk paused (draw window) or the gather
// staging was too small, the device-count gather/scatter were no-ops and the
// batch is finished on the host-driven path. On return the reports are in
// rep_host (if given). *n_ok: inserts applied (the first with a bucket out of
// range when unchecked).
static int insert_impl(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, const uint8_t* d_payload,
                       uint64_t n, uint32_t* d_reports, cudaStream_t s, uint8_t* rep_host, bool checked,
                       uint64_t* n_ok) {
    int rc = walk_impl(t, d_b1, d_b2, n, d_reports, s, true, checked, n_ok);
    if (rc) return rc;
    const ShardMap none{};
    bool done = false;
    if (t->state_on_device) {
        if ((rc = gather_impl(t, none, s)) || (rc = scatter_impl(t, d_payload, s))) return rc;
        if (rep_host && d_reports && *n_ok) XCK(cudaMemcpyAsync(rep_host, d_reports, 16 * *n_ok,
                                                                cudaMemcpyDeviceToHost, s));
        if ((rc = sync_state(t, s))) return rc;
        const uint32_t status = t->h.status;
        *n_ok = t->h.limit < *n_ok ? t->h.limit : *n_ok;
        t->h.limit = ~0ull;
        if (status == 0) {
            done = true;
        } else if (status == 1 || status == 2) {  // the walk paused (draws / FIFO ring): resume it
            t->h.status = 0;
            if (status == 2) {
                if ((rc = grow_fifo(t, s))) return rc;
            } else {
                t->h.draw_count = 0;
            }
            if ((rc = walk_loop(t, d_b1, d_b2, t->h.resume_at, *n_ok, d_reports, s))) return rc;
        } else {  // 3: gather staging too small; the walk is complete
            t->h.status = 0;
        }
        if ((rc = push_state(t, s))) return rc;  // the device copy stays authoritative
    }
    if (!done) {
        if ((rc = gather_impl(t, none, s)) || (rc = scatter_impl(t, d_payload, s))) return rc;
        if (rep_host && d_reports && *n_ok) {
            XCK(cudaMemcpyAsync(rep_host, d_reports, 16 * *n_ok, cudaMemcpyDeviceToHost, s));
            XCK(cudaStreamSynchronize(s));
        }
    }
    return XPIR_OK;
}

extern "C" {

int xpir_table_insert_batch_dev(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2,
                                const uint8_t* d_payload, uint64_t n, uint32_t* d_reports,
                                void* stream) {
    if (!t) return fail(XPIR_EINVAL, "table_insert: null table");
    if (n == 0) return XPIR_OK;
    if (!d_b1 || !d_b2 || !d_payload) return fail(XPIR_EINVAL, "table_insert: null buffer");
    if (t->sharded())
        return fail(XPIR_EINVAL, "table_insert: payload shard: use insert_walk + apply_gather (all shards) + apply_scatter");
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    // items before the first bad one are inserted, as a loop of Table::insert calls would
    uint64_t ok = n;
    int rc = insert_impl(t, d_b1, d_b2, d_payload, n, d_reports, s, nullptr, false, &ok);
    if (rc) return rc;
    if (!stream) XCK(cudaStreamSynchronize(s));
    if (ok < n) return fail(XPIR_EINVAL, "cuckoo: bucket index out of range");
    return XPIR_OK;
}

int xpir_table_insert_batch_async(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2,
                                  const uint8_t* d_payload, uint64_t n, uint32_t* d_reports, void* stream,
                                  void* prefix_done) {
    if (!t) return fail(XPIR_EINVAL, "table_insert: null table");
    if (!d_b1 || !d_b2 || !d_payload || !stream) return fail(XPIR_EINVAL, "table_insert_async: null argument");
    if (t->sharded()) return fail(XPIR_EINVAL, "table_insert_async: whole tables only");
    if (t->state_on_device || t->async_pending)
        return fail(XPIR_ESTATE, "table_insert_async: finish the previous batch first");
    if (n == 0) return XPIR_OK;
    DeviceGuard g(t->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // everything from and into the device state: capturable in a CUDA graph
    XCK(cuckoo_parallel_prefix(t->d, t->dstate, d_b1, d_b2, n, d_reports, t->par, s));
    if (prefix_done) XCK(cudaEventRecord(static_cast<cudaEvent_t>(prefix_done), s));
    XCK(launch_cuckoo_walk(t->d, t->dstate, d_b1, d_b2, WALK_FROM_STATE, n, d_reports, s));
    count_launches(1);
    t->walked = true;
    t->state_on_device = true;
    t->max_touched = uint32_t(t->slots());
    const ShardMap none{};
    int rc = gather_impl(t, none, s);
    if (!rc) rc = scatter_impl(t, d_payload, s);
    if (rc) return rc;
    t->async_pending = true;
    t->async = {d_b1, d_b2, d_payload, d_reports, n, s};
    return XPIR_OK;
}

int xpir_table_finish(xpir_table* t, uint64_t* n_applied) {
    if (!t) return fail(XPIR_EINVAL, "table_finish: null table");
    if (!t->async_pending) {
        if (n_applied) *n_applied = 0;
        return XPIR_OK;
    }
    DeviceGuard g(t->device);
    const auto a = t->async;
    t->async_pending = false;
    cudaStream_t s = a.s;
    int rc = sync_state(t, s);
    if (rc) return rc;
    const uint32_t status = t->h.status;
    uint64_t ok = t->h.limit < a.n ? t->h.limit : a.n;
    t->h.limit = ~0ull;
    t->h.status = 0;
    if (status != 0) {
        if (status == 1 || status == 2) {  // the walk paused (draws / FIFO ring): resume it
            if (status == 2) {
                if ((rc = grow_fifo(t, s))) return rc;
            } else {
                t->h.draw_count = 0;
            }
            if ((rc = walk_loop(t, a.b1, a.b2, t->h.resume_at, ok, a.reports, s))) return rc;
        }
        const ShardMap none{};
        if ((rc = gather_impl(t, none, s)) || (rc = scatter_impl(t, a.payload, s))) return rc;
    }
    if ((rc = push_state(t, s))) return rc;
    XCK(cudaStreamSynchronize(s));
    if (n_applied) *n_applied = ok;
    if (ok < a.n) return fail(XPIR_EINVAL, "cuckoo: bucket index out of range");
    return XPIR_OK;
}

int xpir_table_insert_walk_dev(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, uint64_t n,
                               uint32_t* d_reports, void* stream) {
    if (!t) return fail(XPIR_EINVAL, "table_insert: null table");
    if (n == 0) return XPIR_OK;
    if (!d_b1 || !d_b2) return fail(XPIR_EINVAL, "table_insert: null buffer");
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    uint64_t ok = n;
    int rc = walk_impl(t, d_b1, d_b2, n, d_reports, s, false, false, &ok);
    if (rc) return rc;
    if (!stream) XCK(cudaStreamSynchronize(s));
    // EINVAL with the valid prefix walked: the caller still applies gather/scatter
    if (ok < n) return fail(XPIR_EINVAL, "cuckoo: bucket index out of range");
    return XPIR_OK;
}

int xpir_table_apply_gather_dev(xpir_table* t, const xpir_shard_map* map, void* stream) {
    if (!t) return fail(XPIR_EINVAL, "table_apply: null table");
    ShardMap m{};
    if (map) {
        if (map->n > 8) return fail(XPIR_EINVAL, "table_apply: at most 8 shards");
        m.n = map->n;
        for (uint32_t k = 0; k <= map->n; ++k) m.lo[k] = map->bucket_lo[k];
        for (uint32_t k = 0; k < map->n; ++k) m.data[k] = map->data[k];
        if (m.n && (m.lo[0] != 0 || m.lo[m.n] != t->d.buckets))
            return fail(XPIR_EINVAL, "table_apply: shard map must cover every bucket");
    } else if (t->sharded()) {
        return fail(XPIR_EINVAL, "table_apply: a payload shard needs the shard map");
    }
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    int rc = sync_state(t, s);
    if (!rc) rc = gather_impl(t, m, s);
    if (rc) return rc;
    if (!stream) XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_table_apply_scatter_dev(xpir_table* t, const uint8_t* d_payload, void* stream) {
    if (!t) return fail(XPIR_EINVAL, "table_apply: null table");
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    int rc = sync_state(t, s);
    if (rc) return rc;
    if (t->h.n_touched && !d_payload) return fail(XPIR_EINVAL, "table_apply: null payload");
    if ((rc = scatter_impl(t, d_payload, s))) return rc;
    if (!stream) XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_table_shard(const xpir_table* t, uint32_t* lo, uint32_t* hi) {
    if (!t) return fail(XPIR_EINVAL, "table_shard: null table");
    if (lo) *lo = t->lo;
    if (hi) *hi = t->hi;
    return XPIR_OK;
}

}  // extern "C"

// One host write (ServerCore::apply_write through the drop-in) as a replayed CUDA
// graph: [inputs H2D from the pinned stage, state H2D from the pinned mirror, the
// global-map walk, payload gather, payload scatter, reports D2H, state D2H] —
// one graph launch and one synchronisation per write instead of ~12 runtime
// calls. Captured once per table (its buffers are fixed once reserved); the host
// only packs the write, advances its state mirror and checks the result.
static int insert_one_graph(xpir_table* t, uint32_t b1, uint32_t b2, const uint8_t* payload, uint32_t* report) {
    cudaStream_t s = t->stream;
    const uint64_t item = t->d.item;
    const uint64_t o2 = 16, op = 32, orep = op + round16(item), total = orep + 16;
    if (!t->g1) {
        // fixed buffers: packed write + report (device and pinned), state mirror, gather staging
        XCK(t->g1_stage.ensure(total));
        XCK(t->g1_dev.ensure(total));
        XCK(t->state_h.ensure(sizeof(CuckooState)));
        XCK(t->gather.ensure(502 * item));
        t->d.gather = t->gather.as<uint8_t>();
        uint8_t* dp = t->g1_dev.as<uint8_t>();
        cudaGraph_t graph = nullptr;
        XCK(cudaStreamSynchronize(s));
        XCK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = cudaMemcpyAsync(dp, t->g1_stage.p, orep, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(t->dstate, t->state_h.p, sizeof(CuckooState), cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = launch_cuckoo_walk(t->d, t->dstate, reinterpret_cast<const uint32_t*>(dp),
                                   reinterpret_cast<const uint32_t*>(dp + o2), 0, 1,
                                   reinterpret_cast<uint32_t*>(dp + orep), s);
        const ShardMap none{};
        if (e == cudaSuccess)
            e = launch_cuckoo_gather_sharded(t->d, &t->h, t->lo, t->hi, t->data, none, s, t->dstate, 502, 502);
        if (e == cudaSuccess)
            e = launch_cuckoo_scatter_sharded(t->d, &t->h, t->lo, t->hi, t->data, dp + op, s, t->dstate, 502);
        if (e == cudaSuccess) e = cudaMemcpyAsync(t->g1_stage.p + orep, dp + orep, 16, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(t->state_h.p, t->dstate, sizeof(CuckooState), cudaMemcpyDeviceToHost, s);
        const cudaError_t e2 = cudaStreamEndCapture(s, &graph);
        if (e == cudaSuccess) e = e2;
        if (e == cudaSuccess) e = cudaGraphInstantiate(&t->g1, graph, 0);
        if (graph) cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            t->g1 = nullptr;
            cudaGetLastError();
            return fail(XPIR_ECUDA, std::string("table_insert: single-write graph: ") + cudaGetErrorString(e));
        }
    }
    std::memcpy(t->g1_stage.p, &b1, 4);
    std::memcpy(t->g1_stage.p + o2, &b2, 4);
    std::memcpy(t->g1_stage.p + op, payload, item);
    // the batch starts on the host mirror (as walk_impl's small path), the graph
    // pushes it, walks, moves the payloads and brings the state back
    t->h.batch_id += 1;
    t->h.n_touched = 0;
    t->h.walked = 0;
    t->h.limit = ~0ull;
    t->h.status = 0;
    t->walked = true;
    int rc = refill_draws(t, 2048, s);
    if (rc) return rc;
    XCK(t->state_h.ensure(sizeof(CuckooState)));  // no earlier async copy still reads the mirror
    std::memcpy(t->state_h.p, &t->h, sizeof(CuckooState));
    XCK(cudaGraphLaunch(t->g1, s));
    count_launches(3);
    XCK(cudaStreamSynchronize(s));
    std::memcpy(&t->h, t->state_h.p, sizeof(CuckooState));
    if (t->h.status != 0) {  // the walk paused (draws / FIFO ring): finish on the host-driven path
        const uint32_t st0 = t->h.status;
        t->h.status = 0;
        if (st0 == 2) {
            if ((rc = grow_fifo(t, s))) return rc;
        } else {
            t->h.draw_count = 0;
        }
        uint8_t* dp = t->g1_dev.as<uint8_t>();
        if ((rc = walk_loop(t, reinterpret_cast<const uint32_t*>(dp), reinterpret_cast<const uint32_t*>(dp + o2),
                            t->h.resume_at, 1, reinterpret_cast<uint32_t*>(dp + orep), s)))
            return rc;
        const ShardMap none{};
        if ((rc = gather_impl(t, none, s)) || (rc = scatter_impl(t, dp + op, s))) return rc;
        XCK(cudaMemcpyAsync(t->g1_stage.p + orep, dp + orep, 16, cudaMemcpyDeviceToHost, s));
        XCK(cudaStreamSynchronize(s));
        if ((rc = push_state(t, s))) return rc;
    }
    if (report) std::memcpy(report, t->g1_stage.p + orep, 16);
    return XPIR_OK;
}

extern "C" {

int xpir_table_insert_batch(xpir_table* t, const uint32_t* b1, const uint32_t* b2,
                            const uint8_t* payload, uint64_t n, uint32_t* reports) {
    if (!t) return fail(XPIR_EINVAL, "table_insert: null table");
    if (n == 0) return XPIR_OK;
    if (!b1 || !b2 || !payload) return fail(XPIR_EINVAL, "table_insert: null buffer");
    if (t->sharded())
        return fail(XPIR_EINVAL, "table_insert: payload shard: use insert_walk + apply_gather (all shards) + apply_scatter");
    // cuckoo.cpp:57-58 — validated per item in order; items before the bad one
    // are inserted, exactly as a loop of Table::insert calls would leave them.
    uint64_t ok = n;
    for (uint64_t k = 0; k < n; ++k)
        if (b1[k] >= t->d.buckets || b2[k] >= t->d.buckets) {
            ok = k;
            break;
        }
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    cudaStream_t s = t->stream;
    if (ok == 1 && !t->state_on_device && 256 < t->slots() && walk_w_supported(t->d)) {
        if (int rc = insert_one_graph(t, b1[0], b2[0], payload, reports)) return rc;
    } else if (ok > 0) {
        // [beta1 | beta2 | payload | reports] packed: one pinned staging buffer, one H2D.
        // Large payloads go straight from the caller's memory instead (the driver
        // pipelines pageable copies; one host memcpy of 16 MB into the stage first
        // cost ~2 ms per config-3-sized round)
        const uint64_t o2 = round16(4 * ok), op = o2 + round16(4 * ok), orep = op + round16(ok * t->d.item);
        const uint64_t total = orep + 16 * ok;
        const bool pack_payload = ok * t->d.item <= (uint64_t(1) << 18);
        const uint64_t hrep = pack_payload ? orep : op;  // host offset of the reports
        XCK(t->stage.ensure(hrep + 16 * ok));
        std::memcpy(t->stage.p, b1, 4 * ok);
        std::memcpy(t->stage.p + o2, b2, 4 * ok);
        if (pack_payload) std::memcpy(t->stage.p + op, payload, ok * t->d.item);
        XCK(t->in_pack.ensure(total));
        uint8_t* dp = t->in_pack.as<uint8_t>();
        XCK(cudaMemcpyAsync(dp, t->stage.p, pack_payload ? orep : op, cudaMemcpyHostToDevice, s));
        if (!pack_payload) XCK(cudaMemcpyAsync(dp + op, payload, ok * t->d.item, cudaMemcpyHostToDevice, s));
        uint64_t applied = ok;
        int rc = insert_impl(t, reinterpret_cast<const uint32_t*>(dp), reinterpret_cast<const uint32_t*>(dp + o2),
                             dp + op, ok, reinterpret_cast<uint32_t*>(dp + orep), s, t->stage.p + hrep, true,
                             &applied);
        XCK(t->stage.release_after(s));
        if (rc) return rc;
        if (reports) std::memcpy(reports, t->stage.p + hrep, 16 * ok);
    }
    if (ok < n) return fail(XPIR_EINVAL, "cuckoo: bucket index out of range");
    return XPIR_OK;
}

int xpir_table_reserve(xpir_table* t, uint64_t max_batch) {
    if (!t) return fail(XPIR_EINVAL, "table_reserve: null table");
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    // a round touches its new items' slots plus the slots of the items its
    // eviction chains move: sized for twice the batch (capped at the table)
    const uint64_t n = std::min<uint64_t>(2 * max_batch + 1024, t->slots());
    XCK(t->gather.ensure(n * t->d.item));
    XCK(t->in_b1.ensure(4 * max_batch));
    XCK(t->in_b2.ensure(4 * max_batch));
    XCK(t->in_reports.ensure(16 * max_batch));
    // the packed host-input staging of xpir_table_insert_batch, pinned, for max_batch writes
    // (payloads above 256 KiB are copied from the caller's memory, not staged)
    const uint64_t pack = 2 * round16(4 * max_batch) + round16(max_batch * t->d.item) + 16 * max_batch;
    const bool pack_payload = max_batch * t->d.item <= (uint64_t(1) << 18);
    XCK(t->stage.ensure(pack_payload ? pack : 2 * round16(4 * max_batch) + 16 * max_batch));
    XCK(t->in_pack.ensure(pack));
    XCK(cuckoo_reserve(t->par, max_batch, t->d.buckets, t->stream));  // parallel-prefix scratch
    // a full draw window, so a round's eviction walk rarely has to pause for draws
    int rc = sync_state(t, t->stream);
    if (rc) return rc;
    if ((rc = refill_draws(t, uint64_t(DRAW_CAP) / 2, t->stream)) || (rc = push_state(t, t->stream))) return rc;
    XCK(cudaStreamSynchronize(t->stream));
    return XPIR_OK;
}

int xpir_table_snapshot(const xpir_table* t, uint8_t* host_out) {
    if (!t || !host_out) return fail(XPIR_EINVAL, "table_snapshot: null argument");
    DeviceGuard g(t->device);
    XCK(cudaStreamSynchronize(t->stream));
    XCK(cudaMemcpy(host_out, t->data, t->data_bytes(), cudaMemcpyDeviceToHost));
    return XPIR_OK;
}

void* xpir_table_device_data(const xpir_table* t) { return t ? t->data : nullptr; }

int xpir_table_seal(const xpir_table* t, xpir_store* st, uint64_t epoch, void* stream) {
    if (!t || !st) return fail(XPIR_EINVAL, "table_seal: null argument");
    if (st->N != t->d.buckets || uint64_t(st->S) != uint64_t(t->d.depth) * t->d.item)
        return fail(XPIR_EINVAL, "table_seal: store geometry differs from the table");
    if (st->device != t->device) return fail(XPIR_EINVAL, "table_seal: different devices");
    if (st->lo < t->lo || st->hi > t->hi) return fail(XPIR_EINVAL, "table_seal: store range outside the payload shard");
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    XCK(cudaMemcpyAsync(st->data, t->data + uint64_t(st->lo - t->lo) * st->S, st->bytes(),
                        cudaMemcpyDeviceToDevice, s));
    if (!stream) XCK(cudaStreamSynchronize(s));
    st->epoch = epoch;
    return XPIR_OK;
}

int xpir_table_meta(const xpir_table* t, uint8_t* used, uint32_t* b1, uint32_t* b2,
                    uint64_t* stamp) {
    if (!t) return fail(XPIR_EINVAL, "table_meta: null table");
    DeviceGuard g(t->device);
    XCK(cudaStreamSynchronize(t->stream));
    const uint64_t n = t->slots();
    if (used) XCK(cudaMemcpy(used, t->d.used, n, cudaMemcpyDeviceToHost));
    if (b1) XCK(cudaMemcpy(b1, t->d.beta1, 4 * n, cudaMemcpyDeviceToHost));
    if (b2) XCK(cudaMemcpy(b2, t->d.beta2, 4 * n, cudaMemcpyDeviceToHost));
    if (stamp) XCK(cudaMemcpy(stamp, t->d.stamp, 8 * n, cudaMemcpyDeviceToHost));
    return XPIR_OK;
}

int xpir_table_counters(const xpir_table* t, uint64_t* writes, uint64_t* live, uint64_t* next_stamp) {
    if (!t) return fail(XPIR_EINVAL, "table_counters: null table");
    if (writes) *writes = t->h.writes;
    if (live) *live = t->h.live;
    if (next_stamp) *next_stamp = t->h.next_stamp;
    return XPIR_OK;
}

int xpir_table_slot_used(const xpir_table* t, uint32_t bucket, uint32_t slot) {
    if (!t || bucket >= t->d.buckets || slot >= t->d.depth)
        return fail(XPIR_EINVAL, "slot_used: out of range");
    DeviceGuard g(t->device);
    uint8_t u = 0;
    XCK(cudaStreamSynchronize(t->stream));
    XCK(cudaMemcpy(&u, t->d.used + uint64_t(bucket) * t->d.depth + slot, 1, cudaMemcpyDeviceToHost));
    return u ? 1 : 0;
}

int xpir_table_state_digest(const xpir_table* t, uint8_t out[32]) {
    if (!t || !out) return fail(XPIR_EINVAL, "state_digest: null argument");
    if (t->sharded()) return fail(XPIR_EINVAL, "state_digest: needs the whole table (this is a payload shard)");
    const uint64_t n = t->slots();
    std::vector<uint8_t> data(n * t->d.item), used(n);
    std::vector<uint32_t> b1(n), b2(n);
    std::vector<uint64_t> st(n);
    int rc = xpir_table_snapshot(t, data.data());
    if (rc) return rc;
    rc = xpir_table_meta(t, used.data(), b1.data(), b2.data(), st.data());
    if (rc) return rc;
    HostBlake2b h(32);  // cuckoo.cpp:137-149
    h.update_u64be(t->h.writes);
    h.update_u64be(t->h.live);
    h.update_u64be(t->h.next_stamp);
    h.update(data.data(), data.size());
    for (uint64_t f = 0; f < n; ++f) {
        h.update_u64be(used[f] ? 1 : 0);
        h.update_u64be(uint64_t(b1[f]) << 32 | b2[f]);
        h.update_u64be(st[f]);
    }
    h.final(out);
    return XPIR_OK;
}

}  // extern "C"

